"""Real-GPU backend of the drop-in scenario API.

A scenario with ``"backend": "gpu"`` runs the same task set through the
native dispatcher and the wall-clock executor (runtime.DarisRuntime) instead
of the rate-model event loop: ``build_simulation(cfg)`` returns a
``GpuSimulation`` whose ``run()`` gives the reference's ``SimResult``
(engine.py:223-229 of stagesim) — report, event records, admission audits,
the effective task set (stage nominal times measured on the partition) and
the AFET values measured with random co-runners (timing.py:147-218 made
real). The per-stage trace of the run is attached so it can be replayed
through the rate-model engine's trace mode (``Simulation.run_trace``) for
decision parity.

Each task needs a network: ``model`` on an explicit task, or a workload
profile that names one (presets.DnnProfile.model). There is no CPU fallback:
without a CUDA device ``run()`` raises.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

from .engine import LogRecord, SimResult
from .errors import InvalidScenario
from .gpu import GpuConfig
from .model import TaskSpec
from .scheduler import AblationFlags, SchedulerMode

GPU_MODELS = ("resnet18", "resnet50", "vgg16", "mobilenet_v2")


@dataclass
class GpuTask:
    """Which network a task runs and how many stages it is split into."""
    model: str
    n_stages: int | None = None


@dataclass
class GpuSimResult(SimResult):
    """SimResult plus what only a real run has: the per-stage trace
    (task, job, stage, context, stream, slot, start, end, sampled),
    executor counters and the partitions actually built."""
    trace: list = field(default_factory=list)
    stats: dict = field(default_factory=dict)
    partitions: list = field(default_factory=list)
    phases: list = field(default_factory=list)

    def stage_durations(self) -> dict[tuple[int, int, int], float]:
        """(task, job, stage) -> observed seconds, the input of trace replay."""
        return {(t[0], t[1], t[2]): t[7] - t[6] for t in self.trace}

    def unsampled(self) -> set:
        """(task, job, stage) the run completed without an MRET sample (in
        flight across a detected GPU-wide pause): replay them as such."""
        return {(t[0], t[1], t[2]) for t in self.trace if len(t) > 8 and not t[8]}


class GpuSimulation:
    """One configured run on the real GPU; mirrors Simulation's constructor."""

    def __init__(self, tasks: Sequence[TaskSpec], config: GpuConfig, gpu_tasks: dict[int, GpuTask], *,
                 seed: int = 0, duration: float = 10.0, warmup_frac: float = 0.1, window_size: int = 5,
                 flags: AblationFlags = AblationFlags(), mode: SchedulerMode = SchedulerMode(),
                 phasing: str = "random", placement_order: str = "descending_util",
                 edf_on_job_deadline: bool = False, stage_migration: bool = False, slots: int = 3, e2e: bool = False,
                 calibrate_seconds: float = 0.2, device: int = 0, batch_sizes: dict[int, int] | None = None):
        if flags.no_staging:
            raise InvalidScenario("the gpu backend runs real stage splits; use n_stages=1 instead of "
                                  "the no_staging ablation")
        for t in tasks:
            g = gpu_tasks.get(t.id)
            if g is None:
                raise InvalidScenario(f"task {t.id} has no model; the gpu backend needs one of {GPU_MODELS}")
            if g.model not in GPU_MODELS:
                raise InvalidScenario(f"task {t.id}: no sm_100a network for model {g.model!r}; "
                                      f"known: {GPU_MODELS}")
        self.tasks = list(tasks)
        self.config = config
        self.gpu_tasks = dict(gpu_tasks)
        self.seed = seed
        self.duration = duration
        self.warmup_frac = warmup_frac
        self.window_size = window_size
        self.flags = flags
        self.mode = mode
        self.phasing = phasing
        self.placement_order = placement_order
        self.edf_on_job_deadline = edf_on_job_deadline
        self.stage_migration = stage_migration
        self.slots = slots
        self.e2e = e2e
        self.calibrate_seconds = calibrate_seconds
        self.device = device
        self.batch_sizes = dict(batch_sizes or {})  # images per job (TaskSpec batch_size)
        self.runtime = None

    def build_runtime(self):
        from .runtime import DarisRuntime, TaskDef
        defs = [TaskDef(t.id, self.gpu_tasks[t.id].model, t.priority, 1.0 / t.period,
                        self.gpu_tasks[t.id].n_stages, self.batch_sizes.get(t.id, 1)) for t in self.tasks]
        self.runtime = DarisRuntime(defs, self.config, slots=self.slots, window_size=self.window_size,
                                    flags=self.flags, hpa=self.mode.hpa_enabled,
                                    stage_migration=self.stage_migration, seed=self.seed, e2e=self.e2e,
                                    device=self.device, phasing=self.phasing,
                                    placement_order=self.placement_order,
                                    edf_on_job_deadline=self.edf_on_job_deadline)
        return self.runtime

    def run(self) -> GpuSimResult:
        rt = self.runtime or self.build_runtime()
        full = rt.calibrate_full_load(self.calibrate_seconds)
        res = rt.run(self.duration, self.duration * self.warmup_frac, full_load=full)
        records = [LogRecord(*r) for r in res.records]
        return GpuSimResult(res.report, records, res.admissions, res.tasks, dict(res.full_load),
                            trace=res.trace, stats=res.stats, partitions=res.partitions, phases=res.phases)

    def close(self) -> None:
        if self.runtime is not None:
            self.runtime.close()
            self.runtime = None
