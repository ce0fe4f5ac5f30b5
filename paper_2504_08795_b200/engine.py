"""Simulation entry point of the drop-in API (stagesim/engine.py:61-531).

``Simulation(...).run()`` keeps the reference's signature and result types;
the whole event loop — releases, admission/migration, 8-level + EDF dispatch,
the SM water-fill rate model, completions and the metrics accumulator —
runs inside the native core (``daris_sim_run``). Python only prepares the
seeded randomness (phases, AFET competitor draws) with CPython's own MT19937
so results are bit-identical to the reference.
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass
from enum import IntEnum
from typing import NamedTuple, Sequence

from . import _core
from .errors import InvalidScenario
from .gpu import BatchingCurve, GpuConfig, effective_stage_time, sm_per_context
from .model import Priority, TaskSpec, build_task_set, collapse_stages, spec_to_dict
from .scheduler import AblationFlags, AdmissionDecision, SchedulerMode
from .timing import DEFAULT_FULL_LOAD_REPS, DEFAULT_WINDOW_SIZE, competitor_draws


class EventKind(IntEnum):
    RELEASE = 0
    STAGE_COMPLETE = 1
    SIM_END = 2


class LogRecord(NamedTuple):
    time: float
    kind: str
    task: int | None
    job: int | None
    stage: int | None
    context: int | None
    stream: int | None
    rate: float | None

    def to_dict(self) -> dict:
        return self._asdict()


def format_label(n_contexts: int, n_streams: int, oversubscription: float) -> str:
    """Paper notation contexts x streams _ OS, e.g. 6x1_6."""
    return f"{n_contexts}x{n_streams}_{oversubscription:g}"


def parse_label(label: str) -> tuple[int, int, float]:
    try:
        c, rest = label.split("x", 1)
        s, o = rest.split("_", 1)
        return int(c), int(s), float(o)
    except ValueError as exc:
        raise ValueError(f"malformed config label {label!r}") from exc


@dataclass(frozen=True)
class ResponseStats:
    mean: float = 0.0
    min: float = 0.0
    max: float = 0.0
    p95: float = 0.0
    count: int = 0
    p99: float = 0.0   # new: the north-star metric (nearest rank, like p95)

    @classmethod
    def from_samples(cls, samples: Sequence[float]) -> "ResponseStats":
        if not samples:
            return cls()
        o = sorted(samples)
        n = len(o)
        return cls(sum(o) / n, o[0], o[-1], o[math.ceil(0.95 * n) - 1], n, o[math.ceil(0.99 * n) - 1])

    @classmethod
    def from_native(cls, s: _core.ResponseStatsC) -> "ResponseStats":
        return cls(s.mean, s.min, s.max, s.p95, int(s.count), s.p99)

    def to_dict(self, *, extended: bool = False) -> dict:
        d = {"mean": self.mean, "min": self.min, "max": self.max, "p95": self.p95, "count": self.count}
        if extended:
            d["p99"] = self.p99
        return d


@dataclass(frozen=True)
class MetricsReport:
    label: str
    policy: str
    n_contexts: int
    n_streams: int
    oversubscription: float
    seed: int
    duration: float
    warmup: float
    jps: float
    dmr_hp: float
    dmr_lp: float
    response_hp: ResponseStats
    response_lp: ResponseStats
    released_hp: int
    released_lp: int
    accepted_hp: int
    accepted_lp: int
    rejected_hp: int
    rejected_lp: int
    completed_hp: int
    completed_lp: int
    missed_hp: int
    missed_lp: int

    def to_dict(self, *, extended: bool = False) -> dict:
        out = {}
        for name in self.__dataclass_fields__:
            v = getattr(self, name)
            out[name] = v.to_dict(extended=extended) if isinstance(v, ResponseStats) else v
        return out


@dataclass
class SimResult:
    report: MetricsReport
    records: list[LogRecord]
    admissions: list[AdmissionDecision]
    effective_tasks: list[TaskSpec]
    full_load: dict[int, float]


def report_from_native(r: _core.ReportC, *, label: str, config: GpuConfig, seed: int) -> MetricsReport:
    return MetricsReport(
        label=label, policy=config.policy.value, n_contexts=config.n_contexts, n_streams=config.n_streams,
        oversubscription=config.oversubscription, seed=seed, duration=r.duration, warmup=r.warmup,
        jps=r.jps, dmr_hp=r.dmr_hp, dmr_lp=r.dmr_lp,
        response_hp=ResponseStats.from_native(r.response_hp),
        response_lp=ResponseStats.from_native(r.response_lp),
        released_hp=r.released_hp, released_lp=r.released_lp, accepted_hp=r.accepted_hp,
        accepted_lp=r.accepted_lp, rejected_hp=r.rejected_hp, rejected_lp=r.rejected_lp,
        completed_hp=r.completed_hp, completed_lp=r.completed_lp, missed_hp=r.missed_hp,
        missed_lp=r.missed_lp)


def aggregate_demand(tasks: Sequence[TaskSpec], batch_sizes: dict[int, int] | None = None,
                     curves: dict[int, BatchingCurve] | None = None) -> float:
    """Offered work in full-width seconds per second (engine.py:232-245)."""
    batch_sizes, curves = batch_sizes or {}, curves or {}
    total = 0.0
    for t in tasks:
        b, c = batch_sizes.get(t.id, 1), curves.get(t.id)
        total += sum(effective_stage_time(p, b, c) for p in t.stages) / t.period
    return total


def modeled_capacity(config: GpuConfig, tasks: Sequence[TaskSpec], batch_sizes: dict[int, int] | None = None,
                     curves: dict[int, BatchingCurve] | None = None) -> float:
    """Sustainable full-width work rate for this mix (engine.py:248-271)."""
    batch_sizes, curves = batch_sizes or {}, curves or {}
    width_weighted = rate_sum = 0.0
    for t in tasks:
        b, c = batch_sizes.get(t.id, 1), curves.get(t.id)
        for p in t.stages:
            r = effective_stage_time(p, b, c) / t.period
            width_weighted += r * p.width
            rate_sum += r
    if rate_sum <= 0:
        raise InvalidScenario("cannot size capacity for a task set without demand")
    w = width_weighted / rate_sum
    per_ctx = min(float(config.n_streams), sm_per_context(config) / w)
    return min(config.n_contexts * per_ctx, config.total_sms / w)


def scale_to_overload(tasks: Sequence[TaskSpec], factor: float, capacity: float,
                      batch_sizes: dict[int, int] | None = None,
                      curves: dict[int, BatchingCurve] | None = None) -> list[TaskSpec]:
    """Rescale every period so demand = factor * capacity (engine.py:274-291)."""
    if factor <= 0:
        raise InvalidScenario("overload factor must be positive")
    if capacity <= 0:
        raise InvalidScenario("capacity must be positive")
    ratio = aggregate_demand(tasks, batch_sizes, curves) / (factor * capacity)
    return [TaskSpec(t.id, t.period * ratio, t.deadline * ratio, t.priority, t.stages) for t in tasks]


def _priority(code: int) -> Priority:
    return Priority.HP if code == 0 else Priority.LP


class Simulation:
    """One configured run of the DARIS execution path; call run() once."""

    def __init__(self, tasks: Sequence[TaskSpec], config: GpuConfig, *, seed: int = 0, duration: float = 60.0,
                 warmup_frac: float = 0.1, window_size: int = DEFAULT_WINDOW_SIZE,
                 full_load_reps: int = DEFAULT_FULL_LOAD_REPS, batch_sizes: dict[int, int] | None = None,
                 curves: dict[int, BatchingCurve] | None = None, flags: AblationFlags = AblationFlags(),
                 mode: SchedulerMode = SchedulerMode(), phasing: str = "random",
                 placement_order: str = "descending_util", edf_on_job_deadline: bool = False,
                 collect_log: bool = True, check_invariants: bool = False, stage_migration: bool = False):
        if duration <= 0:
            raise InvalidScenario("duration must be positive")
        if not (0.0 <= warmup_frac < 1.0):
            raise InvalidScenario("warmup fraction must lie in [0, 1)")
        if phasing not in ("random", "zero"):
            raise InvalidScenario(f"unknown phasing mode {phasing!r}")
        for t in tasks:
            for p in t.stages:
                if p.width > config.total_sms:
                    raise InvalidScenario(f"task {t.id} stage width {p.width} exceeds the device "
                                          f"({config.total_sms} SMs)")
        self.tasks = list(tasks)
        self.config = config
        self.seed = seed
        self.duration = duration
        self.warmup_end = duration * warmup_frac
        self.warmup_frac = warmup_frac
        self.window_size = window_size
        self.full_load_reps = full_load_reps
        self.batch_sizes = dict(batch_sizes or {})
        self.curves = dict(curves or {})
        self.flags = flags
        self.mode = mode
        self.phasing = phasing
        self.placement_order = placement_order
        self.edf_on_job_deadline = edf_on_job_deadline
        self.collect_log = collect_log
        self.check_invariants = check_invariants
        self.stage_migration = stage_migration
        self.label = format_label(config.n_contexts, config.n_streams, config.oversubscription)
        self.handle: _core.Handle | None = None

    # offline phase ---------------------------------------------------------
    def _effective(self) -> list[TaskSpec]:
        eff = list(build_task_set(self.tasks).tasks)
        if self.flags.no_staging:
            eff = list(collapse_stages(build_task_set(eff)).tasks)
        return eff

    def _open(self, effective: list[TaskSpec]) -> _core.Handle:
        dicts = [spec_to_dict(t, self.batch_sizes.get(t.id, 1), self.curves.get(t.id)) for t in effective]
        opts = _core.options_struct(window_size=self.window_size, no_staging=False,
                                    no_last=self.flags.no_last, no_prior=self.flags.no_prior,
                                    no_fixed=self.flags.no_fixed, hpa=self.mode.hpa_enabled,
                                    placement_order=self.placement_order,
                                    edf_on_job_deadline=self.edf_on_job_deadline,
                                    check_invariants=self.check_invariants,
                                    stage_migration=self.stage_migration)
        return _core.Handle(self.config.native(), dicts, opts)

    def _measure_full_load(self, h: _core.Handle, effective: list[TaskSpec]) -> dict[int, float]:
        """AFET once per distinct (stages, batch, curve) signature (engine.py:357-375)."""
        memo: dict[tuple, float] = {}
        out: dict[int, float] = {}
        n_slots = self.config.n_contexts * self.config.n_streams
        for t in effective:
            sig = (t.stages, self.batch_sizes.get(t.id, 1), self.curves.get(t.id))
            if sig not in memo:
                seed = self.seed * 7919 + len(memo)
                draws = competitor_draws(len(effective), n_slots, self.full_load_reps, seed)
                memo[sig] = h.full_load_sim(t.id, self.full_load_reps, draws)
            out[t.id] = memo[sig]
        return out

    def phases(self, effective: list[TaskSpec]) -> list[float]:
        """Release offsets (engine.py:417-423): Random(seed).random() * T in id order."""
        rng = random.Random(self.seed)
        return [rng.random() * t.period if self.phasing == "random" else 0.0 for t in effective]

    def prepare(self) -> tuple[_core.Handle, list[TaskSpec], dict[int, float], list[float]]:
        effective = self._effective()
        h = self._open(effective)
        full = self._measure_full_load(h, effective)
        h.set_full_load([full[i] for i in h.task_ids])
        h.populate()
        self.handle = h
        return h, effective, full, self.phases(effective)

    # online phase ----------------------------------------------------------
    def _result(self, h, rep, effective, full) -> SimResult:
        report = report_from_native(rep, label=self.label, config=self.config, seed=self.seed)
        records = [LogRecord(*r) for r in _core.records_from_array(h.log_array())] if self.collect_log else []
        admissions = [AdmissionDecision.from_native(a) for a in h.audits()]
        return SimResult(report, records, admissions, effective, full)

    def run(self) -> SimResult:
        if not self.tasks:
            records = [LogRecord(self.duration, "sim_end", None, None, None, None, None, None)] \
                if self.collect_log else []
            rep = _core.ReportC()
            rep.duration, rep.warmup = self.duration, self.warmup_end
            return SimResult(report_from_native(rep, label=self.label, config=self.config, seed=self.seed),
                             records, [], [], {})
        h, effective, full, phases = self.prepare()
        rep = h.sim_run(self.duration, self.warmup_frac, phases, self.collect_log)
        return self._result(h, rep, effective, full)

    def run_trace(self, durations: dict[tuple[int, int, int], float],
                  full_load: dict[int, float], phases: Sequence[float] | None = None,
                  unsampled=None) -> SimResult:
        """Trace-replay mode: stage (task, job, stage) runs for
        durations[...] seconds at rate 1; AFET baselines are given; `phases`
        (release offsets in task-id order) replace the seeded draw, e.g. the
        ones a real GPU run used; `unsampled` {(task, job, stage)}: stages the
        run completed without an MRET sample (in flight across a GPU pause)."""
        effective = self._effective()
        h = self._open(effective)
        h.set_full_load([full_load[i] for i in h.task_ids])
        h.populate()
        self.handle = h
        ph = list(phases) if phases is not None else self.phases(effective)
        rep = h.trace_run(self.duration, self.warmup_frac, ph, durations, self.collect_log, unsampled)
        return self._result(h, rep, effective, dict(full_load))
