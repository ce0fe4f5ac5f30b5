"""Execution-time tracking (MRET window + AFET baseline) of the drop-in API.

Object-level view with the reference's names and state layout
(stagesim/timing.py:33-218): per-stage ``ExecutionWindow`` rings live on each
``TaskState`` and the utilization cache on the ``TimingTracker``, so callers
that drive the objects directly (the reference's own tests do) see the same
state. Every number is computed by the native decision kernels
(csrc/core/decide.cpp, ``daris_eval_*``) that the stateful dispatcher used by
the engine and the GPU executor also runs on.
"""

from __future__ import annotations

import random
from collections import deque
from typing import TYPE_CHECKING, Sequence

from . import _core
from .errors import NonpositiveSample

if TYPE_CHECKING:  # pragma: no cover
    from .gpu import BatchingCurve, GpuConfig
    from .model import TaskSpec, TaskState

DEFAULT_WINDOW_SIZE = 5        # ws (timing.py:29)
DEFAULT_FULL_LOAD_REPS = 10    # R (timing.py:30)


class ExecutionWindow:
    """The last `capacity` observed execution times of one stage (timing.py:33-62);
    ``peak()`` is the MRET sample."""

    __slots__ = ("capacity", "_ring")

    def __init__(self, capacity: int = DEFAULT_WINDOW_SIZE):
        if capacity < 1:
            raise ValueError("window capacity must be >= 1")
        self.capacity = capacity
        self._ring: deque = deque(maxlen=capacity)

    def record(self, observed_time: float) -> None:
        if not observed_time > 0:
            raise NonpositiveSample(f"observed time must be positive, got {observed_time}")
        self._ring.append(observed_time)

    def peak(self) -> float | None:
        if not self._ring:
            return None
        vals = list(self._ring)
        best = _core.ev_window_peak(vals)
        # hand back the caller's own object (int samples stay ints, like max())
        return next(v for v in vals if v == best)

    @property
    def values(self) -> list[float]:
        return list(self._ring)

    def __len__(self) -> int:
        return len(self._ring)


def competitor_draws(n_pool: int, n_slots: int, repetitions: int, seed: int) -> list[int]:
    """Pool indices the busy-system measurement fills the other streams with:
    repetition r draws from random.Random(seed * 1_000_003 + r) (timing.py:178-190).
    Generated here (CPython's MT19937) and handed to the native loop."""
    draws: list[int] = []
    for rep in range(repetitions):
        rng = random.Random(seed * 1_000_003 + rep)
        draws.extend(rng.randrange(n_pool) for _ in range(1, n_slots))
    return draws


def measure_full_load_time(target: "TaskSpec", pool: Sequence["TaskSpec"], config: "GpuConfig",
                           repetitions: int = DEFAULT_FULL_LOAD_REPS, seed: int = 0, *,
                           batch_sizes: dict[int, int] | None = None,
                           curves: dict[int, "BatchingCurve"] | None = None) -> float:
    """Mean finish time of `target` on ctx 1 / stream 0 with every other stream
    looping random pool tasks (AFET, timing.py:147-181), run natively."""
    from .model import spec_to_dict
    if repetitions < 1:
        raise ValueError("repetitions must be >= 1")
    if not pool:
        raise ValueError("competitor pool must not be empty")
    batch_sizes = batch_sizes or {}
    curves = curves or {}
    tasks = []
    for i, spec in enumerate(list(pool) + [target]):
        d = spec_to_dict(spec, batch_sizes.get(spec.id, 1), curves.get(spec.id))
        d["id"] = i + 1
        d["deadline"] = d["period"]
        tasks.append(d)
    h = _core.Handle(config.native(), tasks, _core.options_struct())
    draws = competitor_draws(len(pool), config.n_contexts * config.n_streams, repetitions, seed)
    return h.full_load_sim(len(tasks), repetitions, draws)


class TimingTracker:
    """Per-task MRET / AFET estimates over TaskState objects (timing.py:64-132)."""

    def __init__(self, states: Sequence["TaskState"]):
        self._states: dict[int, "TaskState"] = {st.task.id: st for st in states}
        self._util_cache: dict[int, float] = {}

    def state(self, task_id: int) -> "TaskState":
        return self._states[task_id]

    def record_execution(self, task_id: int, stage_index: int, observed_time: float) -> None:
        self._states[task_id].windows[stage_index].record(observed_time)

    def stage_estimate(self, task_id: int, stage_index: int) -> float:
        """MRET of the stage, or its nominal share of the AFET while its window is empty."""
        st = self._states[task_id]
        peak = st.windows[stage_index].peak()
        if peak is not None:
            return peak
        spec = st.task
        return _core.ev_stage_fallback(st.full_load_time, spec.stages[stage_index].nominal_time,
                                       spec.nominal_total)

    def stage_estimates(self, task_id: int) -> list[float]:
        return [self.stage_estimate(task_id, j) for j in range(len(self._states[task_id].task.stages))]

    def task_estimate(self, task_id: int) -> float:
        return _core.ev_task_estimate(self.stage_estimates(task_id))

    def utilization(self, task_id: int) -> float:
        """AFET / T before the task's first completed job, MRET_i / T after;
        cached until the next completion of one of its jobs."""
        if task_id in self._util_cache:
            return self._util_cache[task_id]
        st = self._states[task_id]
        est = self.task_estimate(task_id) if st.completed_jobs else 0.0
        u = _core.ev_utilization(st.completed_jobs, st.full_load_time, est, st.task.period)
        self._util_cache[task_id] = u
        return u

    def note_job_complete(self, task_id: int) -> None:
        self._states[task_id].completed_jobs += 1
        self._util_cache.pop(task_id, None)

    def deadline_shares(self, task_id: int) -> list[float]:
        """Stage deadline spans proportional to the estimates, summing to D
        exactly (the last absorbs the rounding residue)."""
        spec = self._states[task_id].task
        return _core.ev_deadline_shares(self.stage_estimates(task_id), spec.deadline, task_id)
