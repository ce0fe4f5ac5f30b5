"""Execution-time tracking (MRET window + AFET baseline) of the drop-in API.

The arithmetic runs in the native core (timing.py:33-132 of the reference is
restated in csrc/core/dispatcher.cpp); this module keeps the names:
``TimingTracker``, ``measure_full_load_time`` and the two defaults.
"""

from __future__ import annotations

import random
from typing import TYPE_CHECKING, Sequence

from . import _core

if TYPE_CHECKING:  # pragma: no cover
    from .gpu import BatchingCurve, GpuConfig
    from .model import TaskSpec, TaskState

DEFAULT_WINDOW_SIZE = 5        # ws (timing.py:29)
DEFAULT_FULL_LOAD_REPS = 10    # R (timing.py:30)


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
    """Per-task MRET/AFET estimates, backed by a native handle.

    Built from TaskStates (their ``full_load_time`` seeds the AFET); the
    Scheduler rebinds it to its own handle so both views share live state.
    """

    def __init__(self, states: Sequence["TaskState"], *, handle: _core.Handle | None = None):
        from .model import spec_to_dict
        self._states = {st.task.id: st for st in states}
        if handle is None:
            ws = next(iter(self._states.values())).window_size if self._states else DEFAULT_WINDOW_SIZE
            handle = _core.Handle(_core.gpu_struct(1, 1, 1, 1.0),
                                  [spec_to_dict(st.task) for st in states],
                                  _core.options_struct(window_size=ws))
            handle.set_full_load([self._states[i].full_load_time for i in handle.task_ids])
        self._h = handle

    def state(self, task_id: int) -> "TaskState":
        return self._states[task_id]

    def record_execution(self, task_id: int, stage_index: int, observed_time: float) -> None:
        self._h.record_execution(task_id, stage_index, observed_time)

    def stage_estimate(self, task_id: int, stage_index: int) -> float:
        return self._h.stage_estimate(task_id, stage_index)

    def task_estimate(self, task_id: int) -> float:
        return self._h.task_estimate(task_id)

    def utilization(self, task_id: int) -> float:
        return self._h.utilization(task_id)

    def note_job_complete(self, task_id: int) -> None:
        self._h.note_job_complete(task_id)
        self._states[task_id].completed_jobs += 1

    def deadline_shares(self, task_id: int) -> list[float]:
        return self._h.deadline_shares(task_id, len(self._states[task_id].task.stages))
