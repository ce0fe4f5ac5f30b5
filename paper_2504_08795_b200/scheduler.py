"""Scheduling core of the drop-in API: placement, admission, migration,
priority dispatch and stage completion, executed by the native dispatcher.

Keeps the reference's public names (stagesim/scheduler.py:26-324):
``AblationFlags``, ``SchedulerMode``, ``PriorityKey``, ``ContextUtilization``,
``AdmissionDecision``, ``Placement`` and ``Scheduler`` with
populate_contexts / context_utilization(s) / admission_test / predicted_finish /
admit_or_migrate / priority_key / dispatch / complete_stage.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Sequence

from . import _core
from .model import Job, Priority, StageJob, StageState, TaskState
from .timing import TimingTracker


@dataclass(frozen=True)
class ContextUtilization:
    hp_total: float
    lp_total: float
    lp_active: float
    hp_active: float

    @property
    def total(self) -> float:
        return self.hp_total + self.lp_total

    @property
    def active(self) -> float:
        return self.hp_total + self.lp_active


@dataclass(frozen=True)
class AblationFlags:
    no_staging: bool = False
    no_last: bool = False
    no_prior: bool = False
    no_fixed: bool = False

    @classmethod
    def from_names(cls, names: Iterable[str]) -> "AblationFlags":
        known = {"no_staging", "no_last", "no_prior", "no_fixed"}
        cleaned = {n.replace("-", "_") for n in names}
        bad = cleaned - known
        if bad:
            raise ValueError(f"unknown ablation flags: {sorted(bad)}")
        return cls(**{n: True for n in cleaned})


@dataclass(frozen=True)
class SchedulerMode:
    hpa_enabled: bool = False


@dataclass(frozen=True, order=True)
class PriorityKey:
    level: int
    edf_key: float
    task_id: int
    job_id: int


@dataclass
class AdmissionDecision:
    time: float
    job_id: int
    task_id: int
    priority: Priority
    context: int
    active_util: float
    job_util: float
    limit: float
    admitted: bool

    @classmethod
    def from_native(cls, a: _core.AuditC) -> "AdmissionDecision":
        return cls(a.time, a.job, a.task, Priority.HP if a.priority == 0 else Priority.LP, a.context,
                   a.active_util, a.job_util, a.limit, bool(a.admitted))


@dataclass
class Placement:
    context: int | None
    migrated_from: int | None = None
    audits: list[AdmissionDecision] = field(default_factory=list)

    @property
    def rejected(self) -> bool:
        return self.context is None


class Scheduler:
    """Object-level view over one native dispatcher handle.

    Jobs are created natively at release (``admit_or_migrate``); the Job /
    StageJob objects passed in are views that this class keeps in sync.
    """

    def __init__(self, tracker: TimingTracker, contexts: Sequence, config, *,
                 flags: AblationFlags = AblationFlags(), mode: SchedulerMode = SchedulerMode(),
                 placement_order: str = "descending_util", edf_on_job_deadline: bool = False,
                 stage_migration: bool = False):
        from .model import spec_to_dict
        if placement_order not in ("descending_util", "insertion"):
            raise ValueError(f"unknown placement order {placement_order!r}")
        self.tracker = tracker
        self.contexts = list(contexts)
        self.config = config
        self.flags = flags
        self.mode = mode
        self.placement_order = placement_order
        self.edf_on_job_deadline = edf_on_job_deadline
        states = list(tracker._states.values())
        ws = states[0].window_size if states else 5
        self._h = _core.Handle(config.native(), [spec_to_dict(st.task) for st in states],
                               _core.options_struct(window_size=ws, no_last=flags.no_last,
                                                    no_prior=flags.no_prior, no_fixed=flags.no_fixed,
                                                    hpa=mode.hpa_enabled, placement_order=placement_order,
                                                    edf_on_job_deadline=edf_on_job_deadline,
                                                    stage_migration=stage_migration))
        self._h.set_full_load([tracker._states[i].full_load_time for i in self._h.task_ids])
        tracker._h = self._h          # one source of truth
        self._jobs: dict[int, Job] = {}

    # --- placement ---
    def populate_contexts(self, states: Sequence[TaskState]) -> None:
        self._h.populate()
        for st in states:
            st.current_context = self._h.home_context(st.task.id)

    def context_utilization(self, ctx_id: int) -> ContextUtilization:
        l = self._h.ledger(ctx_id)
        return ContextUtilization(l.hp_total, l.lp_total, l.lp_active, l.hp_active)

    def context_utilizations(self) -> list[ContextUtilization]:
        return [self.context_utilization(c.id) for c in self.contexts]

    # --- admission ---
    def admission_test(self, job: Job, ctx_id: int, t: float) -> AdmissionDecision:
        return AdmissionDecision.from_native(self._h.admission_test(job.task_id, job.job_id, ctx_id, t))

    def predicted_finish(self, job: Job, ctx_id: int, t: float) -> float:
        return self._h.predicted_finish(job.task_id, ctx_id, t)

    def admit_or_migrate(self, job: Job, t: float) -> Placement:
        n_before = len(self._h.audits())
        work = [s.remaining_work for s in job.stage_jobs] or None
        pl = self._h.release(job.task_id, t, job.job_id, work)
        audits = [AdmissionDecision.from_native(a) for a in self._h.audits()[n_before:]]
        st = self.tracker.state(job.task_id)
        if pl.context == 0:
            return Placement(None, audits=audits)
        job.placement = pl.context
        st.active_jobs += 1
        st.current_context = self._h.home_context(job.task_id)
        if job.stage_jobs:
            job.stage_jobs[0].state = StageState.READY
        self._jobs[job.job_id] = job
        return Placement(pl.context, migrated_from=pl.migrated_from or None, audits=audits)

    # --- dispatch ---
    def priority_key(self, stage: StageJob) -> PriorityKey:
        hp = self.tracker.state(stage.task_id).task.priority is Priority.HP
        is_last = stage.is_last and not self.flags.no_last
        late = stage.predecessor_missed and not self.flags.no_prior
        level = 0 if self.flags.no_fixed else 4 * (not hp) + 2 * (not is_last) + (not late)
        edf = stage.job.absolute_deadline if self.edf_on_job_deadline else stage.virtual_abs_deadline
        return PriorityKey(level, edf, stage.task_id, stage.job_id)

    def dispatch(self, ctx_id: int, t: float, stream: int = 0) -> StageJob | None:
        ref = self._h.dispatch(ctx_id, stream, t)
        if ref is None:
            return None
        job = self._jobs[ref.job]
        st = job.stage_jobs[ref.stage]
        st.state = StageState.RUNNING
        st.started_at, st.context, st.stream = ref.started_at, ref.context, ref.stream
        st.virtual_abs_deadline = ref.virtual_deadline
        return st

    def complete_stage(self, stage: StageJob, t: float) -> tuple[bool, bool]:
        done, missed = self._h.complete(stage.job_id, stage.stage_index, t)
        stage.state = StageState.DONE
        job = stage.job
        if not done:
            nxt = job.stage_jobs[stage.stage_index + 1]
            nxt.predecessor_missed = t > stage.virtual_abs_deadline
            nxt.state = StageState.READY
            return False, False
        job.completion_time = t
        st = self.tracker.state(stage.task_id)
        st.active_jobs -= 1
        st.completed_jobs += 1
        self._jobs.pop(job.job_id, None)
        return True, missed
