"""Scheduling core of the drop-in API: placement, admission, migration,
priority dispatch and stage completion, decided by the native decision kernels.

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
    """Object-level scheduler over Python-owned state (scheduler.py:102-324).

    State lives where the reference keeps it — ``ctx_tasks`` / ``ready`` /
    ``live_jobs`` per context, ``TaskState.current_context`` / ``active_jobs``,
    the tracker's windows — so code that drives or inspects those objects
    directly works unchanged. Each decision (ledgers, admission, Algorithm 1,
    predicted finish, priority level, dispatch pick) is one native decision
    kernel (csrc/core/decide.cpp) — the same functions the stateful dispatcher
    behind the engine and the GPU executor runs, so both views decide alike
    (tests/test_object_api.py drives them in lockstep).

    ``stage_migration`` (extension, off by default as the reference has none):
    a successor stage is queued in its task's current home context instead of
    the job's placement, so a task migrated at release pulls its in-flight job
    along (the native option of the same name, dispatcher.cpp ``complete``).
    """

    def __init__(self, tracker: TimingTracker, contexts: Sequence, config, *,
                 flags: AblationFlags = AblationFlags(), mode: SchedulerMode = SchedulerMode(),
                 placement_order: str = "descending_util", edf_on_job_deadline: bool = False,
                 stage_migration: bool = False):
        if placement_order not in ("descending_util", "insertion"):
            raise ValueError(f"unknown placement order {placement_order!r}")
        self.tracker = tracker
        self.contexts = list(contexts)
        self.config = config
        self.flags = flags
        self.mode = mode
        self.placement_order = placement_order
        self.edf_on_job_deadline = edf_on_job_deadline
        self.stage_migration = stage_migration
        ids = [c.id for c in self.contexts]
        self.ctx_tasks: dict[int, list[int]] = {c: [] for c in ids}
        self.ready: dict[int, list[StageJob]] = {c: [] for c in ids}
        self.live_jobs: dict[int, list[Job]] = {c: [] for c in ids}

    def _is_hp(self, task_id: int) -> bool:
        return self.tracker.state(task_id).task.priority is Priority.HP

    # --- placement (Algorithm 1) ---
    def populate_contexts(self, states: Sequence[TaskState]) -> None:
        """HP tasks first, then LP; within a class heaviest utilization first
        (or insertion order); each to the context with the least total so far."""
        states = list(states)
        utils = [self.tracker.utilization(st.task.id) for st in states]
        homes, order = _core.ev_placement(utils, [st.task.priority is Priority.HP for st in states],
                                          [st.task.id for st in states], len(self.contexts),
                                          self.placement_order == "insertion")
        for i in order:
            ctx_id = self.contexts[homes[i] - 1].id
            states[i].current_context = ctx_id
            self.ctx_tasks[ctx_id].append(states[i].task.id)

    # --- Eq. 4-7 ledgers ---
    def context_utilization(self, ctx_id: int) -> ContextUtilization:
        entries = [(self.tracker.utilization(tid), self._is_hp(tid), self.tracker.state(tid).active_jobs)
                   for tid in self.ctx_tasks[ctx_id]]
        l = _core.ev_ledger(entries)
        ledger = ContextUtilization(l.hp_total, l.lp_total, l.lp_active, l.hp_active)
        self.contexts[ctx_id - 1].util_ledger = ledger
        return ledger

    def context_utilizations(self) -> list[ContextUtilization]:
        return [self.context_utilization(c.id) for c in self.contexts]

    # --- Eq. 10-11 admission ---
    def admission_test(self, job: Job, ctx_id: int, t: float) -> AdmissionDecision:
        ledger = self.context_utilization(ctx_id)
        u = self.tracker.utilization(job.task_id)
        hp = self._is_hp(job.task_id)
        lc = _core.LedgerC(ledger.hp_total, ledger.lp_total, ledger.lp_active, ledger.hp_active)
        active, limit, ok = _core.ev_admission(lc, u, hp, self.config.n_streams)
        return AdmissionDecision(t, job.job_id, job.task_id, Priority.HP if hp else Priority.LP, ctx_id,
                                 active, u, limit, ok)

    def predicted_finish(self, job: Job, ctx_id: int, t: float) -> float:
        """t + (estimated work of live jobs' unfinished stages here) / N_s + the job's own estimate."""
        backlog = [self.tracker.stage_estimate(live.task_id, sj.stage_index)
                   for live in self.live_jobs[ctx_id] for sj in live.stage_jobs if sj.state is not StageState.DONE]
        return _core.ev_predicted_finish(t, backlog, self.config.n_streams, self.tracker.task_estimate(job.task_id))

    def admit_or_migrate(self, job: Job, t: float) -> Placement:
        """HP: home, tested only under HPA. LP: home if it passes, else the
        passing context with the earliest predicted finish (sticky migration),
        else rejected."""
        st = self.tracker.state(job.task_id)
        home = st.current_context
        audits: list[AdmissionDecision] = []

        def passes(ctx_id: int) -> bool:
            d = self.admission_test(job, ctx_id, t)
            audits.append(d)
            return d.admitted

        if self._is_hp(job.task_id):
            if self.mode.hpa_enabled and not passes(home):
                return Placement(None, audits=audits)
            self._place(job, home)
            return Placement(home, audits=audits)
        if passes(home):
            self._place(job, home)
            return Placement(home, audits=audits)
        fits = [c.id for c in self.contexts if c.id != home and passes(c.id)]
        if not fits:
            return Placement(None, audits=audits)
        finish = [self.predicted_finish(job, c, t) for c in fits]
        target = fits[min(range(len(fits)), key=lambda k: (finish[k], fits[k]))]
        self._migrate_task(job.task_id, home, target)
        self._place(job, target)
        return Placement(target, migrated_from=home, audits=audits)

    def _migrate_task(self, task_id: int, old_ctx: int, new_ctx: int) -> None:
        if self._is_hp(task_id):
            raise AssertionError("high-priority tasks never migrate")
        self.ctx_tasks[old_ctx].remove(task_id)
        self.ctx_tasks[new_ctx].append(task_id)
        self.tracker.state(task_id).current_context = new_ctx

    def _place(self, job: Job, ctx_id: int) -> None:
        job.placement = ctx_id
        self.tracker.state(job.task_id).active_jobs += 1
        self.live_jobs[ctx_id].append(job)
        head = job.stage_jobs[0]
        head.transition(StageState.READY)
        self.ready[ctx_id].append(head)

    # --- dispatch (8 fixed levels + EDF) ---
    def priority_key(self, stage: StageJob) -> PriorityKey:
        f = self.flags
        level = _core.ev_priority_level(self._is_hp(stage.task_id), stage.is_last, stage.predecessor_missed,
                                        f.no_last, f.no_prior, f.no_fixed)
        edf = stage.job.absolute_deadline if self.edf_on_job_deadline else stage.virtual_abs_deadline
        return PriorityKey(level, edf, stage.task_id, stage.job_id)

    def dispatch(self, ctx_id: int, t: float) -> StageJob | None:
        """Remove and return the context's highest-priority ready stage (no preemption)."""
        queue = self.ready[ctx_id]
        if not queue:
            return None
        keys = [self.priority_key(s) for s in queue]
        best = queue.pop(_core.ev_pick([(k.level, k.edf_key, k.task_id, k.job_id) for k in keys]))
        return best

    # --- completion ---
    def complete_stage(self, stage: StageJob, t: float) -> tuple[bool, bool]:
        """Record the observed time; promote the successor (late flag = t past
        this stage's virtual deadline) or retire the job. Returns (job_done, missed)."""
        self.tracker.record_execution(stage.task_id, stage.stage_index, t - stage.started_at)
        stage.transition(StageState.DONE)
        job = stage.job
        if not stage.is_last:
            nxt = job.stage_jobs[stage.stage_index + 1]
            nxt.predecessor_missed = t > stage.virtual_abs_deadline
            nxt.transition(StageState.READY)
            ctx = job.placement
            if self.stage_migration:
                home = self.tracker.state(job.task_id).current_context
                if home != ctx:
                    self.live_jobs[ctx].remove(job)
                    self.live_jobs[home].append(job)
                    job.placement = ctx = home
            self.ready[ctx].append(nxt)
            return False, False
        job.completion_time = t
        self.tracker.state(stage.task_id).active_jobs -= 1
        self.tracker.note_job_complete(stage.task_id)
        self.live_jobs[job.placement].remove(job)
        return True, t > job.absolute_deadline
