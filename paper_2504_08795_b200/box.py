"""Box-level layer: tasks shard across the GPUs of one node, one independent
DARIS instance per GPU. No collective on the inference path.

``place_tasks`` applies the reference's Algorithm 1 rule at GPU granularity
(scheduler.py:131-153): HP tasks first, then LP, each class in descending
utilization (ties by id), each task onto the GPU with the lowest total
utilization so far (ties to the lowest GPU index).

``BoxAdmission`` is the box-level admission / re-placement layer above the
per-GPU instances: the reference's context-level rules (admission_test,
scheduler.py:179-200; migration by predicted finish, :202-266) lifted one
level, with a GPU's stream slots (N_c x N_s) as its capacity. Its state is the
per-GPU ledgers each rank publishes (``GpuLedger``), exchanged on the control
plane (``sync``: one all_gather of small host objects) — never on the
inference path.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence


@dataclass(frozen=True)
class BoxTask:
    id: int
    hp: bool
    utilization: float   # demand in fractions of one GPU


def place_tasks(tasks: Sequence[BoxTask], n_gpus: int) -> dict[int, int]:
    """task id -> GPU index (0-based)."""
    if n_gpus < 1:
        raise ValueError("n_gpus must be >= 1")
    totals = [0.0] * n_gpus
    out: dict[int, int] = {}
    for want_hp in (True, False):
        group = sorted((t for t in tasks if t.hp == want_hp), key=lambda t: (-t.utilization, t.id))
        for t in group:
            g = min(range(n_gpus), key=lambda k: (totals[k], k))
            out[t.id] = g
            totals[g] += t.utilization
    return out


def local_tasks(assignment: dict[int, int], rank: int) -> list[int]:
    return sorted(tid for tid, g in assignment.items() if g == rank)


def aggregate(values: Sequence[dict]) -> dict:
    """Whole-box metrics from per-GPU reports (host-side, control plane only)."""
    out = {"completed": 0, "released_hp": 0, "released_lp": 0, "accepted_hp": 0, "accepted_lp": 0,
           "missed_hp": 0, "missed_lp": 0}
    for v in values:
        for k in out:
            out[k] += int(v.get(k, 0))
    out["dmr_hp"] = out["missed_hp"] / out["accepted_hp"] if out["accepted_hp"] else 0.0
    out["dmr_lp"] = out["missed_lp"] / out["accepted_lp"] if out["accepted_lp"] else 0.0
    return out


@dataclass
class GpuLedger:
    """One GPU's Eq. 4-7 ledger summed over its contexts (scheduler.py:26-41,
    157-175), plus what predicted finish needs: `backlog` = the remaining
    stage estimates of its live jobs (s), and `slots` = N_c x N_s."""
    gpu: int
    slots: int
    hp_total: float = 0.0
    lp_total: float = 0.0
    lp_active: float = 0.0
    backlog: float = 0.0
    tasks: dict = field(default_factory=dict)   # task id -> (hp, utilization)


class BoxAdmission:
    """Task admission to the box and release-time LP re-placement across GPUs.

    * ``admit_task``: HP tasks go to the lowest-total GPU (Algorithm 1's rule,
      ties to the lowest index) if its HP total plus u stays below its slots;
      LP tasks to the lowest-total GPU whose LP test passes —
      lp_total + u < slots - hp_total (strict, as scheduler.py:189-199 tests a
      context). A task no GPU can take is rejected at the box (None).
    * ``replace_lp``: an LP task whose GPU rejected its job (that GPU's DARIS
      admission and its own context migration both failed) moves, for its next
      release, to the GPU with the earliest predicted finish
      (t + backlog / slots + MRET_i, scheduler.py:202-213 per GPU) among those
      whose LP test passes with the task's utilisation added; sticky, like the
      reference's task migration (scheduler.py:215-266). The move is not
      zero-delay: the next job's input is staged on the new GPU.
    """

    def __init__(self, n_gpus: int, slots_per_gpu: int):
        if n_gpus < 1 or slots_per_gpu < 1:
            raise ValueError("need >= 1 GPU and >= 1 stream slot per GPU")
        self.ledgers = [GpuLedger(g, slots_per_gpu) for g in range(n_gpus)]
        self.home: dict[int, int] = {}
        self.pending: list[tuple[int, int, int, float]] = []   # moves decided here since the last sync

    def _total(self, g: int) -> float:
        L = self.ledgers[g]
        return L.hp_total + L.lp_total

    def _lp_ok(self, L: GpuLedger, u: float) -> bool:
        return L.lp_total + u < L.slots - L.hp_total

    def admit_task(self, task: BoxTask) -> int | None:
        order = sorted(range(len(self.ledgers)), key=lambda g: (self._total(g), g))
        for g in order:
            L = self.ledgers[g]
            ok = (L.hp_total + task.utilization < L.slots) if task.hp else self._lp_ok(L, task.utilization)
            if ok:
                if task.hp:
                    L.hp_total += task.utilization
                else:
                    L.lp_total += task.utilization
                L.tasks[task.id] = (task.hp, task.utilization)
                self.home[task.id] = g
                return g
            if task.hp:
                break   # HP: the lowest-total GPU only (no test elsewhere), as HP stays home
        return None

    def admit_all(self, tasks: Sequence[BoxTask]) -> dict[int, int | None]:
        """Admit a task set in Algorithm 1's order (HP first, descending u, ties by id)."""
        out = {}
        for want_hp in (True, False):
            for t in sorted((t for t in tasks if t.hp == want_hp), key=lambda t: (-t.utilization, t.id)):
                out[t.id] = self.admit_task(t)
        return out

    def predicted_finish(self, g: int, t: float, mret: float) -> float:
        L = self.ledgers[g]
        return t + L.backlog / L.slots + mret

    def replace_lp(self, task_id: int, t: float, mret: float) -> int | None:
        """Re-home LP task `task_id` after its GPU rejected a job; returns the new
        GPU, or None when no other GPU's LP test passes (the task stays)."""
        src = self.home[task_id]
        hp, u = self.ledgers[src].tasks[task_id]
        if hp:
            raise ValueError("only LP tasks are re-placed (HP tasks stay on their GPU)")
        cands = [g for g in range(len(self.ledgers)) if g != src and self._lp_ok(self.ledgers[g], u)]
        if not cands:
            return None
        dst = min(cands, key=lambda g: (self.predicted_finish(g, t, mret), g))
        self._move(task_id, src, dst, u)
        self.pending.append((task_id, src, dst, u))
        return dst

    def _move(self, task_id: int, src: int, dst: int, u: float) -> None:
        if task_id in self.ledgers[src].tasks:
            del self.ledgers[src].tasks[task_id]
            self.ledgers[src].lp_total -= u
        if task_id not in self.ledgers[dst].tasks:
            self.ledgers[dst].tasks[task_id] = (False, u)
            self.ledgers[dst].lp_total += u
        self.home[task_id] = dst

    def publish(self, g: int, hp_total: float, lp_total: float, lp_active: float, backlog: float,
                tasks: dict | None = None) -> None:
        """A GPU's live ledger (its rank calls this with its dispatcher's numbers)."""
        L = self.ledgers[g]
        L.hp_total, L.lp_total, L.lp_active, L.backlog = hp_total, lp_total, lp_active, backlog
        if tasks is not None:
            L.tasks = dict(tasks)
            for tid in tasks:
                self.home[tid] = g

    def sync(self, rank: int) -> None:
        """Control plane: every rank contributes its own GPU's ledger and the
        re-placements it decided since the last sync; every rank then applies
        the same moves, in rank order, to the same gathered ledgers, so all
        ranks agree on every task's home (torch.distributed all_gather_object,
        gloo or NCCL; host objects of a few hundred bytes)."""
        import torch.distributed as dist
        mine = self.ledgers[rank]
        got: list = [None] * dist.get_world_size()
        dist.all_gather_object(got, ((mine.hp_total, mine.lp_total, mine.lp_active, mine.backlog, mine.tasks),
                                     self.pending))
        for g, ((hp_t, lp_t, lp_a, bl, tasks), _) in enumerate(got):
            self.publish(g, hp_t, lp_t, lp_a, bl, tasks)
        for _, moves in got:
            for task_id, src, dst, u in moves:
                self._move(task_id, src, dst, u)
        self.pending = []
