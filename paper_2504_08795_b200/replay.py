"""Independent checks over an event log (stagesim/replay.py:25-216 names).

Everything is recomputed from the raw records — whether they came from the
native sim backend, the trace-replay backend or a real GPU run — so the same
audits apply to all three. Records may be LogRecord tuples or dicts.
"""

from __future__ import annotations

import math
from typing import Iterable, Mapping, Sequence

from .model import Priority, TaskSpec

FIELDS = ("time", "kind", "task", "job", "stage", "context", "stream", "rate")


def _row(rec) -> tuple:
    return tuple(rec[f] for f in FIELDS) if isinstance(rec, Mapping) else tuple(rec)


def _stats(xs: list[float]) -> dict:
    if not xs:
        return {"mean": 0.0, "min": 0.0, "max": 0.0, "p95": 0.0, "count": 0}
    o = sorted(xs)
    return {"mean": sum(o) / len(o), "min": o[0], "max": o[-1], "p95": o[math.ceil(0.95 * len(o)) - 1],
            "count": len(o)}


def replay_metrics(records: Iterable, tasks: Sequence[TaskSpec], *, duration: float, warmup_end: float,
                   batch_sizes: Mapping[int, int] | None = None) -> dict:
    """Headline metrics rebuilt from the log alone (no accumulator state)."""
    batch_sizes = batch_sizes or {}
    spec = {t.id: t for t in tasks}
    zero = lambda: {Priority.HP: 0, Priority.LP: 0}  # noqa: E731
    rel, acc, rej, cmp_, miss = zero(), zero(), zero(), zero(), zero()
    resp = {Priority.HP: [], Priority.LP: []}
    released_at: dict[int, float] = {}
    counted: dict[int, bool] = {}
    inputs = 0
    for rec in records:
        t, kind, task, job = _row(rec)[:4]
        if kind == "release":
            released_at[job] = t
            counted[job] = t >= warmup_end
            if counted[job]:
                rel[spec[task].priority] += 1
        elif kind in ("admit", "reject"):
            if counted[job]:
                (acc if kind == "admit" else rej)[spec[task].priority] += 1
        elif kind == "job_complete" and counted[job]:
            s = spec[task]
            cmp_[s.priority] += 1
            inputs += batch_sizes.get(task, 1)
            resp[s.priority].append(t - released_at[job])
            if t > released_at[job] + s.deadline:
                miss[s.priority] += 1
    window = duration - warmup_end
    ratio = lambda n, d: n / d if d else 0.0  # noqa: E731
    out = {"jps": inputs / window if window > 0 else 0.0,
           "dmr_hp": ratio(miss[Priority.HP], acc[Priority.HP]), "dmr_lp": ratio(miss[Priority.LP], acc[Priority.LP]),
           "response_hp": _stats(resp[Priority.HP]), "response_lp": _stats(resp[Priority.LP])}
    for name, d in (("released", rel), ("accepted", acc), ("rejected", rej), ("completed", cmp_), ("missed", miss)):
        out[f"{name}_hp"] = d[Priority.HP]
        out[f"{name}_lp"] = d[Priority.LP]
    return out


def compare_with_report(replayed: dict, report) -> list[str]:
    actual = report.to_dict()
    return [f"{k}: log replay {v!r} != accumulator {actual[k]!r}" for k, v in replayed.items() if actual[k] != v]


def check_event_order(records: Iterable, duration: float) -> None:
    """Monotone time, inside the horizon, releases before completions at one instant."""
    last = -math.inf
    completion_at = None
    for rec in records:
        t, kind = _row(rec)[:2]
        if t < last:
            raise AssertionError(f"event log goes backwards at t={t}")
        if t > duration:
            raise AssertionError(f"event at t={t} beyond the horizon {duration}")
        if t > last:
            completion_at = None
        last = t
        if kind in ("stage_complete", "job_complete"):
            completion_at = t
        elif kind in ("release", "admit", "reject") and completion_at == t:
            raise AssertionError(f"release after completion at t={t}")


def check_work_conservation(records: Iterable, tasks: Sequence[TaskSpec], *, n_contexts: int,
                            n_streams: int) -> None:
    """After each instant, no context idles a stream while it holds ready stages."""
    n_stages = {t.id: len(t.stages) for t in tasks}
    where: dict[int, int] = {}
    ready = {k: set() for k in range(1, n_contexts + 1)}
    busy = {k: set() for k in range(1, n_contexts + 1)}

    def settle(at):
        for k in ready:
            if ready[k] and len(busy[k]) < n_streams:
                raise AssertionError(f"context {k} idles {n_streams - len(busy[k])} stream(s) while "
                                     f"{len(ready[k])} stage(s) are ready at t={at}")

    now = None
    for rec in records:
        t, kind, task, job, stage, ctx, stream, _ = _row(rec)
        if now is not None and t != now:
            settle(now)
        now = t
        if kind == "admit":
            where[job] = ctx
            ready[ctx].add((job, 0))
        elif kind == "stage_start":
            ready[ctx].discard((job, stage))
            busy[ctx].add(stream)
        elif kind == "stage_complete":
            busy[ctx].discard(stream)
            if stage + 1 < n_stages[task]:
                ready[where[job]].add((job, stage + 1))
    if now is not None:
        settle(now)


def check_admission_audit(result) -> None:
    """Audit records are self-consistent and every started LP job was admitted."""
    for d in result.admissions:
        if (d.active_util + d.job_util < d.limit) != d.admitted:
            raise AssertionError(f"admission record for job {d.job_id} in context {d.context} is inconsistent")
    admitted = {d.job_id for d in result.admissions if d.admitted}
    lp = {t.id for t in result.effective_tasks if t.priority is Priority.LP}
    for rec in result.records:
        t, kind, task, job = _row(rec)[:4]
        if kind == "stage_start" and task in lp and job not in admitted:
            raise AssertionError(f"low-priority job {job} started at t={t} without a passing admission test")
