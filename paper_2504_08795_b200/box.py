"""Box-level layer: tasks shard across the GPUs of one node, one independent
DARIS instance per GPU. No collective on the inference path.

``place_tasks`` applies the reference's Algorithm 1 rule at GPU granularity
(scheduler.py:131-153): HP tasks first, then LP, each class in descending
utilization (ties by id), each task onto the GPU with the lowest total
utilization so far (ties to the lowest GPU index).
"""

from __future__ import annotations

from dataclasses import dataclass
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
