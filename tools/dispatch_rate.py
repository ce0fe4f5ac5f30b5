"""Dispatcher cost, CPU only ("the dispatcher is CPU- and
latency-bound: report µs/decision"): the same task set through the unmodified
reference (stagesim, from /root/reference) and through this package's native
engine in rate-model mode, one core each; event logs must be identical, then
wall time per scheduling decision (release/admit/stage_start/stage_complete/...)
and stage dispatches per second. Configs: C1 (2 ResNet-18, 2x2 OS 1) and C2
(8 ResNet-50, 4x2 OS 2) at the given per-task rate.
python tools/dispatch_rate.py --seconds 2 --rate 1000"""

from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF = Path("/root/reference/pkg/src")

import paper_2504_08795_b200 as ours  # noqa: E402


def specs(mod, cfg, rate):
    return [mod.TaskSpec.periodic(t.id, 1.0 / rate, mod.Priority.HP if t.priority.value == "hp" else mod.Priority.LP,
                                  tuple(mod.StageProfile(p.nominal_time, p.width) for p in t.stages))
            for t in cfg.tasks]


def timed(mod, cfg, rate, seconds):
    g = cfg.gpu
    sim = mod.Simulation(specs(mod, cfg, rate), mod.GpuConfig(g.total_sms, g.n_contexts, g.n_streams,
                                                              g.oversubscription, mod.Policy.MPS_STR),
                         seed=0, duration=seconds)
    t0 = time.perf_counter()
    res = sim.run()
    return time.perf_counter() - t0, res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=2.0, help="simulated seconds")
    ap.add_argument("--rate", type=float, default=1000.0, help="releases per second per task")
    args = ap.parse_args()
    sys.path.insert(0, str(REF))
    import stagesim as ref
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except OSError:
        pass
    print(f"one core, {args.seconds:g} simulated s at {args.rate:g} releases/s/task; cpu_count={os.cpu_count()}")
    for name, preset in (("C1", "c1_resnet18_b200"), ("C2", "c2_resnet50_b200")):
        cfg = ours.scenario_from_dict({"preset": name.lower() + "_b200", "workload": {"preset": preset}})
        tr, rr = timed(ref, cfg, args.rate, args.seconds)
        tn, rn = timed(ours, cfg, args.rate, args.seconds)
        same = [tuple(r) for r in rr.records] == [tuple(r) for r in rn.records]
        n = len(rr.records)
        starts = sum(1 for r in rr.records if r[1] == "stage_start")
        print(f"{name}: {n} log records ({starts} stage dispatches), logs identical={same}\n"
              f"  reference stagesim : {tr:8.3f} s  {tr / n * 1e6:8.2f} us/decision  {starts / tr:12.0f} dispatches/s\n"
              f"  native engine      : {tn:8.3f} s  {tn / n * 1e6:8.2f} us/decision  {starts / tn:12.0f} dispatches/s"
              f"  ({tr / tn:.0f}x)", flush=True)


if __name__ == "__main__":
    main()
