"""Look for multi-millisecond GPU stalls in a DARIS run: stage executions
(dispatch -> observed completion) above a threshold, with their start times,
per partition mode. python tools/probe_stall.py --modes green,soft --rate 800"""

import argparse
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2504_08795_b200.gpu import GpuConfig, Policy  # noqa: E402
from paper_2504_08795_b200.model import Priority  # noqa: E402
from paper_2504_08795_b200.runtime import DarisRuntime, TaskDef  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", default="green,soft")
    ap.add_argument("--rate", type=float, default=800)
    ap.add_argument("--duration", type=float, default=3.0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--thresh", type=float, default=0.001)
    args = ap.parse_args()
    gpu = GpuConfig(148, 4, 2, 2.0, Policy.MPS_STR)
    for mode in args.modes.split(","):
        tasks = [TaskDef(i + 1, "resnet50", Priority.HP if i < 4 else Priority.LP, args.rate, 4) for i in range(8)]
        rt = DarisRuntime(tasks, gpu, slots=3, partition=mode)
        rt.capture_all()
        afet = rt.calibrate_full_load(0.3)
        for rep in range(args.reps):
            res = rt.run(duration=args.duration, warmup=0.1, full_load=afet)
            long = [t for t in res.trace if t[7] - t[6] > args.thresh]
            starts = sorted({round(t[6], 3) for t in long})
            gt = rt.exec.trace_gpu()
            for i, t in enumerate(res.trace):
                if t[7] - t[6] > args.thresh and gt:
                    g0, g1 = gt[i]
                    print(f"   long: task {t[0]} job {t[1]} st {t[2]} c{t[3]}.{t[4]} host [{t[6] * 1e3:.3f}, "
                          f"{t[7] * 1e3:.3f}] gpu [{g0 * 1e3:.3f}, {g1 * 1e3:.3f}] ms")
                    # what else ran on the GPU around it
                    for j, u in enumerate(res.trace):
                        if j != i and gt[j][1] > g0 - 2e-4 and gt[j][0] < g1:
                            print(f"      other: task {u[0]} st {u[2]} c{u[3]}.{u[4]} gpu [{gt[j][0] * 1e3:.3f}, "
                                  f"{gt[j][1] * 1e3:.3f}] host [{u[6] * 1e3:.3f}, {u[7] * 1e3:.3f}]")
                    break
            r = res.report
            print(f"{mode} rep{rep} env_nohiprio={bool(os.environ.get('DARIS_NO_HIPRIO'))} jps={r.jps:.0f} "
                  f"miss_hp={r.missed_hp} rej_lp={r.rejected_lp} stages={len(res.trace)} long={len(long)} "
                  f"max={max(t[7] - t[6] for t in res.trace) * 1e3:.2f}ms at t={starts[:12]} "
                  f"gap={res.stats['loop_gap_max'] * 1e6:.0f}us", flush=True)
        rt.close()
        del rt


if __name__ == "__main__":
    main()
