"""A/B of an executor environment switch read at every run (default: stage
completion by event polling vs host-mapped flags, DARIS_EXEC_FLAGS=0/1): C2 at
fixed per-task rates around the knee, interleaved windows per value; prints
completed inferences/s, HP misses, LP loss, p99 HP response and poll count.
python tools/flags_ab.py --rates 1500 1650 1800 --windows 4 [--env DARIS_STAGE_INPUT --values 0 1] [--e2e]"""

from __future__ import annotations

import argparse
import os
import statistics as S
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2504_08795_b200.gpu import GpuConfig, Policy  # noqa: E402
from paper_2504_08795_b200.runtime import DarisRuntime  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rates", type=float, nargs="+", default=[1500.0, 1650.0, 1800.0])
    ap.add_argument("--windows", type=int, default=4)
    ap.add_argument("--seconds", type=float, default=1.0)
    ap.add_argument("--env", default="DARIS_EXEC_FLAGS")
    ap.add_argument("--values", nargs="+", default=["0", "1"])
    ap.add_argument("--e2e", action="store_true", help="pinned-host input pools (H2D + D2H every job)")
    args = ap.parse_args()
    gpu = GpuConfig(148, 4, 2, 2.0, Policy.MPS_STR)
    rt = DarisRuntime(bench.c2_tasks(100.0, list(range(8))), gpu, slots=3, seed=0)
    rt.capture_all()
    rt.afet = rt.calibrate_full_load(0.2)
    if args.e2e:
        rt.use_host_io(True)
    for rate in args.rates:
        rt.set_rate(rate)
        rows = {v: [] for v in args.values}
        for _ in range(args.windows):
            for mode in args.values:
                os.environ[args.env] = mode
                res = rt.run(args.seconds, args.seconds * 0.1, full_load=rt.afet)
                rep = res.report
                rows[mode].append((rep.jps, rep.missed_hp, bench.lp_loss(rep), rep.response_hp.p99 * 1e3,
                                   res.stats["polls"], res.stats["stalls"]))
        for mode, r in rows.items():
            bad = sum(1 for x in r if x[1] > 0 or x[2] >= 0.02)
            print(f"rate={rate:.0f} {args.env}={mode} jps={S.median(x[0] for x in r):.0f} failing={bad}/{len(r)} "
                  f"hp_miss={[x[1] for x in r]} lp_loss={[round(x[2], 3) for x in r]} "
                  f"p99_ms={[round(x[3], 3) for x in r]} polls={S.median(x[4] for x in r):.0f} "
                  f"stalls={[x[5] for x in r]}", flush=True)
    os.environ.pop(args.env, None)
    rt.close()


if __name__ == "__main__":
    main()
