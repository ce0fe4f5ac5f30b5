"""Does the in-process NVML clock sampler perturb the schedule? C2 at a fixed
rate near the knee, N windows each with the sampler running and not running
(interleaved); counts windows with HP misses / LP loss and the executor's
worst loop gap. python tools/sampler_ab.py --rate 1500 --windows 8"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2504_08795_b200.gpu import GpuConfig, Policy  # noqa: E402
from paper_2504_08795_b200.runtime import DarisRuntime  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rate", type=float, default=1500.0)
    ap.add_argument("--windows", type=int, default=8)
    ap.add_argument("--seconds", type=float, default=1.3)
    args = ap.parse_args()
    gpu = GpuConfig(148, 4, 2, 2.0, Policy.MPS_STR)
    rt = DarisRuntime(bench.c2_tasks(100.0, list(range(8))), gpu, slots=3, seed=0)
    rt.capture_all()
    rt.afet = rt.calibrate_full_load(0.2)
    rt.set_rate(args.rate)
    stats = {"sampler": [], "none": []}
    for w in range(args.windows):
        for mode in ("sampler", "none"):
            if mode == "sampler":
                with bench.ClockSampler(0):
                    res = rt.run(args.seconds, args.seconds * 0.1, full_load=rt.afet)
            else:
                res = rt.run(args.seconds, args.seconds * 0.1, full_load=rt.afet)
            rep = res.report
            stats[mode].append((rep.missed_hp, bench.lp_loss(rep), res.stats["loop_gap_max"], res.stats["stalls"]))
    for mode, rows in stats.items():
        bad = sum(1 for r in rows if r[0] > 0 or r[1] >= 0.02)
        print(f"{mode:8s} windows={len(rows)} failing={bad} hp_miss={[r[0] for r in rows]} "
              f"loop_gap_max_us={[round(r[2] * 1e6) for r in rows]} stalls={[r[3] for r in rows]}")
    rt.close()


if __name__ == "__main__":
    main()
