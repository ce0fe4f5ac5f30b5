"""Fixed-rate C2 runs with long timed windows: per 0.5-s window, HP misses, LP
loss and GPU-wide stalls (executor stall log). Shows how the knee depends on
the window protocol (bench.py) and on the pool's periodic GPU pauses.

python tools/window_sweep.py --rates 400,800,1200,1500 [--seconds 10] [--step 0.5]
"""

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2504_08795_b200.gpu import GpuConfig, Policy  # noqa: E402
from paper_2504_08795_b200.runtime import DarisRuntime, window_ok  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rates", default="400,800,1200,1500")
    ap.add_argument("--seconds", type=float, default=10.0)
    ap.add_argument("--step", type=float, default=0.5)
    ap.add_argument("--warmup", type=float, default=1.0)
    args = ap.parse_args()
    gpu = GpuConfig(148, 4, 2, 2.0, Policy.MPS_STR)
    rt = DarisRuntime(bench.c2_tasks(100.0, list(range(8))), gpu, slots=3, seed=0)
    rt.capture_all()
    rt.afet = rt.calibrate_full_load(0.3)
    n = int(round(args.seconds / args.step))
    for r in [float(x) for x in args.rates.split(",")]:
        rt.set_rate(r)
        res = rt.run(duration=args.warmup + args.seconds, warmup=args.warmup, full_load=rt.afet)
        ws = res.windows(args.warmup, args.step, n)
        bad = [k for k, w in enumerate(ws) if not window_ok(w)]
        print(json.dumps({"rate_per_task": r, "inf_per_s": round(sum(w["completed_images"] for w in ws) / args.seconds, 1),
                          "windows": n, "windows_failed": len(bad),
                          "failed_with_stall": sum(1 for k in bad if ws[k]["stalls"] > 0),
                          "stalls": len(res.stalls), "stall_ms": [round(b * 1e3, 2) for _, b in res.stalls][:20],
                          "miss_hp": [ws[k]["missed_hp"] for k in bad],
                          "lp_loss": [round(ws[k]["lp_loss"], 4) for k in bad],
                          "p99_hp_ms": round(res.report.response_hp.p99 * 1e3, 3)}), flush=True)
    rt.close()


if __name__ == "__main__":
    main()
