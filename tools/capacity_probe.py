"""Closed-loop capacity of concurrent batch-1 ResNet-50 jobs: every
(context, stream) slot loops whole jobs (stage graphs back to back, no
scheduler, no deadlines) for a few seconds — the busy-system AFET measurement
(timing.py:147-218 made real). capacity = slots / mean job time. Shows how
far concurrency of b1 jobs goes before the SMs saturate, per partition shape.

python tools/capacity_probe.py [--shapes 1x1_1,1x8_1,4x2_2,4x4_2] [--seconds 1.0]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2504_08795_b200.gpu import GpuConfig, Policy  # noqa: E402
from paper_2504_08795_b200.runtime import DarisRuntime  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="1x1_1,1x2_1,1x4_1,1x8_1,1x16_1,2x2_1,4x2_2,4x4_2,8x2_4")
    ap.add_argument("--seconds", type=float, default=1.0)
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--partition", default="green", choices=["green", "soft"])
    args = ap.parse_args()
    for shape in args.shapes.split(","):
        a, os_ = shape.split("_")
        nc, ns = (int(x) for x in a.split("x"))
        n = nc * ns
        gpu = GpuConfig(148, nc, ns, float(os_), Policy.MPS_STR)
        tasks = bench.c2_tasks(100.0, list(range(max(n, 1))))
        for t in tasks:
            t.model = args.model
            t.n_stages = None
        rt = DarisRuntime(tasks, gpu, slots=1, seed=0, partition=args.partition)
        rt.capture_all()
        iso = sum(rt.stage_nominal[args.model])
        job = rt.exec.busy_calibrate([rt.net_of(t).n_stages for t in rt.tasks], [t.id for t in rt.tasks],
                                     args.seconds)
        print(json.dumps({"shape": shape, "slots": n, "partition_sms": rt.exec.partitions[0]["sm_count"],
                          "plan_sms": rt.sm_budget, "partition": args.partition,
                          "isolated_ms": round(iso * 1e3, 4), "loaded_job_ms": round(job * 1e3, 4),
                          "capacity_inf_s": round(n / job, 1), "stretch": round(job / iso, 3)}), flush=True)
        rt.close()


if __name__ == "__main__":
    main()
