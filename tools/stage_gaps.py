"""Where a job's time goes under load: for every completed job of a C2 run,
GPU execution of each stage (CUDA events around the stage graph) vs the gaps
between stages (stage s done on the GPU -> host observes it -> dispatcher ->
graph launch -> stage s+1 starts on the GPU), from the executor trace with
DARIS_GPU_TIMING=1.

DARIS_GPU_TIMING=1 python tools/stage_gaps.py --rate 1500 --duration 1.0
"""

from __future__ import annotations

import argparse
import os
import statistics as S
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("DARIS_GPU_TIMING", "1")

import bench  # noqa: E402
from paper_2504_08795_b200.gpu import GpuConfig, Policy  # noqa: E402
from paper_2504_08795_b200.runtime import DarisRuntime  # noqa: E402


def pct(xs, q):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(q * len(xs)))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rates", default="800,1500")
    ap.add_argument("--duration", type=float, default=1.0)
    args = ap.parse_args()
    gpu = GpuConfig(148, 4, 2, 2.0, Policy.MPS_STR)
    rt = DarisRuntime(bench.c2_tasks(100.0, list(range(8))), gpu, slots=3, seed=0)
    rt.capture_all()
    rt.afet = rt.calibrate_full_load(0.2)
    iso = rt.stage_nominal["resnet50"]
    print("isolated stage graphs (us):", [round(x * 1e6, 1) for x in iso], "sum", round(sum(iso) * 1e6, 1))
    for rate in (float(r) for r in args.rates.split(",")):
        rt.set_rate(rate)
        res = rt.run(args.duration, args.duration * 0.1, full_load=rt.afet)
        per_job = defaultdict(dict)
        gpu_times = rt.exec.trace_gpu()  # aligned with res.trace
        for t, g in zip(res.trace, gpu_times):
            task, job, stage = t[0], t[1], t[2]
            per_job[(task, job)][stage] = (t[6], t[7]) + tuple(g)   # host start, host end, gpu start, gpu end
        execs = defaultdict(list)
        gaps = defaultdict(list)
        host_obs = []
        for stages in per_job.values():
            if len(stages) != 4 or not all(stages[s][2] > 0 for s in range(4)):  # (NaN: no timing)
                continue
            for s in range(4):
                execs[s].append(stages[s][3] - stages[s][2])
                host_obs.append(stages[s][1] - stages[s][3])  # host saw completion after the GPU end event
                if s < 3:
                    gaps[s].append(stages[s + 1][2] - stages[s][3])
        rep = res.report
        print(f"rate {rate:.0f}/task: jps {rep.jps:.0f}, HP p99 {rep.response_hp.p99 * 1e3:.3f} ms, jobs {len(per_job)}")
        for s in range(4):
            e = execs[s]
            if e:
                print(f"  stage {s}: GPU exec p50 {S.median(e) * 1e6:6.1f} p99 {pct(e, .99) * 1e6:6.1f} us", end="")
            if s < 3 and gaps[s]:
                g = gaps[s]
                print(f" | gap to next stage p50 {S.median(g) * 1e6:5.1f} p99 {pct(g, .99) * 1e6:5.1f} us", end="")
            print()
        if host_obs:
            print(f"  host observes a stage end after the GPU: p50 {S.median(host_obs) * 1e6:.1f} "
                  f"p99 {pct(host_obs, .99) * 1e6:.1f} us")
    rt.close()


if __name__ == "__main__":
    main()
