"""Knee diagnostics for the C2 workload: response-time distribution per class
and the stage timeline of the worst HP jobs (queueing vs execution), at a
list of per-task rates.

python tools/diag_knee.py --rates 350,420,500 --duration 2
"""

import argparse
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2504_08795_b200.gpu import GpuConfig, Policy  # noqa: E402
from paper_2504_08795_b200.model import Priority  # noqa: E402
from paper_2504_08795_b200.runtime import DarisRuntime, TaskDef  # noqa: E402


def pct(v, q):
    v = sorted(v)
    return v[min(len(v) - 1, max(0, int(q * len(v) + 0.999999) - 1))] if v else float("nan")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rates", default="350,420,500")
    ap.add_argument("--duration", type=float, default=2.0)
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--worst", type=int, default=3)
    args = ap.parse_args()
    gpu = GpuConfig(148, 4, 2, 2.0, Policy.MPS_STR)
    tasks = [TaskDef(i + 1, args.model, Priority.HP if i < 4 else Priority.LP, 100.0, 4) for i in range(8)]
    rt = DarisRuntime(tasks, gpu, slots=3)
    rt.capture_all()
    afet = rt.calibrate_full_load(0.3)
    print(f"afet={next(iter(afet.values())) * 1e3:.3f} ms  nominal={[round(x * 1e6, 1) for x in rt.stage_nominal[args.model]]} us")
    for rate in [float(r) for r in args.rates.split(",")]:
        rt.set_rate(rate)
        for _ in range(4):  # re-measure windows hit by a GPU-wide stall (see bench.run_clean)
            res = rt.run(duration=args.duration, warmup=0.1 * args.duration, full_load=afet)
            if res.stats["stalls"] == 0:
                break
        rep, st = res.report, res.stats
        rel = {}
        for r in res.records:
            if r[1] == "release":
                rel[r[3]] = r[0]
        stages = defaultdict(list)
        for t in res.trace:
            stages[t[1]].append(t)
        resp = {0: [], 1: []}
        jobs = []
        for job, sts in stages.items():
            sts.sort(key=lambda x: x[2])
            task = sts[0][0]
            hp = 0 if task <= 4 else 1
            if len(sts) == 4 and job in rel:
                r = sts[-1][7] - rel[job]
                resp[hp].append(r)
                jobs.append((r, job, task, rel[job], sts))
        print(f"\nrate={rate:.0f}/task jps={rep.jps:.0f} miss_hp={rep.missed_hp} dmr_lp={rep.dmr_lp:.4f} "
              f"rej_lp={rep.rejected_lp} stalls={st['stalls']} loop_gap_max={st['loop_gap_max'] * 1e6:.0f}us "
              f"release_lag_max={st['release_lag_max'] * 1e6:.0f}us polls={st['polls']}")
        for hp in (0, 1):
            v = resp[hp]
            print(f"  {'HP' if hp == 0 else 'LP'} n={len(v)} p50={pct(v, .5) * 1e3:.3f} p90={pct(v, .9) * 1e3:.3f} "
                  f"p99={pct(v, .99) * 1e3:.3f} max={max(v) * 1e3 if v else 0:.3f} ms  period={1e3 / rate:.3f} ms")
        # stage execution-time distribution (dispatch -> observed completion)
        for s in range(4):
            d = [t[7] - t[6] for t in res.trace if t[2] == s]
            print(f"  stage{s} exec p50={pct(d, .5) * 1e6:.0f} p99={pct(d, .99) * 1e6:.0f} max={max(d) * 1e6:.0f} us")
        for r, job, task, t_rel, sts in sorted(jobs, key=lambda x: -x[0])[:args.worst]:
            parts = []
            prev = t_rel
            for t in sts:
                parts.append(f"s{t[2]}@c{t[3]}.{t[4]} q={(t[6] - prev) * 1e6:.0f} x={(t[7] - t[6]) * 1e6:.0f}")
                prev = t[7]
            print(f"  worst job {job} task {task} resp={r * 1e3:.3f} ms: " + " | ".join(parts))
    rt.close()


if __name__ == "__main__":
    main()
