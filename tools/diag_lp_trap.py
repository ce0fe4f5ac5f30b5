"""LP admission diagnostics for the C2 workload: why LP jobs get rejected near
the knee. For each run: per-window rejections, and for every LP task the
admission audits (active LP load, the job's cached utilisation, the limit
N_s - hp_total) around its first rejection, the GPU-wide pauses before it, and
the MRET samples (dispatch -> observed completion) of its stages just before.

python tools/diag_lp_trap.py --rates 1400,1648 --duration 10 --repeat 2
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rates", default="1400,1648")
    ap.add_argument("--duration", type=float, default=10.0)
    ap.add_argument("--warmup", type=float, default=1.5)
    ap.add_argument("--repeat", type=int, default=2)
    args = ap.parse_args()
    gpu = GpuConfig(148, 4, 2, 2.0, Policy.MPS_STR)
    tasks = [TaskDef(i + 1, "resnet50", Priority.HP if i < 4 else Priority.LP, 100.0, 4) for i in range(8)]
    rt = DarisRuntime(tasks, gpu, slots=3)
    rt.capture_all()
    afet = rt.calibrate_full_load(0.3)
    print(f"afet={ {k: round(v * 1e3, 3) for k, v in afet.items()} } ms", flush=True)
    for rate in [float(r) for r in args.rates.split(",")]:
        for rep_i in range(args.repeat):
            rt.set_rate(rate)
            res = rt.run(duration=args.warmup + args.duration, warmup=args.warmup, full_load=afet)
            ws = res.windows(args.warmup, 0.5, int(args.duration / 0.5))
            rep = res.report
            print(f"\n=== rate={rate:.0f}/task run {rep_i}: jps={rep.jps:.0f} miss_hp={rep.missed_hp} "
                  f"rej_lp={rep.rejected_lp} stalls={[(round(s, 4), round(l * 1e3, 2)) for s, l in res.stalls]}")
            print("  per-window rejected_lp:", [w["rejected_lp"] for w in ws])
            print("  per-window missed_hp:  ", [w["missed_hp"] for w in ws])
            by_task = defaultdict(list)
            for a in res.admissions:
                by_task[a.task_id].append(a)
            samples = defaultdict(list)  # task -> (end, stage, exec, sampled)
            for t in res.trace:
                samples[t[0]].append((t[7], t[2], t[7] - t[6], t[8] if len(t) > 8 else 1))
            for task in sorted(by_task):
                aud = by_task[task]
                pr = "HP" if task <= 4 else "LP"
                us = [a.job_util for a in aud]
                rejected_jobs = sorted({a.job_id for a in aud} - {a.job_id for a in aud if a.admitted})
                print(f"  task {task} {pr}: audits={len(aud)} u_job min/med/max="
                      f"{min(us):.3f}/{sorted(us)[len(us) // 2]:.3f}/{max(us):.3f} rejected_jobs={len(rejected_jobs)}")
                if not rejected_jobs:
                    continue
                j0 = rejected_jobs[0]
                first = [a for a in aud if a.job_id == j0]
                t0 = first[0].time
                for a in first:
                    print(f"    first reject job {j0} t={t0:.5f} ctx={a.context} active={a.active_util:.3f} "
                          f"u_job={a.job_util:.3f} limit={a.limit:.3f}")
                before = [p for p in res.stalls if p[0] < t0]
                if before:
                    s, l = before[-1]
                    print(f"    last pause before: start={s:.5f} len={l * 1e3:.2f} ms, {((t0 - s - l) * 1e3):.2f} ms "
                          f"before the rejection")
                recent = [x for x in samples[task] if x[0] <= t0][-12:]
                print("    last samples (end, stage, exec us, sampled):",
                      [(round(e, 5), s, round(x * 1e6), sm) for e, s, x, sm in recent])
                # does the task ever get admitted again?
                later = [a for a in aud if a.time > t0 and a.admitted]
                print(f"    admitted again later: {len(later)} audits")
    rt.close()


if __name__ == "__main__":
    main()
