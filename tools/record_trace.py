"""Record a real-GPU DARIS run as a trace fixture for P2 parity tests on the CPU.

Workloads (4 contexts x 2 streams, OS=2, zero phasing):
  c2      8 ResNet-50 tasks (4 HP / 4 LP) at --rate jobs/s each
  c3      ResNet-18/50, VGG-16, MobileNetV2, one HP + one LP task each, every task
          at --factor / (its isolated latency) jobs/s (LP release-time migration on)
  c3mig   c3 with stage-level migration (daris_options.stage_migration); --rates gives
          per-task rates (heterogeneous utilisations make LP tasks migrate while
          one of their jobs is still in flight, so its later stages move)
Writes tests/golden/gpu_trace_<tag>.json.gz holding the task set, AFET
baselines, per-stage durations and the executor's event log.
tests/test_reference_trace_replay.py replays it through the oracle and (where
/root/reference exists, and the run did not use stage migration, which the
reference does not have) through the unmodified reference scheduler.

python tools/record_trace.py --config c2 --tag r02_c2 [--rate 1500] [--duration 0.4]
"""

import argparse
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2504_08795_b200.gpu import GpuConfig, Policy  # noqa: E402
from paper_2504_08795_b200.model import Priority  # noqa: E402
from paper_2504_08795_b200.runtime import DarisRuntime, TaskDef  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c3mig"])
    ap.add_argument("--rate", type=float, default=400.0)
    ap.add_argument("--factor", type=float, default=1.0)
    ap.add_argument("--rates", default=None, help="c3/c3mig: comma-separated jobs/s per task id (overrides --factor)")
    ap.add_argument("--duration", type=float, default=0.4)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    gpu = GpuConfig(148, 4, 2, 2.0, Policy.MPS_STR)
    mig = args.config == "c3mig"
    if args.config == "c2":
        tasks = [TaskDef(i + 1, "resnet50", Priority.HP if i < 4 else Priority.LP, args.rate, 4) for i in range(8)]
    else:
        stages = {"resnet18": 3, "resnet50": 4, "vgg16": 4, "mobilenet_v2": 3}
        tasks = []
        for i, m in enumerate(stages):
            tasks.append(TaskDef(2 * i + 1, m, Priority.HP, 100.0, stages[m]))
            tasks.append(TaskDef(2 * i + 2, m, Priority.LP, 100.0, stages[m]))
    rt = DarisRuntime(tasks, gpu, slots=3, phasing="zero", stage_migration=mig)
    if args.config != "c2":
        iso = {m: sum(v) for m, v in rt.stage_nominal.items()}
        rates = [float(x) for x in args.rates.split(",")] if args.rates else None
        for t in rt.tasks:
            t.rate = rates[t.id - 1] if rates else args.factor / iso[t.model]
    res = rt.run(duration=args.duration, warmup=0.1 * args.duration)
    out = {
        "gpu": {"total_sms": 148, "n_contexts": 4, "n_streams": 2, "oversubscription": 2.0, "policy": "mps-str",
                "kappa": 0.0},
        "tasks": [{"id": s.id, "period": s.period, "deadline": s.deadline, "hp": s.priority is Priority.HP,
                   "stages": [[p.nominal_time, p.width] for p in s.stages]} for s in res.tasks],
        "full_load": {str(k): v for k, v in res.full_load.items()},
        "duration": args.duration, "warmup_frac": 0.1, "phasing": "zero",
        "config": args.config, "stage_migration": mig,
        "trace": [list(t) for t in res.trace],
        "records": [list(r) for r in res.records],
        "report": res.report.to_dict(extended=True),
        "partitions": res.partitions,
    }
    path = Path(args.out) if args.out else ROOT / "tests" / "golden" / f"gpu_trace_{args.tag}.json.gz"
    with gzip.open(path, "wt") as fh:
        json.dump(out, fh)
    print(f"wrote {path}: {len(res.trace)} stages, {len(res.records)} records, "
          f"completed {res.report.completed_hp + res.report.completed_lp}, miss_hp {res.report.missed_hp}")
    rt.close()


if __name__ == "__main__":
    main()
