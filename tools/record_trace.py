"""Record a real-GPU DARIS run as a trace fixture for P2 parity tests on the CPU.

Runs a C2-shaped workload (ResNet-50, 4 contexts x 2 streams, OS=2) on the B200
with zero phasing, and writes tests/golden/gpu_trace_<tag>.json.gz holding the
task set, AFET baselines, per-stage durations and the executor's event log.
tests/test_reference_trace_replay.py replays it through the oracle and (where
/root/reference exists) through the unmodified reference scheduler.

python tools/record_trace.py --tag r01 [--rate 400] [--duration 0.4]
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
    ap.add_argument("--rate", type=float, default=400.0)
    ap.add_argument("--duration", type=float, default=0.4)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    gpu = GpuConfig(148, 4, 2, 2.0, Policy.MPS_STR)
    tasks = [TaskDef(i + 1, "resnet50", Priority.HP if i < 4 else Priority.LP, args.rate, 4) for i in range(8)]
    rt = DarisRuntime(tasks, gpu, slots=3, phasing="zero")
    res = rt.run(duration=args.duration, warmup=0.1 * args.duration)
    out = {
        "gpu": {"total_sms": 148, "n_contexts": 4, "n_streams": 2, "oversubscription": 2.0, "policy": "mps-str",
                "kappa": 0.0},
        "tasks": [{"id": s.id, "period": s.period, "deadline": s.deadline, "hp": s.priority is Priority.HP,
                   "stages": [[p.nominal_time, p.width] for p in s.stages]} for s in res.tasks],
        "full_load": {str(k): v for k, v in res.full_load.items()},
        "duration": args.duration, "warmup_frac": 0.1, "phasing": "zero",
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
