"""Unit-level timeline of one persistent stage-kernel launch (globaltimer
stamps written by the kernel): per layer, when its units were claimed,
started, saw their dependency, finished the gather, got the accumulator and
published, and how many units the busiest CTA ran.

python tools/stage_timeline.py --model resnet50 --stage 2 --sms 74
"""

import argparse
import statistics as S
import sys
from collections import Counter
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2504_08795_b200 import nets  # noqa: E402
from paper_2504_08795_b200.runtime import Executor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--stage", type=int, default=2)
    ap.add_argument("--sms", type=int, default=74)
    ap.add_argument("--grid", type=int, default=0)
    args = ap.parse_args()
    ex = Executor(max(1, 148 // args.sms), 1, args.sms, slots=1, max_tasks=1, max_stages=8)
    sm = ex.partitions[0]["sm_count"]
    grid = args.grid or sm
    sp = ex.stream(1, 0)
    s = torch.cuda.ExternalStream(sp)
    net = nets.build_network(args.model, batch=1)
    tb = nets.allocate_buffers(net, sm_budget=sm)
    tb.input.copy_(torch.randn(1, 3, 224, 224).cuda())
    with torch.cuda.stream(s):
        for st in range(net.n_stages):
            nets.stage_program(net, st, tb, grid).launch(sp)
        prog = nets.stage_program(net, args.stage, tb, grid)
        tr = torch.zeros(prog.units, 16, dtype=torch.int64, device="cuda")
        for _ in range(3):
            for st in range(args.stage + 1):
                nets.stage_program(net, st, tb, grid).launch(sp)
        torch.cuda.synchronize()
        for st in range(args.stage):
            nets.stage_program(net, st, tb, grid).launch(sp)
        prog.set_trace(tr)
        prog.launch(sp)
        torch.cuda.synchronize()
        prog.set_trace(None)
    T = tr.cpu().tolist()
    t0 = min(r[0] for r in T)
    a = net.stage_bounds[args.stage]
    names = [getattr(op.layer, "name", op.kind) for op in net.ops[a:net.stage_bounds[args.stage + 1]]]
    u0 = 0
    prev_pub = None
    print(f"{args.model} stage {args.stage}: grid {grid}, {prog.units} units; times in us from first claim")
    print(f"{'layer':26s} {'units':>5s} {'claim0':>7s} {'start50':>7s} {'dep_max':>7s} {'gath50':>6s} "
          f"{'mma50':>6s} {'epi50':>6s} {'pub_last':>8s} {'dep-prev':>8s} {'maxCTA':>6s}  gather: math/empty0/issue0/loop/wait")
    for i, name in enumerate(names):
        n, sp_ = prog.layer_units(i)
        rows = T[u0:u0 + n]
        u0 += n
        us = lambda v: (v - t0) / 1e3  # noqa: E731
        claim0 = us(min(r[0] for r in rows))
        start50 = S.median(us(r[1]) for r in rows)
        dep_max = max(us(r[2]) for r in rows)
        conv = all(r[3] for r in rows)
        gath = S.median((r[3] - r[2]) / 1e3 for r in rows) if conv else 0
        mma = S.median((r[4] - r[3]) / 1e3 for r in rows) if conv else 0
        epi = S.median((r[6] - r[4]) / 1e3 for r in rows) if conv else 0
        pubs = [us(r[5]) for r in rows if r[5]]
        pub_last = max(pubs) if pubs else float("nan")
        per_cta = Counter(r[7] for r in rows).most_common(1)[0][1]
        dep_gap = (dep_max - prev_pub) if prev_pub is not None else 0.0
        print(f"{name[:26]:26s} {n:5d} {claim0:7.2f} {start50:7.2f} {dep_max:7.2f} {gath:6.2f} {mma:6.2f} "
              f"{epi:6.2f} {pub_last:8.2f} {dep_gap:8.2f} {per_cta:6d}  " +
              (f"{S.median((r[11] - r[2]) / 1e3 for r in rows):.2f}/{S.median((r[12] - r[11]) / 1e3 for r in rows):.2f}/"
               f"{S.median((r[8] - r[12]) / 1e3 for r in rows):.2f}/{S.median((r[9] - r[8]) / 1e3 for r in rows):.2f}/"
               f"{S.median((r[10] - r[9]) / 1e3 for r in rows):.2f}" if conv else ""))
        prev_pub = pub_last
    ex.close()


if __name__ == "__main__":
    main()
