"""One eager batch-1 forward of a network on a green-context partition, with
the layer grids planned for the C2 per-job SM share — the launch sequence the
executor captures into stage graphs. Used as the short command for ncu:

  ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 53 -c 53 \\
      -o gpurun_out/prof python tools/one_forward.py --model resnet50 --plan 23 --reps 2
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2504_08795_b200 import nets  # noqa: E402
from paper_2504_08795_b200.runtime import Executor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--sms", type=int, default=74, help="partition size (rounded to whole SM groups)")
    ap.add_argument("--plan", type=int, default=32, help="SMs the layer grids are planned for (C2: 32)")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--batch", type=int, default=1)
    args = ap.parse_args()
    ex = Executor(max(1, 148 // args.sms), 1, args.sms, slots=1, max_tasks=1, max_stages=8)
    net = nets.build_network(args.model, batch=args.batch)
    tb = nets.allocate_buffers(net, sm_budget=args.plan)
    ctx = ex.cluster_partition()
    sp = ex.stream(ctx, 0)
    s = torch.cuda.ExternalStream(sp)
    x = torch.randn(args.batch, 3, 224, 224, generator=torch.Generator().manual_seed(0)).cuda()
    with torch.cuda.stream(s):
        for _ in range(args.reps):
            out = nets.forward(net, tb, x, stream=sp, sm_budget=args.plan)
    s.synchronize()
    print(f"{args.model}: logits[0,:4] = {out[0, :4].tolist()}")
    ex.close()


if __name__ == "__main__":
    main()
