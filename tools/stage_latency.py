"""Per-stage latency of a network in one green-context partition, one CUDA
graph per stage, in both execution modes (persistent stage kernel vs one
launch per layer). python tools/stage_latency.py --model resnet50 --sms 74"""

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
    ap.add_argument("--sms", type=int, default=74)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--modes", default="layers,persistent")
    args = ap.parse_args()
    ex = Executor(max(1, 148 // args.sms), 1, args.sms, slots=1, max_tasks=1, max_stages=8)
    sm = ex.partitions[0]["sm_count"]
    sp = ex.stream(1, 0)
    s = torch.cuda.ExternalStream(sp)
    net = nets.build_network(args.model, batch=args.batch)
    x = torch.randn(args.batch, 3, 224, 224, generator=torch.Generator().manual_seed(0)).cuda()
    for mode in args.modes.split(","):
        tb = nets.allocate_buffers(net, sm_budget=sm)
        tb.input.copy_(x)
        for st in range(net.n_stages):
            if mode == "persistent":
                nets.stage_program(net, st, tb, sm)
        times = []
        with torch.cuda.stream(s):
            for st in range(net.n_stages):
                g = torch.cuda.CUDAGraph()
                nets.run_stage(net, st, tb, sp, sm, mode=mode)
                g.capture_begin()
                nets.run_stage(net, st, tb, sp, sm, mode=mode)
                g.capture_end()
                for _ in range(5):
                    g.replay()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(args.reps):
                    g.replay()
                e1.record(s)
                e1.synchronize()
                times.append(e0.elapsed_time(e1) * 1e3 / args.reps)
        tot = sum(times)
        print(f"{args.model} b{args.batch} {sm} SMs mode={mode:10s} stages(us)={[round(t, 1) for t in times]} "
              f"total={tot:.1f} us  -> {args.batch / tot * 1e6:.0f} inf/s single stream", flush=True)
        if mode == "persistent":
            a = 0
            for st in range(net.n_stages):
                prog = nets.stage_program(net, st, tb, sm)
                print(f"   stage {st}: grid {prog.grid} units {prog.units} smem {prog.smem_bytes} "
                      f"per-op (units,splits)={[prog.layer_units(i) for i in range(prog.n_ops)]}")
    ex.close()


if __name__ == "__main__":
    main()
