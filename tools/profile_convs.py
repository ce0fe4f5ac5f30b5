"""Per-layer timing of a network's stage kernels inside one green-context
partition, with launch overhead removed: each op is captured into a CUDA graph
(repeated R times) on the partition's stream and replayed between CUDA events.

python tools/profile_convs.py [--model resnet50] [--batch 1] [--sms 74] [--json out.json]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2504_08795_b200 import kernels as K  # noqa: E402
from paper_2504_08795_b200 import nets  # noqa: E402
from paper_2504_08795_b200.runtime import Executor  # noqa: E402


def op_bytes(op) -> int:
    """Algorithmic bytes: weights + input activation + output (+ residual)."""
    def n(shape):
        r = 1
        for s in shape:
            r *= s
        return r
    b = 0
    if op.kind in ("conv", "linear", "dwconv"):
        b += op.layer.weight.numel() * 2
    b += n(op.shape_in) * (4 if op.kind == "pack8" else 2)
    b += n(op.shape_out) * (4 if op.dst == "logits" else 2)
    if op.res:
        b += n(op.shape_out) * 2
    return b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--sms", type=int, default=74)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    n_ctx = max(1, 148 // args.sms)
    ex = Executor(n_ctx, 1, args.sms, slots=1, max_tasks=1, max_stages=8)
    net = nets.build_network(args.model, batch=args.batch)
    tb = nets.allocate_buffers(net, sm_budget=args.sms)
    ctx = ex.cluster_partition()
    stream_ptr = ex.stream(ctx, 0)
    s = torch.cuda.ExternalStream(stream_ptr)
    # warm: every op once eagerly (sets kernel attributes before capture)
    for op in net.ops:
        nets.run_op(op, tb, stream_ptr, args.sms)
    torch.cuda.synchronize()
    rows = []
    for i, op in enumerate(net.ops):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            g.capture_begin()
            for _ in range(args.reps):
                nets.run_op(op, tb, s.cuda_stream, args.sms)
            g.capture_end()
        with torch.cuda.stream(s):
            g.replay()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(5):
                g.replay()
            e1.record(s)
        e1.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / (5 * args.reps)
        plan = None
        if op.kind == "conv":
            L = op.layer
            d = K.conv_desc(op.shape_in, L.cout, L.kh, L.kw, L.stride, L.pad, sm_budget=args.sms)
            p = K.conv_plan(d)
            plan = {"bn": p.block_n, "splits": p.splits, "ctas": p.ctas, "kb": p.kb_per_split}
        name = getattr(op.layer, "name", op.kind) if op.layer is not None else op.kind
        rows.append({"i": i, "kind": op.kind, "name": name, "in": list(op.shape_in), "out": list(op.shape_out),
                     "us": t * 1e6, "tflops": op.flops / t / 1e12 if op.flops else 0.0,
                     "gbs": op_bytes(op) / t / 1e9, "flops": op.flops, "bytes": op_bytes(op), "plan": plan})
    # whole stages as graphs
    stages = []
    for st in range(net.n_stages):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            g.capture_begin()
            nets.run_stage(net, st, tb, s.cuda_stream, args.sms)
            g.capture_end()
            g.replay()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(20):
                g.replay()
            e1.record(s)
        e1.synchronize()
        stages.append(e0.elapsed_time(e1) / 1e3 / 20)
    tot = sum(r["us"] for r in rows)
    conv_t = sum(r["us"] for r in rows if r["kind"] == "conv")
    print(f"{args.model} b{args.batch} in {args.sms} SMs: sum of per-op {tot:.1f} us "
          f"(conv {conv_t:.1f} us, {100 * conv_t / tot:.1f}%), stage graphs "
          f"{[round(x * 1e6, 1) for x in stages]} us = {sum(stages) * 1e6:.1f} us")
    for r in rows:
        print(f"{r['i']:3d} {r['kind']:8s} {r['name']:28s} {str(r['in']):22s} {r['us']:8.2f} us "
              f"{r['tflops']:7.2f} TF/s {r['gbs']:8.1f} GB/s {r['plan'] or ''}")
    if args.json:
        Path(args.json).write_text(json.dumps({"rows": rows, "stages_s": stages}, indent=1))
    ex.close()


if __name__ == "__main__":
    main()
