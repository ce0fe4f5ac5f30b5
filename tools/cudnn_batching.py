"""Sanity ceiling for the single-tenant batching baseline:
torchvision ResNet-50 in bf16, channels_last, cuDNN, one CUDA graph per
forward on the whole GPU; inferences/s per batch size. Library code, not the
product path — printed next to bench.py's batching_baseline (our kernels).

python tools/cudnn_batching.py [--batches 1,8,16,32,64,128]
"""

import argparse
import json

import torch
import torchvision


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="1,8,16,32,64,128")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    torch.backends.cudnn.benchmark = True
    m = torchvision.models.resnet50().cuda().eval().to(torch.bfloat16).to(memory_format=torch.channels_last)
    out = {}
    for b in [int(x) for x in args.batches.split(",")]:
        x = torch.randn(b, 3, 224, 224, device="cuda", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
        s = torch.cuda.Stream()
        with torch.no_grad(), torch.cuda.stream(s):
            for _ in range(3):
                m(x)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                y = m(x)
            for _ in range(3):
                g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(args.reps):
                g.replay()
            e1.record(s)
        e1.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / args.reps
        out[b] = {"inf_per_s": round(b / t, 1), "latency_ms": round(t * 1e3, 3),
                  "tflops": round(b * 8.178e9 / t / 1e12, 1)}
        print(json.dumps({"batch": b, **out[b]}), flush=True)
        del y, g


if __name__ == "__main__":
    main()
