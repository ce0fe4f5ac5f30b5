"""Per-CTA phase timeline of the conv kernels of one network forward, captured
as a CUDA graph on a green-context partition (as the executor runs it).

Each conv CTA stamps %globaltimer at: 0 entry, 1 after barrier/TMEM setup,
2 after griddepcontrol.wait, 3 producer done, 4 accumulator ready, 5 epilogue
done, 6 exit. Prints per-layer medians and the gap between a layer's last CTA
exit and the next layer's first released CTA.

python tools/timeline_convs.py [--model resnet50] [--sms 74] [--json out.json]
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2504_08795_b200 import kernels as K  # noqa: E402
from paper_2504_08795_b200 import nets  # noqa: E402
from paper_2504_08795_b200.runtime import Executor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--sms", type=int, default=74)
    ap.add_argument("--json", default=None)
    ap.add_argument("--dump", nargs="*", default=[], help="layer names whose per-CTA stamps to print")
    args = ap.parse_args()
    ex = Executor(max(1, 148 // args.sms), 1, args.sms, slots=1, max_tasks=1, max_stages=8)
    net = nets.build_network(args.model, batch=1)
    tb = nets.allocate_buffers(net, sm_budget=args.sms)
    ctx = ex.cluster_partition()
    sp = ex.stream(ctx, 0)
    s = torch.cuda.ExternalStream(sp)
    args.sms = ex.partitions[ctx - 1]["sm_count"]  # the partition's actual SM count (whole 8-SM groups)
    ts = {}
    for i, op in enumerate(net.ops):
        if op.kind == "conv":
            L = op.layer
            p = K.conv_plan(K.conv_desc(op.shape_in, L.cout, L.kh, L.kw, L.stride, L.pad, sm_budget=args.sms,
                                        padded_input=L.padded_input,
                                        x2_shape=op.shape_in2 if L.dual_cin else None, stride2=L.dual_stride))
            ts[i] = torch.zeros(p.ctas * 16, dtype=torch.int64, device="cuda")

    def forward(stream):
        for i, op in enumerate(net.ops):
            if op.kind == "conv":
                nets.run_op(op, tb, stream, args.sms, timestamps=ts[i])
            else:
                nets.run_op(op, tb, stream, args.sms)

    forward(sp)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        g.capture_begin()
        forward(sp)
        g.capture_end()
        for _ in range(3):
            g.replay()
    torch.cuda.synchronize()
    rows = []
    prev_end = None
    t_origin = None
    for i, op in enumerate(net.ops):
        if op.kind != "conv":
            continue
        raw_sm = ts[i].view(-1, 16)[:, 15].cpu().tolist()
        a = ts[i].view(-1, 16).cpu().double()
        if t_origin is None:
            t_origin = a[:, 0].min().item()
        a = (a - t_origin) / 1e3  # us
        start = a[:, 0].min().item()
        released = a[:, 2].min().item()
        end = a[:, 6].max().item()
        row = {"i": i, "name": op.layer.name, "ctas": a.shape[0], "start": start, "released": released,
               "end": end,
               "setup_us": statistics.median((a[:, 1] - a[:, 0]).tolist()),
               "wait_us": statistics.median((a[:, 2] - a[:, 1]).tolist()),
               "produce_us": statistics.median((a[:, 3] - a[:, 2]).tolist()),
               "mma_tail_us": statistics.median((a[:, 4] - a[:, 3]).tolist()),
               "epilogue_us": statistics.median((a[:, 5] - a[:, 4]).tolist()),
               "epilogue_max_us": (a[:, 5] - a[:, 4]).max().item(),
               "teardown_us": statistics.median((a[:, 6] - a[:, 5]).tolist()),
               "span_us": end - released,
               "gap_from_prev_us": None if prev_end is None else released - prev_end}
        raw = ts[i].view(-1, 16).cpu()
        if (raw[:, 8] > 0).all():  # cluster split-K: sync / push+arrive / reduce / final wait
            row["cluster_us"] = [statistics.median((a[:, 9] - a[:, 8]).tolist()),
                                 statistics.median((a[:, 10] - a[:, 9]).tolist()),
                                 statistics.median((a[:, 11] - a[:, 10]).tolist()),
                                 statistics.median((a[:, 5] - a[:, 11]).tolist()),
                                 statistics.median((a[:, 8] - a[:, 4]).tolist())]
        if op.layer.name in args.dump:
            print(f"--- {op.layer.name}: per CTA (us from the layer's first release): sm start released "
                  f"prod_done acc_ready epi_done exit [cluster: pre_sync post_sync recv_done reduce_done]")
            order = sorted(range(a.shape[0]), key=lambda c: a[c, 0].item())
            for c in order:
                extra = (" | " + " ".join(f"{a[c, k].item() - released:7.2f}" for k in (8, 9, 10, 11))
                         if raw[c, 8] > 0 else "")
                print(f"  cta {c:3d} sm {int(raw_sm[c]):3d} " + " ".join(
                    f"{a[c, k].item() - released:7.2f}" for k in (0, 2, 3, 4, 5, 6)) + extra)
        prev_end = end
        rows.append(row)
    total = rows[-1]["end"] - rows[0]["released"]
    print(f"{args.model} conv timeline in {args.sms} SMs: first release -> last exit {total:.1f} us over "
          f"{len(rows)} convs")
    print(f"{'layer':28s} ctas  span  gap  setup  wait  prod  mma  epi(max)  tear")
    for r in rows:
        print(f"{r['name']:28s} {r['ctas']:4d} {r['span_us']:5.1f} "
              f"{(r['gap_from_prev_us'] if r['gap_from_prev_us'] is not None else 0):5.2f} {r['setup_us']:5.2f} "
              f"{r['wait_us']:6.2f} {r['produce_us']:5.2f} {r['mma_tail_us']:5.2f} {r['epilogue_us']:5.2f}"
              f"({r['epilogue_max_us']:5.2f}) {r['teardown_us']:5.2f}"
              + ("  cluster[pre %.2f sync %.2f push %.2f reduce %.2f wait %.2f]" % (
                  r["cluster_us"][4], *r["cluster_us"][:4]) if "cluster_us" in r else ""))
    gaps = [r["gap_from_prev_us"] for r in rows if r["gap_from_prev_us"] is not None]
    spans = [r["span_us"] for r in rows]
    print(f"sum span {sum(spans):.1f} us, sum gaps {sum(gaps):.1f} us (median gap {statistics.median(gaps):.2f})")
    if args.json:
        Path(args.json).write_text(json.dumps(rows, indent=1))
    ex.close()


if __name__ == "__main__":
    main()
