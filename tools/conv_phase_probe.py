"""Per-CTA phase stamps of ONE conv launch in isolation (stale, L2-resident
inputs, no predecessor kernel), to separate the kernel's own gather/epilogue
cost from inter-layer effects. python tools/conv_phase_probe.py"""
import statistics as S
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2504_08795_b200 import kernels as K  # noqa: E402

CASES = [  # (name, n, h, w, cin, cout, k, stride, pad, splits)
    ("l3.conv1 1x1 K1024 s8", 1, 14, 14, 1024, 256, 1, 1, 0, 8),
    ("l3.conv1 1x1 K1024 s1", 1, 14, 14, 1024, 256, 1, 1, 0, 1),
    ("l3.conv2 3x3 K2304 s8", 1, 14, 14, 256, 256, 3, 1, 1, 8),
    ("l4.conv2 3x3 K4608 s8", 1, 7, 7, 512, 512, 3, 1, 1, 8),
    ("l1.conv2 3x3 K576 s1", 1, 56, 56, 64, 64, 3, 1, 1, 1),
]
for name, n, h, w, cin, cout, k, st, pd, sp in CASES:
    dev = torch.device("cuda")
    x = torch.randn(n, h, w, cin, device=dev).bfloat16()
    wt = (torch.randn(cout, k, k, cin, device=dev) / (k * k * cin) ** 0.5).bfloat16()
    s = torch.ones(cout, device=dev)
    b = torch.zeros(cout, device=dev)
    d = K.conv_desc((n, h, w, cin), cout, k, k, st, pd, splits=sp, sm_budget=72)
    p = K.conv_plan(d)
    ts = torch.zeros(p.ctas * 16, dtype=torch.int64, device=dev)
    for rep in range(3):
        K.conv2d(x, wt, s, b, stride=st, pad=pd, splits=sp, sm_budget=72, timestamps=ts)
    torch.cuda.synchronize()
    a = (ts.view(-1, 16).double() - ts.view(-1, 16)[:, 0].min().double()) / 1e3
    a = a.cpu()
    med = lambda c1, c0: S.median((a[:, c1] - a[:, c0]).tolist())  # noqa: E731
    print(f"{name:24s} ctas {p.ctas:3d} cluster {p.cluster} kb/split {p.kb_per_split:2d}: setup {med(1, 0):.2f} "
          f"wait {med(2, 1):.2f} prod {med(3, 2):.2f} (max {(a[:, 3] - a[:, 2]).max().item():.2f}) "
          f"mma {med(4, 3):.2f} epi {med(5, 4):.2f} (max {(a[:, 5] - a[:, 4]).max().item():.2f}) "
          f"start-skew {(a[:, 0].max() - a[:, 0].min()).item():.2f} total {(a[:, 6].max()).item():.2f} us" +
          (f"\n      cluster epi: tmem->smem {med(8, 4):.2f} sync1 {med(9, 8):.2f} (max {(a[:, 9] - a[:, 8]).max().item():.2f}) "
           f"reduce {med(10, 9):.2f} sync2 {med(11, 10):.2f} teardown {med(6, 11):.2f}" if p.cluster > 1 else ""))
