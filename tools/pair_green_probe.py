"""Does a CTA-pair conv (cta_group::2, (2,1,1) clusters) run inside each green-
context partition of the C2 layout (4 x 74 SMs, OS = 2: partitions 1 and 4 hold
the 28-SM split remainder)? One launch per partition, each in a child process
under a timeout so a launch that never gets scheduled cannot hang the run."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2504_08795_b200 import kernels as K
from paper_2504_08795_b200.runtime import Executor
ctx = int(sys.argv[2])
ex = Executor(4, 2, 74, slots=1, max_tasks=1, max_stages=4)
print("partitions", [(p["context"], p["sm_count"], p["first_group"], p["n_groups"]) for p in ex.partitions], flush=True)
sp = ex.stream(ctx, 0)
s = torch.cuda.ExternalStream(sp)
g = torch.Generator().manual_seed(0)
x = torch.randn(16, 28, 28, 128, generator=g).bfloat16().cuda()
w = (torch.randn(128, 3, 3, 128, generator=g) / 34).bfloat16().cuda()
sc = torch.ones(128, device="cuda"); b = torch.zeros(128, device="cuda")
d = K.conv_desc(tuple(x.shape), 128, 3, 3, 1, 1, sm_budget=23)
print("plan pair", K.conv_plan(d).pair, flush=True)
torch.cuda.synchronize()
with torch.cuda.stream(s):
    y = K.conv2d(x, w, sc, b, stride=1, pad=1, sm_budget=23, stream=sp)
s.synchronize()
print("ctx", ctx, "ok", float(y.float().abs().sum()), flush=True)
"""
for ctx in (1, 2, 3, 4):
    try:
        r = subprocess.run([sys.executable, "-c", CHILD, str(ROOT), str(ctx)], capture_output=True, text=True,
                           timeout=60)
        print(f"partition {ctx}: rc={r.returncode}", r.stdout.strip().replace("\n", " | "), r.stderr[-300:])
    except subprocess.TimeoutExpired as e:
        print(f"partition {ctx}: TIMEOUT (hung)", (e.stdout or b"")[-300:])
