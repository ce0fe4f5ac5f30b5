"""Summarise an `ncu --set full --page raw --csv` export of consecutive conv
launches of one ResNet-50 b1 forward (tools/_ncu_r01.sh) as one row per layer:
time, algorithmic bytes (bench.conv_algorithmic_bytes), DRAM bytes, tensor-pipe
and SM throughput, warps active, achieved TFLOP/s.

python tools/ncu_conv_summary.py RAW.csv[.gz] --first 3 > summary.csv
(--first: index among the forward's convs of the first captured launch)"""

from __future__ import annotations

import argparse
import csv
import gzip
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--first", type=int, default=3)
    ap.add_argument("--model", default="resnet50")
    args = ap.parse_args()
    import torch
    import bench
    from paper_2504_08795_b200 import nets
    net = nets.build_network(args.model, batch=1, n_stages=4, device=torch.device("cpu"))
    convs = [op for op in net.ops if op.kind == "conv"]
    opener = gzip.open if args.raw.endswith(".gz") else open
    with opener(args.raw, "rt") as fh:
        rows = list(csv.reader(fh))
    h, units, data = rows[0], rows[1], rows[2:]
    col = {k: h.index(k) for k in h}

    def val(r, name, scale_to):
        v = float(r[col[name]].replace(",", ""))
        u = units[col[name]]
        f = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3,
             "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "%": 1.0, "": 1.0}.get(u, 1.0)
        return v * f if scale_to else v

    tensor = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
    print("layer,kernel,grid,time_us,algo_MB,dram_MB,dram_GBps,tensor_pct,sm_throughput_pct,warps_active_pct,TFLOPs")
    tot_t = tot_a = tot_d = 0.0
    for i, r in enumerate(data):
        op = convs[(args.first + i) % len(convs)]
        t = val(r, "gpu__time_duration.sum", True)
        dram = val(r, "dram__bytes_read.sum", True) + val(r, "dram__bytes_write.sum", True)
        algo = bench.conv_algorithmic_bytes(op) / 1e6
        kname = "halo" if "halo" in r[col["Kernel Name"]] else "igemm"
        grid = f"({r[col['launch__grid_dim_x']]}x{r[col['launch__grid_dim_y']]}x{r[col['launch__grid_dim_z']]})"
        print(f"{op.layer.name},{kname},{grid},{t:.2f},{algo:.3f},{dram:.3f},{dram / t * 1e3:.0f},"
              f"{val(r, tensor, False):.2f},{val(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed', False):.1f},"
              f"{val(r, 'sm__warps_active.avg.pct_of_peak_sustained_active', False):.1f},"
              f"{op.flops / (t * 1e-6) / 1e12:.2f}")
        tot_t += t
        tot_a += algo
        tot_d += dram
    print(f"# {len(data)} launches: {tot_t:.1f} us, algorithmic {tot_a:.1f} MB, DRAM {tot_d:.1f} MB "
          f"({tot_d / tot_a:.2f}x), mean DRAM bytes per launch {tot_d / len(data) * 1e6:.0f}")


if __name__ == "__main__":
    main()
