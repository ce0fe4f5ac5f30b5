"""Per-launch DRAM traffic of the conv kernel for bench.py's roofline `traffic`
field, from an `ncu --set full --page raw --csv` export of one ResNet-50 b1
forward's conv launches (tools/one_forward.py at the C2 plan):

  ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 49 -c 49 \\
      -o /tmp/prof python tools/one_forward.py --model resnet50 --plan 23 --reps 2
  ncu -i /tmp/prof.ncu-rep --page raw --csv > raw.csv
  python tools/conv_traffic.py raw.csv --plan 23 --capture "<file name>" > profiles/r02_conv_traffic.json

Writes the plan parameters the capture was taken at; bench.py uses the number
only when they match its own run (plan SMs, model, batch, DARIS_* knobs)."""

from __future__ import annotations

import argparse
import csv
import gzip
import json
import os


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--plan", type=int, default=23)
    ap.add_argument("--capture", default="")
    args = ap.parse_args()
    opener = gzip.open if args.raw.endswith(".gz") else open
    with opener(args.raw, "rt") as fh:
        rows = list(csv.reader(fh))
    h, units, data = rows[0], rows[1], rows[2:]
    col = {k: h.index(k) for k in h}
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def b(r, name):
        return float(r[col[name]].replace(",", "")) * scale[units[col[name]]]

    per = [b(r, "dram__bytes_read.sum") + b(r, "dram__bytes_write.sum") for r in data]
    knobs = {k: v for k, v in os.environ.items() if k.startswith("DARIS_") and k != "DARIS_GPU_TIMING"}
    print(json.dumps({"model": "resnet50", "batch": 1, "plan_sms": args.plan, "knobs": knobs,
                      "launches": len(per), "dram_bytes_per_launch": round(sum(per) / len(per)),
                      "dram_bytes_forward": round(sum(per)), "capture": args.capture or os.path.basename(args.raw)},
                     indent=1))


if __name__ == "__main__":
    main()
