"""BASELINE.json configs beyond the headline on one B200 (bench.py runs C2).

  c1      2 ResNet-18 tasks (1 HP, 1 LP) at 30 JPS, 2 contexts x 2 streams, OS=1, 3 stages
  c3      mixed ResNet-18/50, VGG-16, MobileNetV2 (1 HP + 1 LP each), 4x2 OS=2, knee of a
          common rate factor (task rate = factor / isolated latency of its model), stage
          migration off vs on
  c4      OS in {1,1.5,2,3} x contexts {2,4,8} x streams {1,2,4} (OS <= contexts) for the C2 task
          set (8 ResNet-50, 4 HP / 4 LP): knee inferences/s per cell
  tasks   ResNet-50 task count {8,12,16,24} at 4x2 OS=2, knee per count
  c5      C5 on one GPU: task count raised at a fixed per-task rate until the first HP miss

Every knee uses bench.py's protocol: a probe search over runs whose 0.5-s
windows must meet HP miss 0 and LP loss < 2 %, then a continuous confirmation
run (--confirm-seconds) stepping the rate down until all of its windows pass.
No re-measurement at the same rate. --criterion ok_excl (default) exempts the
windows with a GPU-wide pause (bench.py's value_excl_pauses: the environment's
~1.6 ms whole-GPU freezes cap any strict knee near 1 / 2 ms per task); --criterion
ok is the strict one. One JSON object per cell on stdout.

  python tools/configs_gpu.py c1 c3 c4 tasks [--probe-seconds 0.6] [--c4-cells 2x2_1,4x2_2]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2504_08795_b200.gpu import GpuConfig, Policy  # noqa: E402
from paper_2504_08795_b200.model import Priority  # noqa: E402
from paper_2504_08795_b200.runtime import BufferSetsExhausted, DarisRuntime, TaskDef  # noqa: E402


def log(m):
    print(m, file=sys.stderr, flush=True)


def emit(d):
    print(json.dumps(d), flush=True)


STEP = 0.5


CRITERION = "ok_excl"


def summary(res, warm: float, n: int) -> dict:
    w = bench.summarize(res.windows(warm, STEP, n), STEP)
    rep = res.report
    return {"jps": round(w["inf_per_s"], 1), "hp_miss": w["missed_hp"], "lp_loss": round(w["lp_loss"], 4),
            "constraints_met": w[CRITERION], "criterion": CRITERION, "windows": w["windows"],
            "windows_with_pause": w["windows_with_pause"], "windows_failed": w["windows_failed"],
            "gpu_pauses": w["stalls"], "rejected_lp": w["rejected_lp"],
            "p99_hp_ms": round(rep.response_hp.p99 * 1e3, 3), "p99_lp_ms": round(rep.response_lp.p99 * 1e3, 3)}


def knee_factor(rt, set_factor, f0: float, probe: float) -> tuple[float, None]:
    """bench.py's knee: the feasible rate factor with the most completed jobs/s."""
    return bench.knee_search(rt, f0, probe, STEP, log, set_rate=set_factor, criterion=CRITERION), None


def confirm(rt, set_factor, f: float, seconds: float):
    """Continuous confirmation run at the knee: every window must pass, else
    the factor steps down (bench.STEP_DOWN) and the run repeats."""
    n = max(1, int(round(seconds / STEP)))
    res = None
    for _ in range(8):
        set_factor(f)
        try:
            res = rt.run(duration=1.0 + n * STEP, warmup=1.0, full_load=rt.afet)
        except BufferSetsExhausted as e:  # overloaded: fails every window, step down
            log(f"confirm {f:.4g} overloaded: {e}")
            f *= bench.STEP_DOWN
            continue
        row = summary(res, 1.0, n)
        log(f"confirm {f:.4g} {row}")
        if row["constraints_met"]:
            res.row = row
            return f, res
        f *= bench.STEP_DOWN
    res.row = row
    return f, res


def c1(args):
    gpu = GpuConfig(148, 2, 2, 1.0, Policy.MPS_STR)
    tasks = [TaskDef(1, "resnet18", Priority.HP, 30.0, 3), TaskDef(2, "resnet18", Priority.LP, 30.0, 3)]
    rt = DarisRuntime(tasks, gpu, slots=3, seed=0)
    rt.capture_all()
    rt.afet = rt.calibrate_full_load(0.3)
    res = rt.run(duration=1.0 + 10.0, warmup=1.0, full_load=rt.afet)
    out = {"config": "c1", "rate_per_task": 30.0, "partition_sms": [p["sm_count"] for p in rt.exec.partitions],
           "isolated_ms": round(sum(rt.stage_nominal["resnet18"]) * 1e3, 3), **summary(res, 1.0, 20)}
    iso = sum(rt.stage_nominal["resnet18"])
    f, best = knee_factor(rt, rt.set_rate, 0.6 * 4 / max(rt.afet.values()) / 2, args.probe_seconds)
    f, res = confirm(rt, rt.set_rate, f, args.confirm_seconds)
    out["knee"] = {"rate_per_task": round(f, 1), **res.row}
    emit(out)
    rt.close()


def c3(args):
    gpu = GpuConfig(148, 4, 2, 2.0, Policy.MPS_STR)
    models = ["resnet18", "resnet50", "vgg16", "mobilenet_v2"]
    stages = {"resnet18": 3, "resnet50": 4, "vgg16": 4, "mobilenet_v2": 3}
    for mig in (False, True):
        tasks = []
        for i, m in enumerate(models):
            tasks.append(TaskDef(2 * i + 1, m, Priority.HP, 100.0, stages[m]))
            tasks.append(TaskDef(2 * i + 2, m, Priority.LP, 100.0, stages[m]))
        rt = DarisRuntime(tasks, gpu, slots=3, seed=0, stage_migration=mig)
        rt.capture_all()
        rt.afet = rt.calibrate_full_load(0.3)
        iso = {m: sum(v) for m, v in rt.stage_nominal.items()}

        def set_factor(f, rt=rt, iso=iso):
            for t in rt.tasks:
                t.rate = f / iso[t.model]

        # factor f: every task at f / (its isolated latency); start below the loaded capacity
        f0 = 0.6 * 8 / sum(rt.afet[t.id] / iso[t.model] for t in rt.tasks)
        f, best = knee_factor(rt, set_factor, f0, args.probe_seconds)
        f, res = confirm(rt, set_factor, f, args.confirm_seconds)
        per_model = {}
        for t in rt.tasks:
            per_model.setdefault(t.model, 0.0)
            per_model[t.model] += t.rate
        flops = {m: rt.nets[(m, stages[m], 1)].flops_per_image for m in models}
        tflops = sum(per_model[m] * flops[m] for m in models) / 1e12
        emit({"config": "c3", "stage_migration": mig, "knee_factor": round(f, 4),
              "isolated_ms": {m: round(v * 1e3, 3) for m, v in iso.items()},
              "rate_per_task": {m: round(per_model[m] / 2, 1) for m in models},
              "model_tflops": round(tflops, 2), **res.row})
        rt.close()


def c4(args):
    cells = []
    for os_ in (1.0, 1.5, 2.0, 3.0):
        for nc in (2, 4, 8):
            for ns in (1, 2, 4):
                if os_ <= nc:
                    cells.append((nc, ns, os_))
    if args.c4_cells:
        want = set(args.c4_cells.split(","))
        cells = [c for c in cells if f"{c[0]}x{c[1]}_{c[2]:g}" in want]
    for nc, ns, os_ in cells:
        t0 = time.time()
        gpu = GpuConfig(148, nc, ns, os_, Policy.MPS_STR)
        slots = 3 if 8 * 3 >= nc * ns else 4
        rt = DarisRuntime(bench.c2_tasks(100.0, list(range(8))), gpu, slots=slots, seed=0)
        rt.capture_all()
        rt.afet = rt.calibrate_full_load(0.2)
        iso = sum(rt.stage_nominal["resnet50"])
        f, best = knee_factor(rt, rt.set_rate, 0.6 * min(8, nc * ns) / max(rt.afet.values()) / 8,
                              args.probe_seconds)
        f, res = confirm(rt, rt.set_rate, f, args.confirm_seconds)
        emit({"config": "c4", "cell": f"{nc}x{ns}_{os_:g}", "contexts": nc, "streams": ns, "oversubscription": os_,
              "partition_sms": rt.exec.partitions[0]["sm_count"], "isolated_ms": round(iso * 1e3, 3),
              "knee_rate_per_task": round(f, 1), "seconds": round(time.time() - t0, 1), **res.row})
        rt.close()


def task_scaling(args):
    gpu = GpuConfig(148, 4, 2, 2.0, Policy.MPS_STR)
    for n in (8, 12, 16, 24):
        rt = DarisRuntime(bench.c2_tasks(100.0, list(range(n))), gpu, slots=3, seed=0)
        rt.capture_all()
        rt.afet = rt.calibrate_full_load(0.2)
        iso = sum(rt.stage_nominal["resnet50"])
        f, best = knee_factor(rt, rt.set_rate, 0.6 * 8 / max(rt.afet.values()) / n, args.probe_seconds)
        f, res = confirm(rt, rt.set_rate, f, args.confirm_seconds)
        emit({"config": "tasks", "tasks": n, "contexts": 4, "streams": 2, "oversubscription": 2.0,
              "knee_rate_per_task": round(f, 1), **res.row})
        rt.close()


def c5(args):
    """BASELINE config 5 on one GPU: the C2 mix (half HP, half LP) at a fixed
    per-task rate, task count raised until the first HP deadline miss (or LP
    loss >= 2 %); the last feasible count is this GPU's share of the box."""
    gpu = GpuConfig(148, 4, 2, 2.0, Policy.MPS_STR)
    rate = args.c5_rate
    last_ok = None
    for n in range(8, 65, 4):
        rt = DarisRuntime(bench.c2_tasks(rate, list(range(n))), gpu, slots=3, seed=0)
        rt.capture_all()
        rt.afet = rt.calibrate_full_load(0.2)
        nwin = max(1, int(round(args.confirm_seconds / STEP)))
        try:
            res = rt.run(duration=1.0 + nwin * STEP, warmup=1.0, full_load=rt.afet)
            row = {"config": "c5", "tasks": n, "rate_per_task": rate, **summary(res, 1.0, nwin)}
        except BufferSetsExhausted as e:
            row = {"config": "c5", "tasks": n, "rate_per_task": rate, "constraints_met": False, "overloaded": str(e)}
        ok = row["constraints_met"]
        log(f"c5 tasks={n} ok={ok} {row}")
        rt.close()
        if not ok:
            emit({**row, "first_failing": True, "max_feasible_tasks": last_ok["tasks"] if last_ok else 0,
                  "max_feasible_jps": last_ok["jps"] if last_ok else 0.0})
            return
        last_ok = row
        emit(row)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="+", choices=["c1", "c3", "c4", "tasks", "c5"])
    ap.add_argument("--c5-rate", type=float, default=500.0, help="per-task JPS for the c5 task-count scan")
    ap.add_argument("--probe-seconds", type=float, default=1.0)
    ap.add_argument("--confirm-seconds", type=float, default=10.0)
    ap.add_argument("--c4-cells", default="")
    ap.add_argument("--criterion", default="ok_excl", choices=["ok_excl", "ok"])
    args = ap.parse_args()
    global CRITERION
    CRITERION = args.criterion
    for w in args.which:
        {"c1": c1, "c3": c3, "c4": c4, "tasks": task_scaling, "c5": c5}[w](args)


if __name__ == "__main__":
    main()
