"""Generate the golden scheduling fixtures by running the REFERENCE itself.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
Writes tests/golden/sched_golden.json.gz: for each case the exact inputs the
reference simulated (tasks after overload scaling, GPU config, options) and
its outputs (event log, admission audits, metrics report, AFET baselines).
The GPU box never reads /root/reference; it only reads this file.
"""

from __future__ import annotations

import gzip
import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "sched_golden.json.gz"


def _import_ref():
    sys.path.insert(0, str(REF))
    import stagesim  # noqa: F401
    return stagesim


def _task_json(t, batch_sizes, curves):
    c = curves.get(t.id)
    return {"id": t.id, "period": t.period, "deadline": t.deadline, "hp": t.priority.value == "hp",
            "stages": [[p.nominal_time, p.width] for p in t.stages],
            "batch": batch_sizes.get(t.id, 1),
            "curve": None if c is None else [c.reference_batch, c.reference_gain]}


def _run_case(ss, name, scenario: dict):
    cfg = ss.scenario_from_dict(scenario)
    sim = ss.build_simulation(cfg, collect_log=True)
    res = sim.run()
    g = cfg.gpu
    return {
        "name": name,
        "scenario": scenario,
        "gpu": {"total_sms": g.total_sms, "n_contexts": g.n_contexts, "n_streams": g.n_streams,
                "oversubscription": g.oversubscription, "policy": g.policy.value,
                "kappa": g.interference_kappa},
        "tasks": [_task_json(t, cfg.batch_sizes, cfg.curves) for t in sim.tasks],
        "options": {"seed": cfg.seed, "duration": cfg.duration, "warmup_frac": cfg.warmup_frac,
                    "ws": cfg.window_size, "reps": cfg.full_load_reps,
                    "no_staging": cfg.flags.no_staging, "no_last": cfg.flags.no_last,
                    "no_prior": cfg.flags.no_prior, "no_fixed": cfg.flags.no_fixed,
                    "hpa": cfg.hpa, "phasing": cfg.phasing, "placement_order": cfg.placement_order,
                    "edf_on_job_deadline": cfg.edf_on_job_deadline},
        "records": [list(r) for r in res.records],
        "admissions": [[a.time, a.job_id, a.task_id, a.priority.value, a.context, a.active_util,
                        a.job_util, a.limit, a.admitted] for a in res.admissions],
        "report": res.report.to_dict(),
        "full_load": {str(k): v for k, v in res.full_load.items()},
    }


def _random_scenario(rng: random.Random, idx: int) -> dict:
    policy = rng.choice(["mps", "str", "mps-str"])
    if policy == "str":
        nc, ns = 1, rng.randint(2, 4)
    elif policy == "mps":
        nc, ns = rng.randint(2, 6), 1
    else:
        nc, ns = rng.randint(2, 4), rng.randint(2, 3)
    os_ = rng.choice([1.0, 1.5, 2.0, float(nc)])
    os_ = min(os_, float(nc))
    sms = rng.choice([64, 68, 148])
    n_tasks = rng.randint(1, 7)
    tasks = []
    for i in range(n_tasks):
        n_st = rng.randint(1, 4)
        tasks.append({
            "id": i + 1,
            "period": round(rng.uniform(0.004, 0.03), 6),
            "priority": rng.choice(["hp", "lp", "lp"]),
            "stages": [{"nominal_time": round(rng.uniform(0.0003, 0.004), 6),
                        "width": rng.randint(4, sms)} for _ in range(n_st)],
            **({"batch_size": rng.choice([2, 4]),
                "batching": {"reference_batch": 4, "reference_gain": 1.6}} if rng.random() < 0.2 else {}),
        })
    sc = {"gpu": {"total_sms": sms, "n_contexts": nc, "n_streams": ns, "oversubscription": os_,
                  "policy": policy, "kappa": rng.choice([0.0, 0.0, 0.1])},
          "workload": {"tasks": tasks}, "seed": rng.randint(0, 50), "duration": 0.4,
          "full_load_reps": rng.choice([2, 3]),
          "ablations": rng.choice([[], [], ["no_last"], ["no_prior"], ["no_fixed"], ["no_staging"]]),
          "hpa": rng.random() < 0.25,
          "placement_order": rng.choice(["descending_util", "insertion"]),
          "edf_on_job_deadline": rng.random() < 0.2,
          "phasing": rng.choice(["random", "random", "zero"])}
    if rng.random() < 0.5:
        sc["overload_factor"] = rng.choice([0.8, 1.2, 1.5, 2.0])
    return sc


def cases() -> list[tuple[str, dict]]:
    out = [
        ("resnet18_main_1s", {"preset": "resnet18_main", "duration": 1.0}),
        ("unet_main_1s", {"preset": "unet_main", "duration": 1.0}),
        ("inceptionv3_main_1s", {"preset": "inceptionv3_main", "duration": 1.0}),
        ("mixed_main_0.5s", {"preset": "mixed_main", "duration": 0.5}),
        ("resnet18_no_staging", {"preset": "resnet18_main", "duration": 0.5, "ablations": ["no_staging"]}),
        ("resnet18_hpa", {"preset": "resnet18_main", "duration": 0.5, "hpa": True, "overload_factor": 2.5}),
        ("resnet18_str_4", {"preset": "resnet18_main", "duration": 0.5,
                            "gpu": {"n_contexts": 1, "n_streams": 4, "oversubscription": 1, "policy": "str"}}),
        ("resnet18_mpsstr_2x3_os1.5", {"preset": "resnet18_main", "duration": 0.5, "seed": 3,
                                       "gpu": {"n_contexts": 2, "n_streams": 3, "oversubscription": 1.5,
                                               "policy": "mps-str", "kappa": 0.05}}),
        ("inception_batched", {"preset": "inceptionv3_main", "duration": 0.5,
                               "workload": {"batch_size": "profile"}}),
        # C1 analog: 2 ResNet-18 tasks (1 HP, 1 LP), 2 ctx x 2 streams, OS=1, 3 stages, 148 SMs
        ("c1_resnet18_2x2", {"gpu": {"total_sms": 148, "n_contexts": 2, "n_streams": 2,
                                     "oversubscription": 1, "policy": "mps-str"},
                             "workload": {"tasks": [
                                 {"id": 1, "period": 1 / 30, "priority": "hp",
                                  "stages": [{"nominal_time": 0.0005, "width": 60},
                                             {"nominal_time": 0.0005, "width": 60},
                                             {"nominal_time": 0.0005, "width": 60}]},
                                 {"id": 2, "period": 1 / 30, "priority": "lp",
                                  "stages": [{"nominal_time": 0.0005, "width": 60},
                                             {"nominal_time": 0.0005, "width": 60},
                                             {"nominal_time": 0.0005, "width": 60}]}]},
                             "duration": 2.0}),
        # C2 analog: 8 ResNet-50 tasks (4 HP / 4 LP), 4 ctx x 2 streams, OS=2
        ("c2_resnet50_4x2_os2", {"gpu": {"total_sms": 148, "n_contexts": 4, "n_streams": 2,
                                         "oversubscription": 2, "policy": "mps-str"},
                                 "workload": {"tasks": [
                                     {"id": i + 1, "period": 0.004, "priority": "hp" if i < 4 else "lp",
                                      "stages": [{"nominal_time": 0.0011, "width": 70},
                                                 {"nominal_time": 0.0009, "width": 70},
                                                 {"nominal_time": 0.0009, "width": 70},
                                                 {"nominal_time": 0.0006, "width": 70}]}
                                     for i in range(8)]},
                                 "overload_factor": 1.5, "duration": 0.5}),
    ]
    rng = random.Random(2504_08795)
    for i in range(40):
        out.append((f"random_{i:02d}", _random_scenario(rng, i)))
    return out


def main() -> None:
    ss = _import_ref()
    data = []
    for name, sc in cases():
        data.append(_run_case(ss, name, sc))
        print(f"{name}: {len(data[-1]['records'])} records", flush=True)
    with gzip.open(OUT, "wt") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "stagesim 0.1.0",
                   "cases": data}, fh)
    print("wrote", OUT, OUT.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
