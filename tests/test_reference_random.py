"""P1 parity against the UNMODIFIED reference on random scenarios (SURVEY §8c:
">= 1000 random small instances"): the same task set, device model, ablation
flags, batching and seeds go through stagesim (imported from
/root/reference, skipped where it is absent, e.g. on the GPU box) and through
this package's native event loop; event logs, admission audits and metric
reports must be equal field for field (floats included).

DARIS_REF_RANDOM_N sets the number of instances (default 1000; a 5000-instance
sweep also passed in round 1: ~65 s)."""

import os
import random
import sys
from pathlib import Path

import pytest

REF_SRC = Path("/root/reference/pkg/src")
N = int(os.environ.get("DARIS_REF_RANDOM_N", "1000"))
pytestmark = pytest.mark.skipif(not (REF_SRC / "stagesim").exists(), reason="reference tree not present")


def _ref():
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import stagesim
    return stagesim


def _instance(rng):
    nc = rng.randint(1, 4)
    ns = rng.randint(1, 3)
    sms = rng.choice([16, 68, 148])
    os_ = rng.choice([1.0, min(2.0, nc), float(nc), 1.5 if nc >= 2 else 1.0])
    tasks = []
    for i in range(rng.randint(1, 7)):
        stages = [(round(rng.uniform(2e-4, 3e-3), 7), rng.randint(1, sms)) for _ in range(rng.randint(1, 4))]
        tasks.append((i + 1, round(rng.uniform(3e-3, 2e-2), 6), rng.random() < 0.4, stages,
                      rng.choice([1, 1, 1, 2, 4]), rng.random() < 0.3))
    opts = {"kappa": rng.choice([0.0, 0.0, 0.2]), "hpa": rng.random() < 0.3,
            "edf": rng.random() < 0.2, "no_fixed": rng.random() < 0.15, "no_last": rng.random() < 0.15,
            "no_prior": rng.random() < 0.15, "no_staging": rng.random() < 0.1,
            "order": rng.choice(["descending_util", "insertion"]), "phasing": rng.choice(["random", "zero"]),
            "ws": rng.choice([3, 5, 8])}
    return nc, ns, sms, os_, tasks, opts


def _run(mod, inst, seed):
    nc, ns, sms, os_, tasks, o = inst
    specs, batch, curves = [], {}, {}
    for tid, period, hp, stages, b, curved in tasks:
        pri = mod.Priority.HP if hp else mod.Priority.LP
        specs.append(mod.TaskSpec.periodic(tid, period, pri, tuple(mod.StageProfile(n, w) for n, w in stages)))
        batch[tid] = b
        if curved:
            curves[tid] = mod.BatchingCurve(4, 1.6)
    cfg = mod.GpuConfig(sms, nc, ns, os_, mod.Policy.MPS_STR, o["kappa"])
    flags = mod.AblationFlags(no_staging=o["no_staging"], no_last=o["no_last"], no_prior=o["no_prior"],
                              no_fixed=o["no_fixed"])
    sim = mod.Simulation(specs, cfg, seed=seed, duration=0.2, warmup_frac=0.1, window_size=o["ws"],
                         full_load_reps=2, batch_sizes=batch, curves=curves, flags=flags,
                         mode=mod.SchedulerMode(hpa_enabled=o["hpa"]), phasing=o["phasing"],
                         placement_order=o["order"], edf_on_job_deadline=o["edf"])
    res = sim.run()
    recs = [tuple(r) for r in res.records]
    audits = [(a.time, a.job_id, a.task_id, a.priority.value, a.context, a.active_util, a.job_util, a.limit,
               a.admitted) for a in res.admissions]
    return recs, audits, res.report.to_dict(), dict(res.full_load)


@pytest.mark.parametrize("block", range(10))
def test_native_equals_reference_on_random_instances(block):
    import paper_2504_08795_b200 as ours
    ref = _ref()
    per = (N + 9) // 10
    for k in range(block * per, min(N, (block + 1) * per)):
        rng = random.Random(20_000 + k)
        inst = _instance(rng)
        want = _run(ref, inst, seed=k)
        got = _run(ours, inst, seed=k)
        assert got[0] == want[0], f"instance {k}: event logs differ"
        assert got[1] == want[1], f"instance {k}: admission audits differ"
        assert got[2] == want[2], f"instance {k}: reports differ"
        assert got[3] == want[3], f"instance {k}: AFET values differ"


def _trace_instance(rng):
    nc, ns, sms, os_, tasks, _ = _instance(rng)
    tasks = [(tid, period, hp, stages) for tid, period, hp, stages, _, _ in tasks]
    # per-(task, job, stage) durations, like a recorded GPU trace; jobs are numbered
    # globally in release order, so cover every job id the run can reach
    durations = {}
    for job in range(1, 800):
        for tid, _, _, stages in tasks:
            for j, (nom, _) in enumerate(stages):
                durations[(tid, job, j)] = round(nom * rng.uniform(0.6, 2.5), 9)
    full = {tid: round(sum(n for n, _ in st) * rng.uniform(1.0, 2.0), 9) for tid, _, _, st in tasks}
    return nc, ns, sms, os_, tasks, durations, full


@pytest.mark.parametrize("block", range(4))
def test_trace_replay_equals_reference_on_random_traces(block, monkeypatch):
    """P2's replay engine: fixed per-stage durations and given AFETs
    through this package's native trace engine vs the unmodified reference with
    the trace shim (unit rates, traced stage work, traced AFETs)."""
    import paper_2504_08795_b200 as ours
    ref = _ref()
    import stagesim.engine as E
    from stagesim.gpu import RateAllocation

    per = 50
    for k in range(block * per, (block + 1) * per):
        rng = random.Random(40_000 + k)
        nc, ns, sms, os_, tasks, durations, full = _trace_instance(rng)
        orig_make_job = E.make_job

        def traced_make_job(task, release_time, tracker, _orig=orig_make_job, **kw):
            job = _orig(task, release_time, tracker, **kw)
            for st in job.stage_jobs:
                st.remaining_work = durations[(job.task_id, job.job_id, st.stage_index)]
            return job

        monkeypatch.setattr(E, "make_job", traced_make_job)
        monkeypatch.setattr(E, "allocate_rates",
                            lambda active, config: RateAllocation([0.0] * len(active), [1.0] * len(active), 1.0, {}))
        monkeypatch.setattr(E.Simulation, "_measure_full_load", lambda self, eff: {t.id: full[t.id] for t in eff})

        def specs(mod):
            return [mod.TaskSpec.periodic(tid, period, mod.Priority.HP if hp else mod.Priority.LP,
                                          tuple(mod.StageProfile(n, w) for n, w in st))
                    for tid, period, hp, st in tasks]

        ref_res = ref.Simulation(specs(ref), ref.GpuConfig(sms, nc, ns, os_, ref.Policy.MPS_STR), seed=k,
                                 duration=0.2).run()
        monkeypatch.undo()
        ours_res = ours.Simulation(specs(ours), ours.GpuConfig(sms, nc, ns, os_, ours.Policy.MPS_STR), seed=k,
                                   duration=0.2).run_trace(durations, full)
        assert [tuple(r) for r in ours_res.records] == [tuple(r) for r in ref_res.records], f"trace {k}"
        assert ours_res.report.to_dict() == ref_res.report.to_dict(), f"trace {k}"
