"""P2 parity on a trace recorded on the B200 (tests/golden/gpu_trace_*.json.gz,
made by tools/record_trace.py): the per-stage durations of the real run are
replayed through (a) the oracle and (b) the unmodified reference scheduler
(stagesim, imported from /root/reference when present, with the SURVEY §7
shim: unit rates, traced stage work, traced AFETs). Decisions — event kinds,
tasks, jobs, stages, contexts, streams — and their times must equal the real
run's log up to the horizon.

Fixtures (round 2, B200, 4 contexts x 2 streams, OS=2): gpu_trace_r02_c2 (8
ResNet-50 tasks near the knee, LP rejections and release-time migrations),
gpu_trace_r02_c3 (the mixed ResNet-18/50 / VGG-16 / MobileNetV2 set) and
gpu_trace_r02_c3mig* (the same with stage-level migration; replayed through the
oracle's stage-migration mode only — the reference has no such mode)."""

import gzip
import json
import sys
from pathlib import Path

import pytest

from oracle import stagesim_oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden"
TRACES = sorted(GOLDEN.glob("gpu_trace_*.json.gz"))
REF_SRC = Path("/root/reference/pkg/src")


def _load(path):
    with gzip.open(path, "rt") as fh:
        return json.load(fh)


def _decisions(records, horizon):
    return [tuple(r[:7]) for r in records if r[1] != "sim_end" and r[0] <= horizon]


def _durations(data):
    return {(t[0], t[1], t[2]): t[7] - t[6] for t in data["trace"]}


def _unsampled(data):
    """Stages the run completed without an MRET sample (in flight across a
    detected GPU-wide pause; 9th trace field 0). Older traces have no field."""
    return {(t[0], t[1], t[2]) for t in data["trace"] if len(t) > 8 and not t[8]}


@pytest.mark.parametrize("path", TRACES, ids=[p.name for p in TRACES])
def test_gpu_trace_replays_through_oracle(path):
    data = _load(path)
    tasks = [{"id": t["id"], "period": t["period"], "deadline": t["deadline"], "hp": t["hp"],
              "stages": [(n, w) for n, w in t["stages"]], "batch": 1, "curve": None,
              "full_load": data["full_load"][str(t["id"])]} for t in data["tasks"]]
    recs, _, _, _ = O.simulate(tasks, data["gpu"], duration=data["duration"], warmup_frac=data["warmup_frac"],
                               phasing=data["phasing"], durations=_durations(data),
                               stage_migration=data.get("stage_migration", False), unsampled=_unsampled(data))
    assert _decisions(recs, data["duration"]) == _decisions(data["records"], data["duration"])


def _stage_moves(records):
    admit = {(r[2], r[3]): r[5] for r in records if r[1] == "admit"}
    return sum(1 for r in records if r[1] == "stage_start" and admit[(r[2], r[3])] != r[5])


def test_fixtures_cover_rejections_and_migrations():
    """The committed traces exercise the risky paths: LP admission rejections,
    release-time (task) migration, and in-flight stage moves."""
    data = {p.name: _load(p) for p in TRACES}
    assert any(sum(1 for r in d["records"] if r[1] == "reject") > 0 for d in data.values())
    for d in data.values():
        homes, moved = {}, 0
        for r in d["records"]:
            if r[1] == "admit":
                moved += r[2] in homes and homes[r[2]] != r[5]
                homes[r[2]] = r[5]
        assert moved > 0
    assert any(d.get("stage_migration") and _stage_moves(d["records"]) > 0 for d in data.values())


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference sources not mounted (GPU box)")
@pytest.mark.parametrize("path", TRACES, ids=[p.name for p in TRACES])
def test_gpu_trace_replays_through_reference(path, monkeypatch):
    data = _load(path)
    if data.get("stage_migration"):
        pytest.skip("stage-level migration is an extension the reference does not have")
    if _unsampled(data):
        pytest.skip("pause-excluded MRET samples are an executor extension the reference does not have")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import stagesim
    import stagesim.engine as E
    from stagesim.gpu import RateAllocation

    durations = _durations(data)
    full = {int(k): v for k, v in data["full_load"].items()}
    orig_make_job = E.make_job

    def traced_make_job(task, release_time, tracker, **kw):
        job = orig_make_job(task, release_time, tracker, **kw)
        for st in job.stage_jobs:
            key = (job.task_id, job.job_id, st.stage_index)
            if key in durations:
                st.remaining_work = durations[key]
        return job

    def unit_rates(active, config):
        n = len(active)
        return RateAllocation([0.0] * n, [1.0] * n, 1.0, {})

    monkeypatch.setattr(E, "make_job", traced_make_job)
    monkeypatch.setattr(E, "allocate_rates", unit_rates)
    monkeypatch.setattr(E.Simulation, "_measure_full_load", lambda self, eff: {t.id: full[t.id] for t in eff})
    g = data["gpu"]
    gpu = stagesim.GpuConfig(g["total_sms"], g["n_contexts"], g["n_streams"], g["oversubscription"],
                             stagesim.Policy(g["policy"]))
    specs = [stagesim.TaskSpec(t["id"], t["period"], t["deadline"],
                               stagesim.Priority.HP if t["hp"] else stagesim.Priority.LP,
                               tuple(stagesim.StageProfile(n, w) for n, w in t["stages"])) for t in data["tasks"]]
    res = stagesim.Simulation(specs, gpu, duration=data["duration"], warmup_frac=data["warmup_frac"],
                              phasing=data["phasing"]).run()
    assert _decisions([list(r) for r in res.records], data["duration"]) == \
        _decisions(data["records"], data["duration"])


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference sources not mounted (GPU box)")
@pytest.mark.parametrize("path", TRACES, ids=[p.name for p in TRACES])
def test_reference_checkers_audit_real_gpu_log(path):
    """The reference's own log auditors (replay.py:25-190) on the B200 run's
    event log: time order and horizon, every metric recomputed from the log
    equal to the executor's accumulator (the build adds p99, which the
    reference does not report), and — where jobs stay in their admission
    context — no context idling a stream while it has ready work."""
    data = _load(path)
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import stagesim
    from stagesim import replay as R

    recs = [tuple(r) for r in data["records"]]
    specs = [stagesim.TaskSpec(t["id"], t["period"], t["deadline"],
                               stagesim.Priority.HP if t["hp"] else stagesim.Priority.LP,
                               tuple(stagesim.StageProfile(n, w) for n, w in t["stages"])) for t in data["tasks"]]
    horizon = next(r[0] for r in recs if r[1] == "sim_end")   # the executor's 2^-20 s grid
    R.check_event_order(recs, horizon)
    rep = data["report"]
    replayed = R.replay_metrics(recs, specs, duration=horizon, warmup_end=rep["warmup"])
    for key, value in replayed.items():
        want = rep[key]
        if isinstance(value, dict):
            want = {k: v for k, v in want.items() if k != "p99"}
        assert value == want, key
    if not data.get("stage_migration"):   # the checker assumes successors stay in the job's context
        R.check_work_conservation(recs, specs, n_contexts=data["gpu"]["n_contexts"],
                                  n_streams=data["gpu"]["n_streams"])
