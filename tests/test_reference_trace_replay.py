"""P2 parity on a trace recorded on the B200 (tests/golden/gpu_trace_*.json.gz,
made by tools/record_trace.py): the per-stage durations of the real run are
replayed through (a) the oracle and (b) the unmodified reference scheduler
(stagesim, imported from /root/reference when present, with the SURVEY §7
shim: unit rates, traced stage work, traced AFETs). Decisions — event kinds,
tasks, jobs, stages, contexts, streams — and their times must equal the real
run's log up to the horizon."""

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


@pytest.mark.parametrize("path", TRACES, ids=[p.name for p in TRACES])
def test_gpu_trace_replays_through_oracle(path):
    data = _load(path)
    tasks = [{"id": t["id"], "period": t["period"], "deadline": t["deadline"], "hp": t["hp"],
              "stages": [(n, w) for n, w in t["stages"]], "batch": 1, "curve": None,
              "full_load": data["full_load"][str(t["id"])]} for t in data["tasks"]]
    recs, _, _, _ = O.simulate(tasks, data["gpu"], duration=data["duration"], warmup_frac=data["warmup_frac"],
                               phasing=data["phasing"], durations=_durations(data))
    assert _decisions(recs, data["duration"]) == _decisions(data["records"], data["duration"])


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference sources not mounted (GPU box)")
@pytest.mark.parametrize("path", TRACES, ids=[p.name for p in TRACES])
def test_gpu_trace_replays_through_reference(path, monkeypatch):
    data = _load(path)
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
