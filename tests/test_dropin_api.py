"""Drop-in boundary: the reference's public API, end to end through the
native core. Golden fixtures store the reference's own scenario dicts, so
`scenario_from_dict -> build_simulation -> run` must reproduce the reference
event log, audits and report exactly."""

import json

import pytest

import paper_2504_08795_b200 as ds
from golden_cases import case_by_name, case_ids
from paper_2504_08795_b200.errors import InvalidScenario, SchemaError, UnknownPreset

REFERENCE_NAMES = [
    "AblationFlags", "AdmissionDecision", "BatchingCurve", "CSV_COLUMNS", "EventKind", "GpuConfig", "Job",
    "LogRecord", "MetricsReport", "Policy", "Priority", "PROFILES", "ResponseStats", "SCENARIO_PRESETS",
    "ScenarioConfig", "Scheduler", "SchedulerMode", "SimResult", "Simulation", "SimulatorError", "StageJob",
    "StageProfile", "StageState", "SweepSpec", "TaskSet", "TaskSpec", "TaskState", "TimingTracker",
    "allocate_rates", "build_profile_tasks", "build_simulation", "build_task_set", "ceil_even",
    "check_admission_audit", "check_event_order", "check_work_conservation", "collapse_stages",
    "compare_with_report", "effective_stage_time", "emit_report", "expand_cells", "format_label", "get_profile",
    "get_scenario_preset", "load_scenario", "load_sweep", "measure_full_load_time", "modeled_capacity",
    "parse_label", "profile_stages", "render_csv", "render_json", "replay_metrics", "report_row", "run_sweep",
    "scale_to_overload", "scenario_from_dict", "sm_per_context", "water_fill",
]


def test_every_reference_name_is_exported():
    missing = [n for n in REFERENCE_NAMES if not hasattr(ds, n)]
    assert not missing


@pytest.mark.parametrize("name", case_ids())
def test_scenario_to_run_reproduces_reference(name):
    case = case_by_name(name)
    res = ds.build_simulation(ds.scenario_from_dict(case["scenario"])).run()
    assert [list(r) for r in res.records] == case["records"]
    assert res.report.to_dict() == case["report"]
    # log-only audits from the reference's replay module agree with the accumulator
    ds.check_event_order(res.records, res.report.duration)
    rep = ds.replay_metrics(res.records, res.effective_tasks, duration=res.report.duration,
                            warmup_end=res.report.warmup,
                            batch_sizes={t["id"]: t["batch"] for t in case["tasks"]})
    assert ds.compare_with_report(rep, res.report) == []
    ds.check_admission_audit(res)
    g = res.report
    ds.check_work_conservation(res.records, res.effective_tasks, n_contexts=g.n_contexts, n_streams=g.n_streams)


def test_schema_is_fail_closed():
    with pytest.raises(SchemaError):
        ds.scenario_from_dict({"preset": "resnet18_main", "bogus": 1})
    with pytest.raises(SchemaError):
        ds.scenario_from_dict({"gpu": {"total_sms": True}})
    with pytest.raises(UnknownPreset):
        ds.scenario_from_dict({"preset": "nope"})
    from paper_2504_08795_b200.errors import InvalidOversubscription
    with pytest.raises(InvalidOversubscription):   # as the reference: GpuConfig raises it directly
        ds.scenario_from_dict({"gpu": {"n_contexts": 2, "oversubscription": 3}})
    with pytest.raises(InvalidScenario):           # ValueError from GpuConfig -> InvalidScenario
        ds.scenario_from_dict({"gpu": {"n_contexts": 2, "policy": "str"}})
    with pytest.raises(SchemaError):
        ds.scenario_from_dict({"workload": {"preset": "mixed", "hp_count": 2}})


def test_preset_expansion_counts():
    assert len(ds.scenario_from_dict({"preset": "resnet18_main"}).tasks) == 51
    assert len(ds.scenario_from_dict({"preset": "unet_main"}).tasks) == 15
    assert len(ds.scenario_from_dict({"preset": "mixed_main"}).tasks) == 93


def test_sweep_grid_and_parallel_equals_sequential(tmp_path):
    spec = ds.load_sweep(_write(tmp_path, {"policies": ["mps-str"], "pairs": [[2, 2]],
                                           "oversubscription": [1, 2], "seeds": [0, 1]}))
    cells, skipped = ds.expand_cells(spec)
    assert [c.label for c in cells] == ["2x2_1", "2x2_2"]
    base = ds.scenario_from_dict({"preset": "resnet18_main", "duration": 0.2})
    seq = ds.run_sweep(spec, base)
    par = ds.run_sweep(spec, base, processes=2)
    assert [r.to_dict() for r in seq.reports] == [r.to_dict() for r in par.reports]
    text = ds.emit_report(seq.reports, "csv")
    assert text.splitlines()[0].split(",") == list(ds.CSV_COLUMNS)


def test_full_grid_cell_count():
    spec = ds.SweepSpec(list(ds.Policy), [(n, 0) for n in range(2, 11)], [1.0, 1.5, 2.0, "nc"])
    cells, _ = ds.expand_cells(spec)
    assert len(cells) == 72   # reference tests/test_sweep_report.py:125-131


def _write(tmp_path, obj):
    p = tmp_path / "sweep.json"
    p.write_text(json.dumps(obj))
    return p


def test_event_log_wire_format_round_trip(tmp_path):
    """JSONL event log (the reference CLI's --emit-event-log format): written,
    read back and audited by the replay checkers; the log-only replay of the
    metrics equals the run's own report."""
    import paper_2504_08795_b200 as S
    cfg = S.scenario_from_dict({"preset": "c2_b200", "duration": 0.5})
    res = S.build_simulation(cfg).run()
    path = tmp_path / "events.jsonl"
    n = S.write_event_log(path, [res])
    recs = S.read_event_log(path)
    assert n == len(recs) == len(res.records) and recs[0]["kind"] == "release"
    assert set(recs[0]) == {"time", "kind", "task", "job", "stage", "context", "stream", "rate"}
    S.check_event_order(recs, cfg.duration)
    rep = S.replay_metrics(recs, res.effective_tasks, duration=cfg.duration,
                           warmup_end=cfg.duration * cfg.warmup_frac)
    assert S.compare_with_report(rep, res.report) == []
