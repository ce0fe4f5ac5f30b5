"""The drop-in scenario API's real-GPU backend: ``"backend": "gpu"`` in a
scenario runs the task set on the B200 through the native executor and
returns the reference's SimResult shape; its recorded stage trace replays
through the native trace engine (Simulation.run_trace) and the oracle with
identical decisions."""

import pytest

import paper_2504_08795_b200 as S
from oracle import stagesim_oracle as O
from paper_2504_08795_b200.errors import InvalidScenario, SchemaError
from paper_2504_08795_b200.gpu_backend import GpuSimulation


def test_presets_name_networks():
    for name, models in (("c1_b200", {"resnet18"}), ("c2_b200", {"resnet50"}),
                         ("c3_b200", {"resnet18", "resnet50", "vgg16", "mobilenet_v2"})):
        cfg = S.scenario_from_dict({"preset": name, "backend": "gpu"})
        assert cfg.backend == "gpu"
        assert {g.model for g in cfg.models.values()} == models
        assert set(cfg.models) == {t.id for t in cfg.tasks}
    c3 = S.scenario_from_dict({"preset": "c3_b200"})
    hp = sum(t.priority is S.Priority.HP for t in c3.tasks)
    assert hp * 2 == len(c3.tasks) and c3.stage_migration


def test_sim_backend_runs_b200_presets():
    for name in ("c1_b200", "c2_b200", "c3_b200"):
        res = S.build_simulation(S.scenario_from_dict({"preset": name, "duration": 1.0})).run()
        assert res.report.completed_hp > 0


def test_gpu_backend_schema():
    base = {"backend": "gpu", "gpu": {"total_sms": 148, "n_contexts": 2, "n_streams": 2}}
    cfg = S.scenario_from_dict({**base, "workload": {"tasks": [
        {"id": 1, "period": 0.01, "priority": "hp", "model": "vgg16"},
        {"id": 2, "period": 0.01, "priority": "lp", "model": "resnet18", "n_stages": 2}]}})
    assert [len(t.stages) for t in cfg.tasks] == [4, 2]
    assert cfg.models[2].n_stages == 2
    with pytest.raises(SchemaError):
        S.scenario_from_dict({**base, "workload": {"tasks": [
            {"id": 1, "period": 0.01, "priority": "hp", "model": "unet"}]}})
    with pytest.raises(SchemaError):
        S.scenario_from_dict({**base, "backend": "tpu"})
    with pytest.raises(InvalidScenario):      # unet has no network: fail closed, no fallback
        S.scenario_from_dict({**base, "workload": {"preset": "unet"}})
    cfg = S.scenario_from_dict({**base, "workload": {"preset": "c2_resnet50_b200", "batch_size": 4}})
    assert set(cfg.batch_sizes.values()) == {4}   # batched jobs run as real batch-4 networks
    with pytest.raises(InvalidScenario):
        S.scenario_from_dict({**base, "workload": {"preset": "c2_resnet50_b200", "batch_size": 128}})


def test_gpu_backend_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    sim = S.build_simulation(S.scenario_from_dict({"preset": "c1_b200", "backend": "gpu", "duration": 0.2}))
    assert isinstance(sim, GpuSimulation)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sim.run()


def _cut(records, horizon):
    return [tuple(r[:7]) for r in records if r[1] != "sim_end" and r[0] <= horizon]


@pytest.mark.gpu
@pytest.mark.parametrize("preset,rate", [("c1_b200", 200.0), ("c3_b200", 250.0), ("c2_b200", 1500.0)])
def test_gpu_scenario_runs_and_replays(preset, rate):
    """c2_b200 at 1500 JPS/task is BASELINE config C2 at full size near its knee
    (8 ResNet-50 tasks, 4x2 contexts/streams, OS 2: ~7k stage decisions/0.6 s)."""
    cfg = S.scenario_from_dict({"preset": preset, "backend": "gpu", "duration": 0.6,
                                "workload": {"preset": {"c1_b200": "c1_resnet18_b200",
                                                        "c2_b200": "c2_resnet50_b200",
                                                        "c3_b200": "c3_mixed_b200"}[preset]}})
    # one rate for every task so the run is light enough for any box
    from dataclasses import replace
    cfg = replace(cfg, tasks=[replace(t, period=1.0 / rate, deadline=1.0 / rate) for t in cfg.tasks])
    sim = S.build_simulation(cfg)
    res = sim.run()
    rep = res.report
    assert rep.completed_hp > 0 and rep.completed_lp > 0
    assert res.stats["graph_launches"] > 0 and res.trace
    assert all(p["green"] for p in res.partitions)
    # the real run's event log in the reference wire format, audited from the log alone
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        path = f"{d}/events.jsonl"
        S.write_event_log(path, [res])
        recs = S.read_event_log(path)
    from paper_2504_08795_b200.runtime import quantize  # the executor's 2^-20 s time grid
    horizon, warm = quantize(cfg.duration), quantize(cfg.duration * cfg.warmup_frac)
    S.check_event_order(recs, horizon)
    rep = S.replay_metrics(recs, res.effective_tasks, duration=horizon, warmup_end=warm)
    assert S.compare_with_report(rep, res.report) == []
    # same decisions through the native trace engine of the drop-in API ...
    eff = res.effective_tasks
    replay = S.Simulation(eff, cfg.gpu, seed=cfg.seed, duration=cfg.duration, warmup_frac=cfg.warmup_frac,
                          stage_migration=cfg.stage_migration).run_trace(res.stage_durations(), res.full_load,
                                                                          phases=res.phases,
                                                                          unsampled=res.unsampled())
    assert _cut(res.records, cfg.duration) == _cut(replay.records, cfg.duration)
    assert res.report.missed_hp == replay.report.missed_hp
    # ... and through the oracle restatement of the reference scheduler (its
    # independent stage-migration mode for the C3 migration run)
    otasks = [{"id": t.id, "period": t.period, "deadline": t.deadline, "hp": t.priority is S.Priority.HP,
               "stages": [(p.nominal_time, p.width) for p in t.stages], "batch": 1, "curve": None,
               "full_load": res.full_load[t.id]} for t in eff]
    g = cfg.gpu
    ogpu = {"total_sms": g.total_sms, "n_contexts": g.n_contexts, "n_streams": g.n_streams,
            "oversubscription": g.oversubscription, "policy": g.policy.value, "kappa": 0.0}
    recs, _, _, _ = O.simulate(otasks, ogpu, duration=cfg.duration, warmup_frac=cfg.warmup_frac,
                               durations=res.stage_durations(),
                               phases_override={t.id: ph for t, ph in zip(eff, res.phases)},
                               stage_migration=cfg.stage_migration, unsampled=res.unsampled())
    assert _cut(res.records, cfg.duration) == _cut(recs, cfg.duration)
    sim.close()
