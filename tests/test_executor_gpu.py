"""Real-GPU executor: green-context partitions, stage graphs, the wall-clock
DARIS loop, and P2 trace-replay parity (the recorded per-stage durations
replayed through the oracle scheduler give the same decisions)."""

import pytest
import torch

from oracle import stagesim_oracle as O
from paper_2504_08795_b200 import nets
from paper_2504_08795_b200.gpu import GpuConfig, Policy
from paper_2504_08795_b200.model import Priority
from paper_2504_08795_b200.runtime import DarisRuntime, TaskDef, quantize

pytestmark = pytest.mark.gpu


def _runtime(n_ctx=2, n_str=2, os_=1.0, model="resnet18", rate=200.0, n_tasks=4, **kw):
    gpu = GpuConfig(148, n_ctx, n_str, os_, Policy.MPS_STR)
    tasks = [TaskDef(i + 1, model, Priority.HP if i % 2 == 0 else Priority.LP, rate) for i in range(n_tasks)]
    return DarisRuntime(tasks, gpu, slots=2, **kw)


@pytest.mark.parametrize("n_ctx,n_str,os_,target", [(4, 2, 2.0, 74), (2, 2, 1.0, 74), (4, 1, 1.0, 38)])
def test_partitions_are_green_and_sized(n_ctx, n_str, os_, target):
    """Green partitions over the 8-SM co-scheduled groups plus the 28-SM split
    remainder: each within half a group of ceil_even(OS * 148 / N_c), and
    together covering the device OS times (all 148 SMs in use)."""
    rt = _runtime(n_ctx=n_ctx, n_str=n_str, os_=os_)
    parts = rt.exec.partitions
    assert all(p["green"] for p in parts), parts
    for p in parts:
        assert abs(p["sm_count"] - target) <= 8, p  # within one 8-SM group
    assert sum(p["sm_count"] for p in parts) == round(os_ * 148), parts
    rt.close()


def _decisions(records, horizon):
    keep = []
    for r in records:
        if r[1] == "sim_end" or r[0] > horizon:
            continue
        keep.append((r[0], r[1], r[2], r[3], r[4], r[5], r[6]))
    return keep


@pytest.mark.parametrize("model,flags", [("resnet18", "0"), ("resnet50", "0"), ("resnet50", "1")])
def test_real_run_and_trace_replay_parity(model, flags, monkeypatch):
    """flags=1: stage completions observed through host-mapped flags written by
    cuStreamWriteValue32 (DARIS_EXEC_FLAGS=1) instead of event polling."""
    monkeypatch.setenv("DARIS_EXEC_FLAGS", flags)
    rt = _runtime(model=model, rate=150.0)
    res = rt.run(duration=1.0, warmup=0.1)
    rep = res.report
    assert rep.completed_hp + rep.completed_lp > 100
    assert res.stats["graph_launches"] > 0
    # P2: replay the recorded stage durations through the oracle scheduler
    durations = {(t[0], t[1], t[2]): t[7] - t[6] for t in res.trace}
    tasks = []
    for spec in res.tasks:
        tasks.append({"id": spec.id, "period": spec.period, "deadline": spec.deadline,
                      "hp": spec.priority is Priority.HP,
                      "stages": [(p.nominal_time, p.width) for p in spec.stages], "batch": 1, "curve": None,
                      "full_load": res.full_load[spec.id]})
    gpu = {"total_sms": 148, "n_contexts": 2, "n_streams": 2, "oversubscription": 1.0, "policy": "mps-str",
           "kappa": 0.0}
    phases = {spec.id: ph for spec, ph in zip(res.tasks, res.phases)}
    recs, audits, report, _ = O.simulate(tasks, gpu, duration=1.0, warmup_frac=0.1, durations=durations,
                                         phases_override=phases, unsampled=res.unsampled())
    horizon = 1.0
    real = _decisions(res.records, horizon)
    replay = _decisions(recs, horizon)
    assert real == replay
    rt.close()


def test_e2e_mode_copies_inputs_and_outputs():
    rt = _runtime(rate=100.0, e2e=True)
    res = rt.run(duration=0.5, warmup=0.05)
    assert res.stats["copies_h2d"] > 0 and res.stats["copies_d2h"] > 0
    out = rt.host_out[1]
    assert torch.isfinite(out).all() and out.abs().sum() > 0
    rt.close()


def test_batched_jobs_count_images_and_replay():
    """Tasks whose jobs are batches of images (the reference's batch_size): the
    report counts images, and the recorded trace replays to the same decisions."""
    gpu = GpuConfig(148, 2, 2, 1.0, Policy.MPS_STR)
    tasks = [TaskDef(1, "resnet18", Priority.HP, 150.0, 3, 4), TaskDef(2, "resnet18", Priority.LP, 150.0, 3, 4)]
    rt = DarisRuntime(tasks, gpu, slots=2)
    res = rt.run(duration=0.5, warmup=0.05)
    rep = res.report
    jobs = rep.completed_hp + rep.completed_lp
    assert jobs > 0 and rep.missed_hp == 0
    assert abs(rep.jps * (quantize(0.5) - quantize(0.05)) - 4 * jobs) < 1e-6 * 4 * jobs + 1e-9
    assert "resnet18@b4" in rt.stage_nominal
    durations = {(t[0], t[1], t[2]): t[7] - t[6] for t in res.trace}
    otasks = [{"id": s.id, "period": s.period, "deadline": s.deadline, "hp": s.priority is Priority.HP,
               "stages": [(p.nominal_time, p.width) for p in s.stages], "batch": 4, "curve": None,
               "full_load": res.full_load[s.id]} for s in res.tasks]
    ogpu = {"total_sms": 148, "n_contexts": 2, "n_streams": 2, "oversubscription": 1.0, "policy": "mps-str",
            "kappa": 0.0}
    recs, _, _, _ = O.simulate(otasks, ogpu, duration=0.5, warmup_frac=0.1, durations=durations,
                               phases_override={s.id: ph for s, ph in zip(res.tasks, res.phases)},
                               unsampled=res.unsampled())
    assert _decisions(res.records, 0.5) == _decisions(recs, 0.5)
    rt.close()


def test_buffer_sets_never_shared_under_backlog():
    """More live jobs of one task than it has buffer sets (an HP task released
    far faster than it completes; HP jobs are never admission-tested): a job
    takes over a set only after the holder launched its last stage (ordered
    behind it on the GPU), later jobs wait in a FIFO and hold their stage-0
    launch. Every buffer set's final logits must be those of the last job that
    used it, computed from that job's own input image — any overlap of two jobs
    on one set (activations, split-K scratch / counters) would corrupt them —
    and a normal run afterwards must still be exact."""
    gpu = GpuConfig(148, 1, 3, 1.0, Policy.STR)
    tasks = [TaskDef(1, "resnet50", Priority.HP, 20000.0, 4)]
    rt = DarisRuntime(tasks, gpu, slots=2, phasing="zero")
    rt.capture_all()
    rt.afet = {1: 1e-3}
    res = rt.run(duration=0.05, warmup=0.0, full_load=rt.afet)
    st = res.stats
    assert st["slot_deferred"] > 0 and st["slot_backlog_max"] >= 2, st
    assert res.report.completed_hp > 10
    net = rt.net_of(rt.tasks[0])
    pool = rt.pools[1]
    ref_tb = nets.allocate_buffers(net, rt.plan_of(rt.tasks[0]))

    def logits(img_index):
        out = nets.forward(net, ref_tb, pool[img_index:img_index + 1], stream=None,
                           sm_budget=rt.plan_of(rt.tasks[0])).float().cpu().clone()
        torch.cuda.synchronize()
        return out

    last = {}
    n_st = net.n_stages
    for t in res.trace:   # (task, job, stage, ctx, stream, slot, start, end, ...)
        if t[2] == n_st - 1 and (t[5] not in last or t[7] >= last[t[5]][1]):
            last[t[5]] = (t[1], t[7])
    assert len(last) == 2
    for slot, (job, _) in last.items():
        got = rt.buffers[(1, slot)].output.float().cpu()
        want = logits((job - 1) % rt.pool_size)   # one task, no rejections: job j used image j-1
        cos = torch.nn.functional.cosine_similarity(got.flatten(), want.flatten(), dim=0).item()
        assert cos > 0.9999, (slot, job, cos)
    rt.close()
