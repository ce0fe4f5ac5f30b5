"""The object-level drop-in API (Scheduler / TimingTracker / TaskState / make_job
/ build_contexts over Python-owned state, as the reference's tests drive it)
and the stateful native dispatcher behind the engine and the GPU executor make
the same decisions: a trace-replay event loop written against the object API
(the reference engine's loop, engine.py:417-531, with unit rates) produces the
native trace engine's event log record for record on random instances — with
and without stage-level migration — and the native engine's stage-migration
mode equals the oracle's independent restatement of that rule."""

from __future__ import annotations

import heapq
import random

import pytest

from oracle import stagesim_oracle as O
from paper_2504_08795_b200 import Simulation
from paper_2504_08795_b200.gpu import (GpuConfig, Policy, RateAllocation, advance_progress, build_contexts,
                                       next_completion)
from paper_2504_08795_b200.model import Priority, StageProfile, StageState, TaskSpec, TaskState, make_job
from paper_2504_08795_b200.scheduler import AblationFlags, Scheduler, SchedulerMode
from paper_2504_08795_b200.timing import TimingTracker


def _instance(rng):
    nc = rng.randint(2, 4)
    ns = rng.randint(1, 3)
    specs = []
    for i in range(rng.randint(2, 7)):
        period = round(rng.uniform(2e-3, 8e-3), 6)
        stages = tuple(StageProfile(round(rng.uniform(2e-4, 2e-3), 7), 16) for _ in range(rng.randint(1, 4)))
        specs.append(TaskSpec.periodic(i + 1, period, Priority.HP if rng.random() < 0.4 else Priority.LP, stages))
    full = {s.id: round(sum(p.nominal_time for p in s.stages) * rng.uniform(1.0, 2.5), 7) for s in specs}
    phases = [round(rng.random() * s.period, 7) for s in specs]
    durations = {}
    for s in specs:
        for j in range(400):
            for k, p in enumerate(s.stages):
                durations[(s.id, j, k)] = round(p.nominal_time * rng.uniform(0.6, 2.5), 7)
    opts = {"hpa": rng.random() < 0.2, "edf": rng.random() < 0.2,
            "flags": AblationFlags(no_last=rng.random() < 0.15, no_prior=rng.random() < 0.15,
                                   no_fixed=rng.random() < 0.15),
            "order": rng.choice(["descending_util", "insertion"]), "ws": rng.choice([3, 5])}
    return GpuConfig(148, nc, ns, 1.0, Policy.MPS_STR), specs, full, phases, durations, opts


def _object_loop(gpu, specs, full, phases, durations, o, duration, stage_migration):
    """engine.py:417-531 in trace mode (rate 1), driven through the object API."""
    states = [TaskState.fresh(s, o["ws"]) for s in specs]
    for st in states:
        st.full_load_time = full[st.task.id]
    tracker = TimingTracker(states)
    contexts = build_contexts(gpu)
    sched = Scheduler(tracker, contexts, gpu, flags=o["flags"], mode=SchedulerMode(o["hpa"]),
                      placement_order=o["order"], edf_on_job_deadline=o["edf"], stage_migration=stage_migration)
    sched.populate_contexts(states)
    by_id = {st.task.id: st for st in states}
    recs = []
    heap = [(ph, s.id) for s, ph in zip(specs, phases) if ph < duration]
    heapq.heapify(heap)
    nrel = {s.id: 0 for s in specs}
    phase = {s.id: ph for s, ph in zip(specs, phases)}
    running = []       # active stages in (context, stream) order
    jcount = 0
    now = 0.0

    def refill():
        for ctx in contexts:
            while True:
                k = ctx.free_stream_index()
                if k is None:
                    break
                stage = sched.dispatch(ctx.id, now)
                if stage is None:
                    break
                stage.transition(StageState.RUNNING)
                stage.started_at, stage.context, stage.stream = now, ctx.id, k
                ctx.streams[k].occupant = stage
                recs.append((now, "stage_start", stage.task_id, stage.job_id, stage.stage_index, ctx.id, k))
        running[:] = [sl.occupant for c in contexts for sl in c.streams if sl.occupant is not None]

    while True:
        active = [(s, s.context) for s in running]
        unit = RateAllocation([0.0] * len(active), [1.0] * len(active), 1.0, {})
        cands = [(duration, 2)] + ([(heap[0][0], 0)] if heap else [])
        if active:
            _, fin, t_fin = next_completion(active, unit, now)
            cands.append((t_fin, 1))
        t_ev, kind = min(cands)
        if active:
            advance_progress(active, unit, t_ev - now)
        now = t_ev
        if kind == 2:
            break
        if kind == 0:
            _, tid = heapq.heappop(heap)
            jcount += 1
            job = make_job(by_id[tid], now, tracker, job_id=jcount)
            for sj in job.stage_jobs:
                sj.remaining_work = durations[(tid, jcount, sj.stage_index)]
            recs.append((now, "release", tid, jcount, None, None, None))
            pl = sched.admit_or_migrate(job, now)
            recs.append((now, "reject", tid, jcount, None, None, None) if pl.rejected
                        else (now, "admit", tid, jcount, None, pl.context, None))
            nrel[tid] += 1
            nxt = phase[tid] + nrel[tid] * by_id[tid].task.period
            if nxt < duration:
                heapq.heappush(heap, (nxt, tid))
        else:
            contexts[fin.context - 1].streams[fin.stream].occupant = None
            done, _ = sched.complete_stage(fin, now)
            recs.append((now, "stage_complete", fin.task_id, fin.job_id, fin.stage_index, fin.context, fin.stream))
            if done:
                recs.append((now, "job_complete", fin.task_id, fin.job_id, None, fin.context, None))
        refill()
    return recs


def _native(gpu, specs, full, phases, durations, o, duration, stage_migration):
    sim = Simulation(specs, gpu, duration=duration, warmup_frac=0.1, window_size=o["ws"], flags=o["flags"],
                     mode=SchedulerMode(o["hpa"]), placement_order=o["order"], edf_on_job_deadline=o["edf"],
                     stage_migration=stage_migration)
    res = sim.run_trace(durations, full, phases=phases)
    return [tuple(r[:7]) for r in res.records if r[1] != "sim_end"]


def _oracle(gpu, specs, full, phases, durations, o, duration, stage_migration):
    tasks = [{"id": s.id, "period": s.period, "deadline": s.deadline, "hp": s.priority is Priority.HP,
              "stages": [(p.nominal_time, p.width) for p in s.stages], "batch": 1, "curve": None,
              "full_load": full[s.id]} for s in specs]
    g = {"total_sms": gpu.total_sms, "n_contexts": gpu.n_contexts, "n_streams": gpu.n_streams,
         "oversubscription": gpu.oversubscription, "policy": gpu.policy.value, "kappa": 0.0}
    f = o["flags"]
    recs, _, _, _ = O.simulate(tasks, g, duration=duration, warmup_frac=0.1, ws=o["ws"], hpa=o["hpa"],
                               no_last=f.no_last, no_prior=f.no_prior, no_fixed=f.no_fixed,
                               placement_order=o["order"], edf_on_job_deadline=o["edf"], durations=durations,
                               phases_override={s.id: ph for s, ph in zip(specs, phases)},
                               stage_migration=stage_migration)
    return [tuple(r[:7]) for r in recs if r[1] != "sim_end"]


def _stage_moves(recs):
    admit = {(r[2], r[3]): r[5] for r in recs if r[1] == "admit"}
    return sum(1 for r in recs if r[1] == "stage_start" and admit[(r[2], r[3])] != r[5])


@pytest.mark.parametrize("mig", [False, True], ids=["task-migration", "stage-migration"])
def test_object_api_decides_like_the_native_dispatcher(mig):
    rng = random.Random(11 + mig)
    moves = 0
    for _ in range(60):
        inst = _instance(rng)
        ours = _object_loop(*inst, duration=0.06, stage_migration=mig)
        native = _native(*inst, duration=0.06, stage_migration=mig)
        assert ours == native
        moves += _stage_moves(native)
    assert (moves > 0) == mig   # the migration runs really move in-flight jobs


def test_native_stage_migration_matches_oracle_rule():
    rng = random.Random(5)
    moves = 0
    for _ in range(200):
        inst = _instance(rng)
        native = _native(*inst, duration=0.06, stage_migration=True)
        assert native == _oracle(*inst, duration=0.06, stage_migration=True)
        moves += _stage_moves(native)
    assert moves > 50
