"""Box layer: Algorithm-1 placement at GPU granularity and the multi-process
control plane (world_size 2, gloo on CPU) that bench.py uses at N>1."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_08795_b200.box import BoxTask, aggregate, local_tasks, place_tasks


def test_place_tasks_balances_and_breaks_ties_low():
    tasks = [BoxTask(i + 1, (i % 8) < 4, 1.0) for i in range(16)]
    a = place_tasks(tasks, 2)
    assert sorted(local_tasks(a, 0)) == [1, 3, 5, 7, 9, 11, 13, 15]
    assert sorted(local_tasks(a, 1)) == [2, 4, 6, 8, 10, 12, 14, 16]
    # heaviest first, lightest-total GPU, HP before LP
    b = place_tasks([BoxTask(1, True, 0.5), BoxTask(2, True, 0.9), BoxTask(3, False, 0.2)], 2)
    assert b == {2: 0, 1: 1, 3: 1}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tasks = [BoxTask(i + 1, (i % 8) < 4, 1.0) for i in range(8 * world)]
    mine = local_tasks(place_tasks(tasks, world), rank)
    import torch
    # per-GPU "report": completions proportional to local tasks; reduced like bench.py
    t = torch.tensor([float(len(mine) * 100), float(rank)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    mx = torch.tensor([0.5 + rank], dtype=torch.float64)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    q.put((rank, len(mine), t.tolist(), mx.item()))
    dist.destroy_process_group()


def test_world_size_two_gloo_control_plane():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    out = sorted(q.get(timeout=10) for _ in range(2))
    assert [o[1] for o in out] == [8, 8]
    assert all(o[2] == [1600.0, 1.0] for o in out)
    assert all(o[3] == 1.5 for o in out)


def test_aggregate_box_metrics():
    agg = aggregate([{"completed": 10, "accepted_hp": 5, "missed_hp": 0, "accepted_lp": 5, "missed_lp": 1},
                     {"completed": 12, "accepted_hp": 6, "missed_hp": 0, "accepted_lp": 4, "missed_lp": 0}])
    assert agg["completed"] == 22 and agg["dmr_hp"] == 0.0 and agg["dmr_lp"] == pytest.approx(1 / 9)


def test_box_admission_rules():
    from paper_2504_08795_b200.box import BoxAdmission
    box = BoxAdmission(2, slots_per_gpu=8)
    tasks = [BoxTask(i + 1, (i % 8) < 4, 0.9) for i in range(16)]
    got = box.admit_all(tasks)
    # same as Algorithm 1 placement while every GPU has room
    assert got == place_tasks(tasks, 2)
    assert [round(box.ledgers[g].hp_total, 6) for g in range(2)] == [3.6, 3.6]
    # LP test is strict: lp_total + u < slots - hp_total (3.6 + 1.0 >= 4.4 on both GPUs)
    assert box.admit_task(BoxTask(17, False, 1.0)) is None
    # an HP task is tested on the lowest-total GPU only
    assert box.admit_task(BoxTask(18, True, 0.5)) == 0 and round(box.ledgers[0].hp_total, 6) == 4.1


def test_box_replaces_a_rejected_lp_task_by_predicted_finish():
    from paper_2504_08795_b200.box import BoxAdmission
    box = BoxAdmission(3, slots_per_gpu=4)
    box.admit_all([BoxTask(1, True, 1.5), BoxTask(2, False, 1.0), BoxTask(3, False, 0.5)])
    src = box.home[2]
    assert (box.home[1], src, box.home[3]) == (0, 1, 2)
    box.publish(0, 1.5, 0.0, 0.0, backlog=5e-3)     # GPU 0 passes the LP test but has a long queue
    box.publish(2, 0.0, 0.5, 0.0, backlog=0.4e-3)   # GPU 2: shortest predicted finish
    dst = box.replace_lp(2, t=1.0, mret=3e-4)
    assert dst == 2 and box.home[2] == 2 and 2 in box.ledgers[2].tasks and 2 not in box.ledgers[src].tasks
    with pytest.raises(ValueError):
        box.replace_lp(1, 1.0, 3e-4)                 # HP tasks stay home
    # nowhere to go: every other GPU's LP test fails -> stays
    full = BoxAdmission(2, slots_per_gpu=2)
    full.admit_all([BoxTask(1, True, 1.9), BoxTask(2, True, 1.95), BoxTask(3, False, 0.08)])
    assert full.home == {2: 0, 1: 1, 3: 1}
    assert full.replace_lp(3, 0.0, 1e-4) is None and full.home[3] == 1


def _box_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_08795_b200.box import BoxAdmission
    box = BoxAdmission(world, slots_per_gpu=8)
    box.admit_all([BoxTask(i + 1, (i % 8) < 4, 1.0) for i in range(8 * world)])
    # each rank publishes its own GPU's live numbers; rank 0 sheds LP task 5 (its GPU rejected it)
    box.publish(rank, 4.0, 4.0, 2.0, backlog=(3e-3 if rank == 0 else 1e-3))
    if rank == 0:
        box.ledgers[1].lp_total = 2.0   # rank 0's (stale) view of GPU 1 leaves room
        assert box.replace_lp(5, t=0.5, mret=4e-4) == 1
    box.sync(rank)
    q.put((rank, dict(sorted(box.home.items())), [(L.hp_total, L.lp_total, sorted(L.tasks)) for L in box.ledgers]))
    dist.destroy_process_group()


def test_box_sync_world_size_two_agrees_on_moves():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_box_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    (_, home0, led0), (_, home1, led1) = sorted(q.get(timeout=10) for _ in range(2))
    assert home0 == home1 and home0[5] == 1
    assert led0 == led1
    assert 5 in led0[1][2] and 5 not in led0[0][2] and led0[1][1] == 5.0 and led0[0][1] == 3.0
