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
