"""bench.py's multi-rank flow at world size 2 on CPU (gloo): the box placer's
task split, each rank's own knee search, the min-reduce of the knee rate, the
joint timed-run decision (a run counts only if every rank's windows pass) and
the whole-box metric reduction (value = sum over ranks). Each rank's DARIS
runtime is a stand-in with a known capacity cliff (rank 0 at 1000 jobs/s per
task, rank 1 at 800), so the expected line is computable by hand."""

import json
import os
import socket
from types import SimpleNamespace

import torch.multiprocessing as mp


class _Net:
    n_stages = 4
    stage_bounds = [0, 10, 25, 40, 53]
    flops_per_image = 8.178e9


class FakeDaris:
    def __init__(self, tasks, gpu, cliff):
        self.tasks = tasks
        self.gpu = gpu
        self.cliff = cliff
        self.rate = 0.0
        self.afet = None
        self.nets = {("resnet50", 4, 1): _Net()}
        self.stage_nominal = {"resnet50": [1e-4] * 4}
        self.exec = SimpleNamespace(partitions=[{"sm_count": 72, "green": True}] * gpu.n_contexts)
        self.runs = []

    def capture_all(self):
        return 0

    def calibrate_full_load(self, seconds):
        return {t.id: 4e-4 for t in self.tasks}

    def set_rate(self, r):
        self.rate = r

    def use_host_io(self, on):
        pass

    def close(self):
        pass

    def run(self, duration, warmup, full_load=None):
        r, n_tasks = self.rate, len(self.tasks)
        self.runs.append(r)
        ok = r < self.cliff

        def windows(warm, step, n):
            return [{"released_hp": 10, "released_lp": 10, "missed_hp": 0 if ok else 2, "missed_lp": 0,
                     "rejected_lp": 0, "lp_loss": 0.0, "completed_images": int(r * n_tasks * step),
                     "stalls": 0} for _ in range(n)]
        stats = {k: 0 for k in ("graph_launches", "slot_waits", "slot_deferred", "polls", "stalls", "unsampled")}
        stats.update(release_lag_max=0.0, loop_gap_max=0.0, progress_gap_max=0.0, wall_seconds=duration,
                     h2d_bytes=0, d2h_bytes=0)
        trace = [(1, j, s, 1, 0, 0, warmup + 1e-3 * j, warmup + 1e-3 * j + 1e-4) for j in range(10) for s in range(4)]
        rep = SimpleNamespace(response_hp=SimpleNamespace(p99=5e-4, p95=4e-4, mean=3e-4))
        return SimpleNamespace(report=rep, stats=stats, trace=trace, windows=windows, p99_hp=lambda a, b: 5e-4,
                               stalls=[])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), LOCAL_RANK=str(rank),
                      WORLD_SIZE="2")
    import bench
    seen = {}

    def make(tasks, gpu):
        seen["ids"] = [t.id for t in tasks]
        seen["hp"] = sum(t.priority.value == "hp" for t in tasks)
        seen["rt"] = FakeDaris(tasks, gpu, 1000.0 if rank == 0 else 800.0)
        return seen["rt"]

    args = SimpleNamespace(steps=4, warmup=1, step_seconds=0.5, probe_seconds=1.0, timed_attempts=6, no_cpu=True,
                           no_batching=True, no_batched=True, no_roofline=True, verbose=False, batched=[16])
    out = bench.ours(args, make_runtime=make)
    q.put((rank, seen["ids"], seen["hp"], seen["rt"].runs, json.dumps(out) if out else None))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_bench_flow_world_size_two():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(60)
    (_, ids0, hp0, runs0, line0), (_, ids1, hp1, runs1, line1) = res
    # placement: 16 tasks, 8 per GPU (dense local ids for the rank's dispatcher), 4 HP + 4 LP each
    assert ids0 == ids1 == list(range(1, 9)) and hp0 == hp1 == 4
    assert line1 is None
    line = json.loads(line0)
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    knee = line["config"]["knee_rate_per_task"]
    assert knee < 800                      # min over ranks: rank 1's cliff binds both
    # both ranks ran the same timed rates (joint decision), the last one passing everywhere
    assert runs0[-len(line["gpu_pauses"]["attempts"]):] == runs1[-len(line["gpu_pauses"]["attempts"]):]
    assert line["constraints_met"] and line["windows_failed"] == 0 and line["hp_miss"] == 0
    # whole-box value: both ranks' completed images over the timed window
    assert abs(line["value"] - 2 * 8 * knee) < 1e-6 * line["value"] + 1.0
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    # no pauses in the stand-in: the pause-excluded knee is the same cliff
    assert line["value_excl_pauses"]["rate_per_task"] < 800 and line["value_excl_pauses"]["constraints_met"]
