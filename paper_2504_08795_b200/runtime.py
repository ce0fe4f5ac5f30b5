"""Real-GPU DARIS runtime: partitions + stage graphs + the native executor.

This is the B200 replacement of the reference's device model (gpu.py) and
event loop (engine.py): tasks are real DNNs (nets.py) whose stages run as
CUDA graphs of sm_100a kernels inside green-context SM partitions, scheduled
by the native dispatcher (libdaris_core) from the native wall-clock executor
(libdaris_gpu, include/daris_exec.h).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import random
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Sequence

import numpy as np
import torch

from . import _core, nets
from . import kernels as K
from .engine import ResponseStats, report_from_native
from .gpu import GpuConfig, Policy, sm_per_context
from .model import Priority, StageProfile, TaskSpec, spec_to_dict
from .scheduler import AblationFlags, SchedulerMode

QUANTUM = 1.0 / 1048576.0


def quantize(x: float) -> float:
    return math.floor(x / QUANTUM + 0.5) * QUANTUM


class ExecConfigC(C.Structure):
    _fields_ = [("device", C.c_int32), ("n_contexts", C.c_int32), ("n_streams", C.c_int32),
                ("sm_per_context", C.c_int32), ("partition_mode", C.c_int32), ("slots_per_task", C.c_int32),
                ("max_tasks", C.c_int32), ("max_stages", C.c_int32)]


class PartitionC(C.Structure):
    _fields_ = [("context", C.c_int32), ("sm_count", C.c_int32), ("first_group", C.c_int32),
                ("n_groups", C.c_int32), ("green", C.c_int32), ("group_size", C.c_int32)]


class StageTraceC(C.Structure):
    _fields_ = [("task", C.c_int32), ("job", C.c_int32), ("stage", C.c_int32), ("context", C.c_int32),
                ("stream", C.c_int32), ("slot", C.c_int32), ("start", C.c_double), ("end", C.c_double),
                ("gpu_start", C.c_double), ("gpu_end", C.c_double), ("sampled", C.c_int32), ("_pad", C.c_int32)]


class ExecStatsC(C.Structure):
    _fields_ = [("graph_launches", C.c_int64), ("copies_h2d", C.c_int64), ("copies_d2h", C.c_int64),
                ("copies_d2d", C.c_int64), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("slot_waits", C.c_int64), ("polls", C.c_int64), ("wall_seconds", C.c_double),
                ("release_lag_max", C.c_double), ("loop_gap_max", C.c_double),
                ("progress_gap_max", C.c_double), ("stalls", C.c_int64), ("first_stall_at", C.c_double),
                ("slot_deferred", C.c_int64), ("slot_backlog_max", C.c_int64), ("unsampled", C.c_int64)]


_exec_lib = None


def exec_lib() -> C.CDLL:
    global _exec_lib
    if _exec_lib is None:
        _core.lib()  # load the dispatcher first (libdaris_gpu links against it)
        L = K.lib()
        vp, i32, i64, f64, P = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.POINTER
        sig = {
            "daris_exec_create": [P(ExecConfigC), P(vp), C.c_char_p, C.c_size_t],
            "daris_exec_partition_info": [vp, i32, P(PartitionC)],
            "daris_exec_stream": [vp, i32, i32, P(vp)],
            "daris_exec_capture_begin": [vp, i32, P(vp)],
            "daris_exec_capture_end": [vp, i32, i32, i32, i32],
            "daris_exec_graph_count": [vp, P(i64)],
            "daris_exec_set_io": [vp, i32, i32, vp, vp],
            "daris_exec_set_pool": [vp, i32, vp, i32, i32, i64, vp, i64],
            "daris_exec_run": [vp, vp, f64, f64, P(f64), i32, P(_core.ReportC), P(ExecStatsC)],
            "daris_exec_busy_calibrate": [vp, P(i32), i32, P(i32), f64, P(f64), P(i32)],
            "daris_exec_set_stall_threshold": [vp, f64],
            "daris_exec_time_graph": [vp, i32, i32, i32, i32, i32, P(f64)],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.daris_exec_destroy.argtypes = [vp]
        L.daris_exec_destroy.restype = None
        L.daris_exec_last_error.argtypes = [vp]
        L.daris_exec_last_error.restype = C.c_char_p
        L.daris_exec_trace_count.argtypes = [vp]
        L.daris_exec_trace_count.restype = C.c_int64
        L.daris_exec_trace_copy.argtypes = [vp, P(StageTraceC), i64]
        L.daris_exec_trace_copy.restype = C.c_int64
        L.daris_exec_stall_copy.argtypes = [vp, P(f64), i64]
        L.daris_exec_stall_copy.restype = C.c_int64
        L.daris_exec_quantum.argtypes = []
        L.daris_exec_quantum.restype = C.c_double
        _exec_lib = L
    return _exec_lib


class ExecutorError(RuntimeError):
    pass


class BufferSetsExhausted(ExecutorError):
    """The executor stopped a run past the knee: every stream held a stage-0
    launch waiting for a buffer set of its task while the jobs owning those
    sets had nothing on the GPU (more live jobs of a task than its buffer
    slots: an HP backlog, which admission does not bound). The offered rate is
    infeasible; measurement code treats the run as failing every window."""


class Executor:
    """Thin owner of one native daris_exec (partitions, streams, graphs)."""

    def __init__(self, n_contexts: int, n_streams: int, sm_per_ctx: int, *, partition: str = "green",
                 slots: int = 3, max_tasks: int = 64, max_stages: int = 8, device: int = 0):
        L = exec_lib()
        cfg = ExecConfigC(device, n_contexts, n_streams, sm_per_ctx, 0 if partition == "green" else 1, slots,
                          max_tasks, max_stages)
        err = C.create_string_buffer(512)
        h = C.c_void_p()
        rc = L.daris_exec_create(C.byref(cfg), C.byref(h), err, 512)
        if rc != 0:
            raise ExecutorError(f"daris_exec_create failed ({rc}): {err.value.decode()}")
        self._h = h
        self.n_contexts, self.n_streams, self.slots = n_contexts, n_streams, slots
        self.partitions = []
        for k in range(1, n_contexts + 1):
            p = PartitionC()
            L.daris_exec_partition_info(h, k, C.byref(p))
            self.partitions.append({"context": p.context, "sm_count": p.sm_count, "first_group": p.first_group,
                                    "n_groups": p.n_groups, "green": bool(p.green), "group_size": p.group_size})
        # split-K through 8-CTA clusters only where every partition can co-schedule them
        K.CLUSTER_SPLITK = min(p["group_size"] for p in self.partitions) >= 8
        K.CTA_PAIRS = False  # concurrent tenants: one-CTA tiles only (kernels.py)

    def _c(self, rc: int, what: str) -> None:
        if rc != 0:
            msg = exec_lib().daris_exec_last_error(self._h).decode()
            cls = BufferSetsExhausted if "buffer sets exhausted" in msg else ExecutorError
            raise cls(f"{what} failed ({rc}): {msg}")

    def close(self) -> None:
        if getattr(self, "_h", None):
            exec_lib().daris_exec_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def cluster_partition(self) -> int:
        """1-based context of the first partition that holds a co-scheduled SM
        group (8-CTA clusters launch there), e.g. for single-partition tools."""
        ctx = next((p["context"] for p in self.partitions if p["group_size"] >= 8), 1)
        K.CLUSTER_SPLITK = self.partitions[ctx - 1]["group_size"] >= 8   # the tool runs there only
        K.CTA_PAIRS = True  # one stream, no concurrent tenants
        return ctx

    def stream(self, context: int, stream: int) -> int:
        out = C.c_void_p()
        self._c(exec_lib().daris_exec_stream(self._h, context, stream, C.byref(out)), "daris_exec_stream")
        return out.value

    def capture(self, task: int, stage: int, context: int, slot: int, body) -> None:
        s = C.c_void_p()
        self._c(exec_lib().daris_exec_capture_begin(self._h, context, C.byref(s)), "capture_begin")
        try:
            body(s.value)
        except Exception:
            exec_lib().daris_exec_capture_end(self._h, 1, 0, context, 0)
            raise
        self._c(exec_lib().daris_exec_capture_end(self._h, task, stage, context, slot), "capture_end")

    def time_graph(self, task: int, stage: int, context: int, slot: int = 0, reps: int = 20) -> float:
        out = C.c_double()
        self._c(exec_lib().daris_exec_time_graph(self._h, task, stage, context, slot, reps, C.byref(out)),
                "time_graph")
        return out.value

    def graph_count(self) -> int:
        out = C.c_int64()
        exec_lib().daris_exec_graph_count(self._h, C.byref(out))
        return out.value

    def set_io(self, task: int, slot: int, dev_input: int, dev_output: int) -> None:
        self._c(exec_lib().daris_exec_set_io(self._h, task, slot, dev_input, dev_output), "set_io")

    def set_pool(self, task: int, pool_ptr: int, on_host: bool, n_inputs: int, in_bytes: int,
                 host_out_ptr: int | None, out_bytes: int) -> None:
        self._c(exec_lib().daris_exec_set_pool(self._h, task, pool_ptr, int(on_host), n_inputs, in_bytes,
                                               host_out_ptr, out_bytes), "set_pool")

    def run(self, handle: _core.Handle, duration: float, warmup: float, phases: Sequence[float]):
        rep = _core.ReportC()
        st = ExecStatsC()
        ph = (C.c_double * max(1, len(phases)))(*phases)
        rc = exec_lib().daris_exec_run(self._h, handle._h, duration, warmup, ph, 1, C.byref(rep), C.byref(st))
        self._c(rc, "daris_exec_run")
        return rep, st

    def set_stall_threshold(self, seconds: float) -> None:
        self._c(exec_lib().daris_exec_set_stall_threshold(self._h, seconds), "set_stall_threshold")

    def trace(self) -> list[tuple]:
        L = exec_lib()
        n = L.daris_exec_trace_count(self._h)
        arr = (StageTraceC * max(1, n))()
        L.daris_exec_trace_copy(self._h, arr, n)
        self._gpu_times = [(a.gpu_start, a.gpu_end) for a in list(arr)[:n]]
        return [(a.task, a.job, a.stage, a.context, a.stream, a.slot, a.start, a.end, a.sampled)
                for a in list(arr)[:n]]

    def stall_log(self) -> list[tuple[float, float]]:
        """(start, length) of each GPU-wide stall of the last run (executor seconds)."""
        L = exec_lib()
        n = L.daris_exec_stall_copy(self._h, None, 0)
        buf = (C.c_double * max(2, 2 * n))()
        L.daris_exec_stall_copy(self._h, buf, n)
        return [(buf[2 * i], buf[2 * i + 1]) for i in range(n)]

    def trace_gpu(self) -> list[tuple[float, float]]:
        """Device-side (start, end) of each traced stage, aligned with trace()
        (NaN unless the run had DARIS_GPU_TIMING set)."""
        return getattr(self, "_gpu_times", [])

    def busy_calibrate(self, stage_counts: Sequence[int], slot_tasks: Sequence[int], seconds: float,
                       task_hp: Sequence[bool] | None = None) -> float:
        sc = (C.c_int32 * len(stage_counts))(*stage_counts)
        st = (C.c_int32 * len(slot_tasks))(*slot_tasks)
        hp = (C.c_int32 * len(stage_counts))(*[int(bool(x)) for x in task_hp]) if task_hp is not None else None
        out = C.c_double()
        self._c(exec_lib().daris_exec_busy_calibrate(self._h, sc, len(stage_counts), st, seconds, C.byref(out), hp),
                "busy_calibrate")
        return out.value


# ----------------------------------------------------------------------------
# workload description
# ----------------------------------------------------------------------------

@dataclass
class TaskDef:
    """A periodic DNN inference task on the real GPU."""
    id: int
    model: str
    priority: Priority
    rate: float                  # jobs per second (period = 1/rate, quantised)
    n_stages: int | None = None
    batch: int = 1               # images per job (the reference's TaskSpec batch_size)

    @property
    def key(self) -> str:
        """Name of the network a job of this task runs (model, or model@bB)."""
        return self.model if self.batch == 1 else f"{self.model}@b{self.batch}"

    @property
    def period(self) -> float:
        return quantize(1.0 / self.rate)


@dataclass
class RunResult:
    report: object
    stats: dict
    trace: list
    records: list
    admissions: list
    full_load: dict
    phases: list
    tasks: list
    periods: dict
    stage_nominal: dict
    partitions: list
    log: np.ndarray | None = None        # the raw native event log (_core.LOG_DTYPE)
    stalls: list = field(default_factory=list)  # (start, length) of GPU-wide stalls
    batch: dict = field(default_factory=dict)   # images per job, by task id

    def unsampled(self) -> set:
        """(task, job, stage) of traced stages completed without an MRET sample
        (in flight across a detected GPU-wide pause): replay them as such."""
        return {(t[0], t[1], t[2]) for t in self.trace if len(t) > 8 and not t[8]}

    def windows(self, warmup: float, step: float, n_steps: int) -> list[dict]:
        return window_stats(self.log, self.periods, {t.id for t in self.tasks if t.priority is Priority.HP},
                            warmup, step, n_steps, self.stalls, self.batch)

    def p99_hp(self, start: float, end: float) -> float:
        """Nearest-rank p99 (ordered[ceil(0.99 n) - 1]) of the response times of
        HP jobs released in [start, end) that completed."""
        log = self.log
        hp = np.array(sorted(t.id for t in self.tasks if t.priority is Priority.HP))
        kind, t, job = log["kind"], log["time"], log["job"]
        n = int(job.max()) + 1 if len(job) else 1
        rel = np.full(n, np.nan)
        m = (kind == 0) & np.isin(log["task"], hp) & (t >= start) & (t < end)
        rel[job[m]] = t[m]
        m = kind == 5
        resp = np.sort((t[m] - rel[job[m]])[~np.isnan(rel[job[m]])])
        return float(resp[max(0, int(math.ceil(0.99 * len(resp))) - 1)]) if len(resp) else 0.0


def window_stats(log: np.ndarray, periods: dict[int, float], hp_ids: set[int], warmup: float, step: float,
                 n_steps: int, stalls=(), batch: dict[int, int] | None = None) -> list[dict]:
    """Per-window accounting of a run's event log. Window k holds the jobs
    RELEASED in [warmup + k*step, warmup + (k+1)*step). A job misses when it
    completes after release + D (D = T), or when it was admitted, has not
    completed, and its deadline release + D has passed by the end of the log
    (the run's horizon) — a backlog cannot hide misses. LP loss counts misses
    and admission rejections over LP releases. `stalls` are the executor's
    GPU-wide stalls; each window notes how many began inside the time its
    jobs were live (release to deadline)."""
    kind, t, task, job = log["kind"], log["time"], log["task"], log["job"]
    horizon = float(t[kind == 6][0]) if (kind == 6).any() else float(t.max())
    n = int(job.max()) + 1 if len(job) else 1
    rel_t = np.full(n, np.nan)
    rel_task = np.zeros(n, dtype=np.int64)
    done_t = np.full(n, np.nan)
    rejected = np.zeros(n, dtype=bool)
    m = kind == 0
    rel_t[job[m]] = t[m]
    rel_task[job[m]] = task[m]
    rejected[job[kind == 2]] = True
    m = kind == 5
    done_t[job[m]] = t[m]
    ids = np.nonzero(~np.isnan(rel_t))[0]
    per = np.array([periods[int(k)] for k in rel_task[ids]])
    dl = rel_t[ids] + per
    finished = ~np.isnan(done_t[ids])
    missed = ~rejected[ids] & ((finished & (done_t[ids] > dl)) | (~finished & (dl <= horizon)))
    is_hp = np.isin(rel_task[ids], list(hp_ids))
    imgs = np.array([(batch or {}).get(int(k), 1) for k in rel_task[ids]])
    win = np.floor((rel_t[ids] - warmup) / step).astype(np.int64)
    st_start = np.array([a for a, _ in stalls]) if len(stalls) else np.zeros(0)
    out = []
    for k in range(n_steps):
        sel = win == k
        hp, lp = sel & is_hp, sel & ~is_hp
        lo, hi = warmup + k * step, warmup + (k + 1) * step
        rel_lp = int(lp.sum())
        lost_lp = int((lp & (missed | rejected[ids])).sum())
        out.append({"released_hp": int(hp.sum()), "released_lp": rel_lp, "missed_hp": int((hp & missed).sum()),
                    "missed_lp": int((lp & missed).sum()), "rejected_lp": int((lp & rejected[ids]).sum()),
                    "lp_loss": lost_lp / rel_lp if rel_lp else 0.0,
                    "completed_images": int(imgs[sel & finished & (done_t[ids] <= horizon)].sum()),
                    "stalls": int(((st_start >= lo) & (st_start < hi + max(periods.values()))).sum())})
    return out


def window_ok(w: dict) -> bool:
    """HP miss = 0 and LP loss (misses + rejections) < 2 % in one window."""
    return w["missed_hp"] == 0 and w["lp_loss"] < 0.02 and w["released_hp"] + w["released_lp"] > 0


class DarisRuntime:
    """Owns networks, per-task buffers, stage graphs, a dispatcher and the executor."""

    def __init__(self, tasks: Sequence[TaskDef], gpu: GpuConfig, *, slots: int = 3, partition: str = "green",
                 window_size: int = 5, flags: AblationFlags = AblationFlags(), hpa: bool = False,
                 stage_migration: bool = False, seed: int = 0, e2e: bool = False, pool_size: int = 64,
                 device: int = 0, phasing: str = "random", placement_order: str = "descending_util",
                 edf_on_job_deadline: bool = False):
        if not torch.cuda.is_available():
            raise RuntimeError("DarisRuntime needs a CUDA device (there is no CPU fallback)")
        if phasing not in ("random", "zero"):
            raise ValueError(f"unknown phasing {phasing!r}")
        self.phasing = phasing
        self.tasks = sorted(tasks, key=lambda t: t.id)
        self.gpu = gpu
        self.seed = seed
        self.flags, self.hpa, self.window_size = flags, hpa, window_size
        self.stage_migration = stage_migration
        self.placement_order = placement_order
        self.edf_on_job_deadline = edf_on_job_deadline
        self.e2e = e2e
        self.device = torch.device("cuda", device)
        self.sm_per_ctx = sm_per_context(gpu)
        max_stages = 8
        self.exec = Executor(gpu.n_contexts, gpu.n_streams, self.sm_per_ctx, partition=partition, slots=slots,
                             max_tasks=max(t.id for t in self.tasks), max_stages=max_stages, device=device)
        # SMs the layer planner sizes each job's grids (M/N tiles x split-K) for.
        # Not the partition: with n_contexts x n_streams jobs in flight every SM
        # is shared, and a grid sized for the whole partition spends its extra
        # CTAs on split-K fix-ups that buy isolated latency but cost throughput.
        # Planning for the device's share per concurrent job measured +42 %
        # closed-loop capacity at 4x2 OS=2 and ~2x at 16 streams (round 1, x1.25,
        # profiles/r01_capacity_*). With partitions over all 148 SMs and the
        # pulled split-K the best share moved up: x1.75 (C2: 32 SMs) vs x1.25
        # (23): knee 12.9k vs 12.3k inf/s over two runs each, p99 HP 0.38 vs
        # 0.43 ms (profiles/r02_plan_share_ab.txt). Batched jobs keep x1.25: their
        # grids are wide anyway, and the C2 schedule with batch-16 jobs fell
        # 35.9k -> 30.5k inf/s at x1.75 (profiles/r02_bench_plan32.json).
        # DARIS_PLAN_SMS overrides.
        self.partition_sms = min(p["sm_count"] for p in self.exec.partitions)
        factor = 1.75 if max(t.batch for t in self.tasks) == 1 else 1.25
        share = int(round(factor * gpu.total_sms / (gpu.n_contexts * gpu.n_streams)))
        self.sm_budget = int(os.environ.get("DARIS_PLAN_SMS", "0")) or max(8, min(self.partition_sms, share))
        # per-priority planning (experiment knobs): HP jobs' grids may be planned wider
        self.plan_hp = int(os.environ.get("DARIS_PLAN_SMS_HP", "0")) or self.sm_budget
        self.plan_lp = int(os.environ.get("DARIS_PLAN_SMS_LP", "0")) or self.sm_budget
        # one weight copy per model, shared by all tasks running it
        self.nets: dict[tuple, nets.Network] = {}
        for t in self.tasks:
            key = (t.model, t.n_stages, t.batch)
            if key not in self.nets:
                self.nets[key] = nets.build_network(t.model, batch=t.batch, n_stages=t.n_stages, seed=seed,
                                                    device=self.device)
        self.buffers: dict[tuple[int, int], nets.TaskBuffers] = {}
        for t in self.tasks:
            net = self.net_of(t)
            for s in range(slots):
                self.buffers[(t.id, s)] = nets.allocate_buffers(net, self.plan_of(t))
        self.pool_size = pool_size
        self._pool_cache: dict = {}
        self._make_pools(pool_size)
        torch.cuda.synchronize()
        self._warm()
        self._nominal: dict[str, list[float]] | None = None
        self.handle = None
        self.afet: dict[int, float] | None = None

    def plan_of(self, t: TaskDef) -> int:
        """SMs this task's layer grids are planned for."""
        return self.plan_hp if t.priority is Priority.HP else self.plan_lp

    def net_of(self, t: TaskDef) -> nets.Network:
        return self.nets[(t.model, t.n_stages, t.batch)]

    # -- inputs ------------------------------------------------------------
    def _make_pools(self, pool_size: int) -> None:
        """Synthetic images x ~ N(0,1), one pool per task; device
        resident (resident mode) or pinned host memory (end-to-end mode)."""
        self.pools = {}
        self.host_out = {}
        for t in self.tasks:
            key = (t.id, self.e2e)
            if key not in self._pool_cache:
                g = torch.Generator().manual_seed(self.seed * 1000 + t.id)
                imgs = torch.randn((pool_size, 3, 224, 224), generator=g)
                if self.e2e:
                    self._pool_cache[key] = (imgs.pin_memory(),
                                             torch.zeros(self.net_of(t).output_shape,
                                                         dtype=torch.float32).pin_memory())
                else:
                    self._pool_cache[key] = (imgs.to(self.device), None)
            pool, out = self._pool_cache[key]
            self.pools[t.id] = pool
            self.host_out[t.id] = out
            in_bytes = t.batch * 3 * 224 * 224 * 4  # a job copies `batch` consecutive images
            self.exec.set_pool(t.id, pool.data_ptr(), self.e2e, max(1, pool_size // t.batch), in_bytes,
                               out.data_ptr() if out is not None else None,
                               out.numel() * 4 if out is not None else 0)
            for s in range(self.exec.slots):
                tb = self.buffers[(t.id, s)]
                self.exec.set_io(t.id, s, tb.input.data_ptr(), tb.output.data_ptr())

    # -- graphs ------------------------------------------------------------
    def capture_all(self, homes: dict[int, int] | None = None) -> int:
        """Capture one graph per (task, stage, context, slot); HP tasks only in
        their home context when `homes` is given."""
        n = 0
        for t in self.tasks:
            net = self.net_of(t)
            ctxs = range(1, self.gpu.n_contexts + 1)
            if homes is not None and t.priority is Priority.HP:
                ctxs = [homes[t.id]]
            for k in ctxs:
                for s in range(self.exec.slots):
                    tb = self.buffers[(t.id, s)]
                    for st in range(net.n_stages):
                        self.exec.capture(t.id, st, k, s,
                                          lambda stream, st=st, tb=tb, net=net, plan=self.plan_of(t):
                                          nets.run_stage(net, st, tb, stream, plan))
                        n += 1
        return n

    def _warm(self) -> None:
        """One eager pass of every stage (kernel attributes, tensor maps, stage
        programs) before anything is captured."""
        stream = torch.cuda.Stream(device=self.device)
        with torch.cuda.stream(stream):
            for key, net in self.nets.items():
                tb = self.buffers[(next(t.id for t in self.tasks if (t.model, t.n_stages, t.batch) == key), 0)]
                for st in range(net.n_stages):
                    nets.run_stage(net, st, tb, stream.cuda_stream, self.sm_budget)
        stream.synchronize()

    @property
    def stage_nominal(self) -> dict[str, list[float]]:
        """Isolated per-stage time of each model (the StageProfile nominal_time):
        its captured stage graph replayed alone on partition 1, CUDA-event timed."""
        if self._nominal is None:
            if self.exec.graph_count() == 0:
                self.capture_all()
            out = {}
            for t in self.tasks:
                if t.key in out:
                    continue
                out[t.key] = [max(self.exec.time_graph(t.id, st, 1, 0, 20), 2 * QUANTUM)
                                for st in range(self.net_of(t).n_stages)]
            self._nominal = out
        return self._nominal

    # -- dispatcher ----------------------------------------------------------
    def specs(self) -> list[TaskSpec]:
        out = []
        for t in self.tasks:
            nom = self.stage_nominal[t.key]
            stages = tuple(StageProfile(float(x), self.sm_per_ctx) for x in nom)
            out.append(TaskSpec.periodic(t.id, t.period, t.priority, stages))
        return out

    def open_dispatcher(self, full_load: dict[int, float]) -> _core.Handle:
        batch = {t.id: t.batch for t in self.tasks}
        dicts = [spec_to_dict(s, batch[s.id]) for s in self.specs()]
        opts = _core.options_struct(window_size=self.window_size, no_last=self.flags.no_last,
                                    no_prior=self.flags.no_prior, no_fixed=self.flags.no_fixed, hpa=self.hpa,
                                    placement_order=self.placement_order,
                                    edf_on_job_deadline=self.edf_on_job_deadline,
                                    stage_migration=self.stage_migration)
        h = _core.Handle(self.gpu.native(), dicts, opts)
        h.set_full_load([full_load[i] for i in h.task_ids])
        h.populate()
        return h

    def calibrate_full_load(self, seconds: float = 0.2) -> dict[int, float]:
        """AFET on the GPU (timing.py:147-218 made real): each distinct model is
        timed on ctx 1 / stream 0 while every other slot loops random tasks."""
        if self.exec.graph_count() == 0:
            self.capture_all()
        rng = random.Random(self.seed * 7919)
        n_slots = self.gpu.n_contexts * self.gpu.n_streams
        ids = [t.id for t in self.tasks]
        counts = [self.net_of(t).n_stages for t in self.tasks]
        by_model: dict[str, float] = {}
        out = {}
        for t in self.tasks:
            if t.key not in by_model:
                # random co-runners, each task at most `slots` times (one buffer set per concurrent copy)
                if len(ids) * self.exec.slots < n_slots:
                    raise ValueError(f"AFET calibration needs {n_slots} concurrent jobs but {len(ids)} tasks x "
                                     f"{self.exec.slots} buffer slots cannot supply them")
                slot_tasks = [t.id]
                while len(slot_tasks) < n_slots:
                    c = rng.choice(ids)
                    if slot_tasks.count(c) < self.exec.slots:
                        slot_tasks.append(c)
                hp = [x.priority is Priority.HP for x in self.tasks]
                by_model[t.key] = quantize(max(self.exec.busy_calibrate(counts, slot_tasks, seconds, hp),
                                                 2 * QUANTUM))
            out[t.id] = by_model[t.key]
        self.afet = out
        return out

    def phases(self) -> list[float]:
        """Release offsets as the reference draws them (engine.py:417-423), quantised."""
        if self.phasing == "zero":
            return [0.0 for _ in self.tasks]
        rng = random.Random(self.seed)
        return [quantize(rng.random() * t.period) for t in self.tasks]

    def set_rate(self, rate: float) -> None:
        """Same per-task release rate for every task (periods are quantised)."""
        for t in self.tasks:
            t.rate = rate

    def use_host_io(self, on: bool) -> None:
        """Switch between device-resident input pools and pinned-host pools with
        H2D input / D2H logits copies every job (end-to-end mode)."""
        if on != self.e2e:
            self.e2e = on
            self._make_pools(self.pool_size)
            torch.cuda.synchronize()

    def run(self, duration: float, warmup: float, *, full_load: dict[int, float] | None = None) -> RunResult:
        if self.exec.graph_count() == 0:
            self.capture_all()
        if full_load is None:
            full_load = self.afet if self.afet is not None else self.calibrate_full_load()
        h = self.open_dispatcher(full_load)
        torch.cuda.synchronize()
        phases = self.phases()
        # a progress gap this long with stages in flight is a GPU-wide stall, not scheduling
        longest = max(max(v) for v in self.stage_nominal.values())
        self.exec.set_stall_threshold(max(1e-3, 3.0 * longest))
        rep, st = self.exec.run(h, quantize(duration), quantize(warmup), phases)
        self.handle = h
        report = report_from_native(rep, label=f"{self.gpu.n_contexts}x{self.gpu.n_streams}_"
                                                f"{self.gpu.oversubscription:g}", config=self.gpu,
                                    seed=self.seed)
        stats = {f: getattr(st, f) for f, _ in ExecStatsC._fields_}
        log = h.log_array()
        records = _core.records_from_array(log)
        from .scheduler import AdmissionDecision
        admissions = [AdmissionDecision.from_native(a) for a in h.audits()]
        return RunResult(report, stats, self.exec.trace(), records, admissions, full_load, phases,
                         self.specs(), {t.id: t.period for t in self.tasks}, self.stage_nominal,
                         self.exec.partitions, log, self.exec.stall_log(), {t.id: t.batch for t in self.tasks})

    def close(self) -> None:
        self.exec.close()
