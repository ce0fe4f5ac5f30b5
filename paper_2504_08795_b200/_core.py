"""ctypes binding of the native dispatcher (include/daris.h, lib/libdaris_core.so).

``Handle`` is the only object that crosses into C++: it owns one dispatcher
instance and exposes the C ABI one-to-one. Structures mirror the header.
"""

from __future__ import annotations

import ctypes as C
import math
from pathlib import Path
from typing import Sequence

import numpy as np

from .errors import raise_status

_LIB_PATH = Path(__file__).resolve().parent / "lib" / "libdaris_core.so"
_lib = None

KIND_NAMES = ("release", "admit", "reject", "stage_start", "stage_complete", "job_complete", "sim_end")
POLICY_CODES = {"str": 0, "mps": 1, "mps-str": 2}


class GpuConfigC(C.Structure):
    _fields_ = [("total_sms", C.c_int32), ("n_contexts", C.c_int32), ("n_streams", C.c_int32),
                ("policy", C.c_int32), ("oversubscription", C.c_double), ("kappa", C.c_double)]


class StageSpecC(C.Structure):
    _fields_ = [("nominal_time", C.c_double), ("width", C.c_int32), ("_pad", C.c_int32)]


class TaskSpecC(C.Structure):
    _fields_ = [("id", C.c_int32), ("priority", C.c_int32), ("period", C.c_double), ("deadline", C.c_double),
                ("first_stage", C.c_int32), ("n_stages", C.c_int32), ("batch_size", C.c_int32),
                ("curve_ref_batch", C.c_int32), ("curve_ref_gain", C.c_double)]


class OptionsC(C.Structure):
    _fields_ = [("window_size", C.c_int32), ("no_staging", C.c_int32), ("no_last", C.c_int32),
                ("no_prior", C.c_int32), ("no_fixed", C.c_int32), ("hpa", C.c_int32),
                ("placement_insertion", C.c_int32), ("edf_on_job_deadline", C.c_int32),
                ("check_invariants", C.c_int32), ("stage_migration", C.c_int32)]


class StageRefC(C.Structure):
    _fields_ = [("task", C.c_int32), ("job", C.c_int32), ("stage", C.c_int32), ("context", C.c_int32),
                ("stream", C.c_int32), ("started_at", C.c_double), ("virtual_deadline", C.c_double)]


class PlacementC(C.Structure):
    _fields_ = [("context", C.c_int32), ("migrated_from", C.c_int32), ("n_audits", C.c_int32),
                ("_pad", C.c_int32)]


class LedgerC(C.Structure):
    _fields_ = [("hp_total", C.c_double), ("lp_total", C.c_double), ("lp_active", C.c_double),
                ("hp_active", C.c_double)]


class AuditC(C.Structure):
    _fields_ = [("time", C.c_double), ("active_util", C.c_double), ("job_util", C.c_double),
                ("limit", C.c_double), ("job", C.c_int32), ("task", C.c_int32), ("priority", C.c_int32),
                ("context", C.c_int32), ("admitted", C.c_int32), ("_pad", C.c_int32)]


class LogRecordC(C.Structure):
    _fields_ = [("time", C.c_double), ("kind", C.c_int32), ("task", C.c_int32), ("job", C.c_int32),
                ("stage", C.c_int32), ("context", C.c_int32), ("stream", C.c_int32), ("rate", C.c_double)]


class ResponseStatsC(C.Structure):
    _fields_ = [("mean", C.c_double), ("min", C.c_double), ("max", C.c_double), ("p95", C.c_double),
                ("p99", C.c_double), ("count", C.c_int64)]


class ReportC(C.Structure):
    _fields_ = [("duration", C.c_double), ("warmup", C.c_double), ("jps", C.c_double), ("dmr_hp", C.c_double),
                ("dmr_lp", C.c_double), ("response_hp", ResponseStatsC), ("response_lp", ResponseStatsC)] + \
               [(n, C.c_int64) for n in ("released_hp", "released_lp", "accepted_hp", "accepted_lp",
                                         "rejected_hp", "rejected_lp", "completed_hp", "completed_lp",
                                         "missed_hp", "missed_lp")]


class LedgerEntryC(C.Structure):
    _fields_ = [("util", C.c_double), ("hp", C.c_int32), ("active_jobs", C.c_int32)]


class ReadyKeyC(C.Structure):
    _fields_ = [("edf", C.c_double), ("level", C.c_int32), ("task", C.c_int32), ("job", C.c_int32),
                ("_pad", C.c_int32)]


class TraceEntryC(C.Structure):
    _fields_ = [("task", C.c_int32), ("job", C.c_int32), ("stage", C.c_int32), ("flags", C.c_int32),
                ("duration", C.c_double)]


TRACE_UNSAMPLED = 1  # DARIS_TRACE_UNSAMPLED


LOG_DTYPE = np.dtype([("time", "<f8"), ("kind", "<i4"), ("task", "<i4"), ("job", "<i4"), ("stage", "<i4"),
                      ("context", "<i4"), ("stream", "<i4"), ("rate", "<f8")])


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(f"native dispatcher library missing: {_LIB_PATH} "
                              "(run `python -m paper_2504_08795_b200.build`)")
        L = C.CDLL(str(_LIB_PATH))
        P, i32, i64, f64, vp = C.POINTER, C.c_int32, C.c_int64, C.c_double, C.c_void_p
        sig = {
            "daris_create": [P(GpuConfigC), P(TaskSpecC), i32, P(StageSpecC), i32, P(OptionsC), P(vp),
                             C.c_char_p, C.c_size_t],
            "daris_last_error": [vp],
            "daris_sm_per_context": [P(GpuConfigC), P(i32)],
            "daris_n_tasks": [vp, P(i32)],
            "daris_task_ids": [vp, P(i32)],
            "daris_task_stage_count": [vp, i32, P(i32)],
            "daris_full_load_sim": [vp, i32, i32, P(i32), P(f64)],
            "daris_set_full_load": [vp, P(f64)],
            "daris_populate": [vp],
            "daris_home_context": [vp, i32, P(i32)],
            "daris_release": [vp, i32, f64, i32, P(f64), P(PlacementC)],
            "daris_dispatch": [vp, i32, i32, f64, P(StageRefC), P(i32)],
            "daris_complete": [vp, i32, i32, f64, P(i32), P(i32)],
            "daris_complete_ex": [vp, i32, i32, f64, i32, P(i32), P(i32)],
            "daris_partition_layout": [i32, i32, P(i32), i32, P(i32), P(i32), P(i32)],
            "daris_ready_count": [vp, i32, P(i32)],
            "daris_ledger": [vp, i32, P(LedgerC)],
            "daris_admission_test": [vp, i32, i32, i32, f64, P(AuditC)],
            "daris_predicted_finish": [vp, i32, i32, f64, P(f64)],
            "daris_stage_estimate": [vp, i32, i32, P(f64)],
            "daris_task_estimate": [vp, i32, P(f64)],
            "daris_utilization": [vp, i32, P(f64)],
            "daris_deadline_shares": [vp, i32, P(f64)],
            "daris_record_execution": [vp, i32, i32, f64],
            "daris_note_job_complete": [vp, i32],
            "daris_sim_run": [vp, f64, f64, P(f64), i32, P(ReportC)],
            "daris_trace_run": [vp, f64, f64, P(f64), P(TraceEntryC), i64, i32, P(ReportC)],
            "daris_log_count": [vp],
            "daris_log_copy": [vp, vp, i64],
            "daris_audit_count": [vp],
            "daris_audit_copy": [vp, P(AuditC), i64],
            "daris_log_clear": [vp],
            "daris_water_fill": [P(i32), i32, f64, P(f64), P(i32), P(f64), P(i32)],
            "daris_allocate_rates": [P(GpuConfigC), P(i32), P(i32), i32, P(f64), P(f64), P(f64)],
            "daris_py_sum": [P(f64), P(i32), i64],
            "daris_destroy": [vp],
            # stateless decision kernels (include/daris.h, csrc/core/decide.cpp)
            "daris_eval_last_error": [],
            "daris_eval_window_peak": [P(f64), i32, P(f64)],
            "daris_eval_stage_fallback": [f64, f64, f64, P(f64)],
            "daris_eval_utilization": [i64, f64, f64, f64, P(f64)],
            "daris_eval_deadline_shares": [P(f64), i32, f64, i32, P(f64)],
            "daris_eval_virtual_deadlines": [f64, f64, P(f64), i32, P(f64), P(f64)],
            "daris_eval_ledger": [P(LedgerEntryC), i32, P(LedgerC)],
            "daris_eval_admission": [P(LedgerC), f64, i32, i32, P(f64), P(f64), P(i32)],
            "daris_eval_placement": [P(f64), P(i32), P(i32), i32, i32, i32, P(i32), P(i32), P(f64)],
            "daris_eval_predicted_finish": [f64, P(f64), i64, i32, f64, P(f64)],
            "daris_eval_priority_level": [i32, i32, i32, i32, i32, i32, P(i32)],
            "daris_eval_pick": [P(ReadyKeyC), i32, P(i32)],
            "daris_eval_next_completion": [P(f64), P(f64), P(i64), P(i64), i32, f64, P(i32), P(f64)],
            "daris_eval_advance": [P(f64), P(f64), P(i64), P(i64), i32, f64],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.daris_last_error.restype = C.c_char_p
        L.daris_eval_last_error.restype = C.c_char_p
        L.daris_log_count.restype = C.c_int64
        L.daris_log_copy.restype = C.c_int64
        L.daris_audit_count.restype = C.c_int64
        L.daris_audit_copy.restype = C.c_int64
        L.daris_py_sum.restype = C.c_double
        L.daris_destroy.restype = None
        L.daris_log_clear.restype = None
        _lib = L
    return _lib


EXPORTED_SYMBOLS = (
    "daris_create", "daris_destroy", "daris_last_error", "daris_sm_per_context", "daris_n_tasks",
    "daris_task_ids", "daris_task_stage_count", "daris_full_load_sim", "daris_set_full_load",
    "daris_populate", "daris_home_context", "daris_release", "daris_dispatch", "daris_complete", "daris_complete_ex",
    "daris_ready_count", "daris_ledger", "daris_admission_test", "daris_predicted_finish",
    "daris_stage_estimate", "daris_task_estimate", "daris_utilization", "daris_deadline_shares",
    "daris_record_execution", "daris_note_job_complete", "daris_sim_run", "daris_trace_run",
    "daris_log_count", "daris_log_copy", "daris_audit_count", "daris_audit_copy", "daris_log_clear",
    "daris_water_fill", "daris_allocate_rates", "daris_py_sum",
    "daris_eval_last_error", "daris_eval_window_peak", "daris_eval_stage_fallback", "daris_eval_utilization",
    "daris_eval_deadline_shares", "daris_eval_virtual_deadlines", "daris_eval_ledger", "daris_eval_admission",
    "daris_eval_placement", "daris_eval_predicted_finish", "daris_eval_priority_level", "daris_eval_pick",
    "daris_eval_next_completion", "daris_eval_advance", "daris_partition_layout",
)


def partition_layout(n_contexts: int, sm_per_context: int, unit_sms: Sequence[int]) -> list[tuple[int, int, int]]:
    """The executor's SM partition layout (daris_partition_layout): per context
    (first unit, units taken, SMs) over the cyclic unit sequence `unit_sms`."""
    n = len(unit_sms)
    units = (C.c_int32 * n)(*unit_sms)
    first, taken, sms = (C.c_int32 * n_contexts)(), (C.c_int32 * n_contexts)(), (C.c_int32 * n_contexts)()
    _ev(lib().daris_partition_layout(n_contexts, sm_per_context, units, n, first, taken, sms))
    return [(first[k], taken[k], sms[k]) for k in range(n_contexts)]


def gpu_struct(total_sms, n_contexts, n_streams, oversubscription, policy="mps-str", kappa=0.0) -> GpuConfigC:
    return GpuConfigC(int(total_sms), int(n_contexts), int(n_streams), POLICY_CODES[policy],
                      float(oversubscription), float(kappa))


def options_struct(*, window_size=5, no_staging=False, no_last=False, no_prior=False, no_fixed=False, hpa=False,
                   placement_order="descending_util", edf_on_job_deadline=False, check_invariants=False,
                   stage_migration=False) -> OptionsC:
    return OptionsC(int(window_size), int(no_staging), int(no_last), int(no_prior), int(no_fixed), int(hpa),
                    int(placement_order == "insertion"), int(edf_on_job_deadline), int(check_invariants),
                    int(stage_migration))


def task_structs(tasks: Sequence[dict]):
    """tasks: dicts {id, hp, period, deadline, stages[(nominal, width)], batch, curve(ref_b, ref_g)|None}."""
    n_st = sum(len(t["stages"]) for t in tasks)
    tarr = (TaskSpecC * max(1, len(tasks)))()
    sarr = (StageSpecC * max(1, n_st))()
    k = 0
    for i, t in enumerate(tasks):
        curve = t.get("curve")
        tarr[i] = TaskSpecC(int(t["id"]), 0 if t["hp"] else 1, float(t["period"]), float(t["deadline"]), k,
                            len(t["stages"]), int(t.get("batch", 1)), 0 if curve is None else int(curve[0]),
                            1.0 if curve is None else float(curve[1]))
        for nom, w in t["stages"]:
            sarr[k] = StageSpecC(float(nom), int(w), 0)
            k += 1
    return tarr, sarr, n_st


def check(code: int, handle=None, what: str = "") -> None:
    if code != 0:
        msg = lib().daris_last_error(handle).decode() if handle else what
        raise_status(code, msg or what)


class Handle:
    """One native dispatcher instance (not thread-safe)."""

    def __init__(self, gpu: GpuConfigC, tasks: Sequence[dict], opts: OptionsC):
        L = lib()
        tarr, sarr, n_st = task_structs(tasks)
        err = C.create_string_buffer(512)
        h = C.c_void_p()
        rc = L.daris_create(C.byref(gpu), tarr, len(tasks), sarr, n_st, C.byref(opts), C.byref(h), err, 512)
        if rc != 0:
            raise_status(rc, err.value.decode())
        self._h = h
        self.n_contexts = gpu.n_contexts
        n = C.c_int32()
        L.daris_n_tasks(h, C.byref(n))
        ids = (C.c_int32 * max(1, n.value))()
        L.daris_task_ids(h, ids)
        self.task_ids = list(ids)[: n.value]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().daris_destroy(h)
            self._h = None

    def _c(self, rc: int) -> None:
        check(rc, self._h)

    # --- offline ---
    def full_load_sim(self, task_id: int, reps: int, draws: Sequence[int]) -> float:
        arr = (C.c_int32 * max(1, len(draws)))(*draws)
        out = C.c_double()
        self._c(lib().daris_full_load_sim(self._h, task_id, reps, arr, C.byref(out)))
        return out.value

    def set_full_load(self, per_task: Sequence[float]) -> None:
        arr = (C.c_double * len(per_task))(*per_task)
        self._c(lib().daris_set_full_load(self._h, arr))

    def populate(self) -> None:
        self._c(lib().daris_populate(self._h))

    def home_context(self, task_id: int) -> int:
        out = C.c_int32()
        self._c(lib().daris_home_context(self._h, task_id, C.byref(out)))
        return out.value

    # --- online ---
    def release(self, task_id: int, t: float, job_id: int, stage_work=None) -> PlacementC:
        pl = PlacementC()
        w = None if stage_work is None else (C.c_double * len(stage_work))(*stage_work)
        self._c(lib().daris_release(self._h, task_id, t, job_id, w, C.byref(pl)))
        return pl

    def dispatch(self, context: int, stream: int, t: float):
        ref = StageRefC()
        found = C.c_int32()
        self._c(lib().daris_dispatch(self._h, context, stream, t, C.byref(ref), C.byref(found)))
        return ref if found.value else None

    def complete(self, job_id: int, stage: int, t: float, record_sample: bool = True) -> tuple[bool, bool]:
        done, missed = C.c_int32(), C.c_int32()
        if record_sample:
            self._c(lib().daris_complete(self._h, job_id, stage, t, C.byref(done), C.byref(missed)))
        else:
            self._c(lib().daris_complete_ex(self._h, job_id, stage, t, 0, C.byref(done), C.byref(missed)))
        return bool(done.value), bool(missed.value)

    def ready_count(self, context: int) -> int:
        out = C.c_int32()
        self._c(lib().daris_ready_count(self._h, context, C.byref(out)))
        return out.value

    def ledger(self, context: int) -> LedgerC:
        out = LedgerC()
        self._c(lib().daris_ledger(self._h, context, C.byref(out)))
        return out

    def admission_test(self, task_id: int, job_id: int, context: int, t: float) -> AuditC:
        out = AuditC()
        self._c(lib().daris_admission_test(self._h, task_id, job_id, context, t, C.byref(out)))
        return out

    def predicted_finish(self, task_id: int, context: int, t: float) -> float:
        out = C.c_double()
        self._c(lib().daris_predicted_finish(self._h, task_id, context, t, C.byref(out)))
        return out.value

    def stage_estimate(self, task_id: int, stage: int) -> float:
        out = C.c_double()
        self._c(lib().daris_stage_estimate(self._h, task_id, stage, C.byref(out)))
        return out.value

    def task_estimate(self, task_id: int) -> float:
        out = C.c_double()
        self._c(lib().daris_task_estimate(self._h, task_id, C.byref(out)))
        return out.value

    def utilization(self, task_id: int) -> float:
        out = C.c_double()
        self._c(lib().daris_utilization(self._h, task_id, C.byref(out)))
        return out.value

    def deadline_shares(self, task_id: int, n_stages: int) -> list[float]:
        out = (C.c_double * n_stages)()
        self._c(lib().daris_deadline_shares(self._h, task_id, out))
        return list(out)

    def record_execution(self, task_id: int, stage: int, observed: float) -> None:
        self._c(lib().daris_record_execution(self._h, task_id, stage, observed))

    def note_job_complete(self, task_id: int) -> None:
        self._c(lib().daris_note_job_complete(self._h, task_id))

    # --- engines ---
    def sim_run(self, duration: float, warmup_frac: float, phases: Sequence[float], collect_log=True) -> ReportC:
        rep = ReportC()
        ph = (C.c_double * max(1, len(phases)))(*phases)
        self._c(lib().daris_sim_run(self._h, duration, warmup_frac, ph, int(collect_log), C.byref(rep)))
        return rep

    def trace_run(self, duration: float, warmup_frac: float, phases: Sequence[float], trace: dict,
                  collect_log=True, unsampled=None) -> ReportC:
        """unsampled: {(task, job, stage)} completing without an MRET sample (daris_trace_entry.flags)."""
        rep = ReportC()
        ph = (C.c_double * max(1, len(phases)))(*phases)
        items = list(trace.items())
        arr = (TraceEntryC * max(1, len(items)))()
        skip = unsampled or ()
        for i, ((task, job, stage), dur) in enumerate(items):
            arr[i] = TraceEntryC(task, job, stage, TRACE_UNSAMPLED if (task, job, stage) in skip else 0, dur)
        self._c(lib().daris_trace_run(self._h, duration, warmup_frac, ph, arr, len(items), int(collect_log),
                                      C.byref(rep)))
        return rep

    def log_array(self) -> np.ndarray:
        n = lib().daris_log_count(self._h)
        buf = np.empty(n, dtype=LOG_DTYPE)
        if n:
            lib().daris_log_copy(self._h, buf.ctypes.data, n)
        return buf

    def audits(self) -> list[AuditC]:
        n = lib().daris_audit_count(self._h)
        arr = (AuditC * max(1, n))()
        if n:
            lib().daris_audit_copy(self._h, arr, n)
        return list(arr)[:n]

    def clear_log(self) -> None:
        lib().daris_log_clear(self._h)


def records_from_array(arr: np.ndarray) -> list[tuple]:
    """Native log -> reference LogRecord field tuples (None for absent fields)."""
    out = []
    times = arr["time"].tolist()
    kinds = arr["kind"].tolist()
    tasks = arr["task"].tolist()
    jobs = arr["job"].tolist()
    stages = arr["stage"].tolist()
    ctxs = arr["context"].tolist()
    streams = arr["stream"].tolist()
    rates = arr["rate"].tolist()
    for i in range(len(times)):
        r = rates[i]
        out.append((times[i], KIND_NAMES[kinds[i]],
                    None if tasks[i] < 0 else tasks[i], None if jobs[i] < 0 else jobs[i],
                    None if stages[i] < 0 else stages[i], None if ctxs[i] < 0 else ctxs[i],
                    None if streams[i] < 0 else streams[i], None if math.isnan(r) else r))
    return out


# ----------------------------------------------------------------------------- stateless kernels
# Thin typed wrappers over daris_eval_* (csrc/core/decide.cpp): the object-level
# drop-in API keeps its state in Python objects, like the reference, and makes
# every decision through these, the same functions the native handle uses.

def _ev(code: int) -> None:
    if code != 0:
        raise_status(code, lib().daris_eval_last_error().decode())


def _f64(vals) -> C.Array:
    vals = list(vals)
    return (C.c_double * max(1, len(vals)))(*vals)


def ev_window_peak(values: Sequence[float]) -> float:
    out = C.c_double()
    _ev(lib().daris_eval_window_peak(_f64(values), len(values), C.byref(out)))
    return out.value


def ev_stage_fallback(full_load: float, nominal: float, nominal_total: float) -> float:
    out = C.c_double()
    _ev(lib().daris_eval_stage_fallback(float(full_load), float(nominal), float(nominal_total), C.byref(out)))
    return out.value


def ev_utilization(completed_jobs: int, full_load: float, task_estimate: float, period: float) -> float:
    out = C.c_double()
    _ev(lib().daris_eval_utilization(int(completed_jobs), float(full_load), float(task_estimate), float(period),
                                     C.byref(out)))
    return out.value


def ev_task_estimate(stage_estimates: Sequence[float]) -> float:
    """builtin sum() of the stage estimates (timing.py:88-90), CPython-exact."""
    return lib().daris_py_sum(_f64(stage_estimates), None, len(stage_estimates))


def ev_deadline_shares(estimates: Sequence[float], deadline: float, task_id: int) -> list[float]:
    n = len(estimates)
    out = (C.c_double * max(1, n))()
    _ev(lib().daris_eval_deadline_shares(_f64(estimates), n, float(deadline), int(task_id), out))
    return list(out)[:n]


def ev_virtual_deadlines(release: float, deadline: float, shares: Sequence[float]) -> tuple[float, list[float]]:
    n = len(shares)
    out = (C.c_double * max(1, n))()
    absd = C.c_double()
    _ev(lib().daris_eval_virtual_deadlines(float(release), float(deadline), _f64(shares), n, C.byref(absd), out))
    return absd.value, list(out)[:n]


def ev_ledger(entries: Sequence[tuple[float, bool, int]]) -> LedgerC:
    n = len(entries)
    arr = (LedgerEntryC * max(1, n))(*[LedgerEntryC(float(u), int(bool(hp)), int(min(a, 2 ** 30)))
                                       for u, hp, a in entries])
    out = LedgerC()
    _ev(lib().daris_eval_ledger(arr, n, C.byref(out)))
    return out


def ev_admission(ledger: LedgerC, job_util: float, hp: bool, n_streams: int) -> tuple[float, float, bool]:
    active, limit, ok = C.c_double(), C.c_double(), C.c_int32()
    _ev(lib().daris_eval_admission(C.byref(ledger), float(job_util), int(bool(hp)), int(n_streams),
                                   C.byref(active), C.byref(limit), C.byref(ok)))
    return active.value, limit.value, bool(ok.value)


def ev_placement(utils: Sequence[float], hps: Sequence[bool], ids: Sequence[int], n_contexts: int,
                 insertion: bool) -> tuple[list[int], list[int]]:
    """Algorithm 1: (home context per input index, input indices in placement order)."""
    n = len(utils)
    ctx = (C.c_int32 * max(1, n))()
    order = (C.c_int32 * max(1, n))()
    totals = (C.c_double * max(1, n_contexts))()
    _ev(lib().daris_eval_placement(_f64(utils), (C.c_int32 * max(1, n))(*[int(bool(h)) for h in hps]),
                                   (C.c_int32 * max(1, n))(*[int(i) for i in ids]), n, int(n_contexts),
                                   int(bool(insertion)), ctx, order, totals))
    return list(ctx)[:n], list(order)[:n]


def ev_predicted_finish(t: float, backlog: Sequence[float], n_streams: int, task_estimate: float) -> float:
    out = C.c_double()
    _ev(lib().daris_eval_predicted_finish(float(t), _f64(backlog), len(backlog), int(n_streams),
                                          float(task_estimate), C.byref(out)))
    return out.value


def ev_priority_level(hp: bool, is_last: bool, predecessor_missed: bool, no_last: bool, no_prior: bool,
                      no_fixed: bool) -> int:
    out = C.c_int32()
    _ev(lib().daris_eval_priority_level(int(bool(hp)), int(bool(is_last)), int(bool(predecessor_missed)),
                                        int(bool(no_last)), int(bool(no_prior)), int(bool(no_fixed)),
                                        C.byref(out)))
    return out.value


def ev_pick(keys: Sequence[tuple[int, float, int, int]]) -> int:
    """Index of the minimal (level, edf, task, job) key, first minimum kept."""
    n = len(keys)
    arr = (ReadyKeyC * max(1, n))(*[ReadyKeyC(float(e), int(lv), int(t), int(j), 0) for lv, e, t, j in keys])
    out = C.c_int32()
    _ev(lib().daris_eval_pick(arr, n, C.byref(out)))
    return out.value


def ev_next_completion(remaining: Sequence[float], rates: Sequence[float], job_ids: Sequence[int],
                       stage_indices: Sequence[int], now: float) -> tuple[int, float]:
    n = len(remaining)
    idx, t = C.c_int32(), C.c_double()
    _ev(lib().daris_eval_next_completion(_f64(remaining), _f64(rates), (C.c_int64 * max(1, n))(*job_ids),
                                         (C.c_int64 * max(1, n))(*stage_indices), n, float(now), C.byref(idx),
                                         C.byref(t)))
    return idx.value, t.value


def ev_advance(remaining: list[float], rates: Sequence[float], job_ids: Sequence[int],
               stage_indices: Sequence[int], dt: float) -> tuple[list[float], tuple[int, str] | None]:
    """New remaining work; on overshoot raises after the stages before it were
    advanced (the caller applies `remaining` element-wise, see gpu.advance_progress)."""
    n = len(remaining)
    rem = _f64(remaining)
    code = lib().daris_eval_advance(rem, _f64(rates), (C.c_int64 * max(1, n))(*job_ids),
                                    (C.c_int64 * max(1, n))(*stage_indices), n, float(dt))
    out = list(rem)[:n]
    if code != 0:
        err = lib().daris_eval_last_error().decode()
        return out, (code, err)
    return out, None
