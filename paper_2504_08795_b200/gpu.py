"""GPU partition configuration and the parity rate model of the drop-in API.

``GpuConfig`` / ``Policy`` / ``ceil_even`` / ``sm_per_context`` /
``ContextState`` / ``StreamState`` / ``build_contexts`` keep the reference's
names and rules (stagesim/gpu.py:36-115). ``water_fill``, ``allocate_rates``,
``next_completion`` and ``advance_progress`` call the native rate model (the
sim backend kept for bit-exact parity, csrc/core/sim.cpp + decide.cpp); on
real hardware the executor replaces it entirely.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from enum import Enum
from typing import Sequence

from . import _core
from .errors import InvalidBatch, InvalidOversubscription, raise_status

_EPS = 1e-9


class Policy(Enum):
    STR = "str"          # one context, several streams
    MPS = "mps"          # several contexts, one stream each
    MPS_STR = "mps-str"  # several contexts with several streams


@dataclass(frozen=True)
class GpuConfig:
    total_sms: int
    n_contexts: int
    n_streams: int
    oversubscription: float
    policy: Policy = Policy.MPS_STR
    interference_kappa: float = 0.0

    def __post_init__(self) -> None:   # gpu.py:53-68
        if self.total_sms < 1:
            raise ValueError("total_sms must be >= 1")
        if self.n_contexts < 1 or self.n_streams < 1:
            raise ValueError("n_contexts and n_streams must be >= 1")
        if not (1.0 <= self.oversubscription <= self.n_contexts + _EPS):
            raise InvalidOversubscription(
                f"oversubscription must lie in [1, n_contexts], got {self.oversubscription} "
                f"with {self.n_contexts} contexts")
        if self.policy is Policy.STR and self.n_contexts != 1:
            raise ValueError("the stream-only policy uses a single context")
        if self.policy is Policy.MPS and self.n_streams != 1:
            raise ValueError("the context-only policy uses a single stream per context")
        if self.interference_kappa < 0:
            raise ValueError("interference_kappa must be >= 0")

    @property
    def n_parallel(self) -> int:
        return self.n_contexts * self.n_streams

    def native(self) -> _core.GpuConfigC:
        return _core.gpu_struct(self.total_sms, self.n_contexts, self.n_streams, self.oversubscription,
                                self.policy.value, self.interference_kappa)


def ceil_even(x: float) -> int:
    """Smallest even integer >= x, tolerant of float dust (gpu.py:76-78)."""
    return 2 * math.ceil(x / 2.0 - _EPS)


def sm_per_context(config: GpuConfig) -> int:
    """ceil_even(OS * SMs / N_c), computed by the native core."""
    out = C.c_int32()
    _core.check(_core.lib().daris_sm_per_context(C.byref(config.native()), C.byref(out)),
                what=f"oversubscription {config.oversubscription} outside [1, {config.n_contexts}]")
    return out.value


@dataclass
class StreamState:
    """One stream slot of a context; `occupant` is the stage running on it (gpu.py:89-93)."""

    occupant: object | None = None


@dataclass
class ContextState:
    """A context (SM partition) and its stream slots (gpu.py:96-108)."""

    id: int                      # 1-based
    sms: int                     # SMs granted (sm_per_context)
    streams: list[StreamState]
    util_ledger: object | None = None  # last ContextUtilization computed for it

    def free_stream_index(self) -> int | None:
        """Lowest free stream slot, None when all are occupied."""
        return next((k for k, s in enumerate(self.streams) if s.occupant is None), None)


def build_contexts(config: GpuConfig) -> list[ContextState]:
    """N_c contexts of sm_per_context SMs with N_s empty stream slots each (gpu.py:111-115)."""
    sms = sm_per_context(config)
    return [ContextState(cid, sms, [StreamState() for _ in range(config.n_streams)])
            for cid in range(1, config.n_contexts + 1)]


def water_fill(widths: Sequence[float], capacity: float) -> tuple[list[float], float | None]:
    """Split `capacity` SMs over stages capped at their widths (gpu.py:118-152)."""
    n = len(widths)
    if capacity <= 0:
        raise ValueError("capacity must be positive")
    if n == 0:
        return [], None
    w = (C.c_int32 * n)(*[int(x) for x in widths])
    alloc = (C.c_double * n)()
    is_int = (C.c_int32 * n)()
    level = C.c_double()
    has = C.c_int32()
    _core.check(_core.lib().daris_water_fill(w, n, float(capacity), alloc, is_int, C.byref(level), C.byref(has)),
                what="water_fill")
    vals = [int(alloc[i]) if is_int[i] else alloc[i] for i in range(n)]
    return vals, (level.value if has.value else None)


@dataclass
class RateAllocation:
    allocated: list[float]
    rates: list[float]
    scale: float
    water_levels: dict[int, float | None]

    @property
    def total_allocated(self) -> float:
        return sum(self.allocated)


def allocate_rates(active: Sequence[tuple], config: GpuConfig) -> RateAllocation:
    """Rates of (stage, context_id) pairs under the two-level water fill (gpu.py:167-205)."""
    n = len(active)
    w = (C.c_int32 * max(1, n))(*[int(s.width) for s, _ in active])
    c = (C.c_int32 * max(1, n))(*[int(ctx) for _, ctx in active])
    alloc = (C.c_double * max(1, n))()
    rates = (C.c_double * max(1, n))()
    scale = C.c_double()
    _core.check(_core.lib().daris_allocate_rates(C.byref(config.native()), w, c, n, alloc, rates,
                                                 C.byref(scale)), what="allocate_rates")
    levels: dict[int, float | None] = {}
    per = sm_per_context(config)
    for ctx in dict.fromkeys(ctx for _, ctx in active):
        levels[ctx] = water_fill([s.width for s, cc in active if cc == ctx], per)[1]
    return RateAllocation(list(alloc)[:n], list(rates)[:n], scale.value, levels)


def next_completion(active: Sequence[tuple], allocation: RateAllocation, now: float):
    """(index, stage, time) of the earliest finisher at the current rates, ties
    on (job id, stage index) (gpu.py:208-226); native decide.cpp."""
    stages = [s for s, _ in active]
    idx, t = _core.ev_next_completion([s.remaining_work for s in stages], allocation.rates[:len(stages)],
                                      [s.job_id for s in stages], [s.stage_index for s in stages], now)
    return idx, stages[idx], t


def advance_progress(active: Sequence[tuple], allocation: RateAllocation, dt: float) -> None:
    """Integrate remaining work over `dt` at constant rates, in list order,
    raising OvershootBeyondCompletion past the 1e-9 tolerance (gpu.py:229-240)."""
    stages = [s for s, _ in active]
    rem, err = _core.ev_advance([s.remaining_work for s in stages], allocation.rates[:len(stages)],
                                [s.job_id for s in stages], [s.stage_index for s in stages], dt)
    if err is not None and err[0] != 9:   # ValueError (dt < 0): nothing advanced
        raise_status(*err)
    for s, left in zip(stages, rem):
        s.remaining_work = left
    if err is not None:
        raise_status(*err)


@dataclass(frozen=True)
class BatchingCurve:
    """Log-linear batching gain anchored at one measured point (gpu.py:243-268)."""

    reference_batch: int
    reference_gain: float

    def __post_init__(self) -> None:
        if self.reference_batch < 1:
            raise InvalidBatch(f"reference batch must be >= 1, got {self.reference_batch}")
        if self.reference_gain <= 0:
            raise ValueError("reference gain must be positive")

    def gain(self, batch_size: int) -> float:
        if not isinstance(batch_size, int) or batch_size < 1:
            raise InvalidBatch(f"batch size must be an integer >= 1, got {batch_size!r}")
        if batch_size == 1 or self.reference_batch == 1:
            return 1.0
        return max(1.0, self.reference_gain ** (math.log(batch_size) / math.log(self.reference_batch)))


UNIT_BATCHING = BatchingCurve(1, 1.0)


def effective_stage_time(profile, batch_size: int = 1, curve: BatchingCurve | None = None) -> float:
    """Full-width seconds a stage needs for a batch: nominal * B / gain(B) (gpu.py:273-284)."""
    if not isinstance(batch_size, int) or batch_size < 1:
        raise InvalidBatch(f"batch size must be an integer >= 1, got {batch_size!r}")
    return profile.nominal_time * batch_size / (curve or UNIT_BATCHING).gain(batch_size)
