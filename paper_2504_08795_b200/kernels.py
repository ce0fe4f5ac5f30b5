"""ctypes binding of the sm_100a stage kernels (include/daris_kernels.h).

Torch tensors are used only as device-memory owners: every call passes raw
pointers and sizes across the C ABI. There is no fallback path — if the
native library is missing these functions raise.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import torch

_LIB_PATH = Path(__file__).resolve().parent / "lib" / "libdaris_gpu.so"
_lib = None


class KernelError(RuntimeError):
    pass


class ConvDesc(C.Structure):
    _fields_ = [
        ("x", C.c_void_p), ("y", C.c_void_p), ("residual", C.c_void_p), ("weight", C.c_void_p),
        ("scale", C.c_void_p), ("bias", C.c_void_p), ("workspace", C.c_void_p), ("counters", C.c_void_p),
        ("n", C.c_int32), ("h", C.c_int32), ("w", C.c_int32), ("cin", C.c_int32), ("cout", C.c_int32),
        ("kh", C.c_int32), ("kw", C.c_int32), ("stride", C.c_int32), ("pad", C.c_int32),
        ("ho", C.c_int32), ("wo", C.c_int32), ("relu", C.c_int32), ("block_n", C.c_int32),
        ("splits", C.c_int32), ("sm_budget", C.c_int32), ("flags", C.c_int32), ("timestamps", C.c_void_p),
        ("x2", C.c_void_p), ("h2", C.c_int32), ("w2", C.c_int32), ("cin2", C.c_int32), ("stride2", C.c_int32),
    ]


class ConvPlan(C.Structure):
    _fields_ = [
        ("block_n", C.c_int32), ("splits", C.c_int32), ("kb_per_split", C.c_int32),
        ("tiles_m", C.c_int32), ("tiles_n", C.c_int32), ("workspace_floats", C.c_int64),
        ("counters", C.c_int32), ("ctas", C.c_int32), ("cluster", C.c_int32), ("tma_rows", C.c_int32),
        ("pair", C.c_int32),
    ]


class LinearDesc(C.Structure):
    _fields_ = [
        ("x", C.c_void_p), ("w", C.c_void_p), ("bias", C.c_void_p), ("y", C.c_void_p),
        ("workspace", C.c_void_p), ("counters", C.c_void_p),
        ("batch", C.c_int32), ("k", C.c_int32), ("o", C.c_int32), ("relu", C.c_int32),
        ("y_bf16", C.c_int32), ("splits", C.c_int32), ("sm_budget", C.c_int32),
    ]


class LinearPlan(C.Structure):
    _fields_ = [
        ("block_n", C.c_int32), ("splits", C.c_int32), ("kb_per_split", C.c_int32),
        ("tiles_m", C.c_int32), ("tiles_n", C.c_int32), ("workspace_floats", C.c_int64),
        ("counters", C.c_int32), ("ctas", C.c_int32),
    ]


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise KernelError(f"native stage-kernel library missing: {_LIB_PATH} "
                              "(run `python -m paper_2504_08795_b200.build`)")
        L = C.CDLL(str(_LIB_PATH))
        vp, i32 = C.c_void_p, C.c_int32
        L.daris_conv_plan.argtypes = [C.POINTER(ConvDesc), C.POINTER(ConvPlan)]
        L.daris_conv2d.argtypes = [C.POINTER(ConvDesc), vp]
        L.daris_stem_im2col.argtypes = [vp, vp] + [i32] * 11 + [vp]
        L.daris_pack_nhwc.argtypes = [vp, vp] + [i32] * 5 + [vp]
        L.daris_pack_nhwc_bordered.argtypes = [vp, vp] + [i32] * 7 + [vp]
        L.daris_maxpool.argtypes = [vp, vp] + [i32] * 9 + [vp]
        L.daris_avgpool.argtypes = [vp, vp, i32, i32, i32, vp]
        L.daris_linear.argtypes = [vp, i32, vp, vp, vp, i32, i32, i32, i32, i32, vp]
        L.daris_dwconv.argtypes = [vp, vp, vp, vp, vp] + [i32] * 10 + [vp]
        L.daris_device_sms.argtypes = []
        L.daris_linear_plan.argtypes = [C.POINTER(LinearDesc), C.POINTER(LinearPlan)]
        L.daris_linear_tc.argtypes = [C.POINTER(LinearDesc), vp]
        L.daris_avgpool_bf16.argtypes = [vp, vp, i32, i32, i32, vp]
        L.daris_debug_pair_watch.argtypes = [vp]
        for name in ("daris_conv_plan", "daris_conv2d", "daris_stem_im2col", "daris_pack_nhwc",
                     "daris_maxpool", "daris_avgpool", "daris_linear", "daris_dwconv",
                     "daris_pack_nhwc_bordered", "daris_device_sms", "daris_linear_plan", "daris_linear_tc",
                     "daris_avgpool_bf16", "daris_debug_pair_watch"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise KernelError(f"{what} failed with status {rc}")


# split-K through thread-block clusters + DSMEM; needs partitions whose SM
# groups can co-schedule 8-CTA clusters (the executor's default green contexts)
CLUSTER_SPLITK = True
# CTA pairs (cta_group::2) for large-M launches. The executor turns them off for
# its stage graphs: under many concurrent tenants' streams a run with pairs hung
# twice; single-tenant launches (batching baseline, tools) keep them.
CTA_PAIRS = True


def conv_desc(x_shape, cout, kh, kw, stride, pad, *, relu=1, block_n=0, splits=0, sm_budget=0,
              cluster: bool | None = None, padded_input: bool = False, x2_shape=None, stride2: int = 1) -> ConvDesc:
    n, h, w, cin = x_shape
    ho = (h + 2 * pad - kh) // stride + 1
    wo = (w + 2 * pad - kw) // stride + 1
    d = ConvDesc()
    d.n, d.h, d.w, d.cin, d.cout = n, h, w, cin, cout
    d.kh, d.kw, d.stride, d.pad, d.ho, d.wo = kh, kw, stride, pad, ho, wo
    d.relu, d.block_n, d.splits, d.sm_budget = relu, block_n, splits, sm_budget
    d.flags = ((1 if (CLUSTER_SPLITK if cluster is None else cluster) else 0) | (2 if padded_input else 0) |
               (0 if CTA_PAIRS else 8))
    if x2_shape is not None:  # DARIS_CONV_DUAL: 1x1 branch over x2 as extra K blocks
        d.flags |= 4
        _, d.h2, d.w2, d.cin2 = x2_shape
        d.stride2 = stride2
    return d


def conv_plan(d: ConvDesc) -> ConvPlan:
    p = ConvPlan()
    _check(lib().daris_conv_plan(C.byref(d), C.byref(p)), "daris_conv_plan")
    return p


def conv2d(x: torch.Tensor, weight: torch.Tensor, scale: torch.Tensor, bias: torch.Tensor, *,
           stride: int = 1, pad: int = 0, relu: int = 1, residual: torch.Tensor | None = None,
           out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
           counters: torch.Tensor | None = None, block_n: int = 0, splits: int = 0,
           sm_budget: int = 0, stream=None, timestamps: torch.Tensor | None = None,
           cluster: bool | None = None, padded_input: bool = False, kw: int | None = None,
           x2: torch.Tensor | None = None, stride2: int = 1, kh: int | None = None) -> torch.Tensor:
    """x: [n,h,w,cin] bf16 NHWC; weight: [cout,kh,kw,cin] bf16.
    padded_input (8-channel stems): x's storage is zero-bordered
    [n][h+2pad][w+2pad+8][8] (pack_nhwc(border=pad, extra=8)), weight is
    [cout,kh,8,8] and `kw` gives the real kernel width.
    x2 (DARIS_CONV_DUAL): a 1x1, stride-`stride2` branch over x2 [n,h2,w2,cin2]
    summed into the same accumulator; weight is 2-D [cout, kh*kw*cin + cin2]
    and `kh`/`kw` give the primary kernel."""
    if x2 is not None:
        cout, cin = weight.shape[0], x.shape[3]
        kh, kw = kh or 1, kw or 1
    else:
        cout, kh, kw_w, cin = weight.shape
        kw = kw if (padded_input and kw is not None) else kw_w
    d = conv_desc(tuple(x.shape), cout, kh, kw, stride, pad, relu=relu, block_n=block_n,
                  splits=splits, sm_budget=sm_budget, cluster=cluster, padded_input=padded_input,
                  x2_shape=tuple(x2.shape) if x2 is not None else None, stride2=stride2)
    p = conv_plan(d)
    if out is None:
        out = torch.empty((d.n, d.ho, d.wo, cout), dtype=torch.bfloat16, device=x.device)
    if p.splits > 1:
        if workspace is None or workspace.numel() < p.workspace_floats:
            workspace = torch.zeros(p.workspace_floats, dtype=torch.float32, device=x.device)
        if counters is None or counters.numel() < p.counters:
            counters = torch.zeros(p.counters, dtype=torch.int32, device=x.device)
    d.x, d.y, d.residual, d.weight = _ptr(x), _ptr(out), _ptr(residual), _ptr(weight)
    d.scale, d.bias = _ptr(scale), _ptr(bias)
    d.workspace, d.counters = _ptr(workspace), _ptr(counters)
    d.timestamps = _ptr(timestamps)
    d.x2 = _ptr(x2)
    _check(lib().daris_conv2d(C.byref(d), _stream(stream)), "daris_conv2d")
    return out


def stem_im2col(x: torch.Tensor, kh: int, kw: int, stride: int, pad: int, kpad: int,
                out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    n, c, h, w = x.shape
    ho = (h + 2 * pad - kh) // stride + 1
    wo = (w + 2 * pad - kw) // stride + 1
    if out is None:
        out = torch.empty((n, ho, wo, kpad), dtype=torch.bfloat16, device=x.device)
    _check(lib().daris_stem_im2col(_ptr(x), _ptr(out), n, c, h, w, kh, kw, stride, pad, ho, wo, kpad,
                                   _stream(stream)), "daris_stem_im2col")
    return out


def pack_nhwc(x: torch.Tensor, cpad: int, out: torch.Tensor | None = None, stream=None, *, border: int = 0,
              extra: int = 0) -> torch.Tensor:
    """NCHW fp32 -> NHWC bf16 with cpad channels; with border/extra into the
    interior of a zero-bordered [n][h+2b][w+2b+extra][cpad] buffer."""
    n, c, h, w = x.shape
    if out is None:
        out = torch.zeros((n, h + 2 * border, w + 2 * border + extra, cpad), dtype=torch.bfloat16, device=x.device)
    if border == 0 and extra == 0:
        _check(lib().daris_pack_nhwc(_ptr(x), _ptr(out), n, c, h, w, cpad, _stream(stream)), "daris_pack_nhwc")
    else:
        _check(lib().daris_pack_nhwc_bordered(_ptr(x), _ptr(out), n, c, h, w, cpad, border, extra,
                                              _stream(stream)), "daris_pack_nhwc_bordered")
    return out


def maxpool(x: torch.Tensor, k: int, stride: int, pad: int, out: torch.Tensor | None = None,
            stream=None) -> torch.Tensor:
    n, h, w, c = x.shape
    ho = (h + 2 * pad - k) // stride + 1
    wo = (w + 2 * pad - k) // stride + 1
    if out is None:
        out = torch.empty((n, ho, wo, c), dtype=torch.bfloat16, device=x.device)
    _check(lib().daris_maxpool(_ptr(x), _ptr(out), n, h, w, c, k, stride, pad, ho, wo, _stream(stream)),
           "daris_maxpool")
    return out


def avgpool(x: torch.Tensor, out: torch.Tensor | None = None, stream=None, *, out_bf16: bool = False) -> torch.Tensor:
    """NHWC bf16 -> [n, c] mean over pixels, fp32 (or bf16: the tensor-core linear's input)."""
    n, h, w, c = x.shape
    if out is None:
        out = torch.empty((n, c), dtype=torch.bfloat16 if out_bf16 else torch.float32, device=x.device)
    if out.dtype == torch.bfloat16:
        _check(lib().daris_avgpool_bf16(_ptr(x), _ptr(out), n, h * w, c, _stream(stream)), "daris_avgpool_bf16")
    else:
        _check(lib().daris_avgpool(_ptr(x), _ptr(out), n, h * w, c, _stream(stream)), "daris_avgpool")
    return out


def linear_desc(batch: int, k: int, o: int, *, relu: int = 0, y_bf16: bool = False, splits: int = 0,
                sm_budget: int = 0) -> LinearDesc:
    d = LinearDesc()
    d.batch, d.k, d.o, d.relu, d.y_bf16, d.splits, d.sm_budget = batch, k, o, relu, int(y_bf16), splits, sm_budget
    return d


def linear_plan(d: LinearDesc) -> LinearPlan:
    p = LinearPlan()
    _check(lib().daris_linear_plan(C.byref(d), C.byref(p)), "daris_linear_plan")
    return p


def linear_tc(x: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None, *, relu: int = 0,
              out_bf16: bool = False, out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
              counters: torch.Tensor | None = None, splits: int = 0, sm_budget: int = 0,
              stream=None) -> torch.Tensor:
    """Tensor-core linear (daris_linear_tc): x [b, k] bf16, weight [o, k] bf16, k % 64 == 0."""
    if x.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise KernelError("linear_tc needs bf16 input and weight")
    b, k = x.shape[0], x[0].numel()
    o = weight.shape[0]
    if out is None:
        out = torch.empty((b, o), dtype=torch.bfloat16 if out_bf16 else torch.float32, device=x.device)
    d = linear_desc(b, k, o, relu=relu, y_bf16=out.dtype == torch.bfloat16, splits=splits, sm_budget=sm_budget)
    p = linear_plan(d)
    if p.splits > 1:
        if workspace is None or workspace.numel() < p.workspace_floats:
            workspace = torch.zeros(p.workspace_floats, dtype=torch.float32, device=x.device)
        if counters is None or counters.numel() < p.counters:
            counters = torch.zeros(p.counters, dtype=torch.int32, device=x.device)
    d.x, d.w, d.bias, d.y = _ptr(x), _ptr(weight), _ptr(bias), _ptr(out)
    d.workspace, d.counters = _ptr(workspace), _ptr(counters)
    _check(lib().daris_linear_tc(C.byref(d), _stream(stream)), "daris_linear_tc")
    return out


def linear(x: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None, *, relu: int = 0,
           out_bf16: bool = False, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    b, k = x.shape[0], x[0].numel()
    o = weight.shape[0]
    if out is None:
        out = torch.empty((b, o), dtype=torch.bfloat16 if out_bf16 else torch.float32, device=x.device)
    _check(lib().daris_linear(_ptr(x), int(x.dtype == torch.bfloat16), _ptr(weight), _ptr(bias), _ptr(out),
                              int(out.dtype == torch.bfloat16), b, k, o, relu, _stream(stream)), "daris_linear")
    return out


def dwconv(x: torch.Tensor, weight: torch.Tensor, scale: torch.Tensor, bias: torch.Tensor, *, stride: int,
           pad: int, relu: int = 6, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """weight: [k,k,c] bf16."""
    n, h, w, c = x.shape
    k = weight.shape[0]
    ho = (h + 2 * pad - k) // stride + 1
    wo = (w + 2 * pad - k) // stride + 1
    if out is None:
        out = torch.empty((n, ho, wo, c), dtype=torch.bfloat16, device=x.device)
    _check(lib().daris_dwconv(_ptr(x), _ptr(out), _ptr(weight), _ptr(scale), _ptr(bias), n, h, w, c, k, stride,
                              pad, ho, wo, relu, _stream(stream)), "daris_dwconv")
    return out


def device_sms() -> int:
    return lib().daris_device_sms()


