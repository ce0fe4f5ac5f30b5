"""DNN stage bodies for DARIS tasks, executed only through the sm_100a kernels.

The reference models a DNN as opaque stage quanta (presets.py:20-55,
``StageProfile(nominal_time, width)``). Here a task runs a real network —
ResNet-18 / ResNet-50 / VGG-16 / MobileNetV2 with torchvision's architecture
and seeded random weights — split into synchronisation-delimited stages
(PAPER.md:55). Conv + BatchNorm pairs are folded into (bf16 weight, fp32
scale, fp32 bias); activations live in NHWC bf16; every layer is one launch
of a kernel from include/daris_kernels.h. Torch is used for weight creation
and device memory only.

A ``Network`` holds the device weights (shared by every task running the
same model); a ``TaskBuffers`` holds one job's activations; ``Network.stage_ops``
returns the launch list of a stage for a given buffer set and SM budget,
which the executor captures into one CUDA graph per (task, stage, partition,
buffer set).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import torch
import torch.nn as nn

from . import kernels as K

MODELS = ("resnet18", "resnet50", "vgg16", "mobilenet_v2")


def _pad64(c: int) -> int:
    return (c + 63) // 64 * 64


def randomize_bn(model: nn.Module, seed: int) -> None:
    """Give every BatchNorm non-trivial statistics so folding is exercised."""
    g = torch.Generator().manual_seed(seed)
    for m in model.modules():
        if isinstance(m, nn.BatchNorm2d):
            c = m.num_features
            m.running_mean.copy_(torch.randn(c, generator=g) * 0.1)
            m.running_var.copy_(torch.rand(c, generator=g) * 0.5 + 0.75)
            m.weight.data.copy_(torch.rand(c, generator=g) * 0.5 + 0.75)
            m.bias.data.copy_(torch.randn(c, generator=g) * 0.1)


def make_torch_model(name: str, seed: int = 0) -> nn.Module:
    import torchvision.models as tvm
    torch.manual_seed(seed)
    ctor = {"resnet18": tvm.resnet18, "resnet50": tvm.resnet50, "vgg16": tvm.vgg16,
            "mobilenet_v2": tvm.mobilenet_v2}[name]
    model = ctor(weights=None)
    randomize_bn(model, seed + 1)
    return model.eval()


def fold_bn(conv: nn.Conv2d, bn: nn.BatchNorm2d | None):
    w = conv.weight.detach().float()
    cout = w.shape[0]
    if bn is None:
        scale = torch.ones(cout)
        bias = conv.bias.detach().float() if conv.bias is not None else torch.zeros(cout)
    else:
        inv = torch.rsqrt(bn.running_var.float() + bn.eps)
        scale = bn.weight.detach().float() * inv
        bias = bn.bias.detach().float() - bn.running_mean.float() * scale
        if conv.bias is not None:
            bias = bias + conv.bias.detach().float() * scale
    return w, scale, bias


@dataclass
class ConvLayer:
    """One folded conv (+BN) with its launch geometry; channels padded to 64."""
    name: str
    weight: torch.Tensor          # [cout_p, kh, kw, cin_p] bf16 on device
    scale: torch.Tensor           # [cout_p] fp32
    bias: torch.Tensor
    kh: int
    kw: int
    stride: int
    pad: int
    cin: int                      # padded
    cout: int                     # padded
    relu: int
    flops_per_image: int          # 2*MAC of the unpadded layer at 224x224 input
    padded_input: bool = False    # 8-channel stem read by TMA from a zero-bordered input (DARIS_CONV_PADDED_INPUT)
    dual_cin: int = 0             # > 0: a fused 1x1 branch over cin2 = dual_cin channels (DARIS_CONV_DUAL);
    dual_stride: int = 1          #      weight is then 2-D [cout][kh*kw*cin + dual_cin], scale folded in


@dataclass
class DwLayer:
    name: str
    weight: torch.Tensor          # [k, k, c_p] bf16
    scale: torch.Tensor
    bias: torch.Tensor
    k: int
    stride: int
    pad: int
    c: int
    relu: int
    flops_per_image: int


@dataclass
class LinearLayer:
    name: str
    weight: torch.Tensor          # [out, in] bf16
    bias: torch.Tensor            # fp32
    relu: int
    out_bf16: bool
    flops_per_image: int


def _conv_layer(name, conv, bn, relu, device, hw_out, cin_pad=None) -> ConvLayer:
    w, scale, bias = fold_bn(conv, bn)
    cout, cin, kh, kw = w.shape
    cin_p = cin_pad if cin_pad is not None else _pad64(cin)
    cout_p = _pad64(cout)
    wt = torch.zeros(cout_p, kh, kw, cin_p)
    wt[:cout, :, :, :cin] = w.permute(0, 2, 3, 1)
    sc = torch.zeros(cout_p)
    bi = torch.zeros(cout_p)
    sc[:cout] = scale
    bi[:cout] = bias
    flops = 2 * cout * cin * kh * kw * hw_out
    return ConvLayer(name, wt.to(device=device, dtype=torch.bfloat16).contiguous(), sc.to(device),
                     bi.to(device), kh, kw, conv.stride[0], conv.padding[0], cin_p, cout_p, relu, flops)


def _stem_layer(name, conv, bn, relu, device, hw_out, padded: bool = False) -> ConvLayer:
    """kxk stem over 3 input channels: input packed to NHWC with 8 channels (3 real).
    padded=False: weights [cout][kh][kw][8]; the conv kernel's pixel-chunk mode
    gathers one kernel position (8 channels = 16 B) per chunk.
    padded=True: the input is packed zero-bordered and weights are [cout][kh][8][8]
    (kw padded to 8 pixel slots): one K block per kernel row, loaded as one TMA box
    of overlapping 128-B windows (no gather, no im2col)."""
    w, scale, bias = fold_bn(conv, bn)
    cout, cin, kh, kw = w.shape
    cout_p = _pad64(cout)
    wt = torch.zeros(cout_p, kh, 8 if padded else kw, 8)
    wt[:cout, :, :kw, :cin] = w.permute(0, 2, 3, 1)
    sc = torch.zeros(cout_p)
    bi = torch.zeros(cout_p)
    sc[:cout] = scale
    bi[:cout] = bias
    return ConvLayer(name, wt.to(device=device, dtype=torch.bfloat16).contiguous(), sc.to(device), bi.to(device),
                     kh, kw, conv.stride[0], conv.padding[0], 8, cout_p, relu, 2 * cout * cin * kh * kw * hw_out,
                     padded)


def _dual_layer(name, conv, bn, ds_conv, ds_bn, relu, device, hw_out) -> ConvLayer:
    """A bottleneck's last 1x1 conv with its downsample branch as one GEMM:
    y = relu(A_x * (W*s) + A_in[::stride] * (W_ds*s_ds) + b + b_ds) — the two
    BN scales folded into the bf16 weights, K = [cin | cin_ds], no residual read
    and no separate downsample launch."""
    w, scale, bias = fold_bn(conv, bn)
    wd, sd, bd = fold_bn(ds_conv, ds_bn)
    cout, cin = w.shape[0], w.shape[1]
    cin_d = wd.shape[1]
    cin_p, cind_p, cout_p = _pad64(cin), _pad64(cin_d), _pad64(cout)
    wt = torch.zeros(cout_p, cin_p + cind_p)
    wt[:cout, :cin] = w[:, :, 0, 0] * scale[:, None]
    wt[:cout, cin_p:cin_p + cin_d] = wd[:, :, 0, 0] * sd[:, None]
    sc = torch.zeros(cout_p)
    bi = torch.zeros(cout_p)
    sc[:cout] = 1.0
    bi[:cout] = bias + bd
    flops = 2 * cout * (cin + cin_d) * hw_out
    return ConvLayer(name, wt.to(device=device, dtype=torch.bfloat16).contiguous(), sc.to(device), bi.to(device),
                     1, 1, 1, 0, cin_p, cout_p, relu, flops, False, cind_p, ds_conv.stride[0])


def _stem(b: "_Builder", name, conv, bn, relu, device, batch: int):
    """pack8 + the stem conv; the TMA-window form when the shape allows it."""
    kh, kw = conv.kernel_size
    st, pd = conv.stride[0], conv.padding[0]
    wo = (224 + 2 * pd - kw) // st + 1
    padded = kw <= 8 and wo <= 128
    layer = _stem_layer(name, conv, bn, relu, device, wo * wo, padded)
    b.need("input", batch * 3 * 224 * 224)
    if padded:
        hp, wp = 224 + 2 * pd, 224 + 2 * pd + 8
        b.need("packed", batch * hp * wp * 8)
        b.ops.append(Op("pack8", (pd, 8), "input", "packed", None, (batch, 3, 224, 224), (batch, hp, wp, 8)))
    else:
        b.need("packed", batch * 224 * 224 * 8)
        b.ops.append(Op("pack8", None, "input", "packed", None, (batch, 3, 224, 224), (batch, 224, 224, 8)))
    return b.conv(layer, "packed", (batch, 224, 224, 8))


@dataclass
class Op:
    """One kernel launch of a stage program."""
    kind: str
    layer: object
    src: str
    dst: str
    res: str | None = None
    shape_in: tuple = ()
    shape_out: tuple = ()
    flops: int = 0
    shape_in2: tuple | None = None   # conv with a fused 1x1 branch: the branch input ("res" names it)


@dataclass
class Network:
    name: str
    batch: int
    device: torch.device
    ops: list[Op]
    stage_bounds: list[int]          # op index where each stage starts (+ end sentinel)
    buffer_elems: dict[str, int]     # element counts of the named activation buffers
    input_shape: tuple
    output_shape: tuple
    flops_per_image: int
    torch_model: nn.Module | None = None
    weight_bytes: int = 0

    @property
    def n_stages(self) -> int:
        return len(self.stage_bounds) - 1

    def stage_flops(self) -> list[int]:
        return [sum(op.flops for op in self.ops[a:b]) for a, b in zip(self.stage_bounds, self.stage_bounds[1:])]


@dataclass
class TaskBuffers:
    """Activations + scratch of one job in flight (one 'buffer slot')."""
    bufs: dict[str, torch.Tensor]
    workspace: torch.Tensor
    counters: torch.Tensor

    @property
    def input(self) -> torch.Tensor:
        return self.bufs["input"]

    @property
    def output(self) -> torch.Tensor:
        return self.bufs["logits"]


class _Builder:
    """Assigns activation tensors to a small rotating set of named buffers."""

    def __init__(self, batch: int):
        self.batch = batch
        self.ops: list[Op] = []
        self.sizes: dict[str, int] = {}
        self.free = [f"act{i}" for i in range(6)]
        self.stage_bounds = [0]

    def need(self, name: str, elems: int) -> None:
        self.sizes[name] = max(self.sizes.get(name, 0), elems)

    def take(self, avoid=()) -> str:
        for i, b in enumerate(self.free):
            if b not in avoid:
                return self.free.pop(i)
        raise RuntimeError("activation buffer pool exhausted")

    def give(self, name: str) -> None:
        if name.startswith("act") and name not in self.free:
            self.free.append(name)

    def stage_break(self) -> None:
        self.stage_bounds.append(len(self.ops))

    def conv(self, layer: ConvLayer, src: str, shape, res: str | None = None, dst: str | None = None):
        n, h, w, c = shape
        ho = (h + 2 * layer.pad - layer.kh) // layer.stride + 1
        wo = (w + 2 * layer.pad - layer.kw) // layer.stride + 1
        out_shape = (n, ho, wo, layer.cout)
        if dst is None:
            dst = self.take(avoid=(src, res))
        self.need(dst, n * ho * wo * layer.cout)
        self.ops.append(Op("conv", layer, src, dst, res, shape, out_shape, layer.flops_per_image * n))
        return dst, out_shape


def _pool_classifier(b: "_Builder", lin: LinearLayer, x: str, shape, batch: int) -> None:
    """Global average pool + the final linear layer (two launches)."""
    feat = shape[3]
    b.need("pooled", batch * feat)
    b.need("logits", batch * lin.weight.shape[0])
    out_shape = (batch, lin.weight.shape[0])
    b.ops.append(Op("avgpool", None, x, "pooled", None, shape, (batch, feat)))
    b.ops.append(Op("linear", lin, "pooled", "logits", None, (batch, feat), out_shape, lin.flops_per_image * batch))


def _resnet_ops(model, name, batch, device, split) -> Network:
    b = _Builder(batch)
    x, shape = _stem(b, "conv1", model.conv1, model.bn1, 1, device, batch)
    y = b.take(avoid=(x,))
    b.need(y, batch * 56 * 56 * 64)
    b.ops.append(Op("maxpool", None, x, y, None, shape, (batch, 56, 56, shape[3])))
    b.give(x)
    x, shape = y, (batch, 56, 56, shape[3])
    blocks = []
    for li, layer in enumerate((model.layer1, model.layer2, model.layer3, model.layer4)):
        for bi, blk in enumerate(layer):
            blocks.append((f"layer{li + 1}.{bi}", blk))
    hw = 56
    for idx, (bname, blk) in enumerate(blocks):
        if idx in split:
            b.stage_break()
        stride = blk.conv2.stride[0] if hasattr(blk, "conv3") else blk.conv1.stride[0]
        hw_out = hw // stride
        identity = x
        ds = None
        # the downsample branch rides in the block's last conv as extra K blocks
        # (bottlenecks); otherwise it is its own launch
        fuse_ds = blk.downsample is not None and hasattr(blk, "conv3")
        if blk.downsample is not None and not fuse_ds:
            dl = _conv_layer(f"{bname}.downsample", blk.downsample[0], blk.downsample[1], 0, device, hw_out * hw_out)
            ds, _ = b.conv(dl, x, shape)
            identity = ds
        if hasattr(blk, "conv3"):  # bottleneck
            l1 = _conv_layer(f"{bname}.conv1", blk.conv1, blk.bn1, 1, device, hw * hw)
            t1, s1 = b.conv(l1, x, shape)
            l2 = _conv_layer(f"{bname}.conv2", blk.conv2, blk.bn2, 1, device, hw_out * hw_out)
            t2, s2 = b.conv(l2, t1, s1)
            b.give(t1)
            if fuse_ds:
                l3 = _dual_layer(f"{bname}.conv3+downsample", blk.conv3, blk.bn3, blk.downsample[0],
                                 blk.downsample[1], 1, device, hw_out * hw_out)
                out, s3 = b.conv(l3, t2, s2, res=x)
                b.ops[-1].shape_in2 = shape
            else:
                l3 = _conv_layer(f"{bname}.conv3", blk.conv3, blk.bn3, 1, device, hw_out * hw_out)
                out, s3 = b.conv(l3, t2, s2, res=identity)
            b.give(t2)
        else:
            l1 = _conv_layer(f"{bname}.conv1", blk.conv1, blk.bn1, 1, device, hw_out * hw_out)
            t1, s1 = b.conv(l1, x, shape)
            l2 = _conv_layer(f"{bname}.conv2", blk.conv2, blk.bn2, 1, device, hw_out * hw_out)
            out, s3 = b.conv(l2, t1, s1, res=identity)
            b.give(t1)
        if ds is not None:
            b.give(ds)
        b.give(x)
        x, shape, hw = out, s3, hw_out
    fc = model.fc
    feat = shape[3]
    lin = LinearLayer("fc", fc.weight.detach().to(device=device, dtype=torch.bfloat16).contiguous(),
                      fc.bias.detach().float().to(device), 0, False, 2 * fc.in_features * fc.out_features)
    _pool_classifier(b, lin, x, shape, batch)
    b.stage_break()
    flops = sum(op.flops for op in b.ops) // batch
    return Network(name, batch, device, b.ops, b.stage_bounds, b.sizes, (batch, 3, 224, 224),
                   (batch, fc.out_features), flops)


def _vgg_ops(model, batch, device, n_stages) -> Network:
    b = _Builder(batch)
    feats = list(model.features)
    convs = [(i, m) for i, m in enumerate(feats) if isinstance(m, nn.Conv2d)]
    pools = [i for i, m in enumerate(feats) if isinstance(m, nn.MaxPool2d)]
    # stage boundaries at the maxpools (VGG "splits at its maxpools", SURVEY §8a')
    breaks_after = set(pools[:-1][: max(0, n_stages - 1)]) if n_stages > 1 else set()
    b.need("input", batch * 3 * 224 * 224)
    hw = 224
    x, shape = None, None
    for i, m in enumerate(feats):
        if isinstance(m, nn.Conv2d):
            if x is None:
                stem = _stem_layer(f"features.{i}", m, None, 1, device, hw * hw)
                b.need("packed", batch * 224 * 224 * 8)
                b.ops.append(Op("pack8", None, "input", "packed", None, (batch, 3, 224, 224), (batch, 224, 224, 8)))
                x, shape = b.conv(stem, "packed", (batch, 224, 224, 8))
            else:
                layer = _conv_layer(f"features.{i}", m, None, 1, device, hw * hw)
                nx, shape = b.conv(layer, x, shape)
                b.give(x)
                x = nx
        elif isinstance(m, nn.MaxPool2d):
            y = b.take(avoid=(x,))
            hw //= 2
            b.need(y, batch * hw * hw * shape[3])
            b.ops.append(Op("maxpool2", None, x, y, None, shape, (batch, hw, hw, shape[3])))
            b.give(x)
            x, shape = y, (batch, hw, hw, shape[3])
            if i in breaks_after:
                b.stage_break()
    # classifier: NHWC flatten order -> permute FC1 columns from torch's NCHW order
    lins = [m for m in model.classifier if isinstance(m, nn.Linear)]
    c = shape[3]
    w1 = lins[0].weight.detach().reshape(-1, c, 7, 7).permute(0, 2, 3, 1).reshape(lins[0].out_features, -1)
    src = x
    for k, lin in enumerate(lins):
        w = w1 if k == 0 else lin.weight.detach()
        last = k == len(lins) - 1
        L = LinearLayer(f"classifier.{k}", w.to(device=device, dtype=torch.bfloat16).contiguous(),
                        lin.bias.detach().float().to(device), 0 if last else 1, not last,
                        2 * lin.in_features * lin.out_features)
        dst = "logits" if last else f"fc{k}"
        b.need(dst, batch * lin.out_features)
        b.ops.append(Op("linear", L, src, dst, None, (batch, lin.in_features), (batch, lin.out_features),
                        L.flops_per_image * batch))
        src = dst
    b.stage_break()
    flops = sum(op.flops for op in b.ops) // batch
    return Network("vgg16", batch, device, b.ops, b.stage_bounds, b.sizes, (batch, 3, 224, 224),
                   (batch, lins[-1].out_features), flops)


def _mbv2_ops(model, batch, device, n_stages) -> Network:
    b = _Builder(batch)
    feats = list(model.features)
    b.need("input", batch * 3 * 224 * 224)
    first = feats[0]
    x, shape = _stem(b, "features.0", first[0], first[1], 6, device, batch)
    blocks = feats[1:-1]
    # split the inverted-residual sequence into n_stages groups of roughly equal count
    per = max(1, (len(blocks) + n_stages - 1) // n_stages) if n_stages > 1 else len(blocks) + 1
    hw = 112
    for bi, blk in enumerate(blocks):
        if bi > 0 and bi % per == 0 and len(b.stage_bounds) < n_stages:
            b.stage_break()
        layers = list(blk.conv)
        src = x
        k = 0
        cur, cshape = x, shape
        owned = []
        if len(layers) == 4:  # expand 1x1 + dw + project
            exp = layers[0]
            L = _conv_layer(f"features.{bi + 1}.expand", exp[0], exp[1], 6, device, hw * hw)
            cur, cshape = b.conv(L, cur, cshape)
            owned.append(cur)
            k = 1
        dw = layers[k]
        conv = dw[0]
        stride = conv.stride[0]
        hw_out = hw // stride
        w, scale, bias = fold_bn(conv, dw[1])
        c = w.shape[0]
        cp = _pad64(c)
        wt = torch.zeros(3, 3, cp)
        wt[:, :, :c] = w[:, 0].permute(1, 2, 0)
        sc = torch.zeros(cp)
        bi_ = torch.zeros(cp)
        sc[:c] = scale
        bi_[:c] = bias
        D = DwLayer(f"features.{bi + 1}.dw", wt.to(device=device, dtype=torch.bfloat16).contiguous(), sc.to(device),
                    bi_.to(device), 3, stride, 1, cp, 6, 2 * 9 * c * hw_out * hw_out)
        dst = b.take(avoid=(cur, src))
        out_shape = (batch, hw_out, hw_out, cp)
        b.need(dst, batch * hw_out * hw_out * cp)
        b.ops.append(Op("dwconv", D, cur, dst, None, cshape, out_shape, D.flops_per_image * batch))
        for o in owned:
            b.give(o)
        proj_conv, proj_bn = layers[k + 1], layers[k + 2]
        P = _conv_layer(f"features.{bi + 1}.project", proj_conv, proj_bn, 0, device, hw_out * hw_out)
        res = src if blk.use_res_connect else None
        out, oshape = b.conv(P, dst, out_shape, res=res)
        b.give(dst)
        b.give(src)
        x, shape, hw = out, oshape, hw_out
    last = feats[-1]
    L = _conv_layer("features.18", last[0], last[1], 6, device, hw * hw)
    nx, shape = b.conv(L, x, shape)
    b.give(x)
    x = nx
    fc = [m for m in model.classifier if isinstance(m, nn.Linear)][0]
    lin = LinearLayer("classifier", fc.weight.detach().to(device=device, dtype=torch.bfloat16).contiguous(),
                      fc.bias.detach().float().to(device), 0, False, 2 * fc.in_features * fc.out_features)
    _pool_classifier(b, lin, x, shape, batch)
    b.stage_break()
    flops = sum(op.flops for op in b.ops) // batch
    return Network("mobilenet_v2", batch, device, b.ops, b.stage_bounds, b.sizes, (batch, 3, 224, 224),
                   (batch, fc.out_features), flops)


# default stage splits: block indices (in the flattened residual-block list) that open a new stage
RESNET18_SPLITS = {1: [], 2: [4], 3: [2, 5], 4: [2, 4, 6]}   # 3 stages: FLOP-balanced (SURVEY §8a')
RESNET50_SPLITS = {1: [], 2: [7], 3: [3, 10], 4: [3, 7, 13]}  # 4 stages: layer1..layer4


def build_network(name: str, *, batch: int = 1, n_stages: int | None = None, seed: int = 0,
                  device: torch.device | str = "cuda", keep_torch: bool = False,
                  model: nn.Module | None = None) -> Network:
    """The network as a list of kernel launches (Op) with stage boundaries,
    BN folded into bf16 weights + fp32 scale/bias, the TMA-window stem and the
    downsample branch fused into each bottleneck's last conv."""
    device = torch.device(device)
    if model is None:
        model = make_torch_model(name, seed)
    with torch.no_grad():
        if name == "resnet18":
            n_stages = n_stages or 3
            net = _resnet_ops(model, name, batch, device, set(RESNET18_SPLITS[n_stages]))
        elif name == "resnet50":
            n_stages = n_stages or 4
            net = _resnet_ops(model, name, batch, device, set(RESNET50_SPLITS[n_stages]))
        elif name == "vgg16":
            net = _vgg_ops(model, batch, device, n_stages or 4)
        elif name == "mobilenet_v2":
            net = _mbv2_ops(model, batch, device, n_stages or 3)
        else:
            raise ValueError(f"unknown model {name!r}; known: {MODELS}")
    if keep_torch:
        net.torch_model = model
    seen = set()
    wb = 0
    for op in net.ops:
        L = op.layer
        if L is not None and id(L) not in seen and hasattr(L, "weight"):
            seen.add(id(L))
            wb += L.weight.numel() * 2
    net.weight_bytes = wb
    return net


def allocate_buffers(net: Network, sm_budget: int = 0) -> TaskBuffers:
    bufs = {}
    for name, elems in net.buffer_elems.items():
        if name == "input":
            bufs[name] = torch.zeros(net.input_shape, dtype=torch.float32, device=net.device)
        elif name == "logits":
            bufs[name] = torch.zeros(elems, dtype=torch.float32, device=net.device)
        else:
            bufs[name] = torch.zeros(elems, dtype=torch.bfloat16, device=net.device)
    ws = 1
    ctr = 1
    for op in net.ops:
        if op.kind == "conv":
            L = op.layer
            d = K.conv_desc(op.shape_in, L.cout, L.kh, L.kw, L.stride, L.pad, relu=L.relu, sm_budget=sm_budget,
                            padded_input=L.padded_input, x2_shape=op.shape_in2 if L.dual_cin else None,
                            stride2=L.dual_stride)
            p = K.conv_plan(d)
            ws = max(ws, p.workspace_floats)
            ctr = max(ctr, p.counters)
        elif op.kind == "linear":
            L = op.layer
            p = K.linear_plan(K.linear_desc(op.shape_in[0], op.shape_in[1], L.weight.shape[0], relu=L.relu,
                                            y_bf16=L.out_bf16, sm_budget=sm_budget))
            ws = max(ws, p.workspace_floats)
            ctr = max(ctr, p.counters)
    return TaskBuffers(bufs, torch.zeros(ws, dtype=torch.float32, device=net.device),
                       torch.zeros(ctr, dtype=torch.int32, device=net.device))


def _view(t: torch.Tensor, shape) -> torch.Tensor:
    n = 1
    for s in shape:
        n *= s
    return t.view(-1)[:n].view(shape)


def run_op(op: Op, tb: TaskBuffers, stream, sm_budget: int = 0, timestamps=None) -> None:
    B = tb.bufs
    if op.kind == "pack8":
        border, extra = op.layer if op.layer else (0, 0)
        K.pack_nhwc(B["input"], 8, out=_view(B["packed"], op.shape_out), border=border, extra=extra,
                    stream=stream)
    elif op.kind == "conv":
        L = op.layer
        if L.dual_cin:  # fused 1x1 branch over the block input (named by op.res)
            K.conv2d(_view(B[op.src], op.shape_in), L.weight, L.scale, L.bias, stride=L.stride, pad=L.pad,
                     relu=L.relu, out=_view(B[op.dst], op.shape_out), workspace=tb.workspace,
                     counters=tb.counters, sm_budget=sm_budget, stream=stream, kh=L.kh, kw=L.kw,
                     x2=_view(B[op.res], op.shape_in2), stride2=L.dual_stride, timestamps=timestamps)
            return
        res = _view(B[op.res], op.shape_out) if op.res else None
        K.conv2d(_view(B[op.src], op.shape_in), L.weight, L.scale, L.bias, stride=L.stride, pad=L.pad,
                 relu=L.relu, residual=res, out=_view(B[op.dst], op.shape_out), workspace=tb.workspace,
                 counters=tb.counters, sm_budget=sm_budget, stream=stream, padded_input=L.padded_input,
                 kw=L.kw, timestamps=timestamps)
    elif op.kind == "maxpool":
        K.maxpool(_view(B[op.src], op.shape_in), 3, 2, 1, out=_view(B[op.dst], op.shape_out), stream=stream)
    elif op.kind == "maxpool2":
        K.maxpool(_view(B[op.src], op.shape_in), 2, 2, 0, out=_view(B[op.dst], op.shape_out), stream=stream)
    elif op.kind == "avgpool":
        K.avgpool(_view(B[op.src], op.shape_in), out=_view(B[op.dst], op.shape_out), stream=stream)
    elif op.kind == "linear":
        L = op.layer
        src = B[op.src]
        x = _view(src, op.shape_in)
        out = _view(B[op.dst], op.shape_out)
        if L.out_bf16 and out.dtype != torch.bfloat16:
            raise RuntimeError("bf16 linear output needs a bf16 buffer")
        K.linear_tc(x, L.weight, L.bias, relu=L.relu, out=out, workspace=tb.workspace, counters=tb.counters,
                    sm_budget=sm_budget, stream=stream)
    elif op.kind == "dwconv":
        L = op.layer
        K.dwconv(_view(B[op.src], op.shape_in), L.weight, L.scale, L.bias, stride=L.stride, pad=L.pad, relu=L.relu,
                 out=_view(B[op.dst], op.shape_out), stream=stream)
    else:
        raise ValueError(op.kind)


def stage_launches(net: Network, stage: int) -> int:
    """Kernel launches one execution of the stage issues."""
    return net.stage_bounds[stage + 1] - net.stage_bounds[stage]


def run_stage(net: Network, stage: int, tb: TaskBuffers, stream, sm_budget: int = 0) -> int:
    """Launch one stage (one kernel per op); returns the number of launches issued."""
    a, b = net.stage_bounds[stage], net.stage_bounds[stage + 1]
    for op in net.ops[a:b]:
        run_op(op, tb, stream, sm_budget)
    return b - a


def forward(net: Network, tb: TaskBuffers, x: torch.Tensor | None = None, stream=None, sm_budget: int = 0):
    if x is not None:
        tb.input.copy_(x)
    for s in range(net.n_stages):
        run_stage(net, s, tb, stream, sm_budget)
    return _view(tb.output, net.output_shape)
