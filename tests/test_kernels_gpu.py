"""Numerics of the sm_100a stage kernels against a plain PyTorch fp32
reference of the same op (inputs rounded to bf16 first, so the only error
left is fp32-vs-tensor-core accumulation order and the bf16 output rounding).

Tolerance (stated per SURVEY §8c P3): max |err| <= 1e-2 * max |ref| and
relative L2 error <= 1e-2.
"""

import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu

TOL_MAX = 1e-2
TOL_L2 = 1e-2


def _close(out, ref):
    out = out.float().cpu()
    ref = ref.float().cpu()
    err = (out - ref).abs().max().item()
    scale = ref.abs().max().item() + 1e-6
    l2 = ((out - ref).norm() / (ref.norm() + 1e-6)).item()
    assert err <= TOL_MAX * scale, f"max err {err} vs scale {scale}"
    assert l2 <= TOL_L2, f"rel l2 {l2}"


def _conv_case(n, h, w, cin, cout, k, stride, pad, relu=1, residual=False, block_n=0, splits=0,
               sm_budget=0, seed=0, cluster=None):
    from paper_2504_08795_b200 import kernels as K
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(n, h, w, cin, generator=g).bfloat16()
    wt = (torch.randn(cout, k, k, cin, generator=g) / (k * k * cin) ** 0.5).bfloat16()
    scale = torch.rand(cout, generator=g) + 0.5
    bias = torch.randn(cout, generator=g) * 0.1
    ho = (h + 2 * pad - k) // stride + 1
    wo = (w + 2 * pad - k) // stride + 1
    res = torch.randn(n, ho, wo, cout, generator=g).bfloat16() if residual else None
    ref = F.conv2d(x.float().permute(0, 3, 1, 2), wt.float().permute(0, 3, 1, 2), stride=stride, padding=pad)
    ref = ref.permute(0, 2, 3, 1) * scale + bias
    if res is not None:
        ref = ref + res.float()
    if relu == 1:
        ref = ref.clamp_min(0)
    elif relu == 6:
        ref = ref.clamp(0, 6)
    dev = torch.device("cuda")
    out = K.conv2d(x.to(dev), wt.to(dev), scale.to(dev), bias.to(dev), stride=stride, pad=pad, relu=relu,
                   residual=None if res is None else res.to(dev), block_n=block_n, splits=splits,
                   sm_budget=sm_budget, cluster=cluster)
    torch.cuda.synchronize()
    _close(out, ref)


@pytest.mark.parametrize("bn", [64, 128, 256])
def test_conv3x3_layer1_shapes(bn):
    _conv_case(1, 56, 56, 64, 256 if bn == 256 else 128, 3, 1, 1, block_n=bn, splits=1)


def test_conv3x3_resnet18_layer1_auto():
    _conv_case(1, 56, 56, 64, 64, 3, 1, 1)


def test_conv3x3_stride2():
    _conv_case(1, 56, 56, 64, 128, 3, 2, 1)


def test_conv1x1_downsample_stride2_no_relu():
    _conv_case(1, 56, 56, 256, 512, 1, 2, 0, relu=0)


def test_conv_residual_relu():
    _conv_case(1, 28, 28, 128, 128, 3, 1, 1, residual=True)


def test_conv_relu6():
    _conv_case(1, 14, 14, 64, 128, 1, 1, 0, relu=6)


@pytest.mark.parametrize("cluster", [True, False])
@pytest.mark.parametrize("splits", [2, 3, 8])
def test_conv_split_k_forced(splits, cluster):
    # cluster=True: split-K partials reduced through DSMEM inside one cluster;
    # cluster=False: red.add into a global fp32 tile + last-arriver fix-up
    _conv_case(1, 7, 7, 512, 512, 3, 1, 1, splits=splits, residual=True, cluster=cluster)


@pytest.mark.parametrize("cluster", [True, False])
def test_conv_split_k_auto_small_m(cluster):
    _conv_case(1, 7, 7, 512, 512, 3, 1, 1, sm_budget=74, cluster=cluster)


@pytest.mark.parametrize("cluster", [True, False])
def test_conv_split_k_tail_rows_and_odd_cluster(cluster):
    # M = 196 (two M tiles, the second mostly past the end), 5 splits (odd cluster size)
    _conv_case(1, 14, 14, 256, 256, 3, 1, 1, splits=5, residual=True, cluster=cluster, seed=7)


def test_conv_batch_tail_tile():
    _conv_case(3, 13, 11, 64, 64, 3, 1, 1, seed=3)


def test_conv_split_k_repeat_resets_counters():
    # the same workspace/counters reused by back-to-back launches (CUDA-graph pattern)
    from paper_2504_08795_b200 import kernels as K
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(5)
    x = torch.randn(1, 7, 7, 512, generator=g).bfloat16().to(dev)
    wt = (torch.randn(512, 3, 3, 512, generator=g) / 48).bfloat16().to(dev)
    s = torch.ones(512, device=dev)
    b = torch.zeros(512, device=dev)
    d = K.conv_desc((1, 7, 7, 512), 512, 3, 3, 1, 1, sm_budget=148, cluster=False)
    p = K.conv_plan(d)
    assert p.splits > 1 and p.cluster == 1
    ws = torch.zeros(p.workspace_floats, device=dev)
    ctr = torch.zeros(p.counters, dtype=torch.int32, device=dev)
    outs = [K.conv2d(x, wt, s, b, pad=1, workspace=ws, counters=ctr, sm_budget=148, cluster=False).clone()
            for _ in range(3)]
    torch.cuda.synchronize()
    assert int(ctr.abs().sum()) == 0          # tickets re-armed
    assert float(ws.abs().sum()) == 0.0       # accumulators re-zeroed
    # fp32 atomics reorder the split sums: equal up to bf16 output rounding
    for o in outs[1:]:
        assert (o.float() - outs[0].float()).abs().max().item() <= 2e-2 * outs[0].float().abs().max().item()


def test_stem_im2col_gemm_matches_conv7x7():
    from paper_2504_08795_b200 import kernels as K
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(1)
    x = torch.randn(2, 3, 224, 224, generator=g)
    wt = torch.randn(64, 3, 7, 7, generator=g) / 12
    scale = torch.rand(64, generator=g) + 0.5
    bias = torch.randn(64, generator=g) * 0.1
    xb = x.bfloat16().float()
    wb = wt.bfloat16().float()
    ref = F.conv2d(xb, wb, stride=2, padding=3).permute(0, 2, 3, 1) * scale + bias
    ref = ref.clamp_min(0)
    a = K.stem_im2col(x.to(dev), 7, 7, 2, 3, 192)
    wmat = torch.zeros(64, 192)
    wmat[:, :147] = wt.reshape(64, 147)
    out = K.conv2d(a, wmat.bfloat16().reshape(64, 1, 1, 192).to(dev), scale.to(dev), bias.to(dev))
    torch.cuda.synchronize()
    _close(out, ref)


def test_maxpool_avgpool_linear_dwconv():
    from paper_2504_08795_b200 import kernels as K
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(2)
    x = torch.randn(2, 112, 112, 64, generator=g).bfloat16()
    ref = F.max_pool2d(x.float().permute(0, 3, 1, 2), 3, 2, 1).permute(0, 2, 3, 1)
    out = K.maxpool(x.to(dev), 3, 2, 1)
    torch.cuda.synchronize()
    assert torch.equal(out.float().cpu(), ref.bfloat16().float())

    x = torch.randn(3, 7, 7, 2048, generator=g).bfloat16()
    pooled = K.avgpool(x.to(dev))
    torch.cuda.synchronize()
    _close(pooled, x.float().mean(dim=(1, 2)))

    w = (torch.randn(1000, 2048, generator=g) / 45).bfloat16()
    bias = torch.randn(1000, generator=g)
    xin = torch.randn(5, 2048, generator=g)
    y = K.linear(xin.to(dev), w.to(dev), bias.to(dev))
    torch.cuda.synchronize()
    _close(y, xin @ w.float().t() + bias)

    x = torch.randn(1, 56, 56, 96, generator=g).bfloat16()
    wd = (torch.randn(3, 3, 96, generator=g) / 3).bfloat16()
    sc = torch.rand(96, generator=g) + 0.5
    bi = torch.randn(96, generator=g) * 0.1
    ref = F.conv2d(x.float().permute(0, 3, 1, 2), wd.float().permute(2, 0, 1).unsqueeze(1), stride=2, padding=1,
                   groups=96).permute(0, 2, 3, 1) * sc + bi
    out = K.dwconv(x.to(dev), wd.to(dev), sc.to(dev), bi.to(dev), stride=2, pad=1, relu=6)
    torch.cuda.synchronize()
    _close(out, ref.clamp(0, 6))


@pytest.mark.parametrize("n,hw,c,k,stride,pad", [(3, 57, 64, 3, 2, 1), (1, 112, 64, 3, 2, 1), (2, 14, 512, 2, 2, 0),
                                                 (2, 9, 24, 3, 1, 1)])
def test_maxpool_shapes_exact(n, hw, c, k, stride, pad):
    """max pooling is exact in bf16: the 3x3 fast path (packed bf16 maxima) and
    the generic kernel (VGG's 2x2) equal torch bit for bit, border windows included."""
    from paper_2504_08795_b200 import kernels as K
    g = torch.Generator().manual_seed(n * hw + c + k)
    x = torch.randn(n, hw, hw, c, generator=g).bfloat16()
    ref = F.max_pool2d(x.float().permute(0, 3, 1, 2), k, stride, pad).permute(0, 2, 3, 1)
    out = K.maxpool(x.cuda(), k, stride, pad)
    torch.cuda.synchronize()
    assert torch.equal(out.float().cpu(), ref.bfloat16().float())


@pytest.mark.parametrize("k,stride,pad,hw", [(7, 2, 3, 224), (3, 1, 1, 224), (3, 2, 1, 224)])
def test_stem_pixel_chunk_mode_matches_conv(k, stride, pad, hw):
    """cin == 8 stem mode: NHWC8 input (3 real channels), K = k*k*8 zero-padded by TMA."""
    from paper_2504_08795_b200 import kernels as K
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(k + stride)
    x = torch.randn(2, 3, hw, hw, generator=g)
    wt = torch.randn(64, 3, k, k, generator=g) / (3 * k * k) ** 0.5
    scale = torch.rand(64, generator=g) + 0.5
    bias = torch.randn(64, generator=g) * 0.1
    ref = F.conv2d(x.bfloat16().float(), wt.bfloat16().float(), stride=stride, padding=pad)
    ref = (ref.permute(0, 2, 3, 1) * scale + bias).clamp_min(0)
    packed = K.pack_nhwc(x.to(dev), 8)
    w8 = torch.zeros(64, k, k, 8)
    w8[..., :3] = wt.permute(0, 2, 3, 1)
    out = K.conv2d(packed, w8.bfloat16().to(dev), scale.to(dev), bias.to(dev), stride=stride, pad=pad)
    torch.cuda.synchronize()
    _close(out, ref)


@pytest.mark.parametrize("k,stride,pad,hw,batch", [(7, 2, 3, 224, 2), (3, 2, 1, 224, 1), (7, 2, 3, 64, 3)])
def test_stem_tma_window_mode_matches_conv(k, stride, pad, hw, batch):
    """DARIS_CONV_PADDED_INPUT stems: zero-bordered NHWC8 input, one TMA box of
    overlapping 128-B windows per kernel row, weights [cout][k][8][8]."""
    from paper_2504_08795_b200 import kernels as K
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(100 + k + stride)
    x = torch.randn(batch, 3, hw, hw, generator=g)
    wt = torch.randn(64, 3, k, k, generator=g) / (3 * k * k) ** 0.5
    scale = torch.rand(64, generator=g) + 0.5
    bias = torch.randn(64, generator=g) * 0.1
    ref = F.conv2d(x.bfloat16().float(), wt.bfloat16().float(), stride=stride, padding=pad)
    ref = (ref.permute(0, 2, 3, 1) * scale + bias).clamp_min(0)
    packed = K.pack_nhwc(x.to(dev), 8, border=pad, extra=8)
    assert packed.shape == (batch, hw + 2 * pad, hw + 2 * pad + 8, 8)
    inner = packed[:, pad:pad + hw, pad:pad + hw, :3].float().cpu()
    assert torch.equal(inner, x.bfloat16().float().permute(0, 2, 3, 1))
    assert packed[:, :pad].abs().sum().item() == 0 and packed[:, :, :pad].abs().sum().item() == 0
    w8 = torch.zeros(64, k, 8, 8)
    w8[:, :, :k, :3] = wt.permute(0, 2, 3, 1)
    view = packed.view(-1)[: batch * hw * hw * 8].view(batch, hw, hw, 8)  # logical shape, padded storage
    out = K.conv2d(view, w8.bfloat16().to(dev), scale.to(dev), bias.to(dev), stride=stride, pad=pad,
                   padded_input=True, kw=k)
    torch.cuda.synchronize()
    _close(out, ref)


@pytest.mark.parametrize("n,hw,cin,cout,hw2,cin2,stride2,sm", [(1, 28, 128, 512, 56, 256, 2, 23), (1, 56, 64, 256, 56, 64, 1, 23),
                                                              (2, 7, 512, 2048, 14, 1024, 2, 23), (1, 14, 256, 1024, 28, 512, 2, 72),
                                                              # images stacked along H (flat 1x1 tiling): tiles span images
                                                              (64, 7, 512, 2048, 14, 1024, 2, 148), (5, 14, 256, 1024, 28, 512, 2, 148)])
def test_conv_dual_branch_matches_sum_of_convs(n, hw, cin, cout, hw2, cin2, stride2, sm):
    """DARIS_CONV_DUAL: a 1x1 conv over x plus a 1x1 stride-s branch over x2 in one
    GEMM (the ResNet downsample folded into the block's last conv)."""
    from paper_2504_08795_b200 import kernels as K
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(cin + cin2)
    x = torch.randn(n, hw, hw, cin, generator=g).bfloat16()
    x2 = torch.randn(n, hw2, hw2, cin2, generator=g).bfloat16()
    w = (torch.randn(cout, cin + cin2, generator=g) / (cin + cin2) ** 0.5).bfloat16()
    bias = torch.randn(cout, generator=g) * 0.1
    ref = x.float() @ w[:, :cin].float().t() + x2[:, ::stride2, ::stride2, :].float() @ w[:, cin:].float().t()
    ref = (ref + bias).clamp_min(0)
    out = K.conv2d(x.to(dev), w.to(dev), torch.ones(cout, device=dev), bias.to(dev), relu=1, kh=1, kw=1,
                   x2=x2.to(dev), stride2=stride2, sm_budget=sm)
    torch.cuda.synchronize()
    _close(out, ref)


@pytest.mark.parametrize("batch,k,o,x_bf16,relu", [(1, 25088, 4096, False, 1), (3, 25088, 300, False, 0),
                                                  (1, 4104, 1000, True, 1), (4, 8192, 777, True, 0)])
def test_linear_wide_k(batch, k, o, x_bf16, relu):
    """linear_wide_kernel (K > 4096: VGG's classifier): the input staged in shared
    memory per K tile, weight rows streamed, first tile prefetched before the wait."""
    from paper_2504_08795_b200 import kernels as K
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(k + o)
    x = torch.randn(batch, k, generator=g)
    if x_bf16:
        x = x.bfloat16()
    w = (torch.randn(o, k, generator=g) / k ** 0.5).bfloat16()
    bias = torch.randn(o, generator=g)
    y = K.linear(x.to(dev), w.to(dev), bias.to(dev), relu=relu)
    torch.cuda.synchronize()
    ref = x.float() @ w.float().t() + bias
    _close(y, ref.clamp_min(0) if relu else ref)


@pytest.mark.parametrize("n,h,cin,cout,k,stride,pad,relu,residual,bn", [
    (16, 56, 64, 64, 3, 1, 1, 1, False, 0),      # layer1 conv2 at batch 16 (BN=64)
    (16, 56, 64, 256, 1, 1, 0, 1, True, 128),    # layer1 conv3 + residual (BN=128, short K)
    (8, 56, 256, 128, 3, 2, 1, 6, False, 128),   # strided, ReLU6
    (32, 14, 256, 1024, 1, 1, 0, 0, True, 128),  # two-image-row tiles, no activation
    (4, 28, 128, 128, 3, 1, 1, 1, True, 64),
    # 1x1 convs tiled as a flat pixel GEMM (fewer M tiles than per-image rows)
    (64, 7, 512, 2048, 1, 1, 0, 1, True, 128),   # layer4 conv3 at batch 64: 25 tiles, last one 64 rows
    (8, 7, 2048, 512, 1, 1, 0, 1, False, 0),     # layer4 conv1 at batch 8
    (3, 14, 256, 1024, 1, 1, 0, 1, True, 128),   # 588 px as 14 rows of 42: 5 tiles (was 6), ragged tail
    # 3x3 on 7x7 maps: two whole images per 128-row tile (the last tile holds one)
    (3, 7, 512, 512, 3, 1, 1, 1, True, 128),
    (5, 7, 256, 256, 3, 1, 1, 6, False, 64),
])
def test_conv_large_m(n, h, cin, cout, k, stride, pad, relu, residual, bn):
    """Batched (large-M) launches on a small SM budget: many waves of tiles."""
    _conv_case(n, h, h, cin, cout, k, stride, pad, relu=relu, residual=residual, block_n=bn, sm_budget=8)


@pytest.mark.parametrize("batch,k,o,relu,out_bf16,splits,sm", [
    (1, 2048, 1000, 0, False, 0, 23),      # ResNet-50 classifier, batch 1 (split-K weight stream)
    (64, 2048, 1000, 0, False, 0, 148),    # ... batch 64 (single-tenant batching)
    (17, 2048, 1000, 0, False, 0, 148),    # ragged batch (N tile 32, rows 17..31 zero-filled)
    (3, 512, 1000, 0, False, 1, 0),        # ResNet-18 head, no split
    (100, 1280, 1000, 0, False, 0, 148),   # MobileNetV2 head, batch 100 (N tile 128)
    (300, 512, 200, 1, True, 0, 148),      # two N tiles, bf16 output, ReLU
    (1, 25088, 4096, 1, True, 0, 24),      # VGG-16 FC1 at batch 1 in a 24-SM partition
    (2, 4096, 4096, 1, True, 0, 148),      # VGG-16 FC2
    (32, 4096, 1000, 0, False, 7, 0),      # forced split count
])
def test_linear_tc(batch, k, o, relu, out_bf16, splits, sm):
    """daris_linear_tc (tcgen05 swap-AB) vs a torch fp32 GEMM of the same bf16
    operands; run twice to check the split-K accumulator/tickets re-arm."""
    from paper_2504_08795_b200 import kernels as K
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(batch * 7 + k + o)
    x = torch.randn(batch, k, generator=g).bfloat16()
    w = (torch.randn(o, k, generator=g) / k ** 0.5).bfloat16()
    bias = torch.randn(o, generator=g)
    ref = x.float() @ w.float().t() + bias
    if relu:
        ref = ref.clamp_min(0)
    d = K.linear_desc(batch, k, o, relu=relu, y_bf16=out_bf16, splits=splits, sm_budget=sm)
    p = K.linear_plan(d)
    ws = torch.zeros(max(1, p.workspace_floats), device=dev)
    ctr = torch.zeros(max(1, p.counters), dtype=torch.int32, device=dev)
    xd, wd, bd = x.to(dev), w.to(dev), bias.to(dev)
    for _ in range(2):
        y = K.linear_tc(xd, wd, bd, relu=relu, out_bf16=out_bf16, workspace=ws, counters=ctr, splits=splits,
                        sm_budget=sm)
        torch.cuda.synchronize()
        _close(y, ref)
    assert int(ctr.abs().sum()) == 0 and float(ws.abs().sum()) == 0.0  # scratch re-armed


def test_avgpool_bf16():
    from paper_2504_08795_b200 import kernels as K
    g = torch.Generator().manual_seed(5)
    x = torch.randn(3, 7, 7, 2048, generator=g).bfloat16()
    y = K.avgpool(x.cuda(), out_bf16=True)
    torch.cuda.synchronize()
    assert y.dtype == torch.bfloat16
    _close(y, x.float().mean(dim=(1, 2)))


@pytest.mark.parametrize("n,h,cin,cout,k,stride,pad,residual,bn", [
    (8, 28, 128, 128, 3, 1, 1, True, 128),     # layer2 conv2 shape at batch 8, residual
    (3, 28, 256, 256, 3, 1, 1, True, 256),     # odd M-tile count (21): a phantom tile in the last pair
    (8, 56, 128, 128, 3, 2, 1, False, 128),    # strided
    (16, 14, 256, 256, 3, 1, 1, True, 128),    # layer3 conv2 shape (K = 2304) with a residual
    (16, 7, 512, 512, 3, 1, 1, False, 256),    # layer4 conv2: two whole images per 128-row tile
])
def test_conv_cta_pair(n, h, cin, cout, k, stride, pad, residual, bn):
    """cta_group::2 pairs (UMMA M = 256 over two M tiles, each CTA loading half
    the weight tile): the planner picks them for large-M grids; numerics as the
    one-CTA path."""
    from paper_2504_08795_b200 import kernels as K
    K.CTA_PAIRS = True  # (an executor created earlier in this process turns them off for its tenants)
    d = K.conv_desc((n, h, h, cin), cout, k, k, stride, pad, block_n=bn, sm_budget=8)
    p = K.conv_plan(d)
    assert p.pair == 1 and p.splits == 1, (p.pair, p.splits)
    _conv_case(n, h, h, cin, cout, k, stride, pad, residual=residual, block_n=bn, sm_budget=8, seed=n + h)


def test_conv_cta_pair_dual_branch():
    """The pair path with the fused downsample branch (layer4.0 conv3 at batch 8;
    the default plan keeps 2048-channel convs on one-CTA tiles, so pairs are
    forced with DARIS_CONV_PAIR=2 in a child process: the planner reads it once)."""
    import os
    import subprocess
    import sys
    code = r"""
import sys, torch
sys.path[:0] = [sys.argv[1], sys.argv[1] + '/tests']
import test_kernels_gpu as T
from paper_2504_08795_b200 import kernels as K
dev = torch.device('cuda')
g = torch.Generator().manual_seed(77)
n, hw, cin, cout, hw2, cin2, stride2 = 8, 7, 512, 2048, 14, 1024, 2
d = K.conv_desc((n, hw, hw, cin), cout, 1, 1, 1, 0, sm_budget=8, x2_shape=(n, hw2, hw2, cin2), stride2=stride2)
assert K.conv_plan(d).pair == 1
x = torch.randn(n, hw, hw, cin, generator=g).bfloat16()
x2 = torch.randn(n, hw2, hw2, cin2, generator=g).bfloat16()
w = (torch.randn(cout, cin + cin2, generator=g) / (cin + cin2) ** 0.5).bfloat16()
bias = torch.randn(cout, generator=g) * 0.1
ref = x.float() @ w[:, :cin].float().t() + x2[:, ::stride2, ::stride2, :].float() @ w[:, cin:].float().t()
ref = (ref + bias).clamp_min(0)
out = K.conv2d(x.to(dev), w.to(dev), torch.ones(cout, device=dev), bias.to(dev), relu=1, kh=1, kw=1,
               x2=x2.to(dev), stride2=stride2, sm_budget=8)
torch.cuda.synchronize()
T._close(out, ref)
"""
    root = str(__import__("pathlib").Path(__file__).resolve().parents[1])
    r = subprocess.run([sys.executable, "-c", code, root], env=dict(os.environ, DARIS_CONV_PAIR="2"),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
