"""P3 parity: whole networks run through the sm_100a kernels vs a PyTorch CPU
fp32 forward of the same random-init (BN-randomised) weights.

Tolerance (bf16 storage of every activation, fp32 accumulation):
relative L2 error of the logits <= 5e-2 and cosine similarity >= 0.998.
"""

import pytest
import torch

from paper_2504_08795_b200 import nets

pytestmark = pytest.mark.gpu

REL_L2 = 5e-2
COS = 0.998


@pytest.mark.parametrize("name", ["resnet18", "resnet50", "vgg16", "mobilenet_v2"])
@pytest.mark.parametrize("batch", [1, 2])
@pytest.mark.parametrize("mode", ["persistent", "layers"])
def test_network_matches_torch_cpu(name, batch, mode):
    net = nets.build_network(name, batch=batch, keep_torch=True, stage_mode=mode)
    tb = nets.allocate_buffers(net, sm_budget=74)
    g = torch.Generator().manual_seed(11)
    x = torch.randn(batch, 3, 224, 224, generator=g)
    out = nets.forward(net, tb, x.cuda(), stream=None, sm_budget=74, mode=mode).float().cpu().clone()
    torch.cuda.synchronize()
    with torch.no_grad():
        ref = net.torch_model(x).float()
    rel = ((out - ref).norm() / ref.norm()).item()
    cos = torch.nn.functional.cosine_similarity(out.flatten(), ref.flatten(), dim=0).item()
    print(f"{name} b{batch}: rel_l2={rel:.4f} cos={cos:.5f}")
    assert rel <= REL_L2 and cos >= COS, (rel, cos)
    assert torch.equal(out.argmax(1), ref.argmax(1)) or rel < 1e-2


def test_stage_split_covers_network():
    net = nets.build_network("resnet50", batch=1)
    assert net.n_stages == 4
    assert net.stage_bounds[0] == 0 and net.stage_bounds[-1] == len(net.ops)
    assert abs(net.flops_per_image - 8.18e9) / 8.18e9 < 0.02
    r18 = nets.build_network("resnet18", batch=1)
    assert r18.n_stages == 3
    assert abs(r18.flops_per_image - 3.63e9) / 3.63e9 < 0.02


@pytest.mark.parametrize("grid", [5, 37, 74, 148, 300])
def test_persistent_stage_kernel_grid_and_relaunch(grid):
    """The stage kernel's result must not depend on the grid (claim-order
    scheduling, any co-residency) and its self-resetting counters must make
    back-to-back launches of one program identical; it must also agree with
    the one-launch-per-layer path to bf16 rounding."""
    net = nets.build_network("resnet50", batch=1, stage_mode="persistent")
    tb = nets.allocate_buffers(net, sm_budget=grid)
    x = torch.randn(1, 3, 224, 224, generator=torch.Generator().manual_seed(3)).cuda()
    outs = []
    for _ in range(3):
        tb.input.copy_(x)
        for st in range(net.n_stages):
            nets.run_stage(net, st, tb, None, grid, mode="persistent")
        outs.append(tb.output.clone())
    torch.cuda.synchronize()
    net_l = nets.build_network("resnet50", batch=1, stage_mode="layers")  # same seed, same weights
    tb2 = nets.allocate_buffers(net_l, sm_budget=74)
    ref = nets.forward(net_l, tb2, x, sm_budget=74, mode="layers").clone()
    torch.cuda.synchronize()
    for o in outs[1:]:
        rel_rep = ((o - outs[0]).norm() / outs[0].norm()).item()
        assert rel_rep < 1e-2, rel_rep  # split-K fp32 atomics reorder sums: equal up to bf16 rounding
    rel = ((outs[0] - ref).norm() / ref.norm()).item()
    assert rel < 2e-2, rel


def test_persistent_stage_kernel_concurrent_programs():
    """Several programs running concurrently on different streams (as DARIS
    tenants do) produce the same results as when run alone."""
    net = nets.build_network("resnet18", batch=1, stage_mode="persistent")
    xs = [torch.randn(1, 3, 224, 224, generator=torch.Generator().manual_seed(20 + i)).cuda() for i in range(6)]
    alone = []
    for x in xs:
        tb = nets.allocate_buffers(net, sm_budget=74)
        alone.append(nets.forward(net, tb, x, sm_budget=74, mode="persistent").clone())
    torch.cuda.synchronize()
    tbs = [nets.allocate_buffers(net, sm_budget=74) for _ in xs]
    streams = [torch.cuda.Stream() for _ in xs]
    for _ in range(3):
        for x, tb, s in zip(xs, tbs, streams):
            with torch.cuda.stream(s):
                tb.input.copy_(x)
                for st in range(net.n_stages):
                    nets.run_stage(net, st, tb, s.cuda_stream, 74, mode="persistent")
    torch.cuda.synchronize()
    for a, tb in zip(alone, tbs):
        rel = ((tb.output - a).norm() / a.norm()).item()
        assert rel < 1e-2, rel


@pytest.mark.parametrize("name,batch", [("resnet50", 1), ("resnet50", 2), ("resnet18", 1), ("mobilenet_v2", 1)])
def test_network_at_the_executor_plan(name, batch):
    """Grids planned for the C2 per-job share (23 SMs): 256-row tiles, fused
    downsample, stems by TMA — the forms the executor captures."""
    net = nets.build_network(name, batch=batch, keep_torch=True, stage_mode="layers")
    tb = nets.allocate_buffers(net, sm_budget=23)
    x = torch.randn(batch, 3, 224, 224, generator=torch.Generator().manual_seed(5))
    out = nets.forward(net, tb, x.cuda(), stream=None, sm_budget=23, mode="layers").float().cpu().clone()
    torch.cuda.synchronize()
    with torch.no_grad():
        ref = net.torch_model(x).float()
    rel = ((out - ref).norm() / ref.norm()).item()
    cos = torch.nn.functional.cosine_similarity(out.flatten(), ref.flatten(), dim=0).item()
    assert rel <= REL_L2 and cos >= COS, (rel, cos)
