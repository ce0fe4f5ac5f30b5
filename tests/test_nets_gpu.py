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
def test_network_matches_torch_cpu(name, batch):
    net = nets.build_network(name, batch=batch, keep_torch=True)
    tb = nets.allocate_buffers(net, sm_budget=74)
    g = torch.Generator().manual_seed(11)
    x = torch.randn(batch, 3, 224, 224, generator=g)
    out = nets.forward(net, tb, x.cuda(), stream=None, sm_budget=74).float().cpu().clone()
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


@pytest.mark.parametrize("name,batch", [("resnet50", 1), ("resnet50", 2), ("resnet18", 1), ("mobilenet_v2", 1)])
def test_network_at_the_executor_plan(name, batch):
    """Grids planned for the C2 per-job share (23 SMs): split-K, fused
    downsample, stems by TMA — the forms the executor captures."""
    net = nets.build_network(name, batch=batch, keep_torch=True)
    tb = nets.allocate_buffers(net, sm_budget=23)
    x = torch.randn(batch, 3, 224, 224, generator=torch.Generator().manual_seed(5))
    out = nets.forward(net, tb, x.cuda(), stream=None, sm_budget=23).float().cpu().clone()
    torch.cuda.synchronize()
    with torch.no_grad():
        ref = net.torch_model(x).float()
    rel = ((out - ref).norm() / ref.norm()).item()
    cos = torch.nn.functional.cosine_similarity(out.flatten(), ref.flatten(), dim=0).item()
    assert rel <= REL_L2 and cos >= COS, (rel, cos)
