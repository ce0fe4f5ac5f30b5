"""P3 at scale: the sm_100a path vs PyTorch fp32.

* top-1 on >= 1000 random inputs per model, the inputs batched through the
  GPU path (batch 50: the large-M tile plans), against an fp32 PyTorch
  forward of the same random-init, BN-randomised weights (on the GPU with
  TF32 off — plain fp32 arithmetic like the CPU forward, only fast enough for
  4000 images). Random-init networks put many images' top two logits within
  bf16 rounding of each other (VGG-16: 36 % of images have a top-1/top-2
  margin below twice the image's worst logit error, and 4.3 % flip), so
  top-1 must agree on >= 95 % of all images and on >= 99 % of the images whose
  reference margin exceeds twice that image's worst logit error, and every
  disagreement must be a near-tie: the reference logit of our top-1 class
  within that error bound of the reference maximum. Per-image cosine >= 0.998
  on all 1000 (measured >= 0.99996);
* ResNet-50 logits at batch 16 / 32 / 64 — the shapes the batched DARIS jobs
  and the single-tenant batching baseline run — against a torch CPU fp32
  forward: relative L2 <= 5e-2, cosine >= 0.998 (bf16 activations, fp32
  accumulation), top-1 equal.
"""

import pytest
import torch

from paper_2504_08795_b200 import nets

pytestmark = pytest.mark.gpu

REL_L2 = 5e-2
COS = 0.998


@pytest.fixture(autouse=True)
def _fp32_reference():
    old = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = old


@pytest.mark.parametrize("name", ["resnet18", "resnet50", "vgg16", "mobilenet_v2"])
def test_top1_agreement_on_1000_inputs(name):
    batch, n_batches = 50, 20
    net = nets.build_network(name, batch=batch, keep_torch=True)
    ref_model = net.torch_model.cuda().eval()
    tb = nets.allocate_buffers(net, sm_budget=148)
    g = torch.Generator().manual_seed(1234)
    agree = total = decisive = decisive_agree = 0
    worst_cos = 1.0
    for _ in range(n_batches):
        x = torch.randn(batch, 3, 224, 224, generator=g).cuda()
        out = nets.forward(net, tb, x, stream=None, sm_budget=148).float().clone()
        with torch.no_grad():
            ref = ref_model(x).float()
        torch.cuda.synchronize()
        err = (out - ref).abs().max(dim=1).values                 # worst logit error per image
        top2 = ref.topk(2, dim=1).values
        margin = top2[:, 0] - top2[:, 1]
        ours, theirs = out.argmax(1), ref.argmax(1)
        same = ours == theirs
        dec = margin > 2 * err
        agree += int(same.sum())
        total += batch
        decisive += int(dec.sum())
        decisive_agree += int((same & dec).sum())
        # every disagreement is a near-tie within this image's numerical error
        gap = top2[:, 0] - ref.gather(1, ours[:, None])[:, 0]
        assert bool((same | (gap <= 2 * err)).all()), (gap[~same], err[~same])
        worst_cos = min(worst_cos, torch.nn.functional.cosine_similarity(out, ref, dim=1).min().item())
    print(f"{name}: top-1 agreement {agree}/{total} = {agree / total:.4f}; on decisive images "
          f"{decisive_agree}/{decisive}; worst per-image cosine {worst_cos:.5f}")
    assert total >= 1000 and agree >= 0.95 * total and decisive_agree >= 0.99 * decisive
    assert worst_cos >= COS


@pytest.mark.parametrize("batch", [16, 32, 64])
def test_resnet50_batched_matches_torch_cpu(batch):
    net = nets.build_network("resnet50", batch=batch, keep_torch=True)
    tb = nets.allocate_buffers(net, sm_budget=148)
    x = torch.randn(batch, 3, 224, 224, generator=torch.Generator().manual_seed(batch))
    out = nets.forward(net, tb, x.cuda(), stream=None, sm_budget=148).float().cpu().clone()
    torch.cuda.synchronize()
    with torch.no_grad():
        ref = net.torch_model.float()(x).float()
    rel = ((out - ref).norm() / ref.norm()).item()
    cos = torch.nn.functional.cosine_similarity(out.flatten(), ref.flatten(), dim=0).item()
    print(f"resnet50 b{batch}: rel_l2={rel:.4f} cos={cos:.5f}")
    assert rel <= REL_L2 and cos >= COS, (rel, cos)
    assert (out.argmax(1) == ref.argmax(1)).float().mean().item() >= 0.95
