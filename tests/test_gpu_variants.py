"""User-facing variants: the DC-renormalised output
bsf_run_normalized = filter(f) / filter(image indicator)."""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from paper_1109_5114_b200 import bsf
from gpu_util import make_plan, max_rel, oracle_points
from test_gpu_parity import _small_smooth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("in_dtype,r", [("u8", 1), ("f32", 1), ("f32", 2)])
def test_normalized_constant_image_is_exact(in_dtype, r):
    """A constant image comes back as the constant at every pixel, edges
    included (the denominator is the same filter of the indicator)."""
    H, W = 45, 53
    _, _, cov = _small_smooth(H, W, 3.0, seed=31)
    c = 7.0
    img = torch.full((H, W), c, dtype=torch.float32)
    if in_dtype == "u8":
        img = img.to(torch.uint8)
    plan = bsf.Plan(W, H, in_dtype=bsf.BSF_U8 if in_dtype == "u8" else bsf.BSF_F32, order=r, basis=bsf.BSF_DUAL,
                    max_sigma=3.0, anchor=bsf.BSF_ANCHOR_TILE)
    out = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    plan.run_normalized(img[None].cuda().contiguous(), cov.cuda().contiguous(), out)
    torch.cuda.synchronize()
    assert float((out - c).abs().max()) <= 1e-12 * c


def test_normalized_matches_oracle_ratio():
    H, W = 40, 44
    w, img, cov = _small_smooth(H, W, 3.5, seed=32)
    plan = make_plan(w, order=2, anchor=bsf.BSF_ANCHOR_TILE)
    out = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    plan.run_normalized(img[None].cuda().contiguous(), cov.cuda().contiguous(), out)
    torch.cuda.synchronize()
    pts = synth.sample_points(w, 60, seed=4)
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    num = oracle_points(img.numpy(), cov.numpy(), xs, ys, policy=w.basis, r=2)[0]
    den = oracle_points(np.ones_like(img.numpy()), cov.numpy(), xs, ys, policy=w.basis, r=2)[0]
    got = out[0].cpu().numpy()[ys, xs]
    assert max_rel(got, num / den) <= 1e-9


def test_normalized_needs_tile_anchor():
    w = synth.workload(1, width=32, height=32)
    plan = make_plan(w, anchor=bsf.BSF_ANCHOR_GLOBAL)
    img = synth.make_image(w)[None].cuda()
    cov = synth.make_cov(w).cuda()
    out = torch.empty((1, 32, 32), dtype=torch.float64, device="cuda")
    with pytest.raises(bsf.BsfError):
        plan.run_normalized(img, cov, out)
