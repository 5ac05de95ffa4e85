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


@pytest.mark.parametrize("r,policy", [(1, 2), (2, 2), (2, 1), (3, 0)])
def test_replicate_boundary_matches_padded_oracle(r, policy):
    """BSF_BOUNDARY_REPLICATE: f outside the image is its nearest pixel.  The
    oracle is unchanged: filtering the edge-padded image with zero extension
    (pad >= the kernel reach) at the shifted pixels is the same sum."""
    H, W = 38, 42
    w, img, cov = _small_smooth(H, W, 3.0, seed=33)
    plan = bsf.Plan(W, H, in_dtype=bsf.BSF_F32, order=r, basis=policy, max_sigma=3.0, anchor=bsf.BSF_ANCHOR_TILE,
                    boundary=bsf.BSF_BOUNDARY_REPLICATE)
    out = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    plan.run(img[None].cuda().contiguous(), cov.cuda().contiguous(), out)
    torch.cuda.synchronize()
    pad = int(np.ceil(3.0 * np.sqrt(24.0 * r))) + 6 * r + 4
    big = np.pad(img.numpy(), pad, mode="edge")
    ys, xs = np.mgrid[0:H, 0:W]
    xs, ys = xs.ravel(), ys.ravel()
    c = cov.numpy()
    ref, *_ = O.filter_points(big, xs + pad, ys + pad, c[0][ys, xs].astype(np.float64), c[1][ys, xs].astype(np.float64),
                              c[2][ys, xs].astype(np.float64), policy=policy, r=r)
    got = out[0].cpu().numpy().ravel()
    assert max_rel(got, ref) <= 1e-9
    # interior pixels far from the edges do not see the extension
    plan0 = bsf.Plan(W, H, in_dtype=bsf.BSF_F32, order=r, basis=policy, max_sigma=3.0, anchor=bsf.BSF_ANCHOR_TILE)
    out0 = torch.empty_like(out)
    plan0.run(img[None].cuda().contiguous(), cov.cuda().contiguous(), out0)
    torch.cuda.synchronize()
    assert not torch.equal(out, out0)


def test_replicate_boundary_unsupported_paths():
    w = synth.workload(1, width=32, height=32)
    g_plan = bsf.Plan(32, 32, in_dtype=bsf.BSF_U8, order=1, max_sigma=3.0, boundary=bsf.BSF_BOUNDARY_REPLICATE)
    img = synth.make_image(w)[None].cuda()
    with pytest.raises(bsf.BsfError):
        g_plan.preintegrate(img, g_plan.empty_g())


@pytest.mark.parametrize("anchor", [bsf.BSF_ANCHOR_TILE, bsf.BSF_ANCHOR_AUTO])
def test_covariance_planes_layout(anchor):
    """BSF_COV_C11_C12_C22: the covariance given as (C11, C12, C22) planes
     filters like the same covariance in the (sigma_x,
    sigma_y, theta) layout, to the rounding of the eigen-decomposition."""
    from gpu_util import gpu_full
    w = synth.workload(3, order=1, width=200, height=150, extra={"grid_span": 1200})
    img, cov = synth.make_image(w), synth.make_cov(w)
    sx, sy, th = cov.double()
    c, s = torch.cos(th), torch.sin(th)
    C = torch.stack([sx * sx * c * c + sy * sy * s * s, (sx * sx - sy * sy) * s * c,
                     sx * sx * s * s + sy * sy * c * c]).float()
    a = gpu_full(bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8, order=1, basis=2, max_sigma=w.max_sigma,
                          anchor=anchor), img[None], cov)
    b = gpu_full(bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8, order=1, basis=2, max_sigma=w.max_sigma,
                          anchor=anchor, cov_layout=bsf.BSF_COV_C11_C12_C22), img[None], C)
    rel = ((a - b).abs() / a.abs()).max()
    assert float(rel) < 1e-5, float(rel)  # float32 planes: the two layouts round differently
