"""GPU (CUDA path through the C-ABI) vs the CPU oracle, element by element.

Tolerance (north star): max relative error 1e-9 for float64 output, 1e-4 for
float32 output; bit-exact for the integer pre-integration of u8 images.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synth
from paper_1109_5114_b200 import bsf
from gpu_util import gpu_full, gpu_points, make_plan, max_rel, oracle_points

pytestmark = pytest.mark.gpu
TOL64 = 1e-9


# ---------------------------------------------------------------------------
# bit-exact integer pre-integration (north star: "bit-exactly on the integer
# pre-integration of uint8 images")
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("policy", [0, 1])
@pytest.mark.parametrize("r", [1, 2])
def test_exact_preintegration_c1(policy, r):
    w = synth.workload(1)
    img = synth.make_image(w)
    plan = make_plan(w, policy=policy, order=r)
    P, Pb = plan.geometry.margin_x, plan.geometry.margin_y
    g = plan.empty_g_exact()
    plan.preintegrate_exact(img.cuda(), g)
    torch.cuda.synchronize()
    ref = O.preintegrate_u8(img.numpy(), policy, r, P, Pb)
    got = g[0, 0].cpu().numpy().view(np.uint64)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("r", [1, 2])
def test_exact_preintegration_c3_full_size(r):
    """4096^2 u8 (config 3), both bases; r = 2 wraps modulo 2^64."""
    w = synth.workload(3)
    img = synth.make_image(w)
    plan = make_plan(w, policy=bsf.BSF_DUAL, order=r)
    P, Pb = plan.geometry.margin_x, plan.geometry.margin_y
    g = plan.empty_g_exact()
    plan.preintegrate_exact(img.cuda(), g)
    torch.cuda.synchronize()
    for slot, basis in ((0, 0), (1, 1)):
        ref = O.preintegrate_u8(img.numpy(), basis, r, P, Pb)
        got = g[slot, 0].cpu().numpy().view(np.uint64)
        assert np.array_equal(got, ref), basis


def test_exact_preintegration_ragged_and_batch():
    w = synth.workload(1, width=37, height=19, batch=3)
    imgs = torch.stack([synth.make_image(w, frame=i) for i in range(3)])
    plan = make_plan(w, policy=bsf.BSF_DUAL, order=1)
    g = plan.empty_g_exact()
    plan.preintegrate_exact(imgs.cuda(), g)
    torch.cuda.synchronize()
    P, Pb = plan.geometry.margin_x, plan.geometry.margin_y
    for i in range(3):
        for slot in (0, 1):
            ref = O.preintegrate_u8(imgs[i].numpy(), slot, 1, P, Pb)
            assert np.array_equal(g[slot, i].cpu().numpy().view(np.uint64), ref)


# ---------------------------------------------------------------------------
# filter parity at sizes the oracle finishes in seconds
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("policy", [0, 1, 2])
@pytest.mark.parametrize("precision", [bsf.BSF_PREC_DD, bsf.BSF_PREC_FP64])
def test_filter_c1_all_pixels(policy, precision):
    """Config 1 (128^2 u8, sigma = 3, r = 1): every pixel."""
    w = synth.workload(1)
    img, cov = synth.make_image(w), synth.make_cov(w)
    plan = make_plan(w, policy=policy, precision=precision)
    out = gpu_full(plan, img, cov)[0].numpy()
    ys, xs = np.mgrid[0:w.height, 0:w.width]
    ref, bas, cl, sc = oracle_points(img.numpy(), cov.numpy(), xs.ravel(), ys.ravel(), policy=policy, r=1)
    assert max_rel(out.ravel(), ref) <= TOL64
    st = plan.stats()
    assert st["pixels"] == w.width * w.height and st["flags"] == 0


def _small_smooth(H, W, smax, seed=7):
    """Config-2-like smooth field on a small ragged image."""
    w = synth.workload(2, width=W, height=H, max_sigma=smax, seed=seed)
    img = synth.make_image(w)
    X = torch.arange(W, dtype=torch.float64)[None, :]
    Y = torch.arange(H, dtype=torch.float64)[:, None]
    smaj = 0.8 + (smax - 0.8) * X / (W - 1) + 0 * Y
    ratio = 1.0 + 5.0 * Y / (H - 1) + 0 * X
    th = torch.remainder(torch.atan2(Y - H / 2, X - W / 2), math.pi)
    cov = torch.stack([smaj, smaj / torch.sqrt(ratio), th]).to(torch.float32)
    return w, img, cov


@pytest.mark.parametrize("precision", [bsf.BSF_PREC_DD, bsf.BSF_PREC_AUTO])
@pytest.mark.parametrize("policy", [0, 1, 2])
@pytest.mark.parametrize("r", [1, 2])
def test_filter_small_ragged_all_pixels(policy, r, precision):
    """Ragged size (not a multiple of the 16x8 tile), space-variant field
    spanning isotropic to elongation 6, all orientations, zero scales and the
    clamp: every pixel."""
    H, W = 45, 53
    w, img, cov = _small_smooth(H, W, 3.0)
    plan = make_plan(w, policy=policy, order=r, precision=precision)
    out = gpu_full(plan, img, cov)[0].numpy()
    ys, xs = np.mgrid[0:H, 0:W]
    ref, bas, cl, sc = oracle_points(img.numpy(), cov.numpy(), xs.ravel(), ys.ravel(), policy=policy, r=r)
    err = np.abs(out.ravel() - ref) / np.abs(ref)
    assert err.max() <= TOL64, (err.max(), np.unravel_index(err.argmax(), (H, W)))
    st = plan.stats()
    assert st["flags"] == 0
    if policy != 1:
        assert st["zero_scale"] > 0  # elongated pixels reach the min-kurtosis boundary (F5)


def test_filter_u8_batch_channels_and_f32_out():
    """batch x channels sharing a covariance field; float32 output (1e-4)."""
    w = synth.workload(1, width=40, height=33, batch=2, channels=3)
    imgs = torch.stack([synth.make_image(w, frame=b, channel=c) for b in range(2) for c in range(3)])
    covs = torch.stack([synth.make_cov(w) for _ in range(2)])
    covs[1, 0] *= 0.7
    covs[1, 1] *= 0.4
    plan = make_plan(w, out_f32=True)
    out = gpu_full(plan, imgs, covs, out_dtype=torch.float32).numpy()
    ys, xs = np.mgrid[0:33, 0:40]
    for i in range(6):
        ref, *_ = oracle_points(imgs[i].numpy(), covs[i // 3].numpy(), xs.ravel(), ys.ravel(), policy=2, r=1)
        assert max_rel(out[i].ravel(), ref) <= 1e-4


def test_tiny_images_and_single_pixel():
    for H, W in ((1, 1), (1, 17), (13, 1), (3, 2)):
        w = synth.workload(1, width=W, height=H)
        img, cov = synth.make_image(w), synth.make_cov(w)
        plan = make_plan(w)
        out = gpu_full(plan, img, cov)[0].numpy()
        ys, xs = np.mgrid[0:H, 0:W]
        ref, *_ = oracle_points(img.numpy(), cov.numpy(), xs.ravel(), ys.ravel(), policy=2, r=1)
        assert max_rel(out.ravel(), ref) <= TOL64


def test_reject_mode_flags_infeasible():
    """clamp = 0: an elongation beyond the bound gives NaN and BSF_EINFEASIBLE."""
    w = synth.workload(1, width=16, height=16)
    img = synth.make_image(w)
    cov = synth.make_cov(w)
    cov[0] = 6.0
    cov[1] = 6.0 / 4.0  # rho = 16 > 6.17 everywhere at theta = 22.5 deg
    cov[2] = math.radians(22.5)
    plan = make_plan(w, clamp=0, policy=0)
    out = gpu_full(plan, img, cov)
    assert torch.isnan(out).all()
    st = plan.stats()
    assert st["status"] == 4
    plan2 = make_plan(w, clamp=1, policy=0)
    out2 = gpu_full(plan2, img, cov)[0].numpy()
    ys, xs = np.mgrid[0:16, 0:16]
    ref, bas, cl, sc = oracle_points(img.numpy(), cov.numpy(), xs.ravel(), ys.ravel(), policy=0, r=1)
    assert (cl == 1).all() and plan2.stats()["clamped"] == 256
    assert max_rel(out2.ravel(), ref) <= TOL64


# ---------------------------------------------------------------------------
# full-size configs: sampled outputs in the launch configuration bench times
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("precision", [bsf.BSF_PREC_DD, bsf.BSF_PREC_AUTO])
def test_config2_full_size_sampled(precision):
    w = synth.workload(2)
    img, cov = synth.make_image(w), synth.make_cov(w)
    plan = make_plan(w, precision=precision)
    out = gpu_full(plan, img, cov)[0]
    pts = synth.sample_points(w, 160, seed=2)
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    ref, *_ = oracle_points(img.numpy(), cov.numpy(), xs, ys, policy=2, r=2)
    got = out[ys, xs].numpy()
    assert max_rel(got, ref) <= TOL64
    assert plan.stats()["flags"] == 0


@pytest.mark.parametrize("r", [1, 2])
def test_config3_full_size_sampled(r):
    w = synth.workload(3, order=r)
    img, cov = synth.make_image(w), synth.make_cov(w)
    plan = make_plan(w)
    pts = synth.sample_points(w, 120 if r == 1 else 40, seed=3)
    got = gpu_points(plan, img, cov, pts).numpy()
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    ref, *_ = oracle_points(img.numpy(), cov.numpy(), xs, ys, policy=2, r=r)
    assert max_rel(got, ref) <= TOL64


@pytest.mark.parametrize("r", [3, 4])
def test_exact_preintegration_high_orders(r):
    """Orders 3 and 4 (config 3 sweeps r = 1..4), both bases, wrapping mod 2^64."""
    w = synth.workload(3, width=150, height=97)
    img = synth.make_image(w)
    plan = make_plan(w, policy=bsf.BSF_DUAL, order=r)
    P, Pb = plan.geometry.margin_x, plan.geometry.margin_y
    g = plan.empty_g_exact()
    plan.preintegrate_exact(img.cuda(), g)
    torch.cuda.synchronize()
    for slot in (0, 1):
        ref = O.preintegrate_u8(img.numpy(), slot, r, P, Pb)
        assert np.array_equal(g[slot, 0].cpu().numpy().view(np.uint64), ref), slot


@pytest.mark.parametrize("H,W", [(1, 1), (1, 41), (29, 1), (2, 3)])
def test_exact_preintegration_degenerate_shapes(H, W):
    w = synth.workload(1, width=W, height=H)
    img = synth.make_image(w)
    for r in (1, 2):
        plan = make_plan(w, policy=bsf.BSF_DUAL, order=r)
        P, Pb = plan.geometry.margin_x, plan.geometry.margin_y
        g = plan.empty_g_exact()
        plan.preintegrate_exact(img.cuda(), g)
        torch.cuda.synchronize()
        for slot in (0, 1):
            ref = O.preintegrate_u8(img.numpy(), slot, r, P, Pb)
            assert np.array_equal(g[slot, 0].cpu().numpy().view(np.uint64), ref), (r, slot)
