"""Seeded random cases through the fused product path against the oracle:
sizes (ragged, smaller and larger than a super-tile), orders 1-3, the three
basis policies, u8 / f32 input, f64 / f32 output, batch and channels, random
smooth covariance fields with random sigma ranges, elongations and angles."""
import math

import numpy as np
import pytest
import torch

import synth
from paper_1109_5114_b200 import bsf
from gpu_util import max_rel, oracle_points

pytestmark = pytest.mark.gpu


def _rel_scale(img, cov, xs, ys, ref, u8, policy, r):
    """Denominator of the relative error (R26).  u8 images: |ref|
    (the box spline is non-negative, so outputs are positive).  Signed float
    images: the same filter applied to |f| at the same pixels, sum_q |f(q)|
    beta(p - q) >= |ref| -- the magnitude the pixel's sum is formed from, its
    condition scale; equal to |ref| wherever f does not change sign under
    the kernel's support.  No constant floor."""
    if u8:
        return np.abs(ref)
    return oracle_points(np.abs(img), cov, xs, ys, policy=policy, r=r)[0]


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    H, W = int(rng.integers(5, 90)), int(rng.integers(5, 90))
    r = int(rng.integers(1, 4))
    policy = int(rng.integers(0, 3))
    u8 = bool(rng.integers(0, 2))
    batch, channels = int(rng.integers(1, 3)), int(rng.integers(1, 3))
    smax = float(rng.uniform(0.7, 5.0 if r < 3 else 3.0))
    ph = rng.uniform(0, 2 * math.pi, 4)
    X = np.arange(W)[None, :] / max(W - 1, 1)
    Y = np.arange(H)[:, None] / max(H - 1, 1)
    covs, imgs = [], []
    for b in range(batch):
        smaj = 0.6 + (smax - 0.6) * (0.5 + 0.5 * np.sin(3 * X + ph[0] + b) * np.cos(2 * Y + ph[1]))
        ratio = 1.0 + rng.uniform(0, 5.5) * (0.5 + 0.5 * np.cos(2 * X - 3 * Y + ph[2]))
        th = np.mod(ph[3] + 2.0 * X - 1.5 * Y + b, math.pi)
        covs.append(np.stack([smaj, smaj / np.sqrt(ratio), th + 0 * X]).astype(np.float32))
        for c in range(channels):
            if u8:
                imgs.append(rng.integers(0, 256, (H, W)).astype(np.uint8))
            else:
                imgs.append(rng.uniform(-0.5, 1.0, (H, W)).astype(np.float32))
    return dict(H=H, W=W, r=r, policy=policy, u8=u8, batch=batch, channels=channels, smax=smax,
                cov=np.stack(covs), img=np.stack(imgs), out_f32=bool(rng.integers(0, 2)), rng=rng)


@pytest.mark.parametrize("seed", range(32))
def test_fuzz_fused_vs_oracle(seed):
    c = _case(seed)
    H, W = c["H"], c["W"]
    plan = bsf.Plan(W, H, batch=c["batch"], channels=c["channels"],
                    in_dtype=bsf.BSF_U8 if c["u8"] else bsf.BSF_F32,
                    out_dtype=bsf.BSF_F32 if c["out_f32"] else bsf.BSF_F64, order=c["r"], basis=c["policy"],
                    max_sigma=c["smax"], anchor=bsf.BSF_ANCHOR_TILE)
    nimg = c["batch"] * c["channels"]
    out = torch.empty((nimg, H, W), dtype=torch.float32 if c["out_f32"] else torch.float64, device="cuda")
    plan.run(torch.from_numpy(c["img"]).cuda(), torch.from_numpy(c["cov"]).cuda(), out)
    torch.cuda.synchronize()
    assert plan.uses_fused()
    got = out.cpu().numpy().astype(np.float64)
    rng = c["rng"]
    n = min(H * W, 24)
    for i in range(nimg):
        b = i // c["channels"]
        idx = rng.choice(H * W, n, replace=False)
        ys, xs = idx // W, idx % W
        ref = oracle_points(c["img"][i], c["cov"][b], xs, ys, policy=c["policy"], r=c["r"])[0]
        tol = 1e-6 if c["out_f32"] else 1e-9
        scale = _rel_scale(c["img"][i], c["cov"][b], xs, ys, ref, c["u8"], c["policy"], c["r"])
        err = float(np.max(np.abs(got[i][ys, xs] - ref) / scale))
        assert err <= tol, (seed, i, err, {k: c[k] for k in ("H", "W", "r", "policy", "u8", "smax")})


def _case_large(seed):
    """Image sizes that give the persistent kernel several super-tiles per SM
    (the largest-first work order runs) and, for u8 at order 2 with a large
    reach, 64 x 64 super-tiles."""
    rng = np.random.default_rng(5000 + seed)
    H, W = int(rng.integers(480, 720)), int(rng.integers(640, 900))
    r = int(rng.integers(1, 4))
    u8 = bool(rng.integers(0, 2)) if r != 2 else seed % 2 == 0
    smax = float(rng.uniform(3.0, 14.0 if r < 3 else 3.0))
    ph = rng.uniform(0, 2 * math.pi, 4)
    X = np.arange(W)[None, :] / (W - 1)
    Y = np.arange(H)[:, None] / (H - 1)
    smaj = 0.6 + (smax - 0.6) * (0.5 + 0.5 * np.sin(3 * X + ph[0]) * np.cos(2 * Y + ph[1]))
    ratio = 1.0 + rng.uniform(0, 5.5) * (0.5 + 0.5 * np.cos(2 * X - 3 * Y + ph[2]))
    th = np.mod(ph[3] + 2.0 * X - 1.5 * Y, math.pi)
    cov = np.stack([smaj, smaj / np.sqrt(ratio), th + 0 * X]).astype(np.float32)
    img = rng.integers(0, 256, (H, W)).astype(np.uint8) if u8 else rng.uniform(-0.5, 1.0, (H, W)).astype(np.float32)
    return dict(H=H, W=W, r=r, policy=int(rng.integers(0, 3)), u8=u8, smax=smax, cov=cov, img=img, rng=rng)


@pytest.mark.parametrize("seed", range(8))
def test_fuzz_large_images_vs_oracle(seed):
    c = _case_large(seed)
    H, W = c["H"], c["W"]
    plan = bsf.Plan(W, H, in_dtype=bsf.BSF_U8 if c["u8"] else bsf.BSF_F32, order=c["r"], basis=c["policy"],
                    max_sigma=c["smax"], anchor=bsf.BSF_ANCHOR_TILE)
    n0 = plan.launch_count()
    out = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    plan.run(torch.from_numpy(c["img"]).cuda()[None], torch.from_numpy(c["cov"]).cuda(), out)
    torch.cuda.synchronize()
    assert plan.uses_fused()
    st = plan.geometry.super_tile
    items = ((W + st - 1) // st) * ((H + st - 1) // st)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    ordered = c["r"] >= 2 and (items >= 2 * nsm or (st == 64 and c["r"] == 2))  # 64 x 64 order 2: split mode
    assert plan.launch_count() - n0 == (3 if ordered else 1)
    got = out[0].cpu().numpy()
    rng = c["rng"]
    idx = rng.choice(H * W, 24, replace=False)
    ys, xs = idx // W, idx % W
    ref = oracle_points(c["img"], c["cov"], xs, ys, policy=c["policy"], r=c["r"])[0]
    scale = _rel_scale(c["img"], c["cov"], xs, ys, ref, c["u8"], c["policy"], c["r"])
    err = float(np.max(np.abs(got[ys, xs] - ref) / scale))
    assert err <= 1e-9, (seed, err, st, {k: c[k] for k in ("H", "W", "r", "policy", "u8", "smax")})


def _case_global(seed):
    """u8 images at order 1 through global mode (exact int64 sums + the
    integer gather): ragged and thin sizes across the 32 x 32 gather tiles,
    batch and channels, sigma ranges with zero-scale and clamped pixels."""
    rng = np.random.default_rng(9000 + seed)
    H, W = int(rng.integers(1, 200)), int(rng.integers(1, 260))
    batch, channels = int(rng.integers(1, 3)), int(rng.integers(1, 3))
    smax = float(rng.uniform(0.6, 12.0))
    ph = rng.uniform(0, 2 * math.pi, 4)
    X = np.arange(W)[None, :] / max(W - 1, 1)
    Y = np.arange(H)[:, None] / max(H - 1, 1)
    covs, imgs = [], []
    for b in range(batch):
        smaj = 0.5 + (smax - 0.5) * (0.5 + 0.5 * np.sin(4 * X + ph[0] + b) * np.cos(3 * Y + ph[1]))
        ratio = 1.0 + rng.uniform(0, 12.0) * (0.5 + 0.5 * np.cos(2 * X - 3 * Y + ph[2]))
        th = np.mod(ph[3] + 2.5 * X - 1.5 * Y + b, math.pi)
        covs.append(np.stack([smaj, smaj / np.sqrt(ratio), th + 0 * X]).astype(np.float32))
        for c in range(channels):
            imgs.append(rng.integers(0, 256, (H, W)).astype(np.uint8))
    return dict(H=H, W=W, policy=int(rng.integers(0, 3)), batch=batch, channels=channels, smax=smax,
                cov=np.stack(covs), img=np.stack(imgs), out_f32=bool(rng.integers(0, 2)), rng=rng)


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_global_mode_vs_oracle(seed):
    """Relative error against the oracle with no floor (u8 outputs are
    positive): 1e-9 for f64 output, 1e-6 for f32 output."""
    c = _case_global(seed)
    H, W = c["H"], c["W"]
    plan = bsf.Plan(W, H, batch=c["batch"], channels=c["channels"], in_dtype=bsf.BSF_U8,
                    out_dtype=bsf.BSF_F32 if c["out_f32"] else bsf.BSF_F64, order=1, basis=c["policy"],
                    max_sigma=c["smax"], anchor=bsf.BSF_ANCHOR_GLOBAL)
    assert plan.geometry.global_mode == 1
    nimg = c["batch"] * c["channels"]
    out = torch.empty((nimg, H, W), dtype=torch.float32 if c["out_f32"] else torch.float64, device="cuda")
    plan.run(torch.from_numpy(c["img"]).cuda(), torch.from_numpy(c["cov"]).cuda(), out)
    torch.cuda.synchronize()
    st = plan.stats(reset=True)
    assert st["status"] == 0 and st["pixels"] == nimg * H * W
    got = out.cpu().numpy().astype(np.float64)
    rng = c["rng"]
    n = min(H * W, 20)
    for i in range(nimg):
        b = i // c["channels"]
        idx = rng.choice(H * W, n, replace=False)
        ys, xs = idx // W, idx % W
        ref = oracle_points(c["img"][i], c["cov"][b], xs, ys, policy=c["policy"], r=1)[0]
        ok = ref != 0  # an all-zero neighbourhood: both sides exactly 0
        assert np.all(got[i][ys, xs][~ok] == 0.0)
        err = float(np.max(np.abs(got[i][ys, xs][ok] - ref[ok]) / np.abs(ref[ok]), initial=0.0))
        assert err <= (1e-6 if c["out_f32"] else 1e-9), (seed, i, err, {k: c[k] for k in ("H", "W", "policy", "smax")})
