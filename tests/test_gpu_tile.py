"""Tile-anchored fused path (BSF_ANCHOR_TILE) vs the oracle, and against
itself (full-image run vs explicit pixel list)."""
import math

import numpy as np
import pytest
import torch

import synth
from paper_1109_5114_b200 import bsf
from gpu_util import gpu_full, make_plan, max_rel, oracle_points, tile_points
from test_gpu_parity import _small_smooth

pytestmark = pytest.mark.gpu
TOL64 = 1e-9
TILE = bsf.BSF_ANCHOR_TILE


@pytest.mark.parametrize("policy", [0, 1, 2])
def test_tile_c1_all_pixels(policy):
    w = synth.workload(1)
    img, cov = synth.make_image(w), synth.make_cov(w)
    plan = make_plan(w, policy=policy, anchor=TILE)
    out = gpu_full(plan, img, cov)[0].numpy()
    ys, xs = np.mgrid[0:w.height, 0:w.width]
    ref, *_ = oracle_points(img.numpy(), cov.numpy(), xs.ravel(), ys.ravel(), policy=policy, r=1)
    assert max_rel(out.ravel(), ref) <= TOL64
    st = plan.stats()
    assert st["pixels"] == w.width * w.height and st["flags"] == 0


@pytest.mark.parametrize("precision", [bsf.BSF_PREC_DD, bsf.BSF_PREC_AUTO])
@pytest.mark.parametrize("policy", [0, 1, 2])
@pytest.mark.parametrize("r", [1, 2])
def test_tile_small_ragged_all_pixels(policy, r, precision):
    H, W = 45, 53
    w, img, cov = _small_smooth(H, W, 3.0)
    plan = make_plan(w, policy=policy, order=r, anchor=TILE, precision=precision)
    out = gpu_full(plan, img, cov)[0].numpy()
    ys, xs = np.mgrid[0:H, 0:W]
    ref, *_ = oracle_points(img.numpy(), cov.numpy(), xs.ravel(), ys.ravel(), policy=policy, r=r)
    err = np.abs(out.ravel() - ref) / np.abs(ref)
    assert err.max() <= TOL64, (err.max(), np.unravel_index(err.argmax(), (H, W)))
    assert plan.stats()["flags"] == 0


def test_tile_points_equal_full_run_bitwise():
    """bsf_run_points gives exactly the values of the full tile run."""
    H, W = 70, 90
    w, img, cov = _small_smooth(H, W, 4.0)
    plan = make_plan(w, order=2, anchor=TILE)
    full = gpu_full(plan, img, cov)[0]
    pts = synth.sample_points(w, 50, seed=4)
    got = tile_points(plan, img[None], cov, pts)
    ref = full[pts[:, 2].long(), pts[:, 1].long()]
    assert torch.equal(got, ref)


def test_tile_batch_channels_f32_out():
    w = synth.workload(1, width=40, height=33, batch=2, channels=3)
    imgs = torch.stack([synth.make_image(w, frame=b, channel=c) for b in range(2) for c in range(3)])
    covs = torch.stack([synth.make_cov(w) for _ in range(2)])
    covs[1, 0] *= 0.7
    covs[1, 1] *= 0.4
    plan = make_plan(w, out_f32=True, anchor=TILE)
    out = gpu_full(plan, imgs, covs, out_dtype=torch.float32).numpy()
    ys, xs = np.mgrid[0:33, 0:40]
    for i in range(6):
        ref, *_ = oracle_points(imgs[i].numpy(), covs[i // 3].numpy(), xs.ravel(), ys.ravel(), policy=2, r=1)
        assert max_rel(out[i].ravel(), ref) <= 1e-4


@pytest.mark.parametrize("precision", [bsf.BSF_PREC_DD, bsf.BSF_PREC_AUTO])
def test_tile_config2_full_size_sampled(precision):
    w = synth.workload(2)
    img, cov = synth.make_image(w), synth.make_cov(w)
    plan = make_plan(w, anchor=TILE, precision=precision)
    out = gpu_full(plan, img, cov)[0]
    pts = synth.sample_points(w, 160, seed=2)
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    ref, *_ = oracle_points(img.numpy(), cov.numpy(), xs, ys, policy=2, r=2)
    assert max_rel(out[ys, xs].numpy(), ref) <= TOL64
    assert plan.stats()["flags"] == 0


@pytest.mark.parametrize("r", [1, 2])
def test_tile_config3_full_size_sampled(r):
    w = synth.workload(3, order=r)
    img, cov = synth.make_image(w), synth.make_cov(w)
    plan = make_plan(w, anchor=TILE)
    pts = synth.sample_points(w, 120 if r == 1 else 40, seed=3)
    got, aux = tile_points(plan, img[None], cov, pts, aux=True)
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    ref, bas, cl, sc = oracle_points(img.numpy(), cov.numpy(), xs, ys, policy=2, r=r)
    assert (aux[:, 0].numpy() == bas).all()  # basis decisions agree
    assert max_rel(got.numpy(), ref) <= TOL64
