"""Higher orders and the large configurations (sampled outputs).

Config 5 (32768^2) and config 3 at orders 3-4 are checked on tile-aligned
windows: a point's 16x16 tile only reads the image inside its halo (half-
extent <= sigma_max sqrt(24 r)), so a window with origin on the tile grid that
contains the halo gives exactly the full-image values."""
import math
import os

import numpy as np
import pytest
import torch

import synth
from paper_1109_5114_b200 import bsf, lut
from gpu_util import gpu_full, make_plan, max_rel, oracle_points, tile_points
from test_gpu_parity import _small_smooth

pytestmark = pytest.mark.gpu
TOL64 = 1e-9
TILE = bsf.BSF_ANCHOR_TILE


def _need(r):
    for b in (0, 1):
        if not os.path.exists(lut.path(b, r)):
            pytest.skip("no order-%d tables (run lut/gen_lut.py %d)" % (r, r))


@pytest.mark.parametrize("anchor", [bsf.BSF_ANCHOR_GLOBAL, TILE])
@pytest.mark.parametrize("policy", [0, 1, 2])
def test_order3_small_all_pixels(anchor, policy):
    _need(3)
    H, W = 30, 37
    w, img, cov = _small_smooth(H, W, 2.5, seed=9)
    plan = make_plan(w, policy=policy, order=3, anchor=anchor)
    out = gpu_full(plan, img, cov)[0].numpy()
    ys, xs = np.mgrid[0:H, 0:W]
    ref, *_ = oracle_points(img.numpy(), cov.numpy(), xs.ravel(), ys.ravel(), policy=policy, r=3)
    err = np.abs(out.ravel() - ref) / np.abs(ref)
    assert err.max() <= TOL64, (err.max(), np.unravel_index(err.argmax(), (H, W)))
    assert plan.stats()["flags"] == 0


@pytest.mark.parametrize("policy", [0, 1, 2])
def test_order4_small_points(policy):
    """Order 4 (625 taps; the double-double tile kernel, both bases' tables)
    on a small space-variant field, sampled pixels against the oracle."""
    _need(4)
    H, W = 24, 28
    w, img, cov = _small_smooth(H, W, 2.0, seed=13)
    plan = make_plan(w, policy=policy, order=4, anchor=TILE)
    pts = synth.sample_points(w, 24, seed=17)
    got = tile_points(plan, img[None], cov, pts).numpy()
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    ref, *_ = oracle_points(img.numpy(), cov.numpy(), xs, ys, policy=policy, r=4)
    assert max_rel(got, ref) <= TOL64
    assert plan.stats()["flags"] == 0


def _window_points(w, n, seed, order, frame=0):
    """Sample points and, for each, a tile-aligned window containing its halo."""
    pts = synth.sample_points(w, n, seed=seed)
    halo = int(math.ceil(w.max_sigma * math.sqrt(24.0 * order))) + 3 * order + 8
    res = []
    for _, x, y in pts.tolist():
        x0 = max(0, ((x // 16) * 16 - halo) // 16 * 16)
        y0 = max(0, ((y // 16) * 16 - halo) // 16 * 16)
        x1 = min(w.width, (x // 16) * 16 + 16 + halo)
        y1 = min(w.height, (y // 16) * 16 + 16 + halo)
        res.append((x, y, (y0, y1, x0, x1)))
    return res


def _run_windows(w, order, n, seed, frame=0, channel=0):
    got, ref = [], []
    for x, y, win in _window_points(w, n, seed, order):
        y0, y1, x0, x1 = win
        img = synth.make_image(w, frame=frame, channel=channel, window=win)
        cov = synth.make_cov(w, frame=frame, window=win)
        # the window is the image the plan sees; its true edges coincide with
        # the full image's wherever the halo reaches them
        ww = synth.workload(int(w.name[1]), width=x1 - x0, height=y1 - y0, batch=1, channels=1, order=order,
                            max_sigma=w.max_sigma, seed=w.seed)
        plan = make_plan(ww, order=order, anchor=TILE)
        pt = torch.tensor([[0, x - x0, y - y0]], dtype=torch.int32)
        got.append(float(tile_points(plan, img[None], cov, pt)[0]))
        r, *_ = oracle_points(img.numpy(), cov.numpy(), [x - x0], [y - y0], policy=2, r=order)
        ref.append(r[0])
    return np.array(got), np.array(ref)


@pytest.mark.parametrize("order", [3])
def test_config3_orders_windows(order):
    _need(order)
    w = synth.workload(3, order=order)
    got, ref = _run_windows(w, order, 12, seed=31)
    assert max_rel(got, ref) <= TOL64


def test_config4_frames_sampled():
    """Config 4 (r = 3): sampled pixels of two frames (scale factors differ)."""
    _need(3)
    w = synth.workload(4)
    for frame in (0, 5):
        got, ref = _run_windows(w, 3, 6, seed=40 + frame, frame=frame, channel=frame % 3)
        assert max_rel(got, ref) <= TOL64


def test_config5_windows():
    """Config 5 (32768^2, r = 3, sigma up to 64): sampled pixels."""
    _need(3)
    w = synth.workload(5)
    got, ref = _run_windows(w, 3, 8, seed=50)
    assert max_rel(got, ref) <= TOL64
