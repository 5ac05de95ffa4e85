"""Order 3 with the exact limbs on the 5th-generation tensor cores (plan
option "i8_tc": tcgen05.mma kind::i8 byte-slice products, s32 accumulators in
TMEM, bsf_i8_gather.cuh): the same filter as the DMMA path
(the exact part is exact on both; only the rounded G0 limb and the final
double-double rounding differ) and the oracle's within 1e-9 (PAPER.md:161-166
for the orders, Eq. (11) PAPER.md:345-352 for the contraction)."""
import numpy as np
import pytest
import torch

import synth
from paper_1109_5114_b200 import bsf
from gpu_util import gpu_full, make_plan, oracle_points
from test_gpu_parity import _small_smooth

pytestmark = pytest.mark.gpu
TILE = bsf.BSF_ANCHOR_TILE


def _run(w, img, cov, i8, policy=None, order=3):
    plan = make_plan(w, policy=policy, order=order, anchor=TILE)
    plan.debug_option("i8_tc", i8)
    out = gpu_full(plan, img, cov)
    st = plan.stats()
    assert st["status"] == 0 and st["flags"] == 0
    return out, st


@pytest.mark.parametrize("policy", [0, 1, 2])
def test_i8_order3_small_all_pixels(policy):
    H, W = 30, 37
    w, img, cov = _small_smooth(H, W, 2.5, seed=9)
    a, _ = _run(w, img, cov, 0, policy)
    b, st = _run(w, img, cov, 1, policy)
    rel = ((a - b).abs() / a.abs()).max().item()
    assert rel <= 1e-12, rel
    ys, xs = np.mgrid[0:H, 0:W]
    ref, *_ = oracle_points(img.numpy(), cov.numpy(), xs.ravel(), ys.ravel(), policy=policy, r=3)
    err = np.abs(b[0].numpy().ravel() - ref) / np.abs(ref)
    assert err.max() <= 1e-9, err.max()


def test_i8_order3_config3_crop():
    """A 256 x 192 crop of config 3 (u8, sigma up to 40): both paths agree and
    sampled pixels match the oracle."""
    w = synth.workload(3, width=256, height=192, extra={"grid_span": 4096})
    img, cov = synth.make_image(w), synth.make_cov(w)
    a, _ = _run(w, img[None], cov, 0)
    b, st = _run(w, img[None], cov, 1)
    rel = ((a - b).abs() / a.abs()).max().item()
    assert rel <= 1e-12, rel
    ys, xs = np.mgrid[5:192:37, 3:256:41]
    ref, *_ = oracle_points(img.numpy(), cov.numpy(), xs.ravel(), ys.ravel(), policy=w.basis, r=3)
    err = np.abs(b[0].numpy()[ys.ravel(), xs.ravel()] - ref) / np.abs(ref)
    assert err.max() <= 1e-9, err.max()
