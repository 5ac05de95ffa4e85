"""Parity at the BASELINE.json configs' full size, through the real full-image
launches, on stratified pixels (tests/strata.py: corners and edges, strip /
frame boundaries, min and max sigma, clamped, zero-scale and sector-switch
pixels, uniform), against the oracle at the 1e-9 contract with no tolerance
floor (north star; PAPER.md:161-166 for the orders).

* config 3 (4096^2 u8) at order 1 is in test_gpu_global.py (global mode);
  orders 2 and 3 here run bsf_run on the whole image; order 4 runs
  bsf_run_tiles on the anchoring tiles of the sampled pixels (the same kernel
  and anchoring as a whole-image run, which takes tens of minutes).
* config 4: one 3-channel 2048^2 frame (frame-scaled field) through bsf_run.
* config 5: one row strip (rank 3 of 8) of the 32768^2 image through a
  multi-GPU plan (block input, own rows computed), boundary rows included.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synth
from paper_1109_5114_b200 import bsf
from strata import stratified_points

pytestmark = pytest.mark.gpu
TOL = 1e-9
DEV = torch.device("cuda:0")


def _oracle(img_view, origin, shape, cov_pts, xs, ys, policy, r):
    out = O.filter_points(img_view, xs, ys, cov_pts[0], cov_pts[1], cov_pts[2], policy=policy, r=r,
                          full_shape=shape, origin=origin)[0]
    return out


def _report(rel, labels):
    return {k: float(rel[v].max()) for k, v in labels.items() if len(v)}


@pytest.mark.parametrize("r,n", [(2, 200), (3, 200)])
def test_config3_full_image_orders_2_3(r, n):
    w = synth.workload(3, order=r)
    img = synth.make_image(w, device=DEV).contiguous()
    cov = synth.make_cov(w, device=DEV).contiguous()
    plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8, order=r, basis=w.basis, max_sigma=w.max_sigma,
                    anchor=bsf.BSF_ANCHOR_AUTO)
    assert plan.geometry.global_mode == 0
    out = torch.empty((1, w.height, w.width), dtype=torch.float64, device=DEV)
    plan.run(img[None], cov, out)
    st = plan.stats()
    assert st["status"] == 0 and st["pixels"] == w.width * w.height
    pts, labels = stratified_points(w, n, seed=20 + r, r=r)
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    got = out[0].cpu().numpy()[ys, xs]
    c = synth.cov_at(w, xs, ys).numpy().astype(np.float64)
    ref = _oracle(img.cpu().numpy(), (0, 0), (w.height, w.width), c, xs, ys, w.basis, r)
    rel = np.abs(got - ref) / np.abs(ref)
    assert rel.max() <= TOL, _report(rel, labels)


def test_config3_order4_sampled_tiles():
    r = 4
    w = synth.workload(3, order=r)
    img = synth.make_image(w, device=DEV).contiguous()
    cov = synth.make_cov(w, device=DEV).contiguous()
    plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8, order=r, basis=w.basis, max_sigma=w.max_sigma,
                    anchor=bsf.BSF_ANCHOR_AUTO)
    u = plan.geometry.tile_unit
    pts, labels = stratified_points(w, 24, seed=31, r=r, per_stratum=3)
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    ntx = (w.width + u - 1) // u
    tiles = torch.tensor(sorted({int((y // u) * ntx + x // u) for x, y in zip(xs, ys)}), dtype=torch.int32)
    out = torch.full((1, w.height, w.width), float("nan"), dtype=torch.float64, device=DEV)
    plan.run_tiles(img[None], cov, out, tiles.to(DEV))
    assert plan.stats()["status"] == 0
    got = out[0].cpu().numpy()[ys, xs]
    c = synth.cov_at(w, xs, ys).numpy().astype(np.float64)
    ref = _oracle(img.cpu().numpy(), (0, 0), (w.height, w.width), c, xs, ys, w.basis, r)
    rel = np.abs(got - ref) / np.abs(ref)
    assert rel.max() <= TOL, _report(rel, labels)


def test_config4_one_frame_three_channels():
    w = synth.workload(4)
    frame = 5
    img = torch.stack([synth.make_image(w, frame=frame, channel=c, device=DEV) for c in range(3)]).contiguous()
    cov = synth.make_cov(w, frame=frame, device=DEV)[None].contiguous()
    plan = bsf.Plan(w.width, w.height, batch=1, channels=3, in_dtype=bsf.BSF_F32, order=w.order, basis=w.basis,
                    max_sigma=w.max_sigma, anchor=bsf.BSF_ANCHOR_AUTO)
    out = torch.empty((3, w.height, w.width), dtype=torch.float64, device=DEV)
    plan.run(img, cov, out)
    assert plan.stats()["status"] == 0
    pts, labels = stratified_points(w, 200, seed=41, r=w.order)
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    ch = np.arange(len(xs)) % 3  # the three channels share the frame's covariance field
    c = synth.cov_at(w, xs, ys, frame=frame).numpy().astype(np.float64)
    got = out.cpu().numpy()[ch, ys, xs]
    ref = np.zeros(len(xs))
    imgs = img.cpu().numpy()
    for k in range(3):
        m = ch == k
        ref[m] = _oracle(imgs[k], (0, 0), (w.height, w.width), c[:, m], xs[m], ys[m], w.basis, w.order)
    rel = np.abs(got - ref) / np.abs(ref)
    assert rel.max() <= TOL, _report(rel, labels)


def test_config5_one_row_strip():
    """Rank 3 of 8: the block (own rows + halo, what the NCCL exchange
    delivers) through a multi-GPU plan without communicator; own rows only."""
    w = synth.workload(5)
    world, rank = 8, 3
    plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_F32, order=w.order, basis=w.basis, max_sigma=w.max_sigma,
                    anchor=bsf.BSF_ANCHOR_TILE, rank=rank, nranks=world)
    g = plan.geometry
    y0, y1, b0, b1 = g.row0, g.row0 + g.row_count, g.block_row0, g.block_row0 + g.block_rows
    f_blk = synth.make_image(w, window=(b0, b1, 0, w.width), device=DEV)[None].contiguous()
    cov_own = synth.make_cov(w, window=(y0, y1, 0, w.width), device=DEV).contiguous()
    out = torch.empty((1, y1 - y0, w.width), dtype=torch.float64, device=DEV)
    plan.run(f_blk, cov_own, out)
    assert plan.stats()["status"] == 0
    del cov_own
    pts, labels = stratified_points(w, 200, seed=51, r=w.order, strip_rows=(1, y1 - y0 - 1), rows=(y0, y1))
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    c = synth.cov_at(w, xs, ys).numpy().astype(np.float64)
    got = out[0].cpu().numpy()[ys - y0, xs]
    ref = _oracle(f_blk[0].cpu().numpy(), (0, b0), (w.height, w.width), c, xs, ys, w.basis, w.order)
    rel = np.abs(got - ref) / np.abs(ref)
    assert rel.max() <= TOL, _report(rel, labels)
