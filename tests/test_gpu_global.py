"""Global mode: the paper's single global pre-integration
(Alg. 3 step 2) as exact int64 running
sums, gathered by the fused kernel with an exact two-limb contraction.  Parity
with the oracle at 1e-9 through the full-image launch (bsf_run), at config
scale on stratified pixels."""
import numpy as np
import pytest
import torch

import synth
from paper_1109_5114_b200 import bsf
from gpu_util import gpu_full, make_plan, oracle_points
from strata import stratified_points

pytestmark = pytest.mark.gpu


def _check(w, img, cov, pts, out, r=1, policy=None):
    policy = w.basis if policy is None else policy
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    ref, *_ = oracle_points(img.numpy(), cov.numpy(), xs, ys, policy=policy, r=r)
    got = out[0].numpy()[ys, xs]
    rel = np.abs(got - ref) / np.abs(ref)
    return float(rel.max()), rel


def test_global_mode_config1_every_pixel():
    w = synth.workload(1)
    img, cov = synth.make_image(w), synth.make_cov(w)
    for anchor in (bsf.BSF_ANCHOR_GLOBAL, bsf.BSF_ANCHOR_AUTO):
        plan = make_plan(w, anchor=anchor)
        assert plan.geometry.global_mode == 1
        out = gpu_full(plan, img[None], cov)
        ys, xs = np.mgrid[0:w.height, 0:w.width]
        pts = torch.tensor(np.stack([0 * xs.ravel(), xs.ravel(), ys.ravel()], 1), dtype=torch.int32)
        err, _ = _check(w, img, cov, pts, out)
        assert err <= 1e-9, err
        st = plan.stats(reset=True)
        assert st["status"] == 0 and st["pixels"] == w.width * w.height and st["double_double"] == 0


@pytest.mark.parametrize("policy", [0, 1, 2])
def test_global_mode_space_variant_small(policy):
    """Every pixel of a ragged 150 x 97 u8 image, config-3 field (large
    sigma relative to the image, zero-scale variants, both bases)."""
    w = synth.workload(3, width=150, height=97, max_sigma=40.0, extra={"grid_span": 300})
    img, cov = synth.make_image(w), synth.make_cov(w)
    plan = make_plan(w, policy=policy, anchor=bsf.BSF_ANCHOR_GLOBAL)
    assert plan.geometry.global_mode == 1
    out = gpu_full(plan, img[None], cov)
    ys, xs = np.mgrid[0:w.height:3, 0:w.width:3]
    pts = torch.tensor(np.stack([0 * xs.ravel(), xs.ravel(), ys.ravel()], 1), dtype=torch.int32)
    err, _ = _check(w, img, cov, pts, out, policy=policy)
    assert err <= 1e-9, err
    st = plan.stats(reset=True)
    assert st["status"] == 0 and st["zero_scale"] > 0


def test_global_mode_config3_full_size_stratified():
    """Config 3 at full size (4096^2 u8, order 1) through bsf_run: >= 300
    stratified pixels against the oracle, no tolerance floor."""
    w = synth.workload(3)
    img, cov = synth.make_image(w), synth.make_cov(w)
    plan = make_plan(w, anchor=bsf.BSF_ANCHOR_AUTO)
    assert plan.geometry.global_mode == 1
    out = gpu_full(plan, img[None], cov)
    pts, labels = stratified_points(w, 320, seed=3, r=1)
    err, rel = _check(w, img, cov, pts, out)
    worst = {k: float(rel[v].max()) for k, v in labels.items() if v}
    assert err <= 1e-9, worst
    st = plan.stats()
    assert st["status"] == 0 and st["double_double"] == 0 and st["pixels"] == w.width * w.height


def test_global_mode_matches_tile_path():
    """The global (paper-literal) and the tile-anchored paths compute the same
    filter: agreement far inside the 1e-9 contract on a 512^2 crop."""
    w = synth.workload(3, width=512, height=512, extra={"grid_span": 4096})
    img, cov = synth.make_image(w), synth.make_cov(w)
    a = gpu_full(make_plan(w, anchor=bsf.BSF_ANCHOR_GLOBAL), img[None], cov)
    b = gpu_full(make_plan(w, anchor=bsf.BSF_ANCHOR_TILE), img[None], cov)
    rel = ((a - b).abs() / b.abs()).max()
    assert float(rel) <= 1e-11, float(rel)


def test_global_mode_not_taken_when_sums_could_overflow():
    """Order 2 at config-3 size: the int64 sums would wrap, so AUTO anchors
    per super-tile and GLOBAL keeps the double-double global path."""
    w = synth.workload(3, order=2)
    assert make_plan(w, anchor=bsf.BSF_ANCHOR_AUTO).geometry.global_mode == 0
    w2 = synth.workload(2)  # float input: never global mode
    assert make_plan(w2, anchor=bsf.BSF_ANCHOR_AUTO).geometry.global_mode == 0


def test_filter_exact_is_run_split_in_two_calls():
    """bsf_preintegrate_exact + bsf_filter_exact (the two-call form bench.py
    times) give bsf_run's output bit for bit; non-global plans refuse it."""
    w = synth.workload(3, width=256, height=200, extra={"grid_span": 4096})
    img, cov = synth.make_image(w), synth.make_cov(w)
    plan = make_plan(w, anchor=bsf.BSF_ANCHOR_AUTO)
    a = gpu_full(plan, img[None], cov)
    dev = torch.device("cuda:0")
    g = plan.empty_g_exact()
    out = torch.empty((1, w.height, w.width), dtype=torch.float64, device=dev)
    plan.preintegrate_exact(img[None].to(dev).contiguous(), g)
    plan.filter_exact(g, cov.to(dev).contiguous(), out)
    torch.cuda.synchronize()
    assert torch.equal(a, out.cpu())
    tp = make_plan(w, anchor=bsf.BSF_ANCHOR_TILE)
    with pytest.raises(bsf.BsfError):
        tp.filter_exact(g, cov.to(dev).contiguous(), out)


def test_run_host_banded_scans_config3_full_size():
    """bsf_run_host at config 3's full size (one 4096^2 u8 image): the image
    arrives in row bands and each band is pre-integrated as soon as it is in
    (scan carries between bands, TMA-fed rows); the output equals the
    device-resident run bit for bit."""
    w = synth.workload(3)
    img, cov = synth.make_image(w), synth.make_cov(w)
    plan = make_plan(w, anchor=bsf.BSF_ANCHOR_AUTO)
    assert plan.geometry.global_mode == 1
    dev = gpu_full(plan, img[None], cov)
    f_h = img[None].contiguous().pin_memory()
    c_h = cov.contiguous().pin_memory()
    o_h = torch.full((1, w.height, w.width), float("nan"), dtype=torch.float64).pin_memory()
    plan.run_host(f_h, c_h, o_h)
    torch.cuda.synchronize()
    assert torch.equal(o_h, dev)


@pytest.mark.parametrize("out_f32", [False, True])
def test_run_host_pipeline_global_mode(out_f32):
    """bsf_run_host in global mode overlaps the copies with the compute (image,
    then covariance row bands on a copy-in stream; the gather band by band;
    output bands back on a copy-out stream): bit-identical to the device run,
    with 2 covariance fields x 2 channels and uneven bands (H = 301)."""
    W, H = 230, 301
    w = synth.workload(3, width=W, height=H, extra={"grid_span": 1500})
    img = torch.stack([synth.make_image(w, frame=f, channel=c) for f in range(2) for c in range(2)])
    cov = torch.stack([synth.make_cov(w), synth.make_cov(w, window=(0, H, 1, W + 1))]).contiguous()
    plan = bsf.Plan(W, H, batch=2, channels=2, in_dtype=bsf.BSF_U8, out_dtype=bsf.BSF_F32 if out_f32 else bsf.BSF_F64,
                    order=1, basis=2, max_sigma=w.max_sigma, anchor=bsf.BSF_ANCHOR_AUTO)
    assert plan.geometry.global_mode == 1
    dt = torch.float32 if out_f32 else torch.float64
    dev = gpu_full(plan, img, cov, out_dtype=dt)
    f_h = img.contiguous().pin_memory()
    c_h = cov.contiguous().pin_memory()
    o_h = torch.full((4, H, W), float("nan"), dtype=dt).pin_memory()
    plan.run_host(f_h, c_h, o_h)
    torch.cuda.synchronize()
    assert torch.equal(o_h, dev)
    for _ in range(2):  # repeated calls reuse the streams and events
        plan.run_host(f_h, c_h, o_h)
    torch.cuda.synchronize()
    assert torch.equal(o_h, dev)
    # one image (H = 301: image bands of 96 rows, the last one shorter and
    # holding the bottom margin)
    p1 = bsf.Plan(W, H, in_dtype=bsf.BSF_U8, out_dtype=bsf.BSF_F32 if out_f32 else bsf.BSF_F64, order=1, basis=2,
                  max_sigma=w.max_sigma, anchor=bsf.BSF_ANCHOR_AUTO)
    d1 = gpu_full(p1, img[:1], cov[0], out_dtype=dt)
    o1 = torch.full((1, H, W), float("nan"), dtype=dt).pin_memory()
    p1.run_host(img[:1].contiguous().pin_memory(), cov[0].contiguous().pin_memory(), o1)
    torch.cuda.synchronize()
    assert torch.equal(o1, d1)


@pytest.mark.parametrize("policy", [0, 1, 2])
def test_gx1_dp4a_contraction_is_bit_identical(policy):
    """The byte-plane dp4a contraction (bsf_gx1.cuh gx1_tap_dp) and the
    three-limb IMAD contraction both form E_mu exactly, so the outputs agree
    bit for bit (ragged 150 x 97 image with sums reaching above row 0,
    zero-scale variants, both bases), and both match the oracle at 1e-9."""
    w = synth.workload(3, width=150, height=97, max_sigma=40.0, extra={"grid_span": 300})
    img, cov = synth.make_image(w), synth.make_cov(w)
    outs = []
    for dp in (0, 1):
        plan = make_plan(w, policy=policy, anchor=bsf.BSF_ANCHOR_GLOBAL)
        plan.debug_option("gx1_dp4a", dp)
        outs.append(gpu_full(plan, img[None], cov))
        st = plan.stats(reset=True)
        assert st["status"] == 0 and st["double_double"] == 0
    assert torch.equal(outs[0], outs[1])
    ys, xs = np.mgrid[0:w.height:5, 0:w.width:5]
    pts = torch.tensor(np.stack([0 * xs.ravel(), xs.ravel(), ys.ravel()], 1), dtype=torch.int32)
    err, _ = _check(w, img, cov, pts, outs[1], policy=policy)
    assert err <= 1e-9, err


def test_gx1_dp4a_config3_full_size_bit_identical():
    """Config 3 at full size (sums up to 2^57: all eight byte planes live):
    the dp4a and IMAD contractions give the same image bit for bit."""
    w = synth.workload(3)
    img, cov = synth.make_image(w), synth.make_cov(w)
    outs = []
    for dp in (0, 1):
        plan = make_plan(w, anchor=bsf.BSF_ANCHOR_AUTO)
        assert plan.geometry.global_mode == 1
        plan.debug_option("gx1_dp4a", dp)
        outs.append(gpu_full(plan, img[None], cov))
    assert torch.equal(outs[0], outs[1])
