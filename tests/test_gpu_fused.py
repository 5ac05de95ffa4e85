"""The fused exact-split path (bsf_fused.cuh) against the double-double tile
kernel and against itself: its double-double fallback, its work counter and
its dispatch.  (Parity with the oracle is in test_gpu_tile.py /
test_gpu_orders.py, which run the fused path by default.)"""
import math

import numpy as np
import pytest
import torch

import synth
from paper_1109_5114_b200 import bsf, lut
from gpu_util import gpu_full, make_plan, tile_points
from test_gpu_parity import _small_smooth

pytestmark = pytest.mark.gpu
TILE = bsf.BSF_ANCHOR_TILE


def test_dispatch():
    w = synth.workload(2)
    plan = make_plan(w, anchor=TILE)
    pts = synth.sample_points(w, 4, seed=1)
    tile_points(plan, synth.make_image(w)[None], synth.make_cov(w), pts)
    assert plan.uses_fused()
    # Theta' at r = 3: a 4-bit exact limb unsplit -> split numerators, still fused
    w3 = synth.workload(1, width=40, height=40)
    p3 = make_plan(w3, policy=1, order=3, anchor=TILE)
    tile_points(p3, synth.make_image(w3)[None], synth.make_cov(w3), synth.sample_points(w3, 2, seed=1))
    assert p3.uses_fused()
    # order 4: double-double tile kernel
    p4 = make_plan(w3, policy=0, order=4, anchor=TILE)
    tile_points(p4, synth.make_image(w3)[None], synth.make_cov(w3), synth.sample_points(w3, 2, seed=1))
    assert not p4.uses_fused()
    p0 = make_plan(w, anchor=TILE)
    p0.debug_option("fused", 0)
    tile_points(p0, synth.make_image(w)[None], synth.make_cov(w), pts)
    assert not p0.uses_fused()


@pytest.mark.parametrize("config,order,n", [(2, 2, 3000), (3, 1, 3000), (3, 2, 600), (4, 3, 60)])
def test_fused_matches_double_double_kernel(config, order, n):
    """Split contraction vs the all-double-double tile kernel on the same
    (full-size) workload: both are far more accurate than the 1e-9 contract,
    so they must agree to ~1e-12."""
    w = synth.workload(config, order=order)
    img, cov = synth.make_image(w), synth.make_cov(w)
    pts = synth.sample_points(w, n, seed=5)
    a = tile_points(make_plan(w, anchor=TILE), img[None], cov, pts)
    pb = make_plan(w, anchor=TILE)
    pb.debug_option("fused", 0)
    b = tile_points(pb, img[None], cov, pts)
    rel = (a - b).abs() / b.abs()
    # at r = 3 the double-double kernel's own error reaches ~1e-12 on the most
    # ill-conditioned pixels (u^2 times a condition number ~1e20)
    assert float(rel.max()) <= (1e-12 if order < 3 else 1e-11), float(rel.max())


@pytest.mark.parametrize("r", [1, 2, 3])
def test_forced_fallback_matches_split_path(r):
    """split_tol = 0 sends every pixel to the warp-cooperative double-double
    fallback (mesh_warp on the split planes); it must agree with the split
    path and be counted."""
    H, W = 45, 53
    w, img, cov = _small_smooth(H, W, 3.0)
    plan = make_plan(w, order=r, anchor=TILE)
    a = gpu_full(plan, img, cov)[0]
    st = plan.stats(reset=True)
    assert st["double_double"] < st["pixels"] // 10
    plan.debug_option("split_tol", 0.0)
    b = gpu_full(plan, img, cov)[0]
    st = plan.stats(reset=True)
    assert st["double_double"] == st["pixels"] == H * W
    rel = (a - b).abs() / b.abs()
    assert float(rel.max()) <= (1e-12 if r < 3 else 1e-11), float(rel.max())


def test_macs_counter_is_the_algorithmic_work():
    """bsf_stats.macs = sum over taps of (window slots of the tap's region) x
    (monomials of the table), recomputed on the host from the per-pixel scales
    (aux) and the tables' region classification."""
    H, W, r = 20, 24, 2
    w, img, cov = _small_smooth(H, W, 2.5)
    plan = make_plan(w, order=r, anchor=TILE)
    ys, xs = np.mgrid[0:H, 0:W]
    pts = torch.tensor(np.stack([np.zeros(H * W), xs.ravel(), ys.ravel()], 1), dtype=torch.int32)
    plan.stats(reset=True)
    _, aux = tile_points(plan, img[None], cov, pts, aux=True)
    got = plan.stats()["macs"]
    steps = {0: [(1, 0), (1, 1), (0, 1), (-1, 1)], 1: [(2, 1), (1, 2), (-1, 2), (-2, 1)]}
    tabs = {b: lut.load(b, r) for b in (0, 1)}
    want = 0
    for row in aux.numpy():
        b, drop, ap = int(row[0]), int(row[1]), row[4:8]
        v = tabs[b]["variants"][drop + 1]
        dirs = [k for k in range(4) if k != drop]
        for t in range((r + 1) ** len(dirs)):
            tt, Dx, Dy = t, 0.0, 0.0
            for k in dirs:
                j = tt % (r + 1)
                tt //= r + 1
                m = 0.5 * r - j
                Dx += (m * steps[b][k][0]) * ap[k]
                Dy += (m * steps[b][k][1]) * ap[k]
            reg = lut.region_of(tabs[b], Dx - math.floor(Dx), Dy - math.floor(Dy))
            want += int(v["counts"][reg]) * v["nmon"]
    assert got == want


def test_super_tile_64_matches_32():
    """Order 1 with a large reach anchors the running sums on 64 x 64
    super-tiles (plan geometry); the whole image (ragged in both directions,
    batch of 2) must agree with the 32 x 32 anchoring to ~1e-12, and with the
    oracle at sampled pixels to the 1e-9 contract."""
    w = synth.workload(3, order=1, width=300, height=170)
    img = torch.stack([synth.make_image(w), synth.make_image(w, frame=1)])
    cov = synth.make_cov(w)[None].expand(2, -1, -1, -1).contiguous()
    p64 = make_plan(w, anchor=TILE, batch=2)
    assert p64.geometry.super_tile == 64
    a = gpu_full(p64, img, cov)
    p32 = make_plan(w, anchor=TILE, batch=2, super_tile=32)
    assert p32.geometry.super_tile == 32
    b = gpu_full(p32, img, cov)
    rel = ((a - b).abs() / b.abs()).max()
    assert float(rel) <= 1e-12, float(rel)
    from gpu_util import oracle_points
    pts = synth.sample_points(w, 40, seed=9)
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    ref = oracle_points(img[0].numpy(), cov[0].numpy(), xs, ys, policy=w.basis, r=1)[0]
    got = a[0].cpu().numpy()[ys, xs]
    err = np.max(np.abs(got - ref) / np.abs(ref))
    assert err <= 1e-9, err


@pytest.mark.parametrize("r", [1, 2, 3])
def test_fused_tiny_and_thin_images(r):
    """Degenerate shapes through the fused product path (a super-tile larger
    than the image, single rows/columns, one pixel) against the oracle."""
    for H, W in ((1, 1), (1, 37), (29, 1), (3, 2), (33, 65)):
        w = synth.workload(1, width=W, height=H)
        img, cov = synth.make_image(w), synth.make_cov(w)
        plan = make_plan(w, order=r, anchor=TILE)
        out = gpu_full(plan, img[None], cov)[0].cpu().numpy()
        assert plan.uses_fused()
        ys, xs = np.mgrid[0:H, 0:W]
        from gpu_util import oracle_points, max_rel
        ref, *_ = oracle_points(img.numpy(), cov.numpy(), xs.ravel(), ys.ravel(), policy=2, r=r)
        assert max_rel(out.ravel(), ref) <= 1e-9, (H, W)


def test_run_host_matches_device_run():
    """bsf_run_host (the e2e path of bench.py: pinned host buffers, copies on
    the stream) gives the device run's output bit for bit."""
    w, img, cov = _small_smooth(80, 96, 6.0, seed=12)
    plan = make_plan(w, anchor=TILE)
    dev = gpu_full(plan, img[None], cov).cpu()
    assert torch.isfinite(dev).all()
    f_h = img[None].contiguous().pin_memory()
    c_h = cov.contiguous().pin_memory()
    o_h = torch.empty((1, 80, 96), dtype=torch.float64).pin_memory()
    plan.run_host(f_h, c_h, o_h)
    torch.cuda.synchronize()
    assert torch.equal(o_h, dev)


@pytest.mark.parametrize("r", [2, 3])
def test_work_order_changes_nothing_but_the_schedule(r):
    """The largest-first hand-out of super-tiles (fused_cost_kernel /
    fused_order_kernel) only changes which CTA computes a super-tile and when:
    the output is bit-identical to the raster hand-out, and the two scheduling
    launches are counted."""
    if r == 2:
        w = synth.workload(2, width=640, height=480)  # 300 super-tiles
        img = synth.make_image(w)[None]
    else:
        w = synth.workload(4, width=608, height=512)  # 3 channels x 304 super-tiles
        img = torch.stack([synth.make_image(w, channel=c) for c in range(w.channels)])
    cov = synth.make_cov(w)
    runs = {}
    for o in ("0", "1"):
        plan = make_plan(w, anchor=TILE, batch=1)
        plan.debug_option("work_order", int(o))
        n0 = plan.launch_count()
        out = gpu_full(plan, img, cov)
        runs[o] = (out, plan.launch_count() - n0, plan.stats())
    assert torch.equal(runs["0"][0], runs["1"][0])
    assert runs["1"][1] == runs["0"][1] + 2
    for k in ("pixels", "macs", "double_double"):
        assert runs["0"][2][k] == runs["1"][2][k], k


def test_order2_u8_super_tile_64():
    """u8 input at order 2 with a large reach anchors on 64 x 64 super-tiles
    (its exact low levels keep the larger domains accurate); the output agrees
    with the 32 x 32 anchoring and with the oracle to the 1e-9 contract, and
    bsf_run_split's float64 passes (which run 32 x 32) agree too."""
    w = synth.workload(3, order=2, width=330, height=200)
    img, cov = synth.make_image(w), synth.make_cov(w)
    dev = torch.device("cuda:0")
    p64 = make_plan(w, anchor=TILE)
    assert p64.geometry.super_tile == 64
    a = gpu_full(p64, img[None], cov)
    p32 = make_plan(w, anchor=TILE, super_tile=32)
    assert p32.geometry.super_tile == 32
    b = gpu_full(p32, img[None], cov)
    rel = ((a - b).abs() / b.abs()).max()
    assert float(rel) <= 2e-9, float(rel)
    from gpu_util import oracle_points
    pts = synth.sample_points(w, 24, seed=11)
    xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
    ref = oracle_points(img.numpy(), cov.numpy(), xs, ys, policy=w.basis, r=2)[0]
    err = np.max(np.abs(a[0].numpy()[ys, xs] - ref) / np.abs(ref))
    assert err <= 1e-9, err
    outs = []
    for p in (p64, p32):
        o = torch.empty((1, w.height, w.width), dtype=torch.float64, device=dev)
        p.run_alg1(img[None].to(dev).contiguous(), cov.to(dev).contiguous(), o)
        torch.cuda.synchronize()
        outs.append(o.cpu())
    rel = ((outs[0] - outs[1]).abs() / outs[1].abs()).max()
    assert float(rel) <= 2e-9, float(rel)


def test_item_diagnostics_are_consistent():
    """bsf_debug_item_cycles: the per-super-tile MACs add up to bsf_stats.macs,
    the fallback counts to bsf_stats.double_double, every super-tile reports
    cycles and a halo, and the CTAs' busy cycles add up to the items' cycles."""
    w = synth.workload(2, width=640, height=480)
    img, cov = synth.make_image(w), synth.make_cov(w)
    plan = make_plan(w, anchor=TILE)
    with pytest.raises(RuntimeError):
        plan.item_cycles(4)  # counters not enabled yet
    plan.phase_cycles(reset=True)
    plan.stats(reset=True)
    gpu_full(plan, img[None], cov)
    st = plan.stats(reset=True)
    n = 20 * 15
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    items, work, ctas = plan.item_cycles(n, nsm)
    assert sum(x[0] for x in work) == st["macs"]
    assert sum(x[1] for x in work) == st["double_double"]
    assert all(c > 0 for c in items) and all(x[2] > 0 and x[3] > 0 for x in work)
    assert sum(ctas) == sum(items)


def test_split_mode_quadrants_small_scales():
    """u8 at order 2 with a large reach (64 x 64 super-tiles) and a region of
    tiny scales: the work order hands the ill-conditioned super-tiles out as
    32 x 32 quadrants (split mode), which keeps their pixels off the
    double-double fallback; the output matches the oracle everywhere sampled,
    the small-scale region included."""
    W, H = 448, 320
    w = synth.workload(3, order=2, width=W, height=H)
    img = synth.make_image(w)
    X = torch.arange(W, dtype=torch.float64)[None, :].expand(H, W)
    Y = torch.arange(H, dtype=torch.float64)[:, None].expand(H, W)
    smaj = 0.45 + 13.5 * (X / (W - 1)) ** 2
    th = torch.remainder(0.7 + 0.004 * X + 0.003 * Y, math.pi)
    cov = torch.stack([smaj, smaj / 1.6, th]).to(torch.float32)
    res = {}
    for o in ("0", "1"):
        plan = make_plan(w, anchor=TILE, batch=1)
        plan.debug_option("work_order", int(o))
        assert plan.geometry.super_tile == 64
        n0 = plan.launch_count()
        out = gpu_full(plan, img[None], cov)
        res[o] = (out, plan.stats()["double_double"], plan.launch_count() - n0)
    assert res["1"][2] == 3 and res["0"][2] == 1
    assert res["1"][1] < res["0"][1], (res["1"][1], res["0"][1])
    from gpu_util import oracle_points
    rng = np.random.default_rng(5)
    xs = np.concatenate([rng.integers(0, 64, 16), rng.integers(0, W, 16)])
    ys = rng.integers(0, H, 32)
    ref = oracle_points(img.numpy(), cov.numpy(), xs, ys, policy=w.basis, r=2)[0]
    for o in ("0", "1"):
        err = np.max(np.abs(res[o][0][0].numpy()[ys, xs] - ref) / np.abs(ref))
        assert err <= 1e-9, (o, err)


def test_split_mode_cost_bin_saturation():
    """A covariance far above the plan's max_sigma in one 64 x 64 super-tile
    of an order-2 u8 plan: its cost estimate saturates the largest bin and it
    is handed out as quadrant units (tiny sigma_min).  Every unit must still
    be scheduled: NaN and BSF_ERANGE there (the documented behaviour), finite
    results elsewhere, no out-of-bounds writes."""
    W, H = 256, 192
    w = synth.workload(3, order=2, width=W, height=H, max_sigma=20.0)
    img = synth.make_image(w)
    cov = torch.stack([torch.full((H, W), 3.0), torch.full((H, W), 2.0), torch.full((H, W), 0.3)])
    cov[0, 64:128, 64:128] = 800.0
    cov[1, 64:128, 64:128] = 0.3
    plan = make_plan(w, anchor=TILE)
    assert plan.geometry.super_tile == 64
    out = gpu_full(plan, img[None], cov.to(torch.float32))[0]
    st = plan.stats(reset=True)
    assert st["status"] == 5  # BSF_ERANGE
    assert torch.isnan(out[64:128, 64:128]).all()
    mask = torch.ones(H, W, dtype=torch.bool)
    mask[64:128, 64:128] = False
    assert torch.isfinite(out[mask]).all()


@pytest.mark.parametrize("r", [2, 4])
def test_run_tiles_equals_run_on_listed_tiles(r):
    """bsf_run_tiles computes exactly bsf_run's values on the listed anchoring
    tiles (same kernel, same anchoring) and leaves the other outputs alone."""
    w = synth.workload(3, order=r, width=160 if r == 4 else 300, height=96 if r == 4 else 200,
                       max_sigma=4.0 if r == 4 else 40.0, extra={"grid_span": 800})
    img, cov = synth.make_image(w), synth.make_cov(w)
    if r == 4:
        cov[0] = cov[0].clamp(max=3.0)
        cov[1] = torch.minimum(cov[1], cov[0])
    plan = make_plan(w, anchor=TILE)
    u = plan.geometry.tile_unit
    assert u in (16, 32, 64)
    ntx, nty = (w.width + u - 1) // u, (w.height + u - 1) // u
    ids = torch.tensor(sorted({0, ntx - 1, ntx * nty - 1, ntx + 1}), dtype=torch.int32)
    dev = torch.device("cuda:0")
    sub = torch.full((1, w.height, w.width), float("nan"), dtype=torch.float64, device=dev)
    plan.run_tiles(img[None].to(dev).contiguous(), cov.to(dev).contiguous(), sub, ids.to(dev))
    torch.cuda.synchronize()
    sub = sub.cpu()[0]
    if r == 4:  # order 4: compare with the oracle on the listed tiles (a full run is slow)
        from gpu_util import oracle_points
        for t in ids.tolist()[:2]:
            ty, tx = divmod(t, ntx)
            ys, xs = np.mgrid[ty * u:min(w.height, ty * u + u):5, tx * u:min(w.width, tx * u + u):5]
            ref = oracle_points(img.numpy(), cov.numpy(), xs.ravel(), ys.ravel(), policy=w.basis, r=4)[0]
            got = sub.numpy()[ys.ravel(), xs.ravel()]
            assert np.max(np.abs(got - ref) / np.abs(ref)) <= 1e-9
    else:
        full = gpu_full(plan, img[None], cov)[0]
        mask = torch.zeros(w.height, w.width, dtype=torch.bool)
        for t in ids.tolist():
            ty, tx = divmod(t, ntx)
            mask[ty * u:(ty + 1) * u, tx * u:(tx + 1) * u] = True
        assert torch.equal(sub[mask], full[mask])
        assert torch.isnan(sub[~mask]).all()
