"""Row-strip partitioning of one image (config 5's multi-GPU scheme) with the
real kernel, simulated in one process: every rank's block (own rows + halo
rows from its neighbours, exactly what parallel.exchange_halos assembles) is
filtered by its own plan, and the kept rows must equal the single-GPU result
bit for bit."""
import math

import numpy as np
import pytest
import torch

import synth
from paper_1109_5114_b200 import bsf
from paper_1109_5114_b200 import parallel as PL

pytestmark = pytest.mark.gpu


def _field(H, W, smax):
    X = torch.arange(W, dtype=torch.float64)[None, :]
    Y = torch.arange(H, dtype=torch.float64)[:, None]
    smaj = 1.0 + (smax - 1.0) * (0.5 + 0.5 * torch.sin(X / 37.0) * torch.cos(Y / 23.0))
    ratio = 1.0 + 4.0 * (0.5 + 0.5 * torch.cos(X / 29.0 + Y / 41.0))
    th = torch.remainder(torch.atan2(Y - H / 3, X - W / 2), math.pi)
    return torch.stack([smaj, smaj / torch.sqrt(ratio), th]).to(torch.float32)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("order,policy,smax", [(2, bsf.BSF_DUAL, 5.0), (3, bsf.BSF_THETA, 5.0),
                                               (1, bsf.BSF_DUAL, 16.0)])
def test_strips_bitwise_equal_single_gpu(world, order, policy, smax):
    """Multi-GPU plans (bsf_plan_desc rank / nranks, no communicator: the
    caller assembles the halo, what parallel.exchange_halos does): each rank's
    bsf_run takes its block of input rows and computes its own rows only; they
    equal the one-GPU run bit for bit.  (order 1, sigma 16: 64 x 64 super-tiles
    and a 128-row halo, so a taller image: every strip holds its neighbours'
    halos)"""
    H, W = (640 if order == 1 else 352), 200
    w = synth.workload(5, width=W, height=H, max_sigma=smax, order=order)
    img = synth.make_image(w).cuda()
    cov = _field(H, W, smax).cuda()

    def plan(rank=0, nranks=1):
        return bsf.Plan(W, H, in_dtype=bsf.BSF_F32, order=order, basis=policy, max_sigma=smax,
                        anchor=bsf.BSF_ANCHOR_TILE, rank=rank, nranks=nranks, super_tile=64 if order == 1 else 32)

    full = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    p_full = plan()
    tile = p_full.geometry.super_tile
    assert tile == (64 if order == 1 else 32)
    p_full.run(img[None].contiguous(), cov.contiguous(), full)
    rows = 0
    for rank in range(world):
        p = plan(rank, world)
        st = PL.strip_plan_of(p)
        assert st.tile == tile and st.halo == PL.halo_rows(smax, order, tile)
        assert (st.y0, st.y1, st.b0, st.b1) == bsf.strip_rows(H, tile, st.halo, rank, world)
        assert st.y0 % tile == 0 and st.b0 % tile == 0
        f_blk = img[st.b0:st.b1]                     # = exchange_halos(own rows)
        out = torch.empty((1, st.y1 - st.y0, W), dtype=torch.float64, device="cuda")
        p.run(f_blk[None].contiguous(), cov[:, st.y0:st.y1].contiguous(), out)
        torch.cuda.synchronize()
        ref = full[0, st.y0:st.y1]
        assert torch.equal(out[0], ref), (rank, float((out[0] - ref).abs().max()))
        assert p.stats()["pixels"] == (st.y1 - st.y0) * W  # own rows only
        rows += st.y1 - st.y0
    assert rows == H


def test_multi_gpu_plan_refuses_other_entry_points_and_nccl_id():
    w = synth.workload(5, width=64, height=256, max_sigma=2.0, order=1)
    p = bsf.Plan(64, 256, in_dtype=bsf.BSF_F32, order=1, basis=2, max_sigma=2.0, anchor=bsf.BSF_ANCHOR_TILE,
                 rank=0, nranks=2)
    g = p.geometry
    assert g.row0 == 0 and g.row_count == 128 and g.block_rows == 128 + g.halo
    img = synth.make_image(w).cuda()
    out = torch.empty((1, 256, 64), dtype=torch.float64, device="cuda")
    with pytest.raises(bsf.BsfError):
        p.run_tiles(img[None].contiguous(), torch.ones(3, 256, 64, device="cuda"), out,
                    torch.zeros(1, dtype=torch.int32, device="cuda"))
    assert len(bsf.get_unique_id()) == 128  # NCCL loads in-process (the id a rank-0 caller broadcasts)


def _global_strips_sequential(make_plan, img, H, Pb, world, exact):
    """Run parallel.preintegrate_strip for every rank of a `world` chain in one
    process, the carries passed through a dict (what the NCCL send/recv of
    preintegrate_global_strips carries)."""
    carries, parts = {}, []
    for rank in range(world):
        st = PL.global_strip(H, Pb, rank, world)
        plan = make_plan(st.height, st.margin_y)
        assert plan.geometry.g_height == st.Y1 - st.Y0
        g = plan.empty_g_exact() if exact else plan.empty_g()
        f = img[:, st.Y0:st.Y0 + st.height].contiguous()

        def recv(slot, level, sy, rank=rank):
            return carries.pop((rank, slot, level)) if rank > 0 else None

        def send(slot, level, rows, rank=rank):
            if rank < world - 1:
                carries[(rank + 1, slot, level)] = rows

        PL.preintegrate_strip(plan, f, g, recv_carry=recv, send_carry=send, exact=exact)
        geo = plan.geometry
        parts.append(g.view(geo.nbases, img.shape[0], geo.g_height, -1))
    assert not carries
    return torch.cat(parts, dim=2)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("order,policy", [(1, bsf.BSF_DUAL), (2, bsf.BSF_DUAL), (3, bsf.BSF_THETA_PRIME)])
def test_global_mode_strips_bit_exact(world, order, policy):
    """SURVEY 8(e) GLOBAL mode: row strips + scan carries down the rank chain
    reproduce the single-plan int64 pre-integration bit for bit (u8 input,
    batch of 2 images, ragged last strip)."""
    H, W, smax = 150, 90, 3.0
    gen = torch.Generator().manual_seed(7)
    img = torch.randint(0, 256, (2, H, W), generator=gen, dtype=torch.uint8).cuda()

    def make_plan(height, margin_y):
        return bsf.Plan(W, height, batch=2, in_dtype=bsf.BSF_U8, order=order, basis=policy, max_sigma=smax,
                        margin_y=margin_y)

    full_plan = make_plan(H, 0)
    Pb = full_plan.geometry.margin_y
    g_full = full_plan.empty_g_exact()
    full_plan.preintegrate_exact(img, g_full)
    g_str = _global_strips_sequential(make_plan, img, H, Pb, world, exact=True)
    torch.cuda.synchronize()
    assert torch.equal(g_str, g_full), "GLOBAL-mode strips differ from the single-plan pre-integration"


def test_global_mode_strips_double_double():
    """Same chain on the double-double running sums (f32 input): equal to the
    single plan up to double-double rounding order."""
    H, W, smax, order = 130, 70, 2.5, 2
    gen = torch.Generator().manual_seed(8)
    img = torch.rand((1, H, W), generator=gen).cuda()

    def make_plan(height, margin_y):
        return bsf.Plan(W, height, in_dtype=bsf.BSF_F32, order=order, basis=bsf.BSF_DUAL, max_sigma=smax,
                        margin_y=margin_y)

    full_plan = make_plan(H, 0)
    geo = full_plan.geometry
    g_full = full_plan.empty_g()
    full_plan.preintegrate(img, g_full)
    g_str = _global_strips_sequential(make_plan, img, H, geo.margin_y, 3, exact=False)
    a = g_full.view(geo.nbases, 1, geo.g_height, geo.g_width, 2).sum(-1)
    b = g_str.reshape(geo.nbases, 1, geo.g_height, geo.g_width, 2).sum(-1)
    assert torch.allclose(a, b, rtol=1e-15, atol=0.0)


def test_row_strip_plan_rejects_filtering():
    plan = bsf.Plan(64, 32, in_dtype=bsf.BSF_U8, order=1, max_sigma=2.0, margin_y=-1)
    assert plan.geometry.margin_y == 0
    g = plan.empty_g()
    cov = torch.ones((1, 3, 32, 64), dtype=torch.float32, device="cuda")
    out = torch.empty((1, 32, 64), dtype=torch.float64, device="cuda")
    with pytest.raises(RuntimeError):
        plan.filter(g, cov, out)
