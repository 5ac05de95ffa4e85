"""Multi-process (gloo, CPU) tests of the partitioning and halo exchange of
paper_1109_5114_b200.parallel.  The compute is replaced by a local stand-in
filter (a box mean with zero extension, reach < halo) so the assembly logic is
checked end to end without a GPU: strips must reproduce the full-image result
exactly."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1109_5114_b200 import parallel as PL


def test_shard_range_partitions():
    for n in (0, 1, 7, 64, 65):
        for world in (1, 2, 3, 8):
            spans = [PL.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_strip_plan_alignment_and_cover():
    H = 1000
    halo = PL.halo_rows(8.0, 3)
    assert halo % PL.TILE == 0 and halo >= 8.0 * (72 ** 0.5)
    # the library's partition arithmetic (bsf_strip_rows, no GPU needed)
    from paper_1109_5114_b200 import bsf
    assert bsf.strip_rows(100, 32, 32, 1, 2) == (64, 100, 32, 100)
    with pytest.raises(bsf.BsfError):
        bsf.strip_rows(100, 32, 64, 1, 3)  # a 32-row strip cannot feed its neighbours' 64-row halos
    for world in (1, 2, 4, 8):
        strips = [PL.strip_plan(H, r, world, halo) for r in range(world)]
        assert strips[0].y0 == 0 and strips[-1].y1 == H
        for s, t in zip(strips, strips[1:]):
            assert s.y1 == t.y0 and s.y0 % PL.TILE == 0 and t.y0 % PL.TILE == 0
        for s in strips:
            assert s.b0 == max(0, s.y0 - halo) and s.b1 == min(H, s.y1 + halo)


class _StandIn:
    """Stand-in for a multi-GPU bsf.Plan without communicator: bsf_run takes
    the strip's block and writes its own rows only; the filter is a 2R+1 box
    mean with zero extension (reach R)."""

    R = 3

    def __init__(self, strip=None):
        self.strip = strip

    def run(self, f, cov, out, stream=None):
        k = 2 * self.R + 1
        x = f.to(torch.float64).reshape(1, 1, f.shape[-2], f.shape[-1])
        w = torch.ones(1, 1, k, k, dtype=torch.float64) / (k * k)
        y = torch.nn.functional.conv2d(x, w, padding=self.R)[0, 0]
        out[0] = y[self.strip.out_slice] if self.strip is not None else y


def _worker(rank, world, port, H, W, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(1)
        full = torch.rand(H, W, generator=g, dtype=torch.float64).float()
        halo = PL.TILE  # >= stand-in reach
        st = PL.strip_plan(H, rank, world, halo)
        own = full[st.y0:st.y1].clone()
        blk = PL.exchange_halos(own, st, H)
        ok_blk = torch.equal(blk, full[st.b0:st.b1])
        cov = torch.ones(3, st.y1 - st.y0, W)
        res = PL.filter_strip(_StandIn(st), own[None], cov, st, H)[0]
        # by value (numpy): a torch tensor travels as a shared-memory handle
        # that dies with this process if it exits before the parent reads it
        q.put((rank, ok_blk, st.y0, st.y1, res.numpy().copy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_row_strips_reproduce_full_image(world):
    H, W = 90, 21
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    g = torch.Generator().manual_seed(1)
    full = torch.rand(H, W, generator=g, dtype=torch.float64).float()
    ref = torch.empty(1, H, W, dtype=torch.float64)
    _StandIn().run(full, None, ref)
    for rank, ok_blk, y0, y1, res in got:
        assert ok_blk, rank
        assert torch.equal(torch.from_numpy(res), ref[0, y0:y1]), rank


class _ScanStandIn:
    """Stand-in for a bsf.Plan in GLOBAL-mode pre-integration: the running-sum
    levels computed by plain loops on CPU int64 tensors (the definition
    G(x, y) = V(x, y) + G(x - sx, y - sy), zero state outside the strip's
    domain unless a carry row supplies it)."""

    STEPS = [(1, 2), (2, 1), (-1, 2), (-2, 1)]  # Theta' order

    class _Geo:
        pass

    def __init__(self, W, P, rows, order):
        self.geometry = self._Geo()
        self.geometry.nbases, self.geometry.g_height, self.geometry.g_width = 1, rows, W + 2 * P
        self.P = P

        class _D:
            pass
        self.desc = _D()
        self.desc.batch, self.desc.channels, self.desc.order = 1, 1, order

    def scan_step(self, slot, level):
        return self.STEPS[level % 4]

    def scan_level(self, slot, level, f, g, carry=None, exact=True, stream=None):
        sx, sy = self.STEPS[level % 4]
        GH, GW = self.geometry.g_height, self.geometry.g_width
        gv = g.view(GH, GW)
        if level == 0:
            gv.zero_()
            gv[:f.shape[-2], self.P:self.P + f.shape[-1]] = f.reshape(f.shape[-2], f.shape[-1]).to(torch.int64)
        for y in range(GH):
            for x in range(GW):
                px, py = x - sx, y - sy
                if 0 <= px < GW:
                    if py >= 0:
                        gv[y, x] += gv[py, px]
                    elif carry is not None:
                        gv[y, x] += carry.view(sy, GW)[py + sy, px]


def _global_worker(rank, world, port, H, W, P, Pb, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gen = torch.Generator().manual_seed(3)
        img = torch.randint(0, 256, (H, W), generator=gen, dtype=torch.uint8)
        st = PL.global_strip(H, Pb, rank, world, unit=4)
        plan = _ScanStandIn(W, P, st.Y1 - st.Y0, order=1)
        g = torch.zeros((st.Y1 - st.Y0) * (W + 2 * P), dtype=torch.int64)
        PL.preintegrate_global_strips(plan, img[st.Y0:st.Y0 + st.height], g, st)
        q.put((rank, st.Y0, st.Y1, g.view(st.Y1 - st.Y0, W + 2 * P).numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_global_mode_carry_chain_gloo():
    """SURVEY 8(e) GLOBAL mode over a gloo rank chain (world 3): the strips'
    running sums, with the scan carries sent down the chain, equal the
    one-strip computation exactly."""
    H, W, P, Pb, world = 22, 9, 3, 5, 3
    gen = torch.Generator().manual_seed(3)
    img = torch.randint(0, 256, (H, W), generator=gen, dtype=torch.uint8)
    ref_plan = _ScanStandIn(W, P, H + Pb, order=1)
    ref = torch.zeros((H + Pb) * (W + 2 * P), dtype=torch.int64)
    PL.preintegrate_strip(ref_plan, img, ref, recv_carry=lambda *a: None, send_carry=lambda *a: None)
    ref = ref.view(H + Pb, W + 2 * P)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_global_worker, args=(r, world, port, H, W, P, Pb, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == 0 and res[-1][2] == H + Pb
    for rank, Y0, Y1, g in res:
        assert torch.equal(torch.from_numpy(g), ref[Y0:Y1]), "rank %d rows [%d, %d) differ" % (rank, Y0, Y1)


@pytest.mark.parametrize("H,unit,halo", [(1000, 32, 96), (4096, 64, 128), (352, 32, 32), (777, 16, 48)])
@pytest.mark.parametrize("world", [2, 3, 4, 5, 8])
def test_library_halo_exchange_plan_assembles_every_block(H, unit, halo, world):
    """The row counts bsf_run sends and receives over NCCL (bsf_strip_exchange,
    the library's own arithmetic, no GPU needed) are consistent between
    neighbours and, replayed on a host image, assemble every rank's block
    rows [b0, b1) exactly."""
    import numpy as np
    from paper_1109_5114_b200 import bsf
    try:
        strips = [bsf.strip_rows(H, unit, halo, r, world) for r in range(world)]
    except bsf.BsfError:
        pytest.skip("strips thinner than the halo: the library refuses this partition")
    img = np.arange(H)[:, None] * 1000 + np.arange(7)[None, :]
    xs = [bsf.strip_exchange(H, unit, halo, r, world) for r in range(world)]
    for r, ((y0, y1, b0, b1), x) in enumerate(zip(strips, xs)):
        own = img[y0:y1]
        blk = np.full((b1 - b0, 7), -1)
        blk[x[7]:x[7] + (y1 - y0)] = own
        if r > 0:
            yp0, yp1, _, _ = strips[r - 1]
            xp = xs[r - 1]
            assert xp[6] == x[1] and xp[4] == x[2]  # what each side sends is what the other receives
            prev_own = img[yp0:yp1]
            blk[0:x[2]] = prev_own[xp[3]:xp[3] + xp[4]]
        if r < world - 1:
            yn0, yn1, _, _ = strips[r + 1]
            xn = xs[r + 1]
            nxt_own = img[yn0:yn1]
            blk[x[5]:x[5] + x[6]] = nxt_own[xn[0]:xn[0] + xn[1]]
        assert np.array_equal(blk, img[b0:b1]), r
