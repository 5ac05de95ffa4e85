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
    for world in (1, 2, 4, 8):
        strips = [PL.strip_plan(H, r, world, halo) for r in range(world)]
        assert strips[0].y0 == 0 and strips[-1].y1 == H
        for s, t in zip(strips, strips[1:]):
            assert s.y1 == t.y0 and s.y0 % PL.TILE == 0 and t.y0 % PL.TILE == 0
        for s in strips:
            assert s.b0 == max(0, s.y0 - halo) and s.b1 == min(H, s.y1 + halo)


class _StandIn:
    """Stand-in for a bsf.Plan: 2R+1 box mean with zero extension (reach R)."""

    R = 3

    def __init__(self, height):
        self.height = height

    def run(self, f, cov, out, stream=None):
        k = 2 * self.R + 1
        x = f.to(torch.float64)[None, None]
        w = torch.ones(1, 1, k, k, dtype=torch.float64) / (k * k)
        out[0] = torch.nn.functional.conv2d(x, w, padding=self.R)[0, 0]


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
        res = PL.filter_strip(_StandIn, own, cov, st, H)
        q.put((rank, ok_blk, st.y0, st.y1, res))
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
    _StandIn(H).run(full, None, ref)
    for rank, ok_blk, y0, y1, res in got:
        assert ok_blk, rank
        assert torch.equal(res, ref[0, y0:y1]), rank
