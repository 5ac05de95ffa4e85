"""Multi-GPU partitioning: one process per GPU.

* Independent images / frames (config 4, and bench's weak scaling): each rank
  filters its own contiguous range of frames; no collective on the data path.
* One huge image (config 5): row strips.  The filtered value at p depends only
  on f inside p's kernel support (half-extent <= R_s = sigma_max sqrt(24 r)),
  so each rank receives the input rows [y0 - R_s, y0) and [y1, y1 + R_s) from
  its neighbours (one NCCL send/recv pair per neighbour) and runs the
  tile-anchored kernel on its block, computing its own rows only.  The
  exchange runs inside the library when the plan has a communicator
  (bsf_plan_desc.nccl_id, include/bsf.h), or here through torch.distributed
  (filter_strip).  Strip and halo boundaries are multiples
  of the super-tile (plan.geometry.super_tile rows) on which the fused kernel
  anchors its running sums -- every rank's plan is created with the full
  image's super_tile (bsf_plan_desc.super_tile), since the automatic choice
  depends on the image size --
  and the halo covers a super-tile's halo domain, so every kept super-tile
  sees exactly the data and domain it sees in a single-GPU run: the outputs
  are bit-identical (tests/test_gpu_strips.py).  No scan carries are
  exchanged (the tile path restarts its sums per super-tile).

Only plumbing lives here (partition arithmetic, halo exchange through
torch.distributed); the compute is the C-ABI library.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

TILE = 32  # the fused kernel's usual super-tile (plan.geometry.super_tile: 16, 32 or 64)


def shard_range(n: int, rank: int, world: int):
    """Contiguous balanced split of n units: [start, stop) for `rank`."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def halo_rows(max_sigma: float, order: int, tile: int = TILE) -> int:
    """Rows a super-tile's halo domain reaches beyond it (tap reach bound
    ceil(sigma_max sqrt(24 r)) + 1 plus the interpolation window, <= 6r + 2
    rows), rounded up to whole super-tiles of side `tile`: the value the
    library uses for multi-GPU plans (bsf_geometry.halo)."""
    rs = int(math.ceil(max_sigma * math.sqrt(24.0 * order))) + 1 + 6 * order + 4
    return tile * ((rs + tile - 1) // tile)


@dataclass
class Strip:
    rank: int
    world: int
    y0: int      # first output row of this rank
    y1: int      # one past the last output row
    b0: int      # first row of the local block (input incl. halo)
    b1: int      # one past the last row of the local block
    halo: int
    tile: int = TILE  # super-tile side the strips align to

    @property
    def rows(self):
        return self.b1 - self.b0

    @property
    def out_slice(self):
        """Rows of the local block that are this rank's outputs."""
        return slice(self.y0 - self.b0, self.y1 - self.b0)


def strip_plan(H: int, rank: int, world: int, halo: int, tile: int = TILE) -> Strip:
    """Row strips aligned to the super-tile grid (side `tile` = the plan's
    geometry.super_tile; every strip but the last has a multiple of it): the
    library's own partition (bsf_strip_rows, host arithmetic, no GPU)."""
    from . import bsf
    y0, y1, b0, b1 = bsf.strip_rows(H, tile, halo, rank, world)
    return Strip(rank, world, y0, y1, b0, b1, halo, tile)


def exchange_halos(own: torch.Tensor, strip: Strip, H: int, group=None) -> torch.Tensor:
    """Assemble the local block [b0, b1) from this rank's rows [y0, y1)
    (`own`, shape (..., y1 - y0, W)) and the neighbours' boundary rows, with
    point-to-point sends/receives (NCCL over NVLink for CUDA tensors, gloo on
    CPU).  Assumes every strip is at least `halo` rows tall (else a halo would
    span two neighbours)."""
    import torch.distributed as dist
    r, n = strip.rank, strip.world
    lead = own.shape[:-2]
    W = own.shape[-1]
    block = own.new_zeros(lead + (strip.rows, W))
    block[..., strip.out_slice, :] = own
    ops = []
    top = strip.y0 - strip.b0          # rows needed from rank - 1
    bot = strip.b1 - strip.y1          # rows needed from rank + 1
    if r > 0:
        prev = strip_plan(H, r - 1, n, strip.halo, strip.tile)
        send_up = prev.b1 - prev.y1    # rows rank-1 needs from me
        ops.append(dist.P2POp(dist.isend, own[..., :send_up, :].contiguous(), r - 1, group))
        recv_top = block.new_empty(lead + (top, W))
        ops.append(dist.P2POp(dist.irecv, recv_top, r - 1, group))
    if r < n - 1:
        nxt = strip_plan(H, r + 1, n, strip.halo, strip.tile)
        send_dn = nxt.y0 - nxt.b0      # rows rank+1 needs from me
        ops.append(dist.P2POp(dist.isend, own[..., own.shape[-2] - send_dn:, :].contiguous(), r + 1, group))
        recv_bot = block.new_empty(lead + (bot, W))
        ops.append(dist.P2POp(dist.irecv, recv_bot, r + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if r > 0:
        block[..., :top, :] = recv_top
    if r < n - 1:
        block[..., strip.rows - bot:, :] = recv_bot
    return block


def filter_strip(plan, f_own: torch.Tensor, cov_own: torch.Tensor, strip: Strip, H: int, group=None,
                 stream=None) -> torch.Tensor:
    """Filter this rank's strip of one image with the halo exchanged through
    torch.distributed (NCCL over NVLink for CUDA tensors, gloo on CPU), then
    the library on the block: `plan` is this rank's multi-GPU plan without a
    communicator (bsf.Plan(..., height=H, rank=, nranks=): its geometry is the
    strip), whose bsf_run takes the block of input rows and computes only the
    strip's own rows.  f_own (C, y1 - y0, W); cov_own (3, y1 - y0, W): this
    rank's rows only.  Returns (C, y1 - y0, W) float64.  (A plan WITH a
    communicator, nccl_id=bsf.get_unique_id() broadcast from rank 0, does the
    same exchange inside the library: plan.run(f_own, cov_own, out).)"""
    f_blk = exchange_halos(f_own, strip, H, group)
    out = torch.empty((f_own.shape[0] if f_own.dim() == 3 else 1, strip.y1 - strip.y0, f_own.shape[-1]),
                      dtype=torch.float64, device=f_own.device)
    plan.run(f_blk.contiguous(), cov_own.contiguous(), out, stream)
    return out


def strip_plan_of(plan) -> Strip:
    """The Strip of a multi-GPU bsf.Plan (its geometry)."""
    g, d = plan.geometry, plan.desc
    return Strip(d.rank, d.nranks, g.row0, g.row0 + g.row_count, g.block_row0, g.block_row0 + g.block_rows, g.halo,
                 g.super_tile)


# ---------------------------------------------------------------------------
# GLOBAL mode: the paper's single global pre-integration of
# one image sharded by row strips, with the scan carries passed down the rank
# chain.  Rank k owns domain rows [Y0, Y1) of the global g; after every
# running-sum level with a vertical step (sy >= 1) it sends its last sy rows
# of that level to rank k + 1, which starts the level's lines from them
# (bsf_scan_level's carry).  Horizontal levels need nothing.  The result is
# the single-GPU bsf_preintegrate_exact g, bit for bit.
# ---------------------------------------------------------------------------
@dataclass
class GlobalStrip:
    rank: int
    world: int
    Y0: int        # first global domain row of this rank
    Y1: int        # one past the last
    height: int    # image rows in the strip (plan height)
    margin_y: int  # plan margin_y: -1 (no bottom margin) except on the last rank


def global_strip(H: int, Pb: int, rank: int, world: int, unit: int = TILE) -> GlobalStrip:
    """Split the H image rows in multiples of `unit` (even: the Theta' steps
    have sy = 2); the last rank also owns the Pb margin rows of the domain."""
    n = (H + unit - 1) // unit
    t0, t1 = shard_range(n, rank, world)
    Y0, y1 = t0 * unit, min(H, t1 * unit)
    last = rank == world - 1
    return GlobalStrip(rank, world, Y0, y1 + (Pb if last else 0), y1 - Y0, Pb if last else -1)


def preintegrate_strip(plan, f, g, *, recv_carry, send_carry, exact=True, stream=None):
    """Run every level of every slot on this strip.

    plan: a bsf.Plan for the strip (height = image rows of the strip,
    margin_y as global_strip says); f the strip's image rows; g its running-sum
    buffer (int64 [nbases][nimg][rows][GW], or the float64 double-double
    buffer).  recv_carry(slot, level, sy) -> tensor [nimg][sy][GW](x2) or None
    (first rank); send_carry(slot, level, rows) is called with this strip's last
    sy rows of the level (skipped by the last rank)."""
    geo = plan.geometry
    nimg = plan.desc.batch * plan.desc.channels
    k = 1 if exact else 2
    gv = g.view(geo.nbases, nimg, geo.g_height, geo.g_width * k)
    for slot in range(geo.nbases):
        for level in range(4 * plan.desc.order):
            sx, sy = plan.scan_step(slot, level)
            carry = recv_carry(slot, level, sy) if sy > 0 else None
            plan.scan_level(slot, level, f, g, carry, exact=exact, stream=stream)
            if sy > 0:
                send_carry(slot, level, gv[slot, :, geo.g_height - sy:, :].clone())  # a copy: g is updated in place


def preintegrate_global_strips(plan, f, g, strip: GlobalStrip, *, exact=True, group=None, stream=None):
    """Multi-process GLOBAL-mode pre-integration: one rank per strip, carries
    by point-to-point send/recv (NCCL over NVLink for CUDA tensors, gloo on
    CPU).  Ranks form a chain, so there is no cycle and no deadlock."""
    import torch.distributed as dist
    geo = plan.geometry
    nimg = plan.desc.batch * plan.desc.channels
    k = 1 if exact else 2

    def recv_carry(slot, level, sy):
        if strip.rank == 0:
            return None
        buf = torch.empty((nimg, sy, geo.g_width * k), dtype=g.dtype, device=g.device)
        dist.recv(buf, strip.rank - 1, group=group)
        return buf

    def send_carry(slot, level, rows):
        if strip.rank < strip.world - 1:
            dist.send(rows, strip.rank + 1, group=group)

    preintegrate_strip(plan, f, g, recv_carry=recv_carry, send_carry=send_carry, exact=exact, stream=stream)
