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
@pytest.mark.parametrize("order,policy", [(2, bsf.BSF_DUAL), (3, bsf.BSF_THETA)])
def test_strips_bitwise_equal_single_gpu(world, order, policy):
    H, W, smax = 352, 200, 5.0
    w = synth.workload(5, width=W, height=H, max_sigma=smax, order=order)
    img = synth.make_image(w).cuda()
    cov = _field(H, W, smax).cuda()

    def plan(height):
        return bsf.Plan(W, height, in_dtype=bsf.BSF_F32, order=order, basis=policy, max_sigma=smax,
                        anchor=bsf.BSF_ANCHOR_TILE)

    full = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    plan(H).run(img[None].contiguous(), cov.contiguous(), full)
    halo = PL.halo_rows(smax, order)
    for rank in range(world):
        st = PL.strip_plan(H, rank, world, halo)
        assert st.y0 % PL.TILE == 0 and st.b0 % PL.TILE == 0
        f_blk = img[st.b0:st.b1]                     # = exchange_halos(own rows)
        cov_blk = torch.ones((3, st.rows, W), dtype=torch.float32, device="cuda")
        cov_blk[:, st.out_slice] = cov[:, st.y0:st.y1]  # halo outputs are discarded
        out = torch.empty((1, st.rows, W), dtype=torch.float64, device="cuda")
        plan(st.rows).run(f_blk[None].contiguous(), cov_blk.contiguous(), out)
        torch.cuda.synchronize()
        got = out[0, st.out_slice]
        ref = full[0, st.y0:st.y1]
        assert torch.equal(got, ref), (rank, float((got - ref).abs().max()))
