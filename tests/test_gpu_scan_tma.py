"""The TMA-fed running-sum strip kernel (bsf_scan.cuh scan_strip_tma_kernel)
against the cp.async one (bsf_debug_option "scan_tma" = 0): identical
pre-integrations, int64 bit for bit and double-double bit for bit (same
arithmetic order), on sizes whose rows do / do not meet TMA's 16-byte pitch
rule (the latter falls back per level), both bases, orders 1-3, two images.
Parity of either against the oracle is test_gpu_parity / test_gpu_global."""
import pytest
import torch

from paper_1109_5114_b200 import bsf

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("W,H", [(1024, 777), (1000, 333), (96, 64)])
@pytest.mark.parametrize("order", [1, 2, 3])
@pytest.mark.parametrize("dtype", [bsf.BSF_U8, bsf.BSF_F32])
def test_tma_scan_identical(W, H, order, dtype):
    torch.manual_seed(W + H + order)
    plan = bsf.Plan(W, H, batch=2, in_dtype=dtype, order=order, basis=bsf.BSF_DUAL, max_sigma=3.0)
    if dtype == bsf.BSF_U8:
        f = torch.randint(0, 256, (2, H, W), dtype=torch.uint8, device="cuda")
    else:
        f = torch.rand((2, H, W), dtype=torch.float32, device="cuda") * 255
    runs = [("dd", plan.preintegrate, plan.empty_g)]
    if dtype == bsf.BSF_U8 and plan.geometry.g_exact_bytes:
        runs.append(("int64", plan.preintegrate_exact, plan.empty_g_exact))
    try:
        for name, fn, mk in runs:
            out = []
            for tma in (0, 1):
                plan.debug_option("scan_tma", tma)
                g = mk()
                fn(f, g)
                torch.cuda.synchronize()
                out.append(g)
            assert torch.equal(out[0], out[1]), name
    finally:
        plan.debug_option("scan_tma", 1)
