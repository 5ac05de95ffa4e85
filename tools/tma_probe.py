"""Small check of the TMA-fed scans against the cp.async ones (one level set on
a small u8 image), synchronising after each call (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1109_5114_b200 import bsf  # noqa: E402

W, H = int(sys.argv[1]) if len(sys.argv) > 1 else 128, int(sys.argv[2]) if len(sys.argv) > 2 else 96
for basis in (0, 1):
    plan = bsf.Plan(W, H, in_dtype=bsf.BSF_U8, order=1, basis=basis, max_sigma=3.0)
    f = torch.randint(0, 256, (1, H, W), dtype=torch.uint8, device="cuda")
    out = {}
    for tma in (0, 1):
        plan.debug_option("scan_tma", tma)
        g = plan.empty_g_exact()
        plan.preintegrate_exact(f, g)
        torch.cuda.synchronize()
        out[tma] = g.clone()
        print("basis", basis, "tma", tma, "ok", flush=True)
    print("identical:", torch.equal(out[0], out[1]), flush=True)
