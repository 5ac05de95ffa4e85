"""Small runs of every library path, for a build with the fused kernel's
operand bounds checks on (BSF_NVCC_EXTRA=-DBSF_CHECK_RANGE: every window read
outside its halo plane raises FLAG_RANGE in the plan's stats) — compute-
sanitizer is not available on the GPU pool: fused r = 1..3 (both super-tile
sizes, both boundaries), the global scans (int64, double-double) and gather,
splitting, the normalised variant, GLOBAL-mode strip levels.  Prints the OR
of the flags (0 = clean)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402

dev = torch.device("cuda:0")
flags = 0
for r in (1, 2, 3):
    for smax in (2.5, 14.0 if r == 1 else 2.5):
        w = synth.workload(3, width=70, height=52, order=r, max_sigma=smax)
        img = synth.make_image(w, device=dev)[None].contiguous()
        cov = synth.make_cov(w, device=dev)
        cov = torch.minimum(cov, torch.tensor([smax, smax, 10.0], device=dev)[:, None, None]).contiguous()
        for boundary in (0, 1):
            p = bsf.Plan(70, 52, in_dtype=bsf.BSF_U8, order=r, max_sigma=smax, anchor=bsf.BSF_ANCHOR_TILE,
                         boundary=boundary)
            out = torch.empty((1, 52, 70), dtype=torch.float64, device=dev)
            p.run(img, cov, out)
            flags |= p.stats(reset=True)["flags"]
        p.run_normalized(img, cov, out)
        if r <= 2:
            p.run_split(img, cov, out, 3)
        flags |= p.stats(reset=True)["flags"]
        pg = bsf.Plan(70, 52, in_dtype=bsf.BSF_U8, order=r, max_sigma=smax)
        g = pg.empty_g()
        pg.preintegrate(img, g)
        if r <= 2:
            pg.filter(g, cov, out)
        ge = pg.empty_g_exact()
        pg.preintegrate_exact(img, ge)
        ps = bsf.Plan(70, 32, in_dtype=bsf.BSF_U8, order=r, max_sigma=smax, margin_y=-1)
        gs = ps.empty_g_exact()
        carry = torch.zeros((1, 2, ps.geometry.g_width), dtype=torch.int64, device=dev)
        for lv in range(4 * r):
            ps.scan_level(0, lv, img[:, :32].contiguous(), gs, carry if lv else None)
torch.cuda.synchronize()
print("probe done, flags %d (FLAG_RANGE = 1)" % flags)
