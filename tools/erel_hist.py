"""Distribution of the fused path's a-posteriori error bound (relative,
aux[9]) over sampled pixels of a workload, per basis: how much headroom the
split contraction has below the fallback threshold (5e-10)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--order", type=int, default=0)
ap.add_argument("--n", type=int, default=20000)
args = ap.parse_args()
kw = {"order": args.order} if args.order else {}
w = synth.workload(args.config, **kw)
plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8 if w.in_dtype == "u8" else bsf.BSF_F32, order=w.order,
                basis=w.basis, max_sigma=w.max_sigma, anchor=bsf.BSF_ANCHOR_TILE)
img = synth.make_image(w, device="cuda").contiguous()
cov = synth.make_cov(w, device="cuda").contiguous()
pts = synth.sample_points(w, args.n, seed=3).cuda().contiguous()
out = torch.empty(pts.shape[0], dtype=torch.float64, device="cuda")
aux = torch.empty(pts.shape[0] * 12, dtype=torch.float64, device="cuda")
plan.run_points(img[None], cov, pts, out, aux)
torch.cuda.synchronize()
ax = aux.view(-1, 12).cpu().numpy()
for b in (0, 1):
    e = ax[ax[:, 0] == b, 9]
    e = e[np.isfinite(e) & (e > 0)]
    if len(e) == 0:
        continue
    q = np.quantile(e, [0.5, 0.9, 0.99, 0.999, 1.0])
    print("%s basis %d: %d px, erel quantiles 50/90/99/99.9/max: %s" % (w.name, b, len(e), " ".join("%.2e" % v for v in q)))
    for thr in (1.7e-17, 1e-16, 1e-15, 1e-14):
        print("   fraction above %.1e: %.4f" % (thr, float((e > thr).mean())))
