"""Fallback pixels per 64 x 64 super-tile against its scales (diagnostics).

Runs a workload with 64 x 64 super-tiles (raster work order) and relates each super-tile's double-double
fallback count (bsf_debug_item_cycles) to the conditioning proxy
(64 + 2 E) / sigma_min, E = sqrt(24 r) max sigma_major over the tile,
sigma_min the smallest minor standard deviation in the tile."""
import argparse
import math
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
ap.add_argument("--width", type=int, default=0)
ap.add_argument("--height", type=int, default=0)
args = ap.parse_args()
kw = {}
if args.width:
    kw["width"], kw["height"] = args.width, args.height
if args.order:
    kw["order"] = args.order
w = synth.workload(args.config, **kw)
dev = torch.device("cuda:0")
plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8 if w.in_dtype == "u8" else bsf.BSF_F32, order=w.order,
                basis=w.basis, max_sigma=w.max_sigma, anchor=bsf.BSF_ANCHOR_TILE, super_tile=64)
plan.debug_option("work_order", 0)
img = synth.make_image(w, device=dev).contiguous()
cov = synth.make_cov(w, device=dev).contiguous()
out = torch.empty((1, w.height, w.width), dtype=torch.float64, device=dev)
plan.phase_cycles(reset=True)
plan.run(img, cov, out)
torch.cuda.synchronize()
st = plan.geometry.super_tile
nx, ny = (w.width + st - 1) // st, (w.height + st - 1) // st
items, work, _ = plan.item_cycles(nx * ny, 0)
fb = np.array([x[1] for x in work], dtype=np.float64).reshape(ny, nx)
c = cov.cpu().numpy().astype(np.float64)
E = math.sqrt(24 * w.order)
rows = []
for ty in range(ny):
    for tx in range(nx):
        blk = c[:, ty * st:(ty + 1) * st, tx * st:(tx + 1) * st]
        smin, smaj = blk[1].min(), blk[0].max()
        rows.append(((st + 2 * E * smaj) / smin, smin, smaj, fb[ty, tx]))
rows = np.array(rows)
print("%s r=%d super-tile %d: %d tiles, fallback pixels %d" % (w.name, w.order, st, len(rows), rows[:, 3].sum()))
edges = np.quantile(rows[:, 0], np.linspace(0, 1, 11))
for lo, hi in zip(edges[:-1], edges[1:]):
    m = (rows[:, 0] >= lo) & (rows[:, 0] <= hi)
    print("cond %8.1f..%8.1f: %4d tiles, sigma_min %.2f..%.2f, fallback px/tile mean %.1f max %d" % (
        lo, hi, m.sum(), rows[m, 1].min(), rows[m, 1].max(), rows[m, 3].mean(), rows[m, 3].max()))
