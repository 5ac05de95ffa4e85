"""One bench step of config 3 at a given order, for ncu captures: order 1 =
bsf_preintegrate_exact + bsf_filter_exact (global mode), orders 2-3 = bsf_run
(tile path), order 4 = bsf_run_tiles on bench.py's sample of anchoring tiles
(--r4-tiles, as bench.py).  --reps steps after one warm-up."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--order", type=int, default=1)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--r4-tiles", type=int, default=2368)
args = ap.parse_args()
w = synth.workload(3, order=args.order)
dev = torch.device("cuda:0")
plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8, order=w.order, basis=w.basis, max_sigma=w.max_sigma,
                anchor=bsf.BSF_ANCHOR_AUTO)
img = synth.make_image(w, device=dev)[None].contiguous()
cov = synth.make_cov(w, device=dev).contiguous()
out = torch.empty((1, w.height, w.width), dtype=torch.float64, device=dev)
g = plan.empty_g_exact() if plan.geometry.global_mode else None
tiles = None
if args.order == 4:
    from bench import _tile_sample  # the bench's order-4 sample (same launch)
    tiles = _tile_sample(w, plan.geometry.tile_unit, args.r4_tiles).to(dev)


def step():
    if g is not None:
        plan.preintegrate_exact(img, g)
        plan.filter_exact(g, cov, out)
    elif tiles is not None:
        plan.run_tiles(img, cov, out, tiles)
    else:
        plan.run(img, cov, out)


for _ in range(args.reps + 1):
    step()
torch.cuda.synchronize()
print("ok", w.name, "order", w.order, "global_mode", plan.geometry.global_mode, plan.stats())
