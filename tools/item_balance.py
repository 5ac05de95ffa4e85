"""Load balance of the fused kernel's persistent CTAs (diagnostics).

Runs a workload, reads the per-super-tile busy cycles and the per-CTA busy
cycles (bsf_debug_item_cycles), and reports: the CTA imbalance (1 - mean/max
busy), the spread of item costs, and the makespan a greedy dynamic scheduler
would reach in the kernel's order (raster) versus cost-descending order
(LPT), simulated on the measured item costs."""
import argparse
import heapq
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402


def greedy(costs, nw):
    h = [0.0] * nw
    for c in costs:
        t = heapq.heappop(h)
        heapq.heappush(h, t + c)
    return max(h)


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
                basis=w.basis, max_sigma=w.max_sigma, anchor=bsf.BSF_ANCHOR_TILE)
img = synth.make_image(w, device=dev).contiguous()
cov = synth.make_cov(w, device=dev).contiguous()
out = torch.empty((1, w.height, w.width), dtype=torch.float64, device=dev)
plan.run(img, cov, out)
plan.phase_cycles(reset=True)
plan.run(img, cov, out)
torch.cuda.synchronize()
st = plan.geometry.super_tile
nitems = ((w.width + st - 1) // st) * ((w.height + st - 1) // st)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
items, work, ctas = plan.item_cycles(min(nitems, 8192), nsm)
work = np.array(work, dtype=np.float64)
items = np.array(items, dtype=np.float64)
ctas = np.array(ctas, dtype=np.float64)
print("workload %s %dx%d super-tile %d: %d items, %d CTAs" % (w.name, w.width, w.height, st, nitems, nsm))
print("CTA busy: mean %.4g max %.4g min %.4g -> imbalance 1-mean/max = %.1f %%" %
      (ctas.mean(), ctas.max(), ctas.min(), 100 * (1 - ctas.mean() / ctas.max())))
print("item cycles: mean %.4g min %.4g max %.4g cv %.2f" % (items.mean(), items.min(), items.max(),
                                                            items.std() / items.mean()))
nx = (w.width + st - 1) // st
grid = items[: (len(items) // nx) * nx].reshape(-1, nx)
print("item cost by super-tile row (mean, first 8 rows):", np.round(grid.mean(1)[:8] / items.mean(), 2))
print("item cost by super-tile col (mean, first 8 cols):", np.round(grid.mean(0)[:8] / items.mean(), 2))
lb = items.sum() / nsm
print("simulated makespan / lower bound: raster %.4f, LPT %.4f, reverse-LPT %.4f" % (
    greedy(items, nsm) / lb, greedy(np.sort(items)[::-1], nsm) / lb, greedy(np.sort(items), nsm) / lb))
macs, fb, halo, planes = work[:, 0], work[:, 1], work[:, 2], work[:, 3]


def fit(cols, names):
    A = np.stack(cols + [np.ones_like(macs)], 1)
    coef, *_ = np.linalg.lstsq(A, items, rcond=None)
    pred = A @ coef
    r2 = 1 - ((items - pred) ** 2).sum() / ((items - items.mean()) ** 2).sum()
    print("fit cycles = " + " + ".join("%.3g*%s" % (c, n) for c, n in zip(coef, names + ["1"])) +
          ": R^2 %.3f; ordering by it: makespan/LB %.4f" % (r2, greedy(items[np.argsort(-pred)], nsm) / lb))


fit([macs], ["MACs"])
fit([macs, fb], ["MACs", "fallbacks"])
fit([macs, halo * planes], ["MACs", "halo*planes"])
fit([macs, halo, halo * planes], ["MACs", "halo", "halo*planes"])
print("fallback pixels: %d in %d items; cycles of those items %.1f %% of total" % (
    fb.sum(), (fb > 0).sum(), 100 * items[fb > 0].sum() / items.sum()))
