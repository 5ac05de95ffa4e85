"""A/B timing of the order-1 gather (bsf_filter_exact) on config 3 with a
bsf_debug_option toggled: CUDA events on the launching stream, L2 flushed
between reps.  Usage: python tools/gx1_ab.py --option gx1_dp4a --values 0 1"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--option", default="gx1_dp4a")
ap.add_argument("--values", type=float, nargs="+", default=[0, 1])
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
w = synth.workload(3, order=1)
dev = torch.device("cuda:0")
img = synth.make_image(w, device=dev)[None].contiguous()
cov = synth.make_cov(w, device=dev).contiguous()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {}
outs = {}
for v in args.values:
    plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8, order=1, basis=w.basis, max_sigma=w.max_sigma,
                    anchor=bsf.BSF_ANCHOR_AUTO)
    plan.debug_option(args.option, v)
    g = plan.empty_g_exact()
    out = torch.empty((1, w.height, w.width), dtype=torch.float64, device=dev)
    plan.preintegrate_exact(img, g)
    plan.filter_exact(g, cov, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.filter_exact(g, cov, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    res[v] = {"median_ms": ts[len(ts) // 2], "min_ms": ts[0]}
    outs[v] = out.clone()
same = all(torch.equal(outs[args.values[0]], o) for o in outs.values())
print(json.dumps({"option": args.option, "results": res, "bit_identical": same}))
