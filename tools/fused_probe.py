"""Run the fused product path on a (cropped) BASELINE workload: one warm-up
run, then timed runs (CUDA events).  For ncu captures of fused_kernel<R>:
ncu --set full -k regex:fused_kernel -s 1 -c 1 python tools/fused_probe.py ..."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--order", type=int, default=0)
ap.add_argument("--width", type=int, default=512)
ap.add_argument("--height", type=int, default=512)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--split", type=int, default=0, help="bsf_run_split with this many passes (order from --order)")
ap.add_argument("--anchor", default="tile", choices=["tile", "global", "auto"])
ap.add_argument("--opt", action="append", default=[], help="bsf_debug_option name=value (diagnostics)")
ap.add_argument("--super-tile", type=int, default=0, help="bsf_plan_desc.super_tile (0: the plan's choice)")
args = ap.parse_args()
kw = {"width": args.width, "height": args.height}
if args.order:
    kw["order"] = args.order
w = synth.workload(args.config, **kw)
dev = torch.device("cuda:0")
plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8 if w.in_dtype == "u8" else bsf.BSF_F32, order=w.order,
                basis=w.basis, max_sigma=w.max_sigma, super_tile=args.super_tile,
                anchor={"tile": bsf.BSF_ANCHOR_TILE, "global": bsf.BSF_ANCHOR_GLOBAL, "auto": bsf.BSF_ANCHOR_AUTO}[args.anchor])
for o in args.opt:
    k, v = o.split("=")
    plan.debug_option(k, float(v))
img = synth.make_image(w, device=dev).contiguous()
cov = synth.make_cov(w, device=dev).contiguous()
out = torch.empty((1, w.height, w.width), dtype=torch.float64, device=dev)
run = (lambda: plan.run_split(img, cov, out, args.split)) if args.split else (lambda: plan.run(img, cov, out))
run()
torch.cuda.synchronize()
plan.stats(reset=True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(args.reps):
    run()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / args.reps
st = plan.stats(reset=True)
npx = w.width * w.height
print("%s %dx%d r=%d%s %s(global_mode=%d): %.3f ms, %.3f Mpx/s, macs/px %.0f, dd fallback %d" % (
    w.name, w.width, w.height, w.order, " split n=%d" % args.split if args.split else "", args.anchor,
    plan.geometry.global_mode, ms, npx / ms / 1e3, st["macs"] / max(st["pixels"], 1), st["double_double"]))
