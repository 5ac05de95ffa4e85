"""Calibrate the exact split contraction's a-posteriori bound (GPU).

For sampled pixels of a config, runs the fused path with the fallback
disabled (bsf_debug_option split_tol = inf) and the double-double tile kernel
(bsf_debug_option fused = 0),
and prints the true relative error of the split path against its bound
(aux[9]).  python tools/calib_split.py --config 2 [--order R] [--n 20000]"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--order", type=int, default=0)
ap.add_argument("--n", type=int, default=20000)
ap.add_argument("--child", default="")
ap.add_argument("--opt", action="append", default=[], help="bsf_debug_option name=value")
args = ap.parse_args()

if args.child:
    import numpy as np
    import torch
    import synth
    from paper_1109_5114_b200 import bsf
    w = synth.workload(args.config, order=args.order) if args.order else synth.workload(args.config)
    dev = torch.device("cuda:0")
    plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8 if w.in_dtype == "u8" else bsf.BSF_F32,
                    order=w.order, basis=w.basis, max_sigma=w.max_sigma, anchor=bsf.BSF_ANCHOR_TILE)
    for kv in args.opt:
        k, v = kv.split("=")
        plan.debug_option(k, float(v))
    img = synth.make_image(w, device=dev).contiguous()
    cov = synth.make_cov(w, device=dev).contiguous()
    pts = synth.sample_points(w, args.n, seed=21).to(dev).contiguous()
    out = torch.empty(args.n, dtype=torch.float64, device=dev)
    aux = torch.empty(args.n * 12, dtype=torch.float64, device=dev)
    plan.run_points(img[None], cov, pts, out, aux)
    torch.cuda.synchronize()
    np.savez(args.child, out=out.cpu().numpy(), aux=aux.cpu().view(-1, 12).numpy(), fused=plan.uses_fused())
    sys.exit(0)

import numpy as np  # noqa: E402
tag = "c%d_r%d" % (args.config, args.order)
f1, f2 = "/tmp/split_%s.npz" % tag, "/tmp/dd_%s.npz" % tag
base = [sys.executable, __file__, "--config", str(args.config), "--order", str(args.order), "--n", str(args.n)]
subprocess.check_call(base + ["--child", f1, "--opt", "split_tol=inf"])
subprocess.check_call(base + ["--child", f2, "--opt", "fused=0"])
a, b = np.load(f1), np.load(f2)
assert bool(a["fused"]) and not bool(b["fused"])
err = np.abs(a["out"] - b["out"]) / np.abs(b["out"])
bound = a["aux"][:, 9]
ok = np.isfinite(err) & np.isfinite(bound)
err, bound = err[ok], bound[ok]
res = {"config": args.config, "order": args.order, "n": int(ok.sum()),
       "true_err_max": float(err.max()), "true_err_p50": float(np.median(err)),
       "bound_p50": float(np.median(bound)), "bound_max": float(bound.max()),
       "ratio_max_true_over_bound": float(np.max(err / np.maximum(bound, 1e-300))),
       "frac_bound_gt": {t: float(np.mean(bound > float(t))) for t in ("1e-12", "1e-10", "1e-9", "1e-8", "1e-6")},
       "frac_true_gt_1e-10": float(np.mean(err > 1e-10))}
print(json.dumps(res))
