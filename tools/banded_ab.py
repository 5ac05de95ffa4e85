"""A/B of bsf_run in global mode on config 3 (order 1, inputs in HBM):
plan option global_banded 0 (all scans, then the gather) vs 1 (scans and
gather in row bands, overlapped).  CUDA events on the launching stream, L2
flushed between reps; outputs compared bit for bit.
Usage: python tools/banded_ab.py [--reps 10]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
w = synth.workload(3, order=1)
dev = torch.device("cuda:0")
img = synth.make_image(w, device=dev)[None].contiguous()
cov = synth.make_cov(w, device=dev).contiguous()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res, outs = {}, {}
for v in (0, 1, 0, 1):
    plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8, order=1, basis=w.basis, max_sigma=w.max_sigma,
                    anchor=bsf.BSF_ANCHOR_AUTO)
    plan.debug_option("global_banded", v)
    out = torch.empty((1, w.height, w.width), dtype=torch.float64, device=dev)
    for _ in range(3):
        plan.run(img, cov, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.run(img, cov, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res.setdefault(v, []).append(sum(ts) / len(ts))
    outs[v] = out.clone()
same = bool(torch.equal(outs[0].view(torch.int64), outs[1].view(torch.int64)))
print(json.dumps({"workload": w.name, "order": 1, "ms": {str(k): v for k, v in res.items()},
                  "bit_identical": same, "reps": args.reps}))
