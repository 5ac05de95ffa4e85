"""A/B of the order-3 exact limbs on tcgen05 kind::i8 (plan option "i8_tc")
against the DMMA path: config 3 at order 3 (whole 4096^2 image) and one
config-4 frame (3 channels of 2048^2 f32), CUDA events, one warm-up + one
timed run each, outputs compared."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402

dev = torch.device("cuda:0")
res = {}
for cfg in (3, 4):
    w = synth.workload(cfg, order=3) if cfg == 3 else synth.workload(4)
    C = w.channels if cfg == 4 else 1
    if cfg == 3:
        img = synth.make_image(w, device=dev)[None].contiguous()
        cov = synth.make_cov(w, device=dev).contiguous()
    else:
        img = torch.stack([synth.make_image(w, frame=0, channel=c, device=dev) for c in range(C)]).contiguous()
        cov = synth.make_cov(w, frame=0, device=dev)[None].contiguous()
    outs, t = {}, {}
    for i8 in (0, 1):
        plan = bsf.Plan(w.width, w.height, batch=1, channels=C,
                        in_dtype=bsf.BSF_U8 if w.in_dtype == "u8" else bsf.BSF_F32, order=3, basis=w.basis,
                        max_sigma=w.max_sigma, anchor=bsf.BSF_ANCHOR_AUTO)
        plan.debug_option("i8_tc", i8)
        out = torch.empty((C, w.height, w.width), dtype=torch.float64, device=dev)
        plan.run(img, cov, out)
        torch.cuda.synchronize()
        plan.stats(reset=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.run(img, cov, out)
        e1.record()
        torch.cuda.synchronize()
        t[i8] = e0.elapsed_time(e1)
        st = plan.stats()
        outs[i8] = out
        res["c%d_i8_%d" % (cfg, i8)] = {"ms": t[i8], "mpx_s": C * w.width * w.height / (t[i8] * 1e3),
                                        "double_double": st["double_double"], "status": st["status"]}
    rel = ((outs[0] - outs[1]).abs() / outs[0].abs()).max().item()
    res["c%d_max_rel_diff" % cfg] = rel
    res["c%d_speedup" % cfg] = t[0] / t[1]
    print(json.dumps(res), flush=True)
