"""sha256 of the fused path's output on a few workloads (checks that a change
meant to be bit-neutral is: run before and after, compare the lines)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402

dev = torch.device("cuda:0")
for cfg, kw in ((2, {"width": 1024, "height": 1024}), (3, {"width": 1024, "height": 1024, "order": 2}),
                (3, {"width": 1024, "height": 1024, "order": 1}), (1, {"order": 2}),
                (4, {"width": 512, "height": 256})):
    w = synth.workload(cfg, **kw)
    plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8 if w.in_dtype == "u8" else bsf.BSF_F32, order=w.order,
                    basis=w.basis, max_sigma=w.max_sigma, anchor=bsf.BSF_ANCHOR_TILE)
    img = synth.make_image(w, device=dev).contiguous()
    cov = synth.make_cov(w, device=dev).contiguous()
    out = torch.empty((1, w.height, w.width), dtype=torch.float64, device=dev)
    plan.run(img, cov, out)
    torch.cuda.synchronize()
    st = plan.stats()
    print(w.name, w.order, hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16], st["macs"], st["double_double"])
