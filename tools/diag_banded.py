import sys, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import synth
from paper_1109_5114_b200 import bsf
from gpu_util import gpu_full
for (W, H, B, C) in [(230, 301, 1, 1), (256, 301, 1, 1), (230, 301, 2, 2), (256, 301, 2, 2), (256, 300, 1, 1), (256, 64, 1, 1), (230, 40, 2, 1)]:
    w = synth.workload(3, width=W, height=H, extra={"grid_span": 1500})
    img = torch.stack([synth.make_image(w, frame=f, channel=c) for f in range(B) for c in range(C)])
    cov = torch.stack([synth.make_cov(w) for _ in range(B)]).contiguous()
    plan = bsf.Plan(W, H, batch=B, channels=C, in_dtype=bsf.BSF_U8, order=1, basis=2, max_sigma=w.max_sigma, anchor=bsf.BSF_ANCHOR_AUTO)
    dev = gpu_full(plan, img, cov)
    o_h = torch.full((B * C, H, W), float("nan"), dtype=torch.float64).pin_memory()
    plan.run_host(img.contiguous().pin_memory(), cov.contiguous().pin_memory(), o_h)
    torch.cuda.synchronize()
    bad = ~(o_h == dev)
    rows = bad.any(dim=2).nonzero()
    print(W, H, B, C, "equal" if not bad.any() else "DIFF", int(bad.sum()), rows[:5].tolist() if bad.any() else "", flush=True)
