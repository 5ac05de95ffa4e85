"""Time the global pre-integration kernels alone (GPU): bsf_preintegrate_exact
(int64, u8 input) and bsf_preintegrate (double-double), with algorithmic HBM
bytes = read f once + write every basis' g once."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6542.4) if os.path.exists(
    "MEASURED_PEAKS.json") else 6542.4
for cfg, r in ((2, 2), (3, 1), (3, 2), (3, 4)):
    w = synth.workload(cfg, order=r)
    plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8 if w.in_dtype == "u8" else bsf.BSF_F32, order=r,
                    basis=w.basis, max_sigma=w.max_sigma)
    f = synth.make_image(w, device="cuda").contiguous()
    res = {"workload": w.name, "order": r}
    for name, fn, g, eb in (("dd", plan.preintegrate, plan.empty_g(), 16),
                            ("int64", plan.preintegrate_exact, plan.empty_g_exact() if w.in_dtype == "u8" else None,
                             8)):
        if g is None:
            continue
        for _ in range(2):
            fn(f, g)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            fn(f, g)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        geo = plan.geometry
        byts = f.numel() * f.element_size() + geo.nbases * geo.g_height * geo.g_width * eb
        res[name] = {"ms": round(ms, 4), "alg_bytes": byts, "gbs": round(byts / ms / 1e6, 1),
                     "frac_hbm": round(byts / ms / 1e6 / peak, 4)}
    print(json.dumps(res))
