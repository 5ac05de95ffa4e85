"""A/B of the running-sum strip kernels: TMA-fed rows vs the cp.async ring
(bsf_debug_option "scan_tma"), config 3, the global int64 and double-double
pre-integrations; checks the two give identical sums."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402

for r in (1, 2):
    w = synth.workload(3, order=r)
    plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8, order=r, basis=w.basis, max_sigma=w.max_sigma)
    f = synth.make_image(w, device="cuda")[None].contiguous()
    res = {}
    for name, fn, g in (("int64", plan.preintegrate_exact, plan.empty_g_exact()), ("dd", plan.preintegrate, plan.empty_g())):
        for tma in (0, 1):
            plan.debug_option("scan_tma", tma)
            for _ in range(3):
                fn(f, g)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                fn(f, g)
            b.record()
            torch.cuda.synchronize()
            res[(name, tma)] = (a.elapsed_time(b) / 10, g.clone())
        same = torch.equal(res[(name, 0)][1], res[(name, 1)][1])
        print("config 3 r=%d %s: cp.async %.3f ms, TMA %.3f ms, identical %s" % (
            r, name, res[(name, 0)][0], res[(name, 1)][0], same))
        res.clear()
