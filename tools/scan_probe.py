"""One bsf_preintegrate_exact (or dd with --dd) call on a config-3 image, for
ncu launch lists of the global scan kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 1
dd = "--dd" in sys.argv
w = synth.workload(3, order=r)
plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8, order=r, basis=w.basis, max_sigma=w.max_sigma)
f = synth.make_image(w, device="cuda").contiguous()
g = plan.empty_g() if dd else plan.empty_g_exact()
fn = plan.preintegrate if dd else plan.preintegrate_exact
fn(f, g)
torch.cuda.synchronize()
fn(f, g)
torch.cuda.synchronize()
print("ok")
