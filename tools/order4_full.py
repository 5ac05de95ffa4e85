"""Config 3 at order 4 over the WHOLE 4096^2 image (one bsf_run launch of the
double-double tile kernel; bench.py times 148 sampled tiles
only), timed with CUDA events, then >= 200 stratified pixels of that output
checked against the oracle (tests/strata.py strata; oracle on all host
cores).  Prints one JSON line.  GPU, ~35 min of kernel time + ~10 min of
oracle time on 16 cores."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import synth  # noqa: E402
from paper_1109_5114_b200 import bsf  # noqa: E402
from strata import stratified_points  # noqa: E402

npts = int(sys.argv[1]) if len(sys.argv) > 1 else 200
r = 4
dev = torch.device("cuda:0")
w = synth.workload(3, order=r)
img = synth.make_image(w, device=dev).contiguous()
cov = synth.make_cov(w, device=dev).contiguous()
plan = bsf.Plan(w.width, w.height, in_dtype=bsf.BSF_U8, order=r, basis=w.basis, max_sigma=w.max_sigma,
                anchor=bsf.BSF_ANCHOR_AUTO)
out = torch.full((1, w.height, w.width), float("nan"), dtype=torch.float64, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
plan.run(img[None], cov, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
st = plan.stats()
pts, labels = stratified_points(w, npts, seed=41, r=r)
xs, ys = pts[:, 1].numpy(), pts[:, 2].numpy()
got = out[0].cpu().numpy()[ys, xs]
c = synth.cov_at(w, xs, ys).numpy().astype(np.float64)
t0 = time.perf_counter()
ref = O.filter_points(img.cpu().numpy(), xs, ys, c[0], c[1], c[2], policy=w.basis, r=r,
                      full_shape=(w.height, w.width), origin=(0, 0))[0]
t_or = time.perf_counter() - t0
rel = np.abs(got - ref) / np.abs(ref)
print(json.dumps({
    "workload": w.name, "order": r, "kernel": "tile_kernel<4, dd> (whole image, one bsf_run)",
    "ms": ms, "mpx_s": w.width * w.height / (ms * 1e3), "stats": {k: int(v) for k, v in st.items()},
    "nan_pixels": int(torch.isnan(out).sum()),
    "parity": {"points": int(len(xs)), "max_rel": float(rel.max()), "tol": 1e-9,
               "per_stratum": {k: float(rel[v].max()) for k, v in labels.items() if len(v)},
               "oracle_s": t_or, "oracle_cores": os.cpu_count()}}))
