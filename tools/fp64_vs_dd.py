"""Config 2, tile anchor: fp64 vs double-double outputs (error distribution)."""
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synth
from paper_1109_5114_b200 import bsf
from gpu_util import make_plan, gpu_full
w = synth.workload(2)
img, cov = synth.make_image(w), synth.make_cov(w)
res = {}
for name, prec, anc in (('dd_tile', bsf.BSF_PREC_DD, 1), ('fp_tile', bsf.BSF_PREC_FP64, 1), ('fp_glob', bsf.BSF_PREC_FP64, 0)):
    plan = make_plan(w, precision=prec, anchor=anc)
    res[name] = gpu_full(plan, img, cov)[0].numpy()
e = np.abs(res['fp_tile'] - res['dd_tile']) / np.abs(res['dd_tile'])
eg = np.abs(res['fp_glob'] - res['dd_tile']) / np.abs(res['dd_tile'])
print('tile fp64 rel err: max %.2e  p99.9 %.2e  median %.2e' % (e.max(), np.quantile(e, 0.999), np.median(e)))
print('global fp64 rel err: max %.2e median %.2e' % (eg.max(), np.median(eg)))
for x0 in range(0, 1024, 128):
    blk = e[:, x0:x0 + 128]
    print('x %4d-%4d sigma %.1f-%.1f: max %.2e frac>1e-10 %.4f' % (x0, x0 + 127, 1 + 15 * x0 / 1023, 1 + 15 * (x0 + 127) / 1023,
          blk.max(), (blk > 1e-10).mean()))
np.save('gpurun_out/fp64_err_tile.npy', e.astype(np.float32))
