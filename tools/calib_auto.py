"""Calibrate the AUTO precision estimator: tile anchor, config 2, fp64 vs dd on
random points, with the fp64 path's cancellation ratios."""
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synth
from paper_1109_5114_b200 import bsf
from gpu_util import make_plan, tile_points
w = synth.workload(2)
img, cov = synth.make_image(w), synth.make_cov(w)
pts = synth.sample_points(w, 200000, seed=77)
p64 = make_plan(w, precision=bsf.BSF_PREC_FP64, anchor=1)
pdd = make_plan(w, precision=bsf.BSF_PREC_DD, anchor=1)
v64, a64 = tile_points(p64, img[None], cov, pts, aux=True)
vdd = tile_points(pdd, img[None], cov, pts)
err = (v64 - vdd).abs() / vdd.abs()
np.savez_compressed('gpurun_out/calib.npz', err=err.numpy(), aux=a64.numpy(), pts=pts.numpy())
print('done', float(err.max()))
