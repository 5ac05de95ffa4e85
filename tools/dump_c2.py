"""Dump config-2 running sums (double-double, exact for this input) and the
GPU's per-pixel scales at sampled points, for offline precision experiments."""
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synth
from gpu_util import make_plan
w = synth.workload(2)
img, cov = synth.make_image(w), synth.make_cov(w)
plan = make_plan(w)
g = plan.empty_g(); plan.preintegrate(img.cuda(), g)
pts = synth.sample_points(w, 64, seed=5).cuda()
out = torch.empty(64, dtype=torch.float64, device='cuda'); aux = torch.empty(64 * 12, dtype=torch.float64, device='cuda')
plan.filter_points_aux(g, cov.cuda(), pts, out, aux); torch.cuda.synchronize()
geo = plan.geometry
np.savez_compressed('gpurun_out/c2_dump.npz', g=g.cpu().numpy().astype(np.float64), pts=pts.cpu().numpy(),
                    out=out.cpu().numpy(), aux=aux.cpu().numpy().reshape(64, 12), P=geo.margin_x, Pb=geo.margin_y,
                    GW=geo.g_width, GH=geo.g_height)
print('ok', geo.margin_x, geo.margin_y)
