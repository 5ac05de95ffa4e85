"""Helpers shared by the GPU parity tests (not a test module)."""
from __future__ import annotations

import numpy as np
import torch

import oracle as O
import synth
from paper_1109_5114_b200 import bsf

DT = {"u8": bsf.BSF_U8, "f32": bsf.BSF_F32}


def make_plan(w: synth.Workload, *, policy=None, order=None, precision=bsf.BSF_PREC_DD, clamp=1, out_f32=False,
              margin_x=0, margin_y=0, batch=None, anchor=bsf.BSF_ANCHOR_GLOBAL, super_tile=0):
    return bsf.Plan(w.width, w.height, batch=batch or w.batch, channels=w.channels, in_dtype=DT[w.in_dtype],
                    out_dtype=bsf.BSF_F32 if out_f32 else bsf.BSF_F64, order=order or w.order,
                    basis=w.basis if policy is None else policy, max_sigma=w.max_sigma, margin_x=margin_x,
                    margin_y=margin_y, clamp=clamp, precision=precision, anchor=anchor, super_tile=super_tile)


def gpu_full(plan: bsf.Plan, img: torch.Tensor, cov: torch.Tensor, out_dtype=torch.float64) -> torch.Tensor:
    dev = torch.device("cuda:0")
    f = img.to(dev).contiguous()
    c = cov.to(dev).contiguous()
    d = plan.desc
    out = torch.empty((d.batch * d.channels, d.height, d.width), dtype=out_dtype, device=dev)
    plan.run(f, c, out)
    torch.cuda.synchronize()
    return out.cpu()


def gpu_points(plan: bsf.Plan, img: torch.Tensor, cov: torch.Tensor, pts: torch.Tensor) -> torch.Tensor:
    dev = torch.device("cuda:0")
    f = img.to(dev).contiguous()
    c = cov.to(dev).contiguous()
    g = plan.empty_g()
    plan.preintegrate(f, g)
    p = pts.to(dev).contiguous()
    out = torch.empty(pts.shape[0], dtype=torch.float64, device=dev)
    plan.filter_points(g, c, p, out)
    torch.cuda.synchronize()
    return out.cpu()


def tile_points(plan: bsf.Plan, img: torch.Tensor, cov: torch.Tensor, pts: torch.Tensor, aux=False):
    dev = torch.device("cuda:0")
    out = torch.empty(pts.shape[0], dtype=torch.float64, device=dev)
    ax = torch.empty(pts.shape[0] * 12, dtype=torch.float64, device=dev) if aux else None
    plan.run_points(img.to(dev).contiguous(), cov.to(dev).contiguous(), pts.to(dev).contiguous(), out, ax)
    torch.cuda.synchronize()
    return (out.cpu(), ax.cpu().view(-1, 12)) if aux else out.cpu()


def oracle_points(img: np.ndarray, cov: np.ndarray, xs, ys, *, policy, r, clamp=1, nthreads=0):
    """img (H, W) exactly as the GPU consumed it; cov (3, H, W) float32."""
    xs = np.asarray(xs)
    ys = np.asarray(ys)
    sx = cov[0, ys, xs].astype(np.float64)
    sy = cov[1, ys, xs].astype(np.float64)
    th = cov[2, ys, xs].astype(np.float64)
    out, bas, cl, sc = O.filter_points(img, xs, ys, sx, sy, th, policy=policy, r=r, clamp=clamp, nthreads=nthreads)
    return out, bas, cl, sc


def max_rel(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.maximum(np.abs(b), 1e-300)
    return float(np.max(np.abs(a - b) / den))
