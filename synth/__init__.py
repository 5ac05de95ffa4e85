"""Seeded synthetic inputs for the five BASELINE.json configurations.

This module holds NO arithmetic of the filter: it only draws images and
covariance fields (sigma_x, sigma_y, theta) with the shapes, value
distributions and structure of the configs.  Both the
CUDA path (tests, bench) and the oracle consume what it returns; for parity the
oracle always reads back the exact arrays the GPU consumed.

Randomness is a counter-based hash (SplitMix64 finaliser) of (seed, stream,
index), so any window of any config can be generated independently and the
same bits come out on CPU and GPU.  The paper uses no dataset (PAPER.md:536
ran an unspecified 256x256 image and impulse images); these stand in for it.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

MASK64 = (1 << 64) - 1


def _i64(c: int) -> int:
    c &= MASK64
    return c - (1 << 64) if c >= 1 << 63 else c


_G = _i64(0x9E3779B97F4A7C15)
_M1 = _i64(0xBF58476D1CE4E5B9)
_M2 = _i64(0x94D049BB133111EB)


def _srl(z: torch.Tensor, k: int) -> torch.Tensor:
    return (z >> k) & ((1 << (64 - k)) - 1)


def hash64(idx: torch.Tensor, seed: int, stream: int) -> torch.Tensor:
    z = idx.to(torch.int64) * _G + _i64((seed * 0x632BE59BD9B4E019 + stream * 0x85EBCA77C2B2AE63) & MASK64)
    z = (z ^ _srl(z, 30)) * _M1
    z = (z ^ _srl(z, 27)) * _M2
    return z ^ _srl(z, 31)


def uniform(idx, seed, stream, dtype=torch.float64):
    """U[0,1) with 53 (float64) or 24 (float32) random bits, exact in dtype."""
    h = hash64(idx, seed, stream)
    if dtype == torch.float32:
        return (_srl(h, 40).to(torch.float32)) * (2.0 ** -24)
    return (_srl(h, 11).to(torch.float64)) * (2.0 ** -53)


def uniform_u8(idx, seed, stream):
    return _srl(hash64(idx, seed, stream), 56).to(torch.uint8)


def normal(idx, seed, stream):
    """N(0,1) by Box-Muller on two hashed uniforms (float64)."""
    u1 = uniform(idx, seed, 2 * stream + 1001)
    u2 = uniform(idx, seed, 2 * stream + 1002)
    return torch.sqrt(-2.0 * torch.log1p(-u1)) * torch.cos(2 * math.pi * u2)


def _grid_idx(y0, y1, x0, x1, W, device):
    ys = torch.arange(y0, y1, device=device, dtype=torch.int64)
    xs = torch.arange(x0, x1, device=device, dtype=torch.int64)
    return ys[:, None] * W + xs[None, :], ys, xs


def _upsample(grid: torch.Tensor, n: int, ys: torch.Tensor, xs: torch.Tensor) -> torch.Tensor:
    """Bilinear, align-corners: grid node i sits at pixel i*(N-1)/(n-1)."""
    g = grid.shape[0]
    fy = ys.to(torch.float64) * (g - 1) / (n - 1)
    fx = xs.to(torch.float64) * (g - 1) / (n - 1)
    iy = torch.clamp(fy.floor().long(), max=g - 2)
    ix = torch.clamp(fx.floor().long(), max=g - 2)
    ty = (fy - iy)[:, None]
    tx = (fx - ix)[None, :]
    a = grid[iy][:, ix]
    b = grid[iy][:, ix + 1]
    c = grid[iy + 1][:, ix]
    d = grid[iy + 1][:, ix + 1]
    return (a * (1 - ty) * (1 - tx) + b * (1 - ty) * tx + c * ty * (1 - tx) + d * ty * tx)


@dataclass
class Workload:
    name: str
    width: int
    height: int
    batch: int
    channels: int
    in_dtype: str          # "u8" | "f32"
    order: int
    basis: int             # 0 Theta, 1 Theta', 2 dual
    max_sigma: float
    seed: int
    desc: str = ""
    extra: dict = field(default_factory=dict)


CONFIGS = {
    1: Workload("c1_128_u8_iso_r1", 128, 128, 1, 1, "u8", 1, 2, 3.0, 1,
                "128x128 u8 U{0..255}; sigma = 3 isotropic everywhere; order 1; f64 out"),
    2: Workload("c2_1024_f32_smooth_r2", 1024, 1024, 1, 1, "f32", 2, 2, 16.0, 2,
                "1024x1024 f32 U[0,1) + 8 rectangles; sigma_major 1..16 in x, ratio 1..4 in y, "
                "theta = atan2(y-512, x-512); order 2; dual basis"),
    3: Workload("c3_4096_u8_grid32", 4096, 4096, 1, 1, "u8", 1, 2, 40.0, 3,
                "4096x4096 u8 U{0..255}; sigma_major U[2,40], ratio U[1,6], theta U[0,pi) on a bilinearly "
                "upsampled 32x32 grid; orders 1..4"),
    4: Workload("c4_64x3x2048_f32_r3", 2048, 2048, 64, 3, "f32", 3, 2, 32.0, 4,
                "64 RGB frames 2048^2 f32 clip(N(0.5,0.15),0,1); config-2 field on 2048 scaled per frame by "
                "U[0.5,2]; order 3"),
    5: Workload("c5_32768_f32_grid256_r3", 32768, 32768, 1, 1, "f32", 3, 2, 64.0, 5,
                "32768^2 f32 U[0,1); sigma_major U[2,64], ratio U[1,6], theta U[0,pi) on a bilinearly "
                "upsampled 256x256 grid; order 3"),
}


def workload(cfg: int, **over) -> Workload:
    w = CONFIGS[cfg]
    d = dict(w.__dict__)
    d.update(over)
    return Workload(**d)


def make_image(w: Workload, frame: int = 0, channel: int = 0, window=None, device="cpu") -> torch.Tensor:
    """Image (H, W) or window (y0, y1, x0, x1) of frame/channel."""
    y0, y1, x0, x1 = window if window is not None else (0, w.height, 0, w.width)
    idx, ys, xs = _grid_idx(y0, y1, x0, x1, w.width, device)
    stream = 10 + 97 * frame + channel
    cfg = int(w.name[1])
    if w.in_dtype == "u8":
        return uniform_u8(idx, w.seed, stream)
    if cfg == 4:
        v = 0.5 + 0.15 * normal(idx, w.seed, stream)
        return v.clamp(0.0, 1.0).to(torch.float32)
    img = uniform(idx, w.seed, stream, torch.float32)
    if cfg == 2:
        # 8 random axis-aligned rectangles of constant intensity, painted in order
        k = torch.arange(8, dtype=torch.int64)
        r = lambda s: uniform(k, w.seed, 500 + s)  # noqa: E731
        rx0 = (r(0) * w.width).floor().long()
        ry0 = (r(1) * w.height).floor().long()
        rw = 16 + (r(2) * 241).floor().long()
        rh = 16 + (r(3) * 241).floor().long()
        val = r(4).to(torch.float32)
        for i in range(8):
            my = (ys >= ry0[i]) & (ys < ry0[i] + rh[i])
            mx = (xs >= rx0[i]) & (xs < rx0[i] + rw[i])
            m = my.to(device)[:, None] & mx.to(device)[None, :]
            img = torch.where(m, val[i].to(device), img)
    return img


def make_cov(w: Workload, frame: int = 0, window=None, device="cpu") -> torch.Tensor:
    """float32 planes (3, h, w): sigma_x, sigma_y, theta.  sigma_x is the major
    axis at angle theta; sigma_y = sigma_major / sqrt(ratio): "ratio" is read as
    the eigenvalue ratio (elongation; R13)."""
    y0, y1, x0, x1 = window if window is not None else (0, w.height, 0, w.width)
    ys = torch.arange(y0, y1, device=device, dtype=torch.int64)
    xs = torch.arange(x0, x1, device=device, dtype=torch.int64)
    cfg = int(w.name[1])
    H, W = w.height, w.width
    if cfg == 1 or w.extra.get("isotropic"):
        s = w.extra.get("sigma", 3.0)
        smaj = torch.full((len(ys), len(xs)), s, dtype=torch.float64, device=device)
        ratio = torch.ones_like(smaj)
        th = torch.zeros_like(smaj)
    elif cfg in (2, 4):
        scale = 1.0
        if cfg == 4:
            scale = 0.5 + 1.5 * float(uniform(torch.tensor([frame]), w.seed, 700)[0])
        X = xs.to(torch.float64)[None, :]
        Y = ys.to(torch.float64)[:, None]
        smaj = (1.0 + 15.0 * X / (W - 1)) * scale + 0 * Y
        ratio = 1.0 + 3.0 * Y / (H - 1) + 0 * X
        th = torch.remainder(torch.atan2(Y - H / 2, X - W / 2), math.pi)
    else:
        n = 32 if cfg == 3 else 256
        smax = 40.0 if cfg == 3 else 64.0
        gi = torch.arange(n * n, dtype=torch.int64)
        gs = (2.0 + (smax - 2.0) * uniform(gi, w.seed, 800)).view(n, n).to(device)
        gr = (1.0 + 5.0 * uniform(gi, w.seed, 801)).view(n, n).to(device)
        gt = (math.pi * uniform(gi, w.seed, 802)).view(n, n).to(device)
        if w.extra.get("grid_side"):
            # reduced-size analogue: same grid, mapped onto a smaller image
            pass
        smaj = _upsample(gs, w.extra.get("grid_span", max(H, W)), ys, xs)
        ratio = _upsample(gr, w.extra.get("grid_span", max(H, W)), ys, xs)
        th = _upsample(gt, w.extra.get("grid_span", max(H, W)), ys, xs)
    smin = smaj / torch.sqrt(ratio)
    return torch.stack([smaj, smin, th]).to(torch.float32)


def sample_points(w: Workload, n: int, seed: int = 0, frames: int = 1):
    """Stratified pixel sample: corners and edges, min/max sigma rows/cols,
    and uniform random pixels.  Returns int32 (n, 3): (image, x, y)."""
    H, W = w.height, w.width
    pts = []
    for (x, y) in ((0, 0), (W - 1, 0), (0, H - 1), (W - 1, H - 1), (W // 2, 0), (0, H // 2), (W - 1, H // 2),
                   (W // 2, H - 1), (W // 2, H // 2)):
        pts.append((0, x, y))
    k = torch.arange(4 * n, dtype=torch.int64)
    ux = uniform(k, 9000 + seed, 1)
    uy = uniform(k, 9000 + seed, 2)
    ui = uniform(k, 9000 + seed, 3)
    i = 0
    while len(pts) < n:
        img = int(ui[i] * frames) if frames > 1 else 0
        pts.append((img, int(ux[i] * W), int(uy[i] * H)))
        i += 1
    return torch.tensor(pts[:n], dtype=torch.int32)


def _upsample_pts(grid: torch.Tensor, n: int, ys: torch.Tensor, xs: torch.Tensor) -> torch.Tensor:
    """_upsample at scattered pixels (ys[i], xs[i]): the same arithmetic per
    element, so the values are bit-identical to the gridded version."""
    g = grid.shape[0]
    fy = ys.to(torch.float64) * (g - 1) / (n - 1)
    fx = xs.to(torch.float64) * (g - 1) / (n - 1)
    iy = torch.clamp(fy.floor().long(), max=g - 2)
    ix = torch.clamp(fx.floor().long(), max=g - 2)
    ty = fy - iy
    tx = fx - ix
    a = grid[iy, ix]
    b = grid[iy, ix + 1]
    c = grid[iy + 1, ix]
    d = grid[iy + 1, ix + 1]
    return (a * (1 - ty) * (1 - tx) + b * (1 - ty) * tx + c * ty * (1 - tx) + d * ty * tx)


def cov_at(w: Workload, xs, ys, frame: int = 0) -> torch.Tensor:
    """make_cov's float32 (sigma_x, sigma_y, theta) at scattered pixels:
    returns (3, n), bit-identical to make_cov(w)[:, ys, xs] without building
    the whole field (config 5 is 32768^2)."""
    xs = torch.as_tensor(xs, dtype=torch.int64)
    ys = torch.as_tensor(ys, dtype=torch.int64)
    cfg = int(w.name[1])
    H, W = w.height, w.width
    if cfg == 1 or w.extra.get("isotropic"):
        s = w.extra.get("sigma", 3.0)
        smaj = torch.full(xs.shape, s, dtype=torch.float64)
        ratio = torch.ones_like(smaj)
        th = torch.zeros_like(smaj)
    elif cfg in (2, 4):
        scale = 1.0
        if cfg == 4:
            scale = 0.5 + 1.5 * float(uniform(torch.tensor([frame]), w.seed, 700)[0])
        X = xs.to(torch.float64)
        Y = ys.to(torch.float64)
        smaj = (1.0 + 15.0 * X / (W - 1)) * scale + 0 * Y
        ratio = 1.0 + 3.0 * Y / (H - 1) + 0 * X
        th = torch.remainder(torch.atan2(Y - H / 2, X - W / 2), math.pi)
    else:
        n = 32 if cfg == 3 else 256
        smax = 40.0 if cfg == 3 else 64.0
        gi = torch.arange(n * n, dtype=torch.int64)
        gs = (2.0 + (smax - 2.0) * uniform(gi, w.seed, 800)).view(n, n)
        gr = (1.0 + 5.0 * uniform(gi, w.seed, 801)).view(n, n)
        gt = (math.pi * uniform(gi, w.seed, 802)).view(n, n)
        span = w.extra.get("grid_span", max(H, W))
        smaj = _upsample_pts(gs, span, ys, xs)
        ratio = _upsample_pts(gr, span, ys, xs)
        th = _upsample_pts(gt, span, ys, xs)
    smin = smaj / torch.sqrt(ratio)
    return torch.stack([smaj, smin, th]).to(torch.float32)


def image_at(w: Workload, xs, ys, frame: int = 0, channel: int = 0) -> torch.Tensor:
    """make_image's values at scattered pixels (configs 1, 3, 4, 5: per-pixel
    hashes; config 2's rectangles are painted by make_image only)."""
    xs = torch.as_tensor(xs, dtype=torch.int64)
    ys = torch.as_tensor(ys, dtype=torch.int64)
    idx = ys * w.width + xs
    stream = 10 + 97 * frame + channel
    cfg = int(w.name[1])
    if w.in_dtype == "u8":
        return uniform_u8(idx, w.seed, stream)
    if cfg == 4:
        return (0.5 + 0.15 * normal(idx, w.seed, stream)).clamp(0.0, 1.0).to(torch.float32)
    if cfg == 2:
        raise ValueError("config 2: use make_image")
    return uniform(idx, w.seed, stream, torch.float32)
