"""Stratified pixel samples for parity at full config size (BASELINE.md "CPU
baseline plan": corners and edges, strip and frame boundaries, min and max
sigma, clamped and zero-scale pixels, dual-basis sector-switch angles, plus
uniform random pixels).  The strata that depend on the method (clamp,
zero-scale, sector) are classified with the ORACLE's own functions, so this
module is test infrastructure (it imports oracle/); the covariance is read
with synth.cov_at, bit-identical to the field the GPU consumes."""
from __future__ import annotations

import math

import numpy as np
import torch

import oracle as O
import synth

SWITCH = (math.atan(2 / 3) / 2, math.atan(4) / 2)  # dual-basis sector switches mod pi/4 (pinned in the oracle pins)


def _classify(c, policy, r):
    """Per pixel: (clamped, zero-scale, near a sector switch) by the oracle."""
    n = c.shape[1]
    clamped = np.zeros(n, bool)
    zero = np.zeros(n, bool)
    switch = np.zeros(n, bool)
    for i in range(n):
        sx, sy, th = (float(v) for v in c[:, i])
        b = O.select(policy, sx, sy, th)
        st, C = O.pixel_cov(b, 1, sx, sy, th)
        clamped[i] = st == 1
        try:
            a, _ = O.solve_scales(b, C / r)
            zero[i] = bool((a <= 1e-5 * a.max()).any())
        except ValueError:
            pass
        phi, _ = O.orient(sx, sy, th)
        m = phi % (math.pi / 4)
        switch[i] = min(abs(m - s) for s in SWITCH) < math.radians(0.5)
    return clamped, zero, switch


def stratified_points(w: synth.Workload, n: int, *, seed: int = 0, frames: int = 1, strip_rows=(), r=None,
                      policy=None, pool: int = 20000, per_stratum: int = 0, rows=None):
    """int32 (m, 3) (image, x, y) with m >= n points and a dict stratum ->
    indices.  `strip_rows`: row-strip boundaries (rows y0 - 1 and y0 are
    sampled); frames > 1: frame-edge pixels of the first and last frames;
    rows = (ya, yb): every point in those image rows (a row strip)."""
    r = r or w.order
    policy = w.basis if policy is None else policy
    ya, yb = rows if rows is not None else (0, w.height)
    H, W = yb - ya, w.width
    rng = np.random.default_rng(1000 + seed)
    k = per_stratum or max(4, n // 10)
    pts, labels = [], {}

    def add(name, img, xs, ys):  # ys relative to the first row ya
        idx = list(range(len(pts), len(pts) + len(xs)))
        pts.extend((int(img), int(x), int(y) + ya) for x, y in zip(xs, ys))
        labels.setdefault(name, []).extend(idx)

    cx = [0, W - 1, 0, W - 1, W // 2, 0, W - 1, W // 2, W // 2]
    cy = [0, 0, H - 1, H - 1, 0, H // 2, H // 2, H - 1, H // 2]
    add("corners_edges", 0, cx, cy)
    ex = rng.integers(0, W, k)
    add("edges", 0, np.concatenate([ex, ex, np.zeros(k, int), np.full(k, W - 1)])[:k],
        np.concatenate([np.zeros(k, int), np.full(k, H - 1), rng.integers(0, H, k), rng.integers(0, H, k)])[:k])
    for y0 in strip_rows:
        xs = rng.integers(0, W, k)
        add("strip_boundary", 0, np.concatenate([xs[: k // 2], xs[k // 2:]]),
            np.concatenate([np.full(k // 2, y0 - 1), np.full(k - k // 2, y0)]))
    if frames > 1:
        for f in (0, frames - 1):
            add("frame_edge", f, [0, W - 1, 0, W - 1], [0, 0, H - 1, H - 1])
    # method-dependent strata from a uniform candidate pool, classified by the oracle
    px = rng.integers(0, W, pool)
    py = rng.integers(0, H, pool)
    c = synth.cov_at(w, px, py + ya).numpy().astype(np.float64)
    clamped, zero, switch = _classify(c, policy, r)
    smaj = np.maximum(c[0], c[1])
    order = np.argsort(smaj)
    add("min_sigma", 0, px[order[:k]], py[order[:k]])
    add("max_sigma", 0, px[order[-k:]], py[order[-k:]])
    for name, m in (("clamped", clamped), ("zero_scale", zero), ("sector_switch", switch)):
        sel = np.nonzero(m)[0][:k]
        add(name, 0, px[sel], py[sel])
    nu = max(0, n - len(pts))
    ui = rng.integers(0, frames, nu) if frames > 1 else np.zeros(nu, int)
    base = len(pts)
    pts.extend((int(i), int(x), int(y) + ya) for i, x, y in zip(ui, rng.integers(0, W, nu), rng.integers(0, H, nu)))
    labels["uniform"] = list(range(base, len(pts)))
    return torch.tensor(pts, dtype=torch.int32), labels
