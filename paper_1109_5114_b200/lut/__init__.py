"""Interpolation-kernel tables (see gen_lut.py for what they hold).

``path(basis, r)`` locates the binary table the C-ABI library loads;
``load(basis, r)`` parses it (used by tests and tooling only).
"""
from __future__ import annotations

import os
import struct

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def path(basis: int, r: int) -> str:
    return os.path.join(HERE, "bsf_lut_b%d_r%d.bin" % (basis, r))


def ensure(basis: int, r: int) -> str:
    p = path(basis, r)
    if not os.path.exists(p):
        from . import gen_lut
        gen_lut.generate(basis, r, HERE)
    return p


def _dd_of_ratio(n: np.ndarray, L: int):
    """Correctly rounded double-double of n / L (n exact integers in float64)."""
    from fractions import Fraction as Fr
    hi = n / float(L)
    lo = np.zeros_like(hi)
    for idx in zip(*np.nonzero(n)):
        lo[idx] = float(Fr(int(n[idx]), L) - Fr(float(hi[idx])))
    return hi, lo


def load(basis: int, r: int):
    """Parse a version-2 table: coefficients n / L with integer numerators."""
    with open(ensure(basis, r), "rb") as fh:
        buf = fh.read()
    off = 0

    def take(fmt):
        nonlocal off
        v = struct.unpack_from(fmt, buf, off)
        off += struct.calcsize(fmt)
        return v

    magic, ver, b, rr, nvar = take("<IIIII")
    assert magic == 0x4C465342 and ver == 2 and b == basis and rr == r
    (nreg,) = take("<I")
    normals = [take("<ii") for _ in range(4)]
    keys, centres = [], []
    for _ in range(nreg):
        keys.append(take("<4i"))
        centres.append(take("<dd"))
    variants = []
    for _ in range(nvar):
        drop, deg, nmon, nmax = take("<iiii")
        (L,) = take("<Q")
        counts = np.zeros(nreg, dtype=np.int32)
        offs = np.zeros((nreg, nmax, 2), dtype=np.int32)
        num = np.zeros((nreg, nmax, nmon))
        coef = np.zeros((nreg, nmax, nmon, 2))
        for ri in range(nreg):
            (counts[ri],) = take("<i")
            for s in range(nmax):
                offs[ri, s] = take("<ii")
                if L:
                    num[ri, s] = np.array(take("<%dd" % nmon))
                else:  # double-double pairs (no exact integer form)
                    coef[ri, s] = np.array(take("<%dd" % (2 * nmon))).reshape(nmon, 2)
        if L:
            hi, lo = _dd_of_ratio(num, L)
            coef = np.stack([hi, lo], axis=-1)
        variants.append(dict(drop=drop, deg=deg, nmon=nmon, nmax=nmax, counts=counts, offs=offs, coef=coef,
                             num=num, L=L))
    return dict(basis=basis, r=r, normals=normals, keys=keys, centres=np.array(centres), variants=variants)


def monomials(deg: int):
    return [(i, j) for i in range(deg, -1, -1) for j in range(deg - i, -1, -1)]


def region_of(tab, x: float, y: float) -> int:
    """Region of phi = (x, y); points exactly on knot lines step into an
    adjacent region (the kernel is continuous there)."""
    import math
    e = 1e-12
    for dx, dy in ((0, 0), (e, 0.37 * e), (-e, 0.61 * e), (0.7 * e, -e), (-0.3 * e, -0.77 * e)):
        xx = min(max(x + dx, 0.0), 1 - 2**-53)
        yy = min(max(y + dy, 0.0), 1 - 2**-53)
        k = tuple(math.floor(nx * xx + ny * yy) for nx, ny in tab["normals"])
        if k in tab["keys"]:
            return tab["keys"].index(k)
    raise ValueError((x, y))


def eval_window(tab, variant: int, x: float, y: float):
    """(offsets, weights) of M(phi - d) at phi = (x, y) in [0,1)^2 (float64)."""
    v = tab["variants"][variant]
    ri = region_of(tab, x, y)
    cx, cy = tab["centres"][ri]
    mons = monomials(v["deg"])
    px, py = x - cx, y - cy
    mv = np.array([px**i * py**j for i, j in mons])
    n = v["counts"][ri]
    w = (v["coef"][ri, :n, :, 0] + v["coef"][ri, :n, :, 1]) @ mv
    return v["offs"][ri, :n], w
