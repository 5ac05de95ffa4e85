"""Exact piecewise-polynomial tables for the interpolation kernel of Eq. (11).

Product-side generator (offline precompute; the oracle never uses it).

Eq. (11) interpolates the running sum g4 with the box
spline beta'_b whose scales are the lattice step lengths, a piecewise
quadratic stored "in a look-up table".  For order r the
same construction uses the r-fold kernel (R4): the lattice box
spline M_Xi with direction multiset Xi = {s_1^r, s_2^r, s_3^r, s_4^r} (or with
one direction removed, for zero scales, R5), supported on
sum_k r[0, s_k] (uncentred: the s_k/2 shifts of Eq. (10) are absorbed, R3).

M_Xi is built exactly in rational arithmetic:
  base  M_{s_a, s_b} = 1/|det(s_a, s_b)| on the half-open parallelogram,
  step  M_{Xi + xi}(x) = int_0^1 M_Xi(x - t xi) dt.
Pieces are (i, j, rho): unit square (i, j) intersected with the cell rho of
the arrangement of knot lines n_k . x = c (c integer, n_k = perp(s_k)).  On a
piece M is one polynomial in the local coordinate phi = x - (i, j).

Output table per (basis, r, variant): for each region rho of the unit cell,
the window offsets d with M(phi - d) != 0 and the coefficients of
M(phi - d) as a polynomial in phi (expansion centre c_rho = 0).
Coefficients are stored as double-double (hi, lo) pairs.
"""
from __future__ import annotations

import itertools
import math
import os
import struct
import sys
from fractions import Fraction as Fr

STEPS = {
    0: [(1, 0), (1, 1), (0, 1), (-1, 1)],     # Theta
    1: [(2, 1), (1, 2), (-1, 2), (-2, 1)],    # Theta' (Table 1)
}

# ----------------------------------------------------------------------------
# bivariate polynomials: dict {(i, j): Fraction}
# ----------------------------------------------------------------------------


def padd(p, q, s=1):
    r = dict(p)
    for k, v in q.items():
        r[k] = r.get(k, 0) + s * v
        if r[k] == 0:
            del r[k]
    return r


def pmul(p, q):
    r = {}
    for (a, b), v in p.items():
        for (c, d), w in q.items():
            k = (a + c, b + d)
            r[k] = r.get(k, 0) + v * w
    return {k: v for k, v in r.items() if v != 0}


class Affine2:
    """phi -> (ax . phi + bx, ay . phi + by) as two linear polynomials."""


def lin(cx, cy, c0):
    p = {}
    if cx:
        p[(1, 0)] = Fr(cx)
    if cy:
        p[(0, 1)] = Fr(cy)
    if c0:
        p[(0, 0)] = Fr(c0)
    return p


def _mul_lin_int(A, a, b, c):
    """(a x + b y + c) * A for a dense integer array A[i, j] (x^i y^j)."""
    import numpy as np
    n = A.shape[0]
    R = np.zeros((n + 1, n + 1), dtype=object)
    if c:
        R[:n, :n] += A * c
    if a:
        R[1:, :n] += A * a
    if b:
        R[:n, 1:] += A * b
    return R


def _lcm(a, b):
    return a // math.gcd(a, b) * b


def compose(P, X, Y, cache=None):
    """P(X(phi), Y(phi)) for linear polynomials X, Y, exactly.

    Integer Horner on dense arrays: with X = Xh/dX, Y = Yh/dY (Xh, Yh integer
    linear forms) and C = den * P integer,
      dX^D dY^D den P(X, Y) = sum_i Xh^i dX^(D-i) dY^i T_i,
      T_i = dY^(D-i) Q_i(Y) = sum_j C_ij Yh^j dY^(D-i-j)."""
    if not P:
        return {}
    import numpy as np
    deg = max(i + j for i, j in P)
    den = 1
    for v in P.values():
        den = _lcm(den, Fr(v).denominator)

    def intlin(L):
        a, b, c = Fr(L.get((1, 0), 0)), Fr(L.get((0, 1), 0)), Fr(L.get((0, 0), 0))
        d = _lcm(_lcm(a.denominator, b.denominator), c.denominator)
        return int(a * d), int(b * d), int(c * d), d

    ax, bx, cx, dX = intlin(X)
    ay, by, cy, dY = intlin(Y)
    C = {k: int(Fr(v) * den) for k, v in P.items()}
    acc = None
    for i in range(deg, -1, -1):
        m = deg - i
        q = np.zeros((1, 1), dtype=object)
        q[0, 0] = C.get((i, m), 0)
        for j in range(m - 1, -1, -1):
            q = _mul_lin_int(q, ay, by, cy)
            q[0, 0] += C.get((i, j), 0) * dY ** (m - j)
        w = dX ** (deg - i) * dY ** i
        if acc is None:
            acc = q * w
        else:
            acc = _mul_lin_int(acc, ax, bx, cx)
            n = q.shape[0]
            acc[:n, :n] += q * w
    scale = den * dX ** deg * dY ** deg
    out = {}
    n = acc.shape[0]
    for i in range(n):
        for j in range(n - i):
            v = acc[i, j]
            if v != 0:
                out[(i, j)] = Fr(int(v), scale)
    return out


def peval(P, x, y):
    return sum(v * x**i * y**j for (i, j), v in P.items())


def antideriv_along(P, xi):
    """G with xi . grad G = P (a polynomial antiderivative along xi)."""
    ax, ay = xi
    # coordinates w, v with x = ax w (+ 0), y = v + ay w  when ax != 0,
    # or x = v + ax w, y = ay w when ay != 0.  d/dw = ax d/dx + ay d/dy.
    if ax != 0:
        # x = ax*w, y = v + ay*w  ->  w = x/ax, v = y - ay x/ax
        Pt = compose(P, lin(ax, 0, 0), lin(ay, 1, 0))  # P(ax w, ay w + v) in vars (w, v)
        Gt = {}
        for (i, j), c in Pt.items():
            Gt[(i + 1, j)] = Gt.get((i + 1, j), 0) + c / (i + 1)
        return compose(Gt, lin(Fr(1, ax), 0, 0), lin(Fr(-ay, ax), 1, 0))
    else:
        # y = ay*w, x = v  -> w = y/ay, v = x ; vars (w, v) -> P(v, ay w)
        Pt = compose(P, {(0, 1): Fr(1)}, lin(ay, 0, 0))
        Gt = {}
        for (i, j), c in Pt.items():
            Gt[(i + 1, j)] = Gt.get((i + 1, j), 0) + c / (i + 1)
        return compose(Gt, lin(0, Fr(1, ay), 0), lin(1, 0, 0))


# ----------------------------------------------------------------------------
# regions of the unit cell
# ----------------------------------------------------------------------------


def normals(basis):
    return [(-sy, sx) for sx, sy in STEPS[basis]]


def region_key(basis, x, y):
    return tuple(math.floor(nx * x + ny * y) for nx, ny in normals(basis))


_REG_CACHE = {}


def unit_regions(basis, n=400):
    """Distinct cells of the knot-line arrangement inside [0,1)^2, with a
    floating representative point (sample centroid) and a rational centre."""
    if (basis, n) in _REG_CACHE:
        return _REG_CACHE[(basis, n)]
    acc = {}
    for a in range(n):
        for b in range(n):
            x = (a + 0.5) / n
            y = (b + 0.5) / n
            k = region_key(basis, x, y)
            s = acc.setdefault(k, [0, 0.0, 0.0])
            s[0] += 1
            s[1] += x
            s[2] += y
    regs = []
    for k in sorted(acc):
        cnt, sx, sy = acc[k]
        cx, cy = sx / cnt, sy / cnt
        # generic interior point (off every crossing-order switch line)
        cx += 0.00131
        cy += 0.00071
        assert region_key(basis, cx, cy) == k
        # expansion centre: the cell origin, so that psi = phi is exact on the
        # GPU (fractional tap offsets are exact doubles, R17)
        rc = (Fr(0), Fr(0))
        regs.append({"key": k, "rep": (cx, cy), "centre": rc, "area": cnt / n / n})
    _REG_CACHE[(basis, n)] = regs
    return regs


# ----------------------------------------------------------------------------
# piecewise polynomials over pieces (i, j, region index)
# ----------------------------------------------------------------------------


class PPoly:
    def __init__(self, basis):
        self.basis = basis
        self.regs = unit_regions(basis)
        self.key2reg = {r["key"]: i for i, r in enumerate(self.regs)}
        self.pieces = {}  # (i, j, ridx) -> poly in local phi

    def locate(self, x, y):
        i, j = math.floor(x), math.floor(y)
        k = region_key(self.basis, x - i, y - j)
        return i, j, self.key2reg[k]


def base_parallelogram(basis, sa, sb):
    P = PPoly(basis)
    det = sa[0] * sb[1] - sa[1] * sb[0]
    val = Fr(1, abs(det))
    xs = [0, sa[0], sb[0], sa[0] + sb[0]]
    ys = [0, sa[1], sb[1], sa[1] + sb[1]]
    for i in range(min(xs) - 1, max(xs) + 1):
        for j in range(min(ys) - 1, max(ys) + 1):
            for ri, reg in enumerate(P.regs):
                x = i + reg["rep"][0]
                y = j + reg["rep"][1]
                # solve x = ta sa + tb sb
                ta = (x * sb[1] - y * sb[0]) / det
                tb = (sa[0] * y - sa[1] * x) / det
                if 0 < ta < 1 and 0 < tb < 1:
                    P.pieces[(i, j, ri)] = {(0, 0): val}
    return P


_W = {}  # worker globals (fork)


def _integrate_piece(key):
    P, xi, fams = _W["P"], _W["xi"], _W["fams"]
    Gcache = _W.setdefault("Gcache", {})
    i, j, ri = key
    reg = P.regs[ri]
    px, py = i + reg["rep"][0], j + reg["rep"][1]
    cuts = []  # (t, nvec, c)
    for nx, ny in fams:
        nd = nx * xi[0] + ny * xi[1]
        if nd == 0:
            continue
        v0 = nx * px + ny * py
        v1 = v0 - nd  # value at t = 1
        lo, hi = min(v0, v1), max(v0, v1)
        for c in range(math.ceil(lo), math.floor(hi) + 1):
            t = (v0 - c) / nd
            if 1e-12 < t < 1 - 1e-12:
                cuts.append((t, (nx, ny), c, nd))
    cuts.sort()
    bounds = [(0.0, None)] + [(t, (n, c, nd)) for t, n, c, nd in cuts] + [(1.0, None)]
    total = {}
    for m in range(len(bounds) - 1):
        ta, ba = bounds[m]
        tb, bb = bounds[m + 1]
        if tb - ta < 1e-9:
            raise RuntimeError("degenerate crossing order at a representative point")
        tm = 0.5 * (ta + tb)
        si, sj, sr = P.locate(px - tm * xi[0], py - tm * xi[1])
        src = P.pieces.get((si, sj, sr))
        if not src:
            continue
        # G: antiderivative of src (in its local coords) along xi
        gk = (si, sj, sr)
        if gk not in Gcache:
            Gcache[gk] = antideriv_along(src, xi)
        G = Gcache[gk]
        # int_{ta}^{tb} src(z - t xi) dt = G(z - ta xi) - G(z - tb xi)
        # with z = phi + (i - si, j - sj) in the source's local coords.
        dx, dy = i - si, j - sj

        def tpoly(b):
            if b is None:
                return None
            (nx, ny), c, nd = b
            # t(phi) = (n.(phi + (i,j)) - c) / nd
            return lin(Fr(nx, nd), Fr(ny, nd), Fr(nx * i + ny * j - c, nd))

        def at(tb_, tconst):
            if tb_ is None:
                X = lin(1, 0, dx - tconst * xi[0])
                Y = lin(0, 1, dy - tconst * xi[1])
            else:
                # phi + d - t(phi) xi
                X = padd(lin(1, 0, dx), {k: -xi[0] * v for k, v in tb_.items()})
                Y = padd(lin(0, 1, dy), {k: -xi[1] * v for k, v in tb_.items()})
            return compose(G, X, Y)

        Ga = at(tpoly(ba), Fr(0) if ba is None and m == 0 else None)
        Gb = at(tpoly(bb), Fr(1) if bb is None else None)
        total = padd(total, padd(Ga, Gb, -1))
    return key, total


def integrate_dir(P, xi, workers=None):
    """M'(x) = int_0^1 M(x - t xi) dt, piece by piece (pieces in parallel)."""
    basis = P.basis
    Q = PPoly(basis)
    Q.regs, Q.key2reg = P.regs, P.key2reg
    if not P.pieces:
        return Q
    I = [k[0] for k in P.pieces]
    J = [k[1] for k in P.pieces]
    i0, i1 = min(I) + min(0, xi[0]) - 1, max(I) + max(0, xi[0]) + 1
    j0, j1 = min(J) + min(0, xi[1]) - 1, max(J) + max(0, xi[1]) + 1
    # line families: knot lines n.x = c and unit-square boundaries x = c, y = c
    fams = []
    for nx, ny in normals(basis) + [(1, 0), (0, 1)]:
        if (nx, ny) not in fams and (-nx, -ny) not in fams:
            fams.append((nx, ny))
    keys = [(i, j, ri) for i in range(i0, i1 + 1) for j in range(j0, j1 + 1) for ri in range(len(P.regs))]
    _W.clear()
    _W.update(P=P, xi=xi, fams=fams)
    workers = workers or int(os.environ.get("BSF_LUT_WORKERS", "0")) or (os.cpu_count() or 1)
    if workers > 1 and len(keys) > 64:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(workers) as pool:
            results = pool.map(_integrate_piece, keys, chunksize=max(1, len(keys) // (8 * workers)))
    else:
        results = [_integrate_piece(k) for k in keys]
    for key, total in results:
        if total:
            Q.pieces[key] = total
    return Q


def box_spline(basis, r, drop=None):
    """M_Xi for Xi = each step repeated r times (minus direction `drop`)."""
    dirs = []
    for k, s in enumerate(STEPS[basis]):
        if k == drop:
            continue
        dirs += [s] * r
    # base on two non-parallel directions
    sa = dirs[0]
    b_idx = next(i for i, s in enumerate(dirs) if s[0] * sa[1] - s[1] * sa[0] != 0)
    sb = dirs[b_idx]
    rest = dirs[1:b_idx] + dirs[b_idx + 1:]
    P = base_parallelogram(basis, sa, sb)
    for xi in rest:
        P = integrate_dir(P, xi)
    return P


def shift_poly(P, cx, cy):
    """P(phi) -> polynomial in psi = phi - c."""
    return compose(P, lin(1, 0, cx), lin(0, 1, cy))


def to_dd(fr):
    hi = float(fr)
    lo = float(fr - Fr(hi))
    return hi, lo


def build_table(basis, r, drop=None):
    P = box_spline(basis, r, drop)
    deg = max(i + j for poly in P.pieces.values() for i, j in poly) if P.pieces else 0
    regs = P.regs
    table = []
    for ri, reg in enumerate(regs):
        cx, cy = reg["centre"]
        win = []
        for (i, j, pr), poly in sorted(P.pieces.items()):
            if pr != ri:
                continue
            # piece at integer part (i, j) = -d
            d = (-i, -j)
            win.append((d, shift_poly(poly, cx, cy)))
        table.append(win)
    return P, deg, table


def monomials(deg):
    """Monomial order used by the GPU Horner scheme: x-major, i desc."""
    return [(i, j) for i in range(deg, -1, -1) for j in range(deg - i, -1, -1)]


MAGIC = 0x4C465342  # 'BSFL'
VERSION = 2


def integer_table(table, nmon_list):
    """Common denominator L and integer numerators n = L * c of every
    coefficient of one variant (the GPU contracts with the integers exactly,
    DESIGN.md "Exact split contraction")."""
    L = 1
    for win in table:
        for _, poly in win:
            for v in poly.values():
                L = _lcm(L, Fr(v).denominator)
    return L


def write_bin(path, basis, r, variants):
    """variants: list of (drop, deg, table, regs).

    Version 2 layout (little endian): header MAGIC, 2, basis, r, nvar; nreg;
    4 knot-line normals; per region key[4] and centre[2]; per variant
    (drop, deg, nmon, nmax), L (uint64, common denominator), then per region
    count and per window slot (dx, dy) and nmon numerators n (float64, exact
    integers |n| < 2^53): coefficient = n / L.  When L or a numerator reaches
    2^53 (Theta' at r = 4) L is written as 0 and the slot holds nmon
    correctly rounded double-double pairs (hi, lo) instead."""
    regs = variants[0][3]
    out = bytearray()
    out += struct.pack("<IIIII", MAGIC, VERSION, basis, r, len(variants))
    nreg = len(regs)
    out += struct.pack("<I", nreg)
    nrm = normals(basis)
    for nx, ny in nrm:
        out += struct.pack("<ii", nx, ny)
    for reg in regs:
        out += struct.pack("<4i", *reg["key"])
        out += struct.pack("<dd", float(reg["centre"][0]), float(reg["centre"][1]))
    for drop, deg, table, _ in variants:
        mons = monomials(deg)
        nmax = max(len(w) for w in table)
        L = integer_table(table, len(mons))
        exact = L < 2**53 and all(abs(v * L) < 2**53 for win in table for _, poly in win for v in poly.values())
        out += struct.pack("<iiii", -1 if drop is None else drop, deg, len(mons), nmax)
        out += struct.pack("<Q", L if exact else 0)  # 0: coefficients stored as double-double pairs
        for win in table:
            out += struct.pack("<i", len(win))
            for slot in range(nmax):
                if slot < len(win):
                    (dx, dy), poly = win[slot]
                else:
                    (dx, dy), poly = (0, 0), {}
                out += struct.pack("<ii", dx, dy)
                for (i, j) in mons:
                    c = poly.get((i, j), Fr(0))
                    if exact:
                        n = c * L
                        assert n.denominator == 1
                        out += struct.pack("<d", float(n.numerator))
                    else:
                        out += struct.pack("<dd", *to_dd(c))
    with open(path, "wb") as fh:
        fh.write(out)


def upgrade_v1(path):
    """Rewrite a version-1 table (double-double coefficients) as version 2.

    Each coefficient is a rational with denominator < 2^50; it is recovered
    exactly from its 106-bit double-double value (continued fractions), and
    the recovered value is checked against the stored pair."""
    buf = open(path, "rb").read()
    off = 0

    def take(fmt):
        nonlocal off
        v = struct.unpack_from(fmt, buf, off)
        off += struct.calcsize(fmt)
        return v

    magic, ver, basis, r, nvar = take("<IIIII")
    assert magic == MAGIC and ver == 1, (path, ver)
    (nreg,) = take("<I")
    nrm = [take("<ii") for _ in range(4)]
    regs = []
    for _ in range(nreg):
        key = take("<4i")
        c = take("<dd")
        regs.append({"key": key, "centre": c})
    variants = []
    for _ in range(nvar):
        drop, deg, nmon, nmax = take("<iiii")
        mons = monomials(deg)
        assert len(mons) == nmon
        table = []
        for _ in range(nreg):
            (cnt,) = take("<i")
            win = []
            for s in range(nmax):
                d = take("<ii")
                vals = take("<%dd" % (2 * nmon))
                if s >= cnt:
                    continue
                poly = {}
                for m, (i, j) in enumerate(mons):
                    hi, lo = vals[2 * m], vals[2 * m + 1]
                    if hi == 0.0 and lo == 0.0:
                        continue
                    exact = Fr(hi) + Fr(lo)
                    f = exact.limit_denominator(2**50)
                    assert abs(f - exact) <= abs(exact) * Fr(1, 2**100), (path, f, exact)
                    assert to_dd(f) == (hi, lo), (path, f)
                    poly[(i, j)] = f
                win.append((d, poly))
            table.append(win)
        variants.append((None if drop < 0 else drop, deg, table, regs))
    assert off == len(buf)
    assert [tuple(v) for v in nrm] == [tuple(v) for v in normals(basis)]
    write_bin(path, basis, r, variants)


def generate(basis, r, outdir):
    variants = []
    for drop in [None, 0, 1, 2, 3]:
        P, deg, table = build_table(basis, r, drop)
        variants.append((drop, deg, table, P.regs))
    path = os.path.join(outdir, "bsf_lut_b%d_r%d.bin" % (basis, r))
    write_bin(path, basis, r, variants)
    return path, variants


if __name__ == "__main__":
    outdir = os.path.dirname(os.path.abspath(__file__))
    if sys.argv[1:2] == ["upgrade"]:
        for p in sys.argv[2:]:
            upgrade_v1(p)
            print("upgraded", p)
        sys.exit(0)
    orders = [int(a) for a in sys.argv[1:]] or [1, 2]
    for r in orders:
        for basis in (0, 1):
            import time
            t = time.time()
            path, v = generate(basis, r, outdir)
            print("%s  regions=%d  window=%s  deg=%s  %.1fs" % (
                os.path.basename(path), len(v[0][3]), [max(len(w) for w in t_[2]) for t_ in v],
                [t_[1] for t_ in v], time.time() - t))
