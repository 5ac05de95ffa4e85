"""CPU float64 oracle for the space-variant box-spline filter (TEST INFRASTRUCTURE).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl
reference`` leg may import this package.  The product path
(``paper_1109_5114_b200``) never imports it and shares no code with it.

The arithmetic lives in ``bsf_oracle.c`` (plain C, fp64, no fast-math); this
module is ctypes marshalling only.  See the C file header for what is computed
and which PAPER.md passages each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bsf_oracle.c")
_LIB = os.path.join(_HERE, "libbsf_oracle.so")

THETA, THETA_PRIME, DUAL = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (fp64, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d, i, p = ctypes.c_double, ctypes.c_int, ctypes.c_void_p
        L.or_bound_e.restype = d
        L.or_bound_e.argtypes = [i, d]
        L.or_eq6_rho.restype = d
        L.or_eq6_rho.argtypes = [d]
        L.or_select.restype = i
        L.or_select.argtypes = [i, d, d, d]
        L.or_decode.argtypes = [d, d, d, p]
        L.or_orient.argtypes = [d, d, d, p, p]
        L.or_pixel_cov.restype = i
        L.or_pixel_cov.argtypes = [i, i, d, d, d, p]
        L.or_cov_of_scales.argtypes = [i, p, p]
        L.or_solve_scales.restype = i
        L.or_solve_scales.argtypes = [i, p, p, p]
        L.or_family_J.restype = d
        L.or_family_J.argtypes = [i, p, d]
        L.or_family_range.restype = i
        L.or_family_range.argtypes = [i, p, p]
        L.or_beta_r1.restype = d
        L.or_beta_r1.argtypes = [i, p, d, d]
        L.or_beta.restype = d
        L.or_beta.argtypes = [i, i, p, d, d]
        L.or_beta_points.argtypes = [i, i, p, i, p, p, p, i]
        L.or_filter_points.restype = i
        L.or_filter_points.argtypes = [p, i, i, i, i, i, ctypes.c_long, i, i, i, i, i, i,
                                       p, p, p, p, p, p, p, p, p, i]
        L.or_preintegrate_u8.restype = i
        L.or_preintegrate_u8.argtypes = [p, i, i, i, i, i, i, p]
        L.or_steps.restype = i
        L.or_steps.argtypes = [i, p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --- basis geometry -----------------------------------------------------------

def steps(basis: int) -> np.ndarray:
    out = np.zeros(8, dtype=np.int32)
    lib().or_steps(basis, _ptr(out))
    return out.reshape(4, 2)


def bound_e(basis: int, phi: float) -> float:
    return lib().or_bound_e(basis, phi)


def bound_rho(basis: int, phi: float) -> float:
    e = bound_e(basis, phi)
    return np.inf if e >= 1 else (1 + e) / (1 - e)


def eq6_rho(phi: float) -> float:
    return lib().or_eq6_rho(phi)


def select(policy: int, sx: float, sy: float, th: float) -> int:
    return lib().or_select(policy, sx, sy, th)


def decode(sx: float, sy: float, th: float) -> np.ndarray:
    C = np.zeros(3)
    lib().or_decode(sx, sy, th, _ptr(C))
    return C


def orient(sx: float, sy: float, th: float):
    phi = np.zeros(1)
    rho = np.zeros(1)
    lib().or_orient(sx, sy, th, _ptr(phi), _ptr(rho))
    return float(phi[0]), float(rho[0])


def pixel_cov(basis: int, clamp: int, sx: float, sy: float, th: float):
    C = np.zeros(3)
    st = lib().or_pixel_cov(basis, clamp, sx, sy, th, _ptr(C))
    return st, C


def cov_of_scales(basis: int, a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    C = np.zeros(3)
    lib().or_cov_of_scales(basis, _ptr(a), _ptr(C))
    return C


def solve_scales(basis: int, C):
    C = np.ascontiguousarray(C, dtype=np.float64)
    a = np.zeros(4)
    t = np.zeros(1)
    st = lib().or_solve_scales(basis, _ptr(C), _ptr(a), _ptr(t))
    if st != 0:
        raise ValueError("infeasible covariance for basis %d: %r" % (basis, C))
    return a, float(t[0])


def family_J(basis: int, C, t: float) -> float:
    C = np.ascontiguousarray(C, dtype=np.float64)
    return lib().or_family_J(basis, _ptr(C), t)


def family_range(basis: int, C):
    C = np.ascontiguousarray(C, dtype=np.float64)
    lh = np.zeros(2)
    st = lib().or_family_range(basis, _ptr(C), _ptr(lh))
    return st, float(lh[0]), float(lh[1])


# --- kernel --------------------------------------------------------------------

def beta(basis: int, r: int, a, x, y, polygon: bool = True) -> np.ndarray:
    """Box spline beta^{(r)}_a at points (x, y) (arrays)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    x = np.ascontiguousarray(np.atleast_1d(x), dtype=np.float64)
    y = np.ascontiguousarray(np.atleast_1d(y), dtype=np.float64)
    x, y = np.broadcast_arrays(x, y)
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    out = np.zeros(x.shape)
    lib().or_beta_points(basis, r, _ptr(a), x.size, _ptr(x), _ptr(y), _ptr(out), 1 if polygon else 0)
    return out


def support_halfwidths(basis: int, r: int, a):
    s = steps(basis).astype(np.float64)
    u = s / np.linalg.norm(s, axis=1, keepdims=True)
    a = np.asarray(a, dtype=np.float64)
    return 0.5 * r * float(np.sum(a * np.abs(u[:, 0]))), 0.5 * r * float(np.sum(a * np.abs(u[:, 1])))


def reach(max_sigma: float, r: int) -> float:
    """Upper bound of the kernel support half-extent for any covariance with
    sigma_major <= max_sigma at order r (used by tests to choose margins)."""
    # support half-extent <= (r/2) sum_k a_k and sum_k a_k <= 2 sqrt(sum u_k)
    # with sum u_k <= 12 trace(C/r) (Theta) / 12 trace (Theta'); trace <= 2 s^2.
    return float(np.sqrt(r) * np.sqrt(12.0 * 2.0) * max_sigma) + 1.0


# --- filter --------------------------------------------------------------------

_DT = {np.dtype(np.uint8): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2}


def filter_points(img: np.ndarray, px, py, sx, sy, th, *, policy: int, r: int, clamp: int = 1,
                  full_shape=None, origin=(0, 0), nthreads: int = 0):
    """Direct-sum filter at pixels (px, py).

    ``img`` is a view of the full image (shape ``full_shape`` = (H, W)) whose
    top-left pixel is ``origin`` = (x0, y0) in full-image coordinates.  Each
    pixel's kernel support (clipped to the full image) must lie in the view.
    Returns (out, basis, clamped, scales[n,4]).
    """
    img = np.ascontiguousarray(img)
    if img.dtype not in _DT:
        raise TypeError(img.dtype)
    vh, vw = img.shape
    H, W = full_shape if full_shape is not None else img.shape
    px = np.ascontiguousarray(px, dtype=np.int32)
    py = np.ascontiguousarray(py, dtype=np.int32)
    n = px.size
    sx = np.ascontiguousarray(np.broadcast_to(np.asarray(sx, dtype=np.float64), (n,)))
    sy = np.ascontiguousarray(np.broadcast_to(np.asarray(sy, dtype=np.float64), (n,)))
    th = np.ascontiguousarray(np.broadcast_to(np.asarray(th, dtype=np.float64), (n,)))
    out = np.zeros(n)
    bas = np.zeros(n, dtype=np.int32)
    cl = np.zeros(n, dtype=np.int32)
    sc = np.zeros((n, 4))
    st = lib().or_filter_points(_ptr(img), _DT[img.dtype], int(origin[0]), int(origin[1]), vw, vh, vw, W, H,
                                policy, r, clamp, n, _ptr(px), _ptr(py), _ptr(sx), _ptr(sy), _ptr(th),
                                _ptr(out), _ptr(bas), _ptr(cl), _ptr(sc), nthreads)
    if st > 0:
        raise ValueError("%d point supports left the image view" % st)
    return out, bas, cl, sc


def preintegrate_u8(f: np.ndarray, basis: int, r: int, P: int, Pb: int) -> np.ndarray:
    """Exact uint64 (wrapping) running sums on the domain [-P, W+P) x [0, H+Pb)."""
    f = np.ascontiguousarray(f, dtype=np.uint8)
    H, W = f.shape
    g = np.zeros((H + Pb, W + 2 * P), dtype=np.uint64)
    st = lib().or_preintegrate_u8(_ptr(f), W, H, basis, r, P, Pb, _ptr(g))
    if st != 0:
        raise ValueError("bad basis")
    return g
