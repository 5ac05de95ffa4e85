"""the paper's accuracy experiments in its own
(continuous-domain) protocol, on CPU with the oracle's exact kernel
evaluator: the normalised L2 error ||beta - g|| / ||g|| against the Gaussian g
of the target covariance, the kernels sampled on a fine grid (pitch h) and
Algorithm 1's two-pass kernel formed as the convolution of its isotropic and
residual box splines (FFT on the same grid, times h^2).  Table 2 (PAPER.md:
456-472) for the size-5 anisotropic columns; the paper's numbers depend on
readings it does not state (basis policy, the rho = 8 column is beyond Theta's
bound at 60 deg), so the test checks its claim -- Algorithm 1 is more
accurate in every case -- and prints the table next to the paper's."""
import math

import numpy as np
import pytest

import oracle as O

PAPER = {(5, 4, 0.0): (18.7, 14.6), (5, 3, math.pi / 8): (23.9, 20.8), (5, 8, math.pi / 3): (19.2, 15.8),
         (5, 5, math.pi / 2): (17.2, 12.6)}


def _bound9(C, basis, phi):
    """Eq. (9): the largest s^2 with C - s^2 I inside the
    basis' elongation bound, with l1 >= l2 the eigenvalues of C."""
    tr, det = C[0] + C[2], C[0] * C[2] - C[1] ** 2
    disc = math.sqrt(max(tr * tr / 4 - det, 0.0))
    l1, l2 = tr / 2 + disc, tr / 2 - disc
    e = min(O.bound_e(basis, phi), 1.0)
    return 0.5 * (l1 + l2 - (l1 - l2) / e)


def _kernel(basis, C, X, Y):
    a, _ = O.solve_scales(basis, C)
    return O.beta(basis, 1, a, X.ravel(), Y.ravel()).reshape(X.shape)


def _errors(s, rho, th, h=0.1, L=22.0):
    sx, sy = s, s / math.sqrt(rho)
    basis = O.select(O.DUAL, sx, sy, th)
    st, C = O.pixel_cov(basis, 1, sx, sy, th)  # (clamped) covariance actually filtered with
    xs = np.arange(-L, L + h / 2, h)
    X, Y = np.meshgrid(xs, xs)
    Ci = np.linalg.inv(np.array([[C[0], C[1]], [C[1], C[2]]]))
    g = np.exp(-0.5 * (Ci[0, 0] * X * X + 2 * Ci[0, 1] * X * Y + Ci[1, 1] * Y * Y))
    g /= 2 * math.pi * math.sqrt(1.0 / np.linalg.det(Ci))
    err = lambda k: 100.0 * math.sqrt(((k - g) ** 2).sum() / (g ** 2).sum())  # noqa: E731
    plain = _kernel(basis, C, X, Y)
    phi, _ = O.orient(sx, sy, th)
    s2 = 0.5 * _bound9(C, basis, phi)  # Algorithm 1 step 1: half the bound (9)
    iso = _kernel(O.THETA, np.array([s2, 0.0, s2]), X, Y)
    res = _kernel(basis, np.array([C[0] - s2, C[1], C[2] - s2]), X, Y)
    from scipy.signal import fftconvolve
    alg1 = fftconvolve(iso, res, mode="same") * h * h  # both centred on the same odd grid
    return err(plain), err(alg1), basis


def test_table2_continuous_protocol():
    lines = []
    for (s, rho, th), (p0, p1) in PAPER.items():
        e0, e1, basis = _errors(s, rho, th)
        lines.append("(%g,%g,%.3f) basis %d: %.1f%% -> %.1f%% (paper %.1f -> %.1f)" % (s, rho, th, basis, e0, e1, p0, p1))
        assert e1 < e0, lines[-1]
    print("\n".join(lines))


def test_table2_column_5_4_0_reproduced():
    """The (s, rho, theta) = (5, 4, 0) column, where the readings are
    unambiguous (Theta at an axis, rho the eigenvalue ratio R13): the paper
    prints 18.7 % for the plain box spline and 14.6 % for Algorithm 1; the
    oracle's exact kernels, Eq. (9) and the two-pass composition give the same
    to the paper's rounding (a pin of Algorithm 1 beyond the isotropic case)."""
    e0, e1, basis = _errors(5.0, 4.0, 0.0)
    assert basis == O.THETA
    assert abs(e0 - 18.7) < 0.3 and abs(e1 - 14.6) < 0.3, (e0, e1)


@pytest.mark.parametrize("s", [1.0, 5.0])
def test_table2_isotropic_columns_algorithm1(s):
    """(s, 1, 0) columns: 10.8 % -> 4.9 %, here with
    Algorithm 1 composed explicitly (isotropic pass at half the bound, then the
    residual) rather than through the order-2 equivalence of R11."""
    h, L = (0.02, 6.0) if s < 2 else (0.1, 22.0)
    e0, e1, _ = _errors(s, 1.0, 0.0, h=h, L=L)
    assert round(e0, 1) == 10.8 and round(e1, 1) == 4.9, (e0, e1)
