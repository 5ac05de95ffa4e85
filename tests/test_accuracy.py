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


# ----------------------------------------------------------------------------
# Tables 3 and 4 and the remaining Table 2 columns,
# recomputed with the oracle in the continuous protocol (tools/accuracy_tables.py
# wrote tests/golden/accuracy_tables_recomputed.json calling only oracle/)
# ----------------------------------------------------------------------------
import json  # noqa: E402
import os  # noqa: E402
import sys  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools"))


def _golden_rows(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append(line.split())
    return rows


def _recomputed():
    return json.load(open(os.path.join(GOLD, "accuracy_tables_recomputed.json")))


def test_table3_sigma_fraction_sweep():
    """Table 3 in the continuous protocol, reading sigma^2 =
    fraction x bound (9) (R21): Algorithm 1 improves at every fraction, the
    improvement rises to a maximum in the 50-70 % range and decreases after it,
    with the 50 % value within one point of the maximum -- the paper's claim
    "the best results are obtained when sigma^2 is roughly 50 % of the bound"
    (PAPER.md:483-487).  The paper's values are lower at small fractions
    (3.5 vs ~16 % at 10 %): its protocol is not stated beyond "numerical
    integration" (its Table 2 columns (1,4,0) and (5,4,0) differ although the
    continuous error is scale-invariant), so the values are not pinned; the
    recomputation is (regression against the stored oracle run)."""
    import accuracy_tables as T
    e0, e1, basis = T.errors(5.0, 3.0, math.pi / 4, fracs=T.TABLE3_FRACS)
    imp = [100 * (e0 - e) / e0 for e in e1]
    paper = [float(v) for _, v in _golden_rows("table3_sigma_fraction.txt")]
    print("Table 3 improvement %:", ["%.1f" % v for v in imp], "paper:", paper)
    assert all(v > 0 for v in imp)
    k = int(np.argmax(imp))
    assert 0.5 <= T.TABLE3_FRACS[k] <= 0.7
    assert all(imp[i] < imp[i + 1] for i in range(k))
    assert all(imp[i] > imp[i + 1] for i in range(k, len(imp) - 1))
    assert imp[4] >= imp[k] - 1.0
    assert max(paper) == paper[4]  # the paper's maximum is at 50 %
    stored = _recomputed()["table3"]["improvement"]
    np.testing.assert_allclose(imp, stored, atol=0.06)


def test_table4_new_bound_row():
    """Table 4's new-bound row recomputed exactly (R7): the dual
    bound max(rho_Theta, rho_Theta') at each orientation.  It agrees where the
    Theta bound wins (0, 5, 40, 45 deg: inf, 13.6, 13.6, inf), is unbounded on
    Theta''s axis (atan 1/2 = 26.565 deg), and at 25 deg (29.05 vs 30.1); the
    paper's empirical values at 13.3-22.5 deg and 30 deg are not those of the
    P:413-416 covariance (B.4: 6.85 / 8.23 / 12.20 / 25.23 vs 8.2 / 9.5 / 10.8 /
    28.8), and its minimum is 6.171 at 16.85 deg (pinned in
    test_oracle_pins.test_dual_sector_switch_angles), not 8.2 at 13.3 deg."""
    paper = {float(d): (math.inf if v == "inf" else float(v)) for d, v in _golden_rows("table4_new_bound.txt")}
    ours = {}
    for d in paper:
        phi = math.radians(26.565051177 if d == 26.6 else d)
        ours[d] = max(O.bound_rho(O.THETA, phi), O.bound_rho(O.THETA_PRIME, phi))
    print("Table 4 new bound:", {d: "%.2f / %s" % (ours[d], paper[d]) for d in paper})
    for d in (0.0, 45.0, 26.6):
        assert ours[d] > 1e6 and math.isinf(paper[d])
    for d in (5.0, 40.0):
        assert round(ours[d], 1) == paper[d]
    assert abs(ours[25.0] - paper[25.0]) / paper[25.0] < 0.05
    for d in (20.0, 22.5, 25.0, 30.0):  # Theta' lifts the Theta bound there, as the paper says
        assert ours[d] > O.bound_rho(O.THETA, math.radians(d)) + 2
    stored = {r["deg"]: r["dual"] for r in _recomputed()["table4_new_bound"]}
    for d, v in stored.items():
        if v is not None and d != 26.6:
            assert round(ours[d], 2) == v


def test_table2_all_columns_recomputed():
    """Every column of Table 2 under the stated readings
    (s = sigma_major, rho = eigenvalue ratio, Algorithm 2's basis): Algorithm 1
    improves every column, the isotropic ones by 54.8 % (10.8 -> 4.9, pinned in
    test_oracle_pins), (5,4,0) matches the paper (pinned above); (1,4,0) equals
    (5,4,0) (the continuous error is scale-invariant; the paper's 19.1 -> 15.3
    differs from its own 18.7 -> 14.6 by its discretisation); the other three
    anisotropic columns are not reproduced under any reading tried (basis Theta
    or dual, rho as sigma or eigenvalue ratio: DESIGN.md R23) -- their stored
    oracle values are a regression pin only."""
    rec = _recomputed()["table2"]
    for r in rec:
        assert r["alg1"] < r["plain"], r
    iso = [r for r in rec if r["rho"] == 1]
    assert all(round(r["plain"], 1) == 10.8 and round(r["alg1"], 1) == 4.9 for r in iso)
    by = {(r["s"], r["rho"]): r for r in rec if r["theta"] == 0.0}
    assert abs(by[(1, 4)]["plain"] - by[(5, 4)]["plain"]) < 0.05 and abs(by[(1, 4)]["alg1"] - by[(5, 4)]["alg1"]) < 0.1
    # spot-recompute one anisotropic column from the oracle
    e0, e1, b = _errors(5.0, 5.0, math.pi / 2)
    r = [x for x in rec if x["rho"] == 5][0]
    assert abs(e0 - r["plain"]) < 0.01 and abs(e1 - r["alg1"]) < 0.01
