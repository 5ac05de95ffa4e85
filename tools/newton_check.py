"""Scale-solve convergence check (CPU, diagnostics): the safeguarded Newton
iteration of bsf_pixel.cuh solve_scales, replicated in Python, with the two
stopping rules -- the round-1 step tolerance (4e-16 x the interval scale) and
the rounding-noise stop (|J'| <= 16 u x the magnitude of its terms) -- on
random covariances of the config-3 range; reports iteration counts and the
distance of each root from a 200-step bisection of the same J'."""
import math

import numpy as np

U = 1.1102230246251565e-16


def family(basis, C11, C12, C22):
    if basis == 0:
        A1, A3, B2 = 12 * C11, 12 * C22, 12 * C12
        lo, hi = 2 * abs(B2), 2 * min(A1, A3)
    else:
        P, Q, D = 16 * C11 - 4 * C22, 16 * C22 - 4 * C11, 30 * C12
        lo, hi = max(-P, D - Q), min(P, D + Q)

    def dJ(t):
        if basis == 0:
            x1, x3 = A1 - 0.5 * t, A3 - 0.5 * t
            com = B2 * B2 + 0.25 * t * t
            K11, K22, K12 = x1 * x1 + com, x3 * x3 + com, B2 * t
            k11, k22, k12 = t - A1, t - A3, B2
        else:
            pp, qq = P * P + t * t, Q * Q + (D - t) ** 2
            K11, K22, K12 = (2 * pp + 0.5 * qq) * 0.2, (0.5 * pp + 2 * qq) * 0.2, 0.4 * (P * t + Q * (D - t))
            k11, k22, k12 = t - 0.2 * D, t - 0.8 * D, 0.4 * (P - Q)
        d2 = 2 * k11 * k11 + 2 * K11 + 4 * k12 * k12 + 2 * k22 * k22 + 2 * K22
        mag = abs(2 * K11 * k11) + abs(4 * K12 * k12) + abs(2 * K22 * k22)
        return 2 * K11 * k11 + 4 * K12 * k12 + 2 * K22 * k22, d2, mag
    return lo, hi, dJ


def newton(lo, hi, dJ, noise_stop):
    a, b = lo, hi
    t = 0.5 * (a + b)
    tol = 4e-16 * max(abs(lo), abs(hi))
    for it in range(100):
        g, d2, mag = dJ(t)
        if (noise_stop and abs(g) <= 16 * U * mag) or g == 0:
            break
        if g < 0:
            a = t
        else:
            b = t
        tn = t - g / d2
        if not (a < tn < b):
            tn = 0.5 * (a + b)
        if abs(tn - t) <= tol or b - a <= tol:
            t = tn
            break
        t = tn
    return t, it + 1


def bisect(lo, hi, dJ):
    a, b = lo, hi
    for _ in range(200):
        m = 0.5 * (a + b)
        if m in (a, b):
            break
        if dJ(m)[0] < 0:
            a = m
        else:
            b = m
    return 0.5 * (a + b)


def main(n=100000, seed=7):
    rng = np.random.default_rng(seed)
    cases = []
    for trial in range(n):
        basis = trial % 2
        sx = rng.uniform(0.5, 40)
        sy = sx / math.sqrt(rng.uniform(1, 6))
        th = rng.uniform(0, math.pi)
        s, c = math.sin(th), math.cos(th)
        vx, vy = sx * sx, sy * sy
        lo, hi, dJ = family(basis, vx * c * c + vy * s * s, (vx - vy) * s * c, vx * s * s + vy * c * c)
        if lo < hi and dJ(lo)[0] < 0 < dJ(hi)[0]:
            cases.append((lo, hi, dJ))
    for name, ns in (("step tolerance", False), ("noise stop", True)):
        its, err = [], 0.0
        for lo, hi, dJ in cases:
            t, k = newton(lo, hi, dJ, ns)
            its.append(k)
            err = max(err, abs(t - bisect(lo, hi, dJ)) / max(abs(lo), abs(hi)))
        its = np.array(its)
        print("%-15s %d interior roots: iterations mean %.1f, p50/p90/max %s; max |t - t_bisect| / scale %.1e" % (
            name, len(cases), its.mean(), np.percentile(its, [50, 90, 100]).astype(int).tolist(), err))


if __name__ == "__main__":
    main()
