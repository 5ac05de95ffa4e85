// Per-pixel steps a1-a4 of the hot path, fused into the
// gather kernel: covariance decode, basis choice (Alg. 2), clamp, and the
// minimum-kurtosis scale solve on C/r.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

namespace bsf {

enum { BASIS_THETA = 0, BASIS_THETA_PRIME = 1, BASIS_DUAL = 2 };
enum { FLAG_RANGE = 1, FLAG_INFEASIBLE = 2, FLAG_TWO_ZERO = 4, FLAG_SOLVER = 8 };

// relative threshold under which a scale is treated as exactly zero (R5)
#define BSF_ZERO_REL 1e-5

struct PixelScales {
    int basis;     // chosen basis
    int clamped;   // elongation clamped
    int drop;      // direction with zero scale, or -1
    int flags;     // FLAG_*
    double ap[4];  // a'_k = a_k / h_k (scale in lattice steps)
};

// Elongation bounds as e = (rho-1)/(rho+1).
// Theta, Eq. (6) with t = |tan phi - cot phi|/2 = |cot 2phi|:
//   e = 1 / (|sin 2phi| + |cos 2phi|).
// Theta', feasibility of the PAPER.md:411-416 covariance with a_k^2 >= 0
// (R7): e |cos 2phi| <= 3/5 and e |sin 2phi| <= 4/5.
__device__ __forceinline__ void bounds_e(double phi, double *eT, double *eP) {
    double s2, c2;
    sincos(2.0 * phi, &s2, &c2);
    s2 = fabs(s2);
    c2 = fabs(c2);
    *eT = 1.0 / (s2 + c2);
    double b1 = c2 > 0.0 ? 0.6 / c2 : INFINITY;
    double b2 = s2 > 0.0 ? 0.8 / s2 : INFINITY;
    *eP = fmin(b1, b2);
}

// Minimum-kurtosis scales (R6):
// u = a^2 lies on a line u(t) through the covariance constraints; J(t), the
// squared Frobenius norm of sum_k u_k^2 n_k n_k^T, is a convex quartic.  We
// find the root of the cubic J'(t) on [lo, hi] by safeguarded Newton.
// Returns 0 or FLAG_INFEASIBLE / FLAG_SOLVER.
__device__ __forceinline__ int solve_scales(int basis, double C11, double C12, double C22, double u[4]) {
    double lo, hi;
    // per basis: J'(t) = 2 K11 K11' + 4 K12 K12' + 2 K22 K22'
    double A1 = 0, A3 = 0, B2 = 0, P = 0, Q = 0, D = 0;
    if (basis == BASIS_THETA) {
        // Eq. (4): u = (A1 - t/2, B2 + t/2, A3 - t/2, t/2 - B2)
        A1 = 12.0 * C11;
        A3 = 12.0 * C22;
        B2 = 12.0 * C12;
        lo = 2.0 * fabs(B2);
        hi = 2.0 * fmin(A1, A3);
    } else {
        // u = ((P+t)/2, (Q+D-t)/2, (Q-D+t)/2, (P-t)/2)
        P = 16.0 * C11 - 4.0 * C22;
        Q = 16.0 * C22 - 4.0 * C11;
        D = 30.0 * C12;
        lo = fmax(-P, D - Q);
        hi = fmin(P, D + Q);
    }
    if (lo > hi) {
        double scale = 60.0 * (fabs(C11) + fabs(C22));
        if (lo - hi > 1e-12 * scale) return FLAG_INFEASIBLE;
        lo = hi = 0.5 * (lo + hi);
    }
    auto dJ = [&](double t, double *d2, double *mag) -> double {
        double K11, K12, K22, k11, k12, k22;
        if (basis == BASIS_THETA) {
            double x1 = A1 - 0.5 * t, x3 = A3 - 0.5 * t;
            double common = B2 * B2 + 0.25 * t * t;
            K11 = x1 * x1 + common;
            K22 = x3 * x3 + common;
            K12 = B2 * t;
            k11 = t - A1;
            k22 = t - A3;
            k12 = B2;
        } else {
            double pp = P * P + t * t, qq = Q * Q + (D - t) * (D - t);
            K11 = (2.0 * pp + 0.5 * qq) * 0.2;
            K22 = (0.5 * pp + 2.0 * qq) * 0.2;
            K12 = 0.4 * (P * t + Q * (D - t));
            k11 = t - 0.2 * D;
            k22 = t - 0.8 * D;
            k12 = 0.4 * (P - Q);
        }
        *d2 = 2.0 * k11 * k11 + 2.0 * K11 + 4.0 * k12 * k12 + 2.0 * k22 * k22 + 2.0 * K22;
        // magnitude of the terms: |J'| below 16 u of it is rounding noise
        *mag = fabs(2.0 * K11 * k11) + fabs(4.0 * K12 * k12) + fabs(2.0 * K22 * k22);
        return 2.0 * K11 * k11 + 4.0 * K12 * k12 + 2.0 * K22 * k22;
    };
    double t, d2, mag;
    int flags = 0;
    if (lo == hi) {
        t = lo;
    } else if (dJ(lo, &d2, &mag) >= 0.0) {
        t = lo;
    } else if (dJ(hi, &d2, &mag) <= 0.0) {
        t = hi;
    } else {
        double a = lo, b = hi;
        t = 0.5 * (a + b);
        double tol = 4e-16 * fmax(fabs(lo), fabs(hi));
        int it = 0;
        for (; it < 100; ++it) {
            double g = dJ(t, &d2, &mag);
            // converged to the rounding noise of J' (a tighter step tolerance
            // alone would bisect down to it: ~50 steps instead of ~5)
            if (fabs(g) <= 16.0 * 1.1102230246251565e-16 * mag) break;
            if (g < 0.0)
                a = t;
            else
                b = t;
            double tn = t - g / d2;
            if (!(tn > a && tn < b)) tn = 0.5 * (a + b);
            if (fabs(tn - t) <= tol || b - a <= tol) {
                t = tn;
                break;
            }
            t = tn;
        }
        if (it == 100) flags |= FLAG_SOLVER;
    }
    if (basis == BASIS_THETA) {
        u[0] = A1 - 0.5 * t;
        u[1] = B2 + 0.5 * t;
        u[2] = A3 - 0.5 * t;
        u[3] = 0.5 * t - B2;
    } else {
        u[0] = 0.5 * (P + t);
        u[1] = 0.5 * (Q + D - t);
        u[2] = 0.5 * (Q - D + t);
        u[3] = 0.5 * (P - t);
    }
    return flags;
}

// BSF_COV_C11_C12_C22: the covariance planes decoded in fp64 to the
// (sigma_x >= sigma_y, theta) form of the sigma/theta layout: eigenvalues of
// [[C11, C12], [C12, C22]] and the angle of the top eigenvector,
// theta = atan2(2 C12, C11 - C22) / 2
__device__ __forceinline__ void cov_from_c(double c11, double c12, double c22, double &sx, double &sy, double &th) {
    const double m = 0.5 * (c11 + c22), d = hypot(0.5 * (c11 - c22), c12);
    sx = sqrt(fmax(m + d, 0.0));
    sy = sqrt(fmax(m - d, 0.0));
    th = 0.5 * atan2(2.0 * c12, c11 - c22);
    if (th < 0.0) th += M_PI;
}

// Steps a1-a4: sigma_x, sigma_y, theta -> basis, a'_k, zero-direction.
__device__ __forceinline__ void pixel_scales(double sx, double sy, double th, int policy, int clamp, int order,
                                             PixelScales &ps) {
    ps.flags = 0;
    ps.clamped = 0;
    ps.drop = -1;
    // orientation of the top eigenvector and elongation
    double phi = th, maj = sx, mn = sy;
    if (sx < sy) {
        phi = th + M_PI / 2;
        maj = sy;
        mn = sx;
    }
    phi = fmod(phi, M_PI);
    if (phi < 0) phi += M_PI;
    double rho = (maj / mn) * (maj / mn);
    double eT, eP;
    bounds_e(phi, &eT, &eP);
    int basis = policy;
    if (policy == BASIS_DUAL) basis = (sx == sy) ? BASIS_THETA : (eP > eT ? BASIS_THETA_PRIME : BASIS_THETA);
    ps.basis = basis;
    // C = R(theta) diag(sx^2, sy^2) R(theta)^T
    double c, s;
    sincos(th, &s, &c);
    double vx = sx * sx, vy = sy * sy;
    double C11 = vx * c * c + vy * s * s;
    double C12 = (vx - vy) * s * c;
    double C22 = vx * s * s + vy * c * c;
    if (sx != sy) {
        double eb = basis == BASIS_THETA ? eT : eP;
        if (eb < 1.0) {
            double rb = (1.0 + eb) / (1.0 - eb);
            if (!clamp) {
                if (rho > rb) ps.flags |= FLAG_INFEASIBLE;
            } else if (rho > 0.95 * rb) {
                // clamp: rho <- 0.95 rho_B at the same trace and orientation (R9)
                double lim = 0.95 * rb;
                double T = vx + vy;
                double e = (lim - 1.0) / (lim + 1.0);
                double l1 = 0.5 * T * (1.0 + e), l2 = 0.5 * T * (1.0 - e);
                double cp, sp;
                sincos(phi, &sp, &cp);
                C11 = l1 * cp * cp + l2 * sp * sp;
                C12 = (l1 - l2) * cp * sp;
                C22 = l1 * sp * sp + l2 * cp * cp;
                ps.clamped = 1;
            }
        }
    }
    if (ps.flags) return;
    double ir = 1.0 / order;
    double u[4];
    ps.flags |= solve_scales(basis, C11 * ir, C12 * ir, C22 * ir, u);
    if (ps.flags & FLAG_INFEASIBLE) return;
    // a'_k = a_k / h_k, h_k^2 = |s_k|^2: Theta (1, 2, 1, 2), Theta' (5, 5, 5, 5)
    double amax = 0.0;
    for (int k = 0; k < 4; ++k) {
        double h2 = basis == BASIS_THETA ? ((k & 1) ? 2.0 : 1.0) : 5.0;
        double uk = u[k] > 0.0 ? u[k] : 0.0;
        ps.ap[k] = sqrt(uk / h2);
        amax = fmax(amax, ps.ap[k]);
    }
    int nz = 0;
    for (int k = 0; k < 4; ++k)
        if (ps.ap[k] <= BSF_ZERO_REL * amax) {
            ps.drop = k;
            ps.ap[k] = 0.0;
            ++nz;
        }
    if (nz > 1) ps.flags |= FLAG_TWO_ZERO;
    // R17: put a'_k on the 2^-40 grid.  Then every tap displacement
    // (R/2 - j) a'_k s_k is a multiple of 2^-41 below 2^12 in magnitude, so
    // displacements, their sums, lattice bases and fractional offsets are
    // exact doubles.  Scale change <= 2^-41 (lattice units).
    for (int k = 0; k < 4; ++k) {
        ps.ap[k] = rint(ps.ap[k] * 0x1p40) * 0x1p-40;
        if (ps.ap[k] == 0.0 && k != ps.drop) ps.flags |= FLAG_TWO_ZERO;  // sigma below ~1e-12
    }
}

}  // namespace bsf
