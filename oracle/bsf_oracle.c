/*
 * oracle/bsf_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU float64 implementation of what the
 * space-variant box-spline filter of Chaudhury & Sanyal (arXiv 1109.5114,
 * cited as PAPER.md:<line>) computes.  It shares NO code with the CUDA path
 * (paper_1109_5114_b200/csrc) and must only be used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
 *
 * What it computes:
 *   out(p) = sum_{q in image} f(q) * beta^{(r)}_{a(p)}(p - q)           (*)
 * i.e. the paper's space-variant filter applied to the
 * sampled image and evaluated at pixel centres, with the box spline of
 * Eq. (2) with N = 4 directions, each direction repeated r
 * times (north star "each direction repeated to the chosen order"), scales
 * a(p) from the minimum-kurtosis rule applied to
 * C(p)/r (Prop. 1).  Zero extension outside the image; no
 * renormalisation.  The O(1) algorithm (Alg. 3) computes
 * the same number in exact arithmetic; the oracle does NOT use it.
 *
 * Kernel evaluation: r = 1 by rectangle overlap (the box
 * spline is the overlap of two rotated rectangles); r >= 2 by exact nested
 * piecewise Gauss-Legendre integration of the convolution of the four r-fold
 * boxes (Eq. 2 written out).  Parity pins: tests/test_oracle_*.py.
 *
 * Compiled with -O2 -fno-fast-math -ffp-contract=off.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_THETA 0
#define OR_THETA_PRIME 1
#define OR_DUAL 2

/* ------------------------------------------------------------------------ */
/* Basis directions.                                                         */
/* Theta  = {0, 45, 90, 135 deg}, lattice steps 1, sqrt2. */
/* Theta' = {26.6, 63.4, 116.6, 153.4 deg}, tangents 1/2, 2, -2, -1/2         */
/* (PAPER.md:296-305); scale a1..a4 <-> steps (2,1),(1,2),(-1,2),(-2,1) by    */
/* Table 1 rows i = 1,2,4,8.                               */
/* ------------------------------------------------------------------------ */
static const int OR_STEP[2][4][2] = {
    {{1, 0}, {1, 1}, {0, 1}, {-1, 1}},
    {{2, 1}, {1, 2}, {-1, 2}, {-2, 1}},
};

static void or_unit_dirs(int basis, double u[4][2]) {
    for (int k = 0; k < 4; k++) {
        double sx = OR_STEP[basis][k][0], sy = OR_STEP[basis][k][1];
        double h = sqrt(sx * sx + sy * sy);
        u[k][0] = sx / h;
        u[k][1] = sy / h;
    }
}

int or_steps(int basis, int *out8) {
    if (basis != OR_THETA && basis != OR_THETA_PRIME) return -1;
    for (int k = 0; k < 4; k++) {
        out8[2 * k] = OR_STEP[basis][k][0];
        out8[2 * k + 1] = OR_STEP[basis][k][1];
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Covariance of the box spline as a function of u = a^2 (elementwise).      */
/* Theta : Eq. (4).                                        */
/* Theta': PAPER.md:411-416.                                                 */
/* Returned as (C11, C12, C22).                                              */
/* ------------------------------------------------------------------------ */
void or_cov_of_scales(int basis, const double *a, double *C) {
    double u1 = a[0] * a[0], u2 = a[1] * a[1], u3 = a[2] * a[2], u4 = a[3] * a[3];
    if (basis == OR_THETA) {
        C[0] = (2 * u1 + u2 + u4) / 24.0;
        C[1] = (u2 - u4) / 24.0;
        C[2] = (2 * u3 + u2 + u4) / 24.0;
    } else {
        C[0] = (4 * u1 + u2 + u3 + 4 * u4) / 60.0;
        C[1] = 2 * (u1 + u2 - u3 - u4) / 60.0;
        C[2] = (u1 + 4 * u2 + 4 * u3 + u4) / 60.0;
    }
}

/* Linear map u -> (C11, C12, C22) as a 3x4 matrix, read off the formulas. */
static void or_cov_matrix(int basis, double A[3][4]) {
    for (int k = 0; k < 4; k++) {
        double a[4] = {0, 0, 0, 0};
        a[k] = 1.0; /* u_k = 1 */
        double C[3];
        or_cov_of_scales(basis, a, C);
        for (int i = 0; i < 3; i++) A[i][k] = C[i];
    }
}

/* Kurtosis matrix with kappa dropped (PAPER.md:426-431 for Theta';      */
/* the Theta matrix by the same construction sum_k a_k^4 u_k u_k^T,      */
/* DESIGN.md reading R6).  Entries (K11, K12, K22) as functions of u.    */
static void or_kurt_of_u(int basis, const double *u, double *K) {
    double q1 = u[0] * u[0], q2 = u[1] * u[1], q3 = u[2] * u[2], q4 = u[3] * u[3];
    if (basis == OR_THETA_PRIME) {
        K[0] = (4 * q1 + q2 + q3 + 4 * q4) / 5.0;
        K[1] = 2 * (q1 + q2 - q3 - q4) / 5.0;
        K[2] = (q1 + 4 * q2 + 4 * q3 + q4) / 5.0;
    } else {
        K[0] = q1 + q2 / 2 + q4 / 2;
        K[1] = (q2 - q4) / 2;
        K[2] = q3 + q2 / 2 + q4 / 2;
    }
}

/* Frobenius norm^2 of the kurtosis matrix (off-diagonal counted twice). */
static double or_J(int basis, const double *u) {
    double K[3];
    or_kurt_of_u(basis, u, K);
    return K[0] * K[0] + 2 * K[1] * K[1] + K[2] * K[2];
}

/* dJ/dt along u(t) = up + t z, by the chain rule on the matrix entries. */
static double or_dJ(int basis, const double *u, const double *z) {
    /* dK/dt = sum_k (dK/du_k) z_k, dK/du_k = 2 u_k * coefficient. */
    double K[3];
    or_kurt_of_u(basis, u, K);
    double dK[3] = {0, 0, 0};
    for (int k = 0; k < 4; k++) {
        /* coefficient of q_k = u_k^2 in each entry: evaluate at unit q. */
        double uk[4] = {0, 0, 0, 0};
        uk[k] = 1.0;
        double Kk[3];
        or_kurt_of_u(basis, uk, Kk);
        for (int i = 0; i < 3; i++) dK[i] += Kk[i] * 2.0 * u[k] * z[k];
    }
    return 2 * (K[0] * dK[0] + 2 * K[1] * dK[1] + K[2] * dK[2]);
}

/* ------------------------------------------------------------------------ */
/* The one-parameter family of scale vectors with covariance C.             */
/* The map u -> C is 3x4 linear; we take a particular solution and the null */
/* vector by plain Gaussian elimination (no closed form retyped).           */
/* Returns 0 and fills up, z, [tlo, thi]; -1 if the family is empty         */
/* (C not reachable with u >= 0: infeasible).             */
/* ------------------------------------------------------------------------ */
int or_family(int basis, const double *C, double *up, double *z, double *tlo, double *thi) {
    double A[3][4];
    or_cov_matrix(basis, A);
    /* Solve with u4 as the free variable: A[:, :3] x = C - A[:,3] t.  */
    double M[3][5];
    for (int i = 0; i < 3; i++) {
        for (int k = 0; k < 4; k++) M[i][k] = A[i][k];
        M[i][4] = C[i];
    }
    /* Gauss-Jordan elimination with partial pivoting on the first 3 columns. */
    for (int c = 0; c < 3; c++) {
        int best = c;
        for (int r = c + 1; r < 3; r++)
            if (fabs(M[r][c]) > fabs(M[best][c])) best = r;
        if (best != c)
            for (int k = 0; k < 5; k++) {
                double t = M[c][k];
                M[c][k] = M[best][k];
                M[best][k] = t;
            }
        for (int r = 0; r < 3; r++) {
            if (r == c) continue;
            double f = M[r][c] / M[c][c];
            for (int k = c; k < 5; k++) M[r][k] -= f * M[c][k];
        }
    }
    /* x_c = (M[c][4] - M[c][3] * t) / M[c][c] for c < 3, x_3 = t.       */
    for (int c = 0; c < 3; c++) {
        up[c] = M[c][4] / M[c][c];
        z[c] = -M[c][3] / M[c][c];
    }
    up[3] = 0.0;
    z[3] = 1.0;
    double lo = -INFINITY, hi = INFINITY;
    for (int k = 0; k < 4; k++) {
        if (z[k] > 0) {
            double b = -up[k] / z[k];
            if (b > lo) lo = b;
        } else if (z[k] < 0) {
            double b = -up[k] / z[k];
            if (b < hi) hi = b;
        } else if (up[k] < 0) {
            *tlo = INFINITY;
            *thi = -INFINITY;
            return -2;
        }
    }
    *tlo = lo;
    *thi = hi;
    if (!(lo <= hi)) return -1;
    return 0;
}

/* Minimum-kurtosis scales for covariance C.
 * J(t) is convex (R6), so: endpoint if the derivative does not
 * change sign, else bisection on the sign of J'(t) to adjacent doubles.
 * Writes a[4] = sqrt(max(u,0)).  Returns 0, or -1 if infeasible.          */
int or_solve_scales(int basis, const double *C, double *a_out, double *t_out) {
    double up[4], z[4], lo, hi;
    int st = or_family(basis, C, up, z, &lo, &hi);
    if (st != 0) {
        /* exactly at the feasibility boundary the interval is a point; allow
           rounding-level slack there, otherwise infeasible. */
        double scale = 60.0 * (fabs(C[0]) + fabs(C[2])) + 1e-300;
        if (isfinite(lo) && isfinite(hi) && lo - hi <= 1e-12 * scale) {
            lo = hi = 0.5 * (lo + hi);
        } else {
            return -1;
        }
    }
    double u[4];
#define OR_U_AT(t)                                               \
    do {                                                         \
        for (int k_ = 0; k_ < 4; k_++) u[k_] = up[k_] + (t)*z[k_]; \
    } while (0)
    double ts;
    OR_U_AT(lo);
    double dlo = or_dJ(basis, u, z);
    OR_U_AT(hi);
    double dhi = or_dJ(basis, u, z);
    if (lo == hi || dlo >= 0) {
        ts = lo;
    } else if (dhi <= 0) {
        ts = hi;
    } else {
        double a = lo, b = hi;
        for (int it = 0; it < 2000; it++) {
            double m = 0.5 * (a + b);
            if (m <= a || m >= b) break;
            OR_U_AT(m);
            double dm = or_dJ(basis, u, z);
            if (dm > 0)
                b = m;
            else if (dm < 0)
                a = m;
            else {
                a = b = m;
                break;
            }
        }
        ts = 0.5 * (a + b);
    }
    OR_U_AT(ts);
#undef OR_U_AT
    for (int k = 0; k < 4; k++) a_out[k] = sqrt(u[k] > 0 ? u[k] : 0.0);
    if (t_out) *t_out = ts;
    return 0;
}

/* J at an arbitrary t of the family (for the dense-sweep optimality pin). */
double or_family_J(int basis, const double *C, double t) {
    double up[4], z[4], lo, hi, u[4];
    or_family(basis, C, up, z, &lo, &hi);
    for (int k = 0; k < 4; k++) u[k] = up[k] + t * z[k];
    return or_J(basis, u);
}

int or_family_range(int basis, const double *C, double *lohi) {
    double up[4], z[4];
    return or_family(basis, C, up, z, &lohi[0], &lohi[1]);
}

/* ------------------------------------------------------------------------ */
/* Covariance decode, orientation/elongation, bounds, selection, clamp.      */
/* ------------------------------------------------------------------------ */

/* C = R(theta) diag(sx^2, sy^2) R(theta)^T: the ellipse (sigma_x, sigma_y,  */
/* theta) of the covariance field (north star; shape parameters, Eq. (3),    */
/* PAPER.md:130-148).                                                        */
void or_decode(double sx, double sy, double th, double *C) {
    double c = cos(th), s = sin(th);
    double vx = sx * sx, vy = sy * sy;
    C[0] = vx * c * c + vy * s * s;
    C[1] = (vx - vy) * s * c;
    C[2] = vx * s * s + vy * c * c;
}

/* Orientation phi of the top eigenvector (in [0, pi)) and elongation rho =  */
/* lambda_max / lambda_min, taken from the input theta.       */
void or_orient(double sx, double sy, double th, double *phi, double *rho) {
    double p = th, maj = sx, mn = sy;
    if (sx < sy) {
        p = th + M_PI / 2;
        maj = sy;
        mn = sx;
    }
    p = fmod(p, M_PI);
    if (p < 0) p += M_PI;
    *phi = p;
    *rho = (maj / mn) * (maj / mn);
}

/* Elongation bound as e_B = (rho_B - 1)/(rho_B + 1).
 * Theta : Eq. (6), rewritten with t = |cot 2phi|:
 *         e = sqrt(1+t^2)/(1+t) = 1/(|sin 2phi| + |cos 2phi|).
 * Theta': the exact feasibility region of the P:411-416 covariance map with
 *         u >= 0 (R7): e|cos 2phi| <= 3/5 and e|sin 2phi| <= 4/5.
 * The Theta one is checked against Eq. (6) verbatim in the pins.           */
double or_bound_e(int basis, double phi) {
    double s2 = fabs(sin(2 * phi)), c2 = fabs(cos(2 * phi));
    if (basis == OR_THETA) return 1.0 / (s2 + c2);
    double b1 = c2 > 0 ? 0.6 / c2 : INFINITY;
    double b2 = s2 > 0 ? 0.8 / s2 : INFINITY;
    return b1 < b2 ? b1 : b2;
}

/* Eq. (6) exactly as printed: rho bound for Theta. */
double or_eq6_rho(double phi) {
    double t = fabs(tan(phi) - 1.0 / tan(phi)) / 2.0;
    double r = sqrt(1 + t * t);
    return (1 + t + r) / (1 + t - r);
}

/* Algorithm 2 sector choice (R8): Theta' iff its
 * bound at phi is strictly larger; isotropic pixels and ties go to Theta.  */
int or_select(int policy, double sx, double sy, double th) {
    if (policy != OR_DUAL) return policy;
    if (sx == sy) return OR_THETA;
    double phi, rho;
    or_orient(sx, sy, th, &phi, &rho);
    return or_bound_e(OR_THETA_PRIME, phi) > or_bound_e(OR_THETA, phi) ? OR_THETA_PRIME : OR_THETA;
}

/* Pixel covariance after basis choice and the clamp policy (R9):
 * rho <- min(rho, 0.95 rho_B(phi)) at the same trace and orientation.
 * Returns 0 ok, 1 ok-and-clamped, -1 infeasible (clamp = 0).             */
int or_pixel_cov(int basis, int clamp, double sx, double sy, double th, double *C) {
    or_decode(sx, sy, th, C);
    if (sx == sy) return 0;
    double phi, rho;
    or_orient(sx, sy, th, &phi, &rho);
    double eb = or_bound_e(basis, phi);
    if (eb >= 1.0) return 0; /* any elongation reachable */
    double rb = (1 + eb) / (1 - eb);
    if (!clamp) return rho <= rb ? 0 : -1;
    double lim = 0.95 * rb;
    if (rho <= lim) return 0;
    double T = sx * sx + sy * sy;
    double e = (lim - 1) / (lim + 1);
    double l1 = T * (1 + e) / 2, l2 = T * (1 - e) / 2;
    double c = cos(phi), s = sin(phi);
    C[0] = l1 * c * c + l2 * s * s;
    C[1] = (l1 - l2) * c * s;
    C[2] = l1 * s * s + l2 * c * c;
    return 1;
}

/* ------------------------------------------------------------------------ */
/* Box-spline kernel, order r = 1: overlap of two rectangles.                */
/* L1*L3 is the uniform density on R13 = {s u1 + t u3 : |s|<=a1/2, |t|<=a3/2}*/
/* (u1 _|_ u3), L2*L4 likewise on R24; beta(x) = |R13 n (x + R24)| / prod a. */
/* ------------------------------------------------------------------------ */
typedef struct {
    double x, y;
} or_pt;

/* Sutherland-Hodgman: clip polygon P (n vertices) by half-plane n.x <= c. */
static int or_clip(const or_pt *P, int n, double nx, double ny, double c, or_pt *Q) {
    int m = 0;
    for (int i = 0; i < n; i++) {
        or_pt A = P[i], B = P[(i + 1) % n];
        double fa = nx * A.x + ny * A.y - c, fb = nx * B.x + ny * B.y - c;
        if (fa <= 0) Q[m++] = A;
        if ((fa < 0 && fb > 0) || (fa > 0 && fb < 0)) {
            double t = fa / (fa - fb);
            Q[m].x = A.x + t * (B.x - A.x);
            Q[m].y = A.y + t * (B.y - A.y);
            m++;
        }
    }
    return m;
}

static double or_shoelace(const or_pt *P, int n) {
    double s = 0;
    for (int i = 0; i < n; i++) {
        or_pt A = P[i], B = P[(i + 1) % n];
        s += A.x * B.y - B.x * A.y;
    }
    return 0.5 * fabs(s);
}

/* length of segment [A,B] inside the convex rectangle {|v.e1|<=h1,|v.e2|<=h2} */
static double or_seg_in_rect(or_pt A, or_pt B, const double *e1, double h1, const double *e2, double h2) {
    double t0 = 0, t1 = 1;
    const double *es[2] = {e1, e2};
    double hs[2] = {h1, h2};
    for (int i = 0; i < 2; i++) {
        double pa = A.x * es[i][0] + A.y * es[i][1];
        double pb = B.x * es[i][0] + B.y * es[i][1];
        double d = pb - pa;
        /* -h <= pa + t d <= h */
        if (d == 0) {
            if (pa < -hs[i] || pa > hs[i]) return 0;
        } else {
            double ta = (-hs[i] - pa) / d, tb = (hs[i] - pa) / d;
            if (ta > tb) {
                double t = ta;
                ta = tb;
                tb = t;
            }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        }
    }
    if (t1 <= t0) return 0;
    double L = hypot(B.x - A.x, B.y - A.y);
    return (t1 - t0) * L;
}

double or_beta_r1(int basis, const double *a, double x, double y) {
    double u[4][2];
    or_unit_dirs(basis, u);
    int z13 = (a[0] == 0) + (a[2] == 0), z24 = (a[1] == 0) + (a[3] == 0);
    if (z13 + z24 > 1) return NAN; /* two zero scales: not supported */
    if (z13 == 0 && z24 == 0) {
        /* x + R24 as a polygon, clipped by the 4 half-planes of R13. */
        or_pt P[16], Q[16];
        int n = 0;
        double h2 = a[1] / 2, h4 = a[3] / 2;
        double sg[4][2] = {{-1, -1}, {1, -1}, {1, 1}, {-1, 1}};
        for (int i = 0; i < 4; i++) {
            P[n].x = x + sg[i][0] * h2 * u[1][0] + sg[i][1] * h4 * u[3][0];
            P[n].y = y + sg[i][0] * h2 * u[1][1] + sg[i][1] * h4 * u[3][1];
            n++;
        }
        double h1 = a[0] / 2, h3 = a[2] / 2;
        n = or_clip(P, n, u[0][0], u[0][1], h1, Q);
        if (n == 0) return 0;
        n = or_clip(Q, n, -u[0][0], -u[0][1], h1, P);
        if (n == 0) return 0;
        n = or_clip(P, n, u[2][0], u[2][1], h3, Q);
        if (n == 0) return 0;
        n = or_clip(Q, n, -u[2][0], -u[2][1], h3, P);
        if (n == 0) return 0;
        return or_shoelace(P, n) / (a[0] * a[1] * a[2] * a[3]);
    }
    if (z13 == 1) {
        /* R13 is the segment {s u_k : |s| <= a_k/2} with line density 1/a_k;
           beta(x) = |{z in seg : z - x in R24}| / (a_k a2 a4). */
        int k = a[0] != 0 ? 0 : 2;
        double hk = a[k] / 2;
        or_pt A = {-hk * u[k][0] - x, -hk * u[k][1] - y};
        or_pt B = {hk * u[k][0] - x, hk * u[k][1] - y};
        double L = or_seg_in_rect(A, B, u[1], a[1] / 2, u[3], a[3] / 2);
        return L / (a[k] * a[1] * a[3]);
    }
    {
        int k = a[1] != 0 ? 1 : 3;
        double hk = a[k] / 2;
        or_pt A = {x - hk * u[k][0], y - hk * u[k][1]};
        or_pt B = {x + hk * u[k][0], y + hk * u[k][1]};
        double L = or_seg_in_rect(A, B, u[0], a[0] / 2, u[2], a[2] / 2);
        return L / (a[0] * a[2] * a[k]);
    }
}

/* ------------------------------------------------------------------------ */
/* Box-spline kernel, general order r: Eq. (2) with each box r-fold.         */
/* x = s1 u1 + s2 u2 + s3 u3 + s4 u4 with s_k ~ b_{a_k} independent, where   */
/* b_a = Box_a^{*r} is the centred B-spline of order r with knot spacing a   */
/* and unit mass.  With (P,Q) an orthogonal pair and (A,B) the other pair,  */
/*   beta(x) = int int b_A(tA) b_B(tB) b_P(x.uP - tA uA.uP - tB uB.uP)      */
/*                             b_Q(x.uQ - tA uA.uQ - tB uB.uQ) dtA dtB.      */
/* Exact piecewise Gauss-Legendre.                      */
/* ------------------------------------------------------------------------ */

/* centred cardinal B-spline of order r (degree r-1), unit mass, spacing a. */
static double or_bspline(int r, double a, double s) {
    /* N_r(x) on [0, r] by Cox-de Boor on integer knots; b_a(s)=N_r(s/a+r/2)/a */
    if (r == 1) return (s > -0.5 * a && s <= 0.5 * a) ? 1.0 / a : 0.0; /* Box_a */
    double xx = s / a + 0.5 * r;
    if (!(xx >= 0 && xx < r)) return 0;
    double N[8];
    int j = (int)floor(xx);
    /* degree-0 basis on [i, i+1) */
    for (int i = 0; i < r; i++) N[i] = (i == j) ? 1.0 : 0.0;
    for (int p = 1; p < r; p++) {
        for (int i = 0; i + p < r; i++) {
            double left = (xx - i) / p * N[i];
            double right = (i + p + 1 - xx) / p * N[i + 1];
            N[i] = left + right;
        }
    }
    return N[0] / a;
}

static const double OR_GL_X[8][8] = {
    {0},
    {0.0},
    {-0.5773502691896257645, 0.5773502691896257645},
    {-0.7745966692414833770, 0.0, 0.7745966692414833770},
    {-0.8611363115940525752, -0.3399810435848562648, 0.3399810435848562648, 0.8611363115940525752},
    {-0.9061798459386639928, -0.5384693101056830910, 0.0, 0.5384693101056830910, 0.9061798459386639928},
    {-0.9324695142031520278, -0.6612093864662645136, -0.2386191860831969086, 0.2386191860831969086,
     0.6612093864662645136, 0.9324695142031520278},
    {-0.9491079123427585245, -0.7415311855993944399, -0.4058451513773971669, 0.0, 0.4058451513773971669,
     0.7415311855993944399, 0.9491079123427585245},
};
static const double OR_GL_W[8][8] = {
    {0},
    {2.0},
    {1.0, 1.0},
    {0.5555555555555555556, 0.8888888888888888889, 0.5555555555555555556},
    {0.3478548451374538574, 0.6521451548625461426, 0.6521451548625461426, 0.3478548451374538574},
    {0.2369268850561890875, 0.4786286704993664680, 0.5688888888888888889, 0.4786286704993664680,
     0.2369268850561890875},
    {0.1713244923791703450, 0.3607615730481386076, 0.4679139345726910474, 0.4679139345726910474,
     0.3607615730481386076, 0.1713244923791703450},
    {0.1294849661688696933, 0.2797053914892766679, 0.3818300505051189449, 0.4179591836734693878,
     0.3818300505051189449, 0.2797053914892766679, 0.1294849661688696933},
};

static int or_cmp_dbl(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

typedef struct {
    int r;
    double aA, aB, aP, aQ;
    double pP, pQ;          /* x.uP, x.uQ */
    double cAP, cBP, cAQ, cBQ; /* uA.uP etc. */
} or_nest;

/* integrand factor for fixed tA as a function of tB */
static double or_inner(const or_nest *S, double tA, int ni) {
    /* breakpoints in tB */
    double bp[64];
    int nb = 0;
    int r = S->r;
    double hB = 0.5 * r * S->aB;
    for (int i = 0; i <= r; i++) bp[nb++] = S->aB * (i - 0.5 * r);
    /* P knots: pP - tA cAP - tB cBP = aP (i - r/2) */
    if (S->cBP != 0)
        for (int i = 0; i <= r; i++) bp[nb++] = (S->pP - tA * S->cAP - S->aP * (i - 0.5 * r)) / S->cBP;
    if (S->cBQ != 0)
        for (int i = 0; i <= r; i++) bp[nb++] = (S->pQ - tA * S->cAQ - S->aQ * (i - 0.5 * r)) / S->cBQ;
    qsort(bp, nb, sizeof(double), or_cmp_dbl);
    double sum = 0;
    for (int i = 0; i + 1 < nb; i++) {
        double lo = bp[i], hi = bp[i + 1];
        if (lo < -hB) lo = -hB;
        if (hi > hB) hi = hB;
        if (!(hi > lo)) continue;
        double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
        for (int g = 0; g < ni; g++) {
            double tB = mid + half * OR_GL_X[ni][g];
            double v = or_bspline(r, S->aB, tB) *
                       or_bspline(r, S->aP, S->pP - tA * S->cAP - tB * S->cBP) *
                       or_bspline(r, S->aQ, S->pQ - tA * S->cAQ - tB * S->cBQ);
            sum += OR_GL_W[ni][g] * half * v;
        }
    }
    return sum;
}

/* inner integral when b_B is a delta (aB = 0): tB = 0 */
static double or_inner_delta(const or_nest *S, double tA) {
    return or_bspline(S->r, S->aP, S->pP - tA * S->cAP) * or_bspline(S->r, S->aQ, S->pQ - tA * S->cAQ);
}

double or_beta(int basis, int r, const double *a, double x, double y) {
    if (r < 1 || r > 4) return NAN;
    double u[4][2];
    or_unit_dirs(basis, u);
    int P = 0, Q = 2, A = 1, B = 3;
    if (a[0] == 0 || a[2] == 0) {
        P = 1;
        Q = 3;
        A = 0;
        B = 2;
    }
    if (a[P] == 0 || a[Q] == 0) return NAN; /* two zero scales */
    or_nest S;
    S.r = r;
    S.aA = a[A];
    S.aB = a[B];
    S.aP = a[P];
    S.aQ = a[Q];
    S.pP = x * u[P][0] + y * u[P][1];
    S.pQ = x * u[Q][0] + y * u[Q][1];
    S.cAP = u[A][0] * u[P][0] + u[A][1] * u[P][1];
    S.cBP = u[B][0] * u[P][0] + u[B][1] * u[P][1];
    S.cAQ = u[A][0] * u[Q][0] + u[A][1] * u[Q][1];
    S.cBQ = u[B][0] * u[Q][0] + u[B][1] * u[Q][1];
    if (S.aB == 0 && S.aA != 0) {
        /* swap so that the delta (if any) is on A */
        double t;
        t = S.aA; S.aA = S.aB; S.aB = t;
        t = S.cAP; S.cAP = S.cBP; S.cBP = t;
        t = S.cAQ; S.cAQ = S.cBQ; S.cBQ = t;
    }
    int ni = (3 * r - 2 + 1) / 2;
    if (ni < 1) ni = 1;
    int no = 2 * r - 1;
    if (S.aA == 0) {
        /* b_A = delta: tA = 0 */
        if (S.aB == 0) return or_inner_delta(&S, 0.0);
        return or_inner(&S, 0.0, ni);
    }
    /* outer breakpoints in tA: knots of b_A, and crossings of the inner lines */
    double lines_a[64], lines_b[64]; /* tB = la + lb * tA */
    int nl = 0;
    for (int i = 0; i <= r; i++) {
        lines_a[nl] = S.aB * (i - 0.5 * r);
        lines_b[nl] = 0;
        nl++;
    }
    {
        for (int i = 0; i <= r; i++) {
            lines_a[nl] = (S.pP - S.aP * (i - 0.5 * r)) / S.cBP;
            lines_b[nl] = -S.cAP / S.cBP;
            nl++;
        }
        for (int i = 0; i <= r; i++) {
            lines_a[nl] = (S.pQ - S.aQ * (i - 0.5 * r)) / S.cBQ;
            lines_b[nl] = -S.cAQ / S.cBQ;
            nl++;
        }
    }
    double hA = 0.5 * r * S.aA;
    double bp[1200];
    int nb = 0;
    for (int i = 0; i <= r; i++) bp[nb++] = S.aA * (i - 0.5 * r);
    for (int i = 0; i < nl; i++)
        for (int j = i + 1; j < nl; j++) {
            double db = lines_b[i] - lines_b[j];
            if (db != 0) {
                double t = (lines_a[j] - lines_a[i]) / db;
                if (t > -hA && t < hA) bp[nb++] = t;
            }
        }
    qsort(bp, nb, sizeof(double), or_cmp_dbl);
    double sum = 0;
    int nq = no;
    for (int i = 0; i + 1 < nb; i++) {
        double lo = bp[i], hi = bp[i + 1];
        if (lo < -hA) lo = -hA;
        if (hi > hA) hi = hA;
        if (!(hi > lo)) continue;
        double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
        for (int g = 0; g < nq; g++) {
            double tA = mid + half * OR_GL_X[nq][g];
            double w = or_bspline(r, S.aA, tA);
            if (w == 0) continue;
            double inner = or_inner(&S, tA, ni);
            sum += OR_GL_W[nq][g] * half * w * inner;
        }
    }
    return sum;
}

/* ------------------------------------------------------------------------ */
/* The filter at one pixel: direct sum (*) over the kernel support.          */
/* ------------------------------------------------------------------------ */
typedef struct {
    const void *f;   /* image view */
    int dtype;       /* 0 u8, 1 f32, 2 f64 */
    int vx0, vy0;    /* view origin in full-image coords */
    int vw, vh;      /* view size */
    long stride;     /* elements per view row */
    int W, H;        /* full image size (zero extension outside) */
} or_image;

static double or_pix(const or_image *im, int x, int y, int *oob) {
    if (x < 0 || y < 0 || x >= im->W || y >= im->H) return 0.0;
    int lx = x - im->vx0, ly = y - im->vy0;
    if (lx < 0 || ly < 0 || lx >= im->vw || ly >= im->vh) {
        *oob = 1;
        return 0.0;
    }
    long i = (long)ly * im->stride + lx;
    if (im->dtype == 0) return (double)((const uint8_t *)im->f)[i];
    if (im->dtype == 1) return (double)((const float *)im->f)[i];
    return ((const double *)im->f)[i];
}

/* half-extents of the zonotope support sum_k [-r a_k/2, r a_k/2] u_k */
static void or_support(int basis, int r, const double *a, double *hx, double *hy) {
    double u[4][2];
    or_unit_dirs(basis, u);
    double sx = 0, sy = 0;
    for (int k = 0; k < 4; k++) {
        sx += 0.5 * r * a[k] * fabs(u[k][0]);
        sy += 0.5 * r * a[k] * fabs(u[k][1]);
    }
    *hx = sx;
    *hy = sy;
}

double or_filter_at(const or_image *im, int basis, int r, const double *a, int px, int py, int *oob) {
    double hx, hy;
    or_support(basis, r, a, &hx, &hy);
    int x0 = (int)floor(px - hx) - 1, x1 = (int)ceil(px + hx) + 1;
    int y0 = (int)floor(py - hy) - 1, y1 = (int)ceil(py + hy) + 1;
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    if (x1 > im->W - 1) x1 = im->W - 1;
    if (y1 > im->H - 1) y1 = im->H - 1;
    /* Neumaier summation of nonnegative-kernel terms */
    double s = 0, c = 0;
    for (int qy = y0; qy <= y1; qy++) {
        for (int qx = x0; qx <= x1; qx++) {
            double b = (r == 1) ? or_beta_r1(basis, a, (double)(px - qx), (double)(py - qy))
                                : or_beta(basis, r, a, (double)(px - qx), (double)(py - qy));
            if (b == 0) continue;
            double v = or_pix(im, qx, qy, oob) * b;
            double t = s + v;
            if (fabs(s) >= fabs(v))
                c += (s - t) + v;
            else
                c += (v - t) + s;
            s = t;
        }
    }
    return s + c;
}

/* ------------------------------------------------------------------------ */
/* Public batch entry: filter at a list of pixels.                           */
/*   image view (see or_image), cov per point (sx, sy, theta) as doubles,   */
/*   policy OR_THETA / OR_THETA_PRIME / OR_DUAL, order r, clamp flag.       */
/* Outputs: out[n]; aux basis[n], clamped[n], scales[4n].                   */
/* Returns the number of points whose support left the image view (0 = ok),*/
/* or -1 on infeasible covariance with clamp = 0 (out = NaN there).         */
/* ------------------------------------------------------------------------ */
int or_filter_points(const void *f, int dtype, int vx0, int vy0, int vw, int vh, long stride, int W, int H,
                     int policy, int r, int clamp, int n, const int *px, const int *py, const double *sx,
                     const double *sy, const double *th, double *out, int *basis_out, int *clamped_out,
                     double *scales_out, int nthreads) {
    or_image im = {f, dtype, vx0, vy0, vw, vh, stride, W, H};
    int bad = 0, infeas = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : bad, infeas)
#endif
    for (int i = 0; i < n; i++) {
        int basis = or_select(policy, sx[i], sy[i], th[i]);
        double C[3], a[4];
        int cl = or_pixel_cov(basis, clamp, sx[i], sy[i], th[i], C);
        if (basis_out) basis_out[i] = basis;
        if (clamped_out) clamped_out[i] = cl;
        if (cl < 0) {
            out[i] = NAN;
            infeas++;
            continue;
        }
        double Cr[3] = {C[0] / r, C[1] / r, C[2] / r};
        if (or_solve_scales(basis, Cr, a, NULL) != 0) {
            out[i] = NAN;
            infeas++;
            continue;
        }
        if (scales_out)
            for (int k = 0; k < 4; k++) scales_out[4 * i + k] = a[k];
        int oob = 0;
        out[i] = or_filter_at(&im, basis, r, a, px[i], py[i], &oob);
        if (oob) bad++;
    }
    if (infeas) return -1;
    return bad;
}

/* Kernel samples on a list of points (for pins and the Fig. 6 test). */
void or_beta_points(int basis, int r, const double *a, int n, const double *x, const double *y, double *out,
                    int use_polygon) {
    for (int i = 0; i < n; i++)
        out[i] = (r == 1 && use_polygon) ? or_beta_r1(basis, a, x[i], y[i]) : or_beta(basis, r, a, x[i], y[i]);
}

/* Scale solve for a list of covariances (C11, C12, C22 per row). */
int or_solve_many(int basis, int n, const double *C, double *a_out, double *t_out) {
    int bad = 0;
    for (int i = 0; i < n; i++)
        if (or_solve_scales(basis, C + 3 * i, a_out + 4 * i, t_out ? t_out + i : NULL) != 0) bad++;
    return bad;
}

/* ------------------------------------------------------------------------ */
/* Integer pre-integration reference (bit-exact contract).                   */
/* Running sums (Alg. 3 step 2) */
/* with integer steps and no sqrt5 factor (R3), uint64 wrapping,  */
/* on the domain x in [-P, W+P), y in [0, H+Pb), zero state outside it.     */
/* Level order: Theta' (a)(b)(c)(d) = steps (1,2),(2,1),(-1,2),(-2,1);       */
/* Theta (1,0),(1,1),(0,1),(-1,1); the 4 levels repeated r times.            */
/* g has (H+Pb) rows of (W+2P) uint64; g[y][x+P].                            */
/* ------------------------------------------------------------------------ */
static const int OR_SCAN_ORDER[2][4][2] = {
    {{1, 0}, {1, 1}, {0, 1}, {-1, 1}},
    {{1, 2}, {2, 1}, {-1, 2}, {-2, 1}},
};

int or_preintegrate_u8(const uint8_t *f, int W, int H, int basis, int r, int P, int Pb, uint64_t *g) {
    if (basis != OR_THETA && basis != OR_THETA_PRIME) return -1;
    int GW = W + 2 * P, GH = H + Pb;
    memset(g, 0, sizeof(uint64_t) * (size_t)GW * GH);
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) g[(size_t)y * GW + x + P] = f[(size_t)y * W + x];
    for (int rep = 0; rep < r; rep++) {
        for (int lv = 0; lv < 4; lv++) {
            int sx = OR_SCAN_ORDER[basis][lv][0], sy = OR_SCAN_ORDER[basis][lv][1];
            /* g(q) <- g(q) + g(q - s), visiting q in an order where q - s is
               already final: increasing y; within a row, increasing x when
               sy = 0 (then sx = 1). */
            for (int y = 0; y < GH; y++) {
                for (int xi = 0; xi < GW; xi++) {
                    int py = y - sy, pxi = xi - sx;
                    if (py < 0 || pxi < 0 || pxi >= GW) continue;
                    g[(size_t)y * GW + xi] += g[(size_t)py * GW + pxi];
                }
            }
        }
    }
    return 0;
}
