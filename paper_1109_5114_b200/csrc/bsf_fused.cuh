// Fused tile path with the exact split contraction.
//
// Included by bsf_kernels.cu inside namespace bsf (uses c_steps, c_scan_order,
// classify, tile_domain, tile_scan_level, comp_step, pixel_scales from there).
//
// Per 16x16 output tile (one persistent CTA per SM, 256 threads):
//  1. a1-a4 per pixel: covariance decode, Alg. 2 basis, clamp, scale solve
//     (bsf_pixel.cuh), tap geometry extents.
//  2. a5: the 4r running sums of every basis in use on the tile's halo domain
//     (double-double, zero state outside; R18), and for every zero-
//     scale variant in use its exact lattice difference (1 - T_{s_k})^r G (R5).
//  3. Exact split of every plane: G = 2^e (G1 + G0), G1 an integer with
//     |G1| <= 2^kbits, where kbits is chosen per table so that
//     sum_slots |G1| |n| <= 2^53: the contraction sum_d G1_d n_{d,mu} of the
//     integer table numerators n is then EXACT in fp64, and only the small part
//     G0 (|G0| <= 1/2) carries rounding.  One fp64 FMA per limb per algorithmic
//     multiply-add gives a result as accurate as double-double.
//  4. a6: the (r+1)^4 (or (r+1)^3) taps of every pixel are bucketed by
//     interpolation key (basis, variant, region of the unit cell) and padded to
//     16-lane groups, so each half-warp reads ONE coefficient table: the table
//     loads are broadcasts, the G loads are per lane.  Per tap:
//       E_mu = sum_d (G1_d + G0_d) n_{d,mu}         (2 DFMA per coefficient)
//       F    = sum_mu E_mu phi^mu                   (compensated Horner, rows)
//  5. a7: per pixel S = sum_j c_j F_j in double-double, out = 2^e S w^r / L.

constexpr int FT = 256;                       // threads per CTA = pixels per sub-tile
constexpr int STILE = 2 * TILE;               // super-tile: the running sums' anchor
constexpr int NKEY = 2 * NVAR * MAX_REG;      // (basis, variant, region)
constexpr int NPLANE = 2 * NVAR;              // (basis, variant)
constexpr uint16_t NOKEY = 0xFFFF;


#ifndef BSF_MT1
#define BSF_MT1 4
#endif
#ifndef BSF_MT3
#define BSF_MT3 1
#endif
#ifndef BSF_G3_NP1
#define BSF_G3_NP1 9  // order >= 3, unsplit numerators: n-tiles per pass (9 = all at degree 10: one pass)
#endif
#ifndef G3_PRESPLIT_MAX
// order 3: halo planes up to this many points are split into their three limbs
// once (the groups then load them); larger ones (config 5's sigma <= 64) are
// split on the fly, where the pass over the whole domain would cost more
#define G3_PRESPLIT_MAX 250000
#endif
#ifndef BSF_G3_NP2
#define BSF_G3_NP2 3  // order >= 3, split numerators (five limb products per tile): 9 = 3 x 3 at degree 10
#endif
template <int R> struct FusedCfg;
// NTAP taps per pixel, P pixels per chunk, MT 8-item m-tiles per group
template <> struct FusedCfg<1> { static constexpr int NTAP = 16, P = 256, MT = BSF_MT1; };
template <> struct FusedCfg<2> { static constexpr int NTAP = 81, P = 256, MT = 4; };
#ifndef BSF_P3
#define BSF_P3 64
#endif
template <> struct FusedCfg<3> { static constexpr int NTAP = 256, P = BSF_P3, MT = BSF_MT3; };
template <> struct FusedCfg<4> { static constexpr int NTAP = 625, P = 16, MT = 1; };

// per-tap interpolated values F (double-double) live in a per-CTA global
// buffer (L2-resident) of fused_fbuf_items() entries, not in shared memory,
// so a chunk can hold a whole sub-tile (less bucket padding)
template <int R>
constexpr int fused_items() { return FusedCfg<R>::P * FusedCfg<R>::NTAP; }

// dynamic shared memory: the chunk buffers of phases 4-5, aliased by the
// pre-integration ring of phase 2 (at least FUSED_SMEM_MIN bytes for it)
constexpr size_t FUSED_SMEM_MIN = 0;
template <int R>
constexpr size_t fused_smem_bytes() {
    constexpr size_t ITEMS = (size_t)FusedCfg<R>::P * FusedCfg<R>::NTAP;
    constexpr size_t GS = 8 * FusedCfg<R>::MT;
    constexpr size_t chunk = FT * 4 * 8 + FT * 5 * 16 + ITEMS * 2 + (ITEMS + GS * NKEY) * 2 + (FT / 32) * NKEY * 4 +
                             FT * 4;
    return chunk > FUSED_SMEM_MIN ? chunk : FUSED_SMEM_MIN;
}

// order 3, i8 route (bsf_i8_gather.cuh): after the chunk buffers, 1 KB
// aligned: seven A slices (4 KB each), eight B slices (1 KB each), the E12
// tile (32 items x E12S columns, double-double)
constexpr size_t I8_SMEM = 7 * 4096 + 8 * 1024 + 32 * 72 * 16;
template <int R>
constexpr size_t i8_smem_off() { return (fused_smem_bytes<R>() + 1023) / 1024 * 1024; }

// pixel info word: bit0 basis, bits1-3 variant (drop + 1), bit4 live, bit5 clamped, bits 8.. flags
__device__ __forceinline__ int info_basis(int w) { return w & 1; }
__device__ __forceinline__ int info_var(int w) { return (w >> 1) & 7; }
__device__ __forceinline__ bool info_live(int w) { return (w >> 4) & 1; }

// C(R, j) for the compile-time order R (no integer division)
template <int R>
__device__ __forceinline__ int binomR(int j) {
    if constexpr (R == 1) return 1;
    if constexpr (R == 2) return j == 1 ? 2 : 1;
    if constexpr (R == 3) return (j == 1 || j == 2) ? 3 : 1;
    if constexpr (R == 4) return j == 2 ? 6 : ((j == 1 || j == 3) ? 4 : 1);
    return 0;
}

// tap t of a pixel: displacement D (exact, R17) and binomial sign weight
template <int R>
__device__ __forceinline__ void fused_tap(const double *ap, int basis, int drop, int t, double &Dx, double &Dy,
                                          int &coef) {
    int tt = t;
    coef = 1;
    Dx = 0.0;
    Dy = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (k == drop) continue;
        int j = tt % (R + 1);
        tt /= (R + 1);
        coef *= binomR<R>(j) * ((j & 1) ? -1 : 1);
        double m = 0.5 * R - j;
        Dx += (m * c_steps[basis][k][0]) * ap[k];
        Dy += (m * c_steps[basis][k][1]) * ap[k];
    }
}

// split running sum (G1, G0) at domain point (lx, ly); zero above the domain.
// Branch-free: the load always reads a valid address and the value is
// selected afterwards (no divergence barriers in the MMA loop).
__device__ __forceinline__ double2 load_split(const double2 *__restrict__ G, int NX, int NY, int lx, int ly,
                                              int &flags) {
#ifndef BSF_CHECK_RANGE
    // the super-tile domain covers every window read by construction
    // (fused_domain); build with -DBSF_CHECK_RANGE to check and flag instead
    (void)NY;
    (void)flags;
    return G[(size_t)ly * NX + lx];
#endif
    const bool inside = lx >= 0 && lx < NX && ly >= 0 && ly < NY;
    flags |= (ly >= 0 && !inside) ? FLAG_RANGE : 0;
    const double2 v = G[inside ? (size_t)ly * NX + lx : 0];
    return inside ? v : make_double2(0.0, 0.0);
}

// Halo domain of a super-tile (as tile_domain, for ST x ST outputs).
__device__ __forceinline__ TileDomain fused_domain(const LutBasis &L, int R, int x0, int y0, int EX, int EY,
                                                   int ST) {
    TileDomain d;
    d.X0 = x0 - EX + L.wxmin - 2 * R - 1;  // zero-scale lattice difference reaches back R|s_x| <= 2R
    const int X1 = x0 + ST - 1 + EX + L.wxmax + 2 * R + 1;
    d.Y0 = y0 - EY;  // no kernel support above: zero state (reads above hit the zero pad rows)
    const int Y1 = y0 + ST - 1 + EY + L.wymax + 1;
    d.NX = X1 - d.X0 + 1;
    d.NY = Y1 - d.Y0 + 1;
    return d;
}

// Region classifier of the unit cell (classify() in bsf_kernels.cu) with its
// tables staged in shared memory once per CTA.
struct ClsTables {
    int2 normal[2][4];
    int kmin[2][4], radix[2][4];
    signed char table[2][81];
};

__device__ __forceinline__ int cls_key(const ClsTables &T, int b, double x, double y) {
    int idx = 0, mul = 1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int f = (int)floor(T.normal[b][k].x * x + T.normal[b][k].y * y) - T.kmin[b][k];
        if (f < 0 || f >= T.radix[b][k]) return -1;
        idx += f * mul;
        mul *= T.radix[b][k];
    }
    return T.table[b][idx];
}

__device__ __forceinline__ int cls_region(const ClsTables &T, int b, double x, double y) {
    const double one_m = 1.0 - 1.1102230246251565e-16;
    x = fmin(fmax(x, 0.0), one_m);
    y = fmin(fmax(y, 0.0), one_m);
    int r = cls_key(T, b, x, y);
    if (r >= 0) return r;
    // exactly on knot lines: any adjacent region gives the same value (the
    // kernel is continuous), step into one -- the same nudges as classify()
    const double e = 1e-12;
    const double dx[4] = {e, -e, 0.7 * e, -0.3 * e};
    const double dy[4] = {0.37 * e, 0.61 * e, -e, -0.77 * e};
    for (int i = 0; i < 4; ++i) {
        r = cls_key(T, b, fmin(fmax(x + dx[i], 0.0), one_m), fmin(fmax(y + dy[i], 0.0), one_m));
        if (r >= 0) return r;
    }
    return 0;
}

// (sigma_x, sigma_y, theta) of a pixel under the covariance mode of the launch
// (Algorithm 1): the planes, s sigma_b^2 I (the global
// isotropic pass, theta = 0), or C - s sigma_b^2 I (same eigenvectors,
// eigenvalues lowered: PAPER.md:228-231); s = sigma2_scale (1 for Algorithm 1,
// the generalised splitting's shares otherwise, R22)
// output row window (row strips): rows of cov / out, and membership
__device__ __forceinline__ int out_rows(const TileArgs &a) { return a.oH ? a.oH : a.H; }
__device__ __forceinline__ bool out_row(const TileArgs &a, int y) {
    return y >= a.oy0 && y < a.oy0 + out_rows(a) && y < a.H;
}
__device__ __forceinline__ long long out_index(const TileArgs &a, int img, int x, int y) {
    return ((long long)img * out_rows(a) + (y - a.oy0)) * a.W + x;
}

__device__ __forceinline__ void load_cov(const TileArgs &a, int img, int x, int y, double &sx, double &sy,
                                         double &th) {
    const size_t ipl = (size_t)out_rows(a) * a.W;
    const int b = img / a.channels;
    if (a.cov_mode == COV_ISO) {
        sx = sy = sqrt(a.sigma2[b] * a.sigma2_scale);
        th = 0.0;
        return;
    }
    const float *cv = a.cov + (size_t)b * 3 * ipl + (size_t)(y - a.oy0) * a.W + x;
    sx = __ldg(cv);
    sy = __ldg(cv + ipl);
    th = __ldg(cv + 2 * ipl);
    if (a.cov_layout == BSF_COV_C11_C12_C22) cov_from_c(sx, sy, th, sx, sy, th);
    if (a.cov_mode == COV_SUB) {
        const double s2 = a.sigma2[b] * a.sigma2_scale;
        sx = sqrt(fmax(sx * sx - s2, 0.0));
        sy = sqrt(fmax(sy * sy - s2, 0.0));
    }
}

__device__ __forceinline__ double load_f(const TileArgs &a, size_t o) {
    if (a.in_f64) return ((const double *)a.f)[o];
    return a.in_u8 ? (double)((const uint8_t *)a.f)[o] : (double)((const float *)a.f)[o];
}

// displacement of tap t from the per-pixel geometry (see the sub-tile scales):
// identical to fused_tap's value, with 4 FMAs per coordinate
template <int R>
__device__ __forceinline__ void fused_tap_v(const double2 *tv, int drop, int t, double &Dx, double &Dy) {
    const double2 c = tv[4];
    Dx = c.x;
    Dy = c.y;
    int tt = t;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (k == drop) continue;
        const double j = (double)(tt % (R + 1));
        tt /= (R + 1);
        const double2 v = tv[k];
        Dx = fma(-j, v.x, Dx);  // exact (R17)
        Dy = fma(-j, v.y, Dy);
    }
}

// binomial sign weight of tap t: prod_k (-1)^{j_k} C(R, j_k)
template <int R>
__device__ __forceinline__ int tap_coef(int t, int drop) {
    int c = 1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (k == drop) continue;
        const int j = t % (R + 1);
        t /= (R + 1);
        c *= binomR<R>(j) * ((j & 1) ? -1 : 1);
    }
    return c;
}

// FP64 tensor-core MMA (DMMA): D(8x8) += A(8x4) B(4x8).  Fragments (PTX ISA,
// m8n8k4 .f64): lane l holds A[l/4][l%4], B[l%4][l/4], C[l/4][2(l%4)+{0,1}].
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int DEG>
struct DegCfg {
    static constexpr int NMON = (DEG + 1) * (DEG + 2) / 2;
    static constexpr int NT = bsf_nt(DEG);  // 8-column n-tiles (bsf_mono_col layout)
};

// Row polynomials R_i(phi_y) of the rows this lane of the quad owns
// (compensated Horner over its accumulator slots, highest y power first).  All
// lanes step through the slots in lock-step; which slots start a row or belong
// to one is a per-lane mask, applied by selects (no divergence).  The q-th row
// of the lane ends in (Rh[q], Rl[q]).
template <int DEG>
struct RowCfg {
    static constexpr int QMAX = bsf_lane_rows(DEG, 0) > bsf_lane_rows(DEG, 1)
                                    ? (bsf_lane_rows(DEG, 0) > bsf_lane_rows(DEG, 3) ? bsf_lane_rows(DEG, 0)
                                                                                     : bsf_lane_rows(DEG, 3))
                                    : (bsf_lane_rows(DEG, 1) > bsf_lane_rows(DEG, 3) ? bsf_lane_rows(DEG, 1)
                                                                                     : bsf_lane_rows(DEG, 3));
};

// NORM (global int64 sums, both limbs exact): the accumulators hold E1 and E0
// of E = 2^k E1 + E0; e = TwoSum(E1, E0 2^-k) is E / 2^k as an exact,
// normalised double-double.  Otherwise (A, B) is taken as it is (below).
template <int DEG, int NT, bool NORM = false>
__device__ __forceinline__ void fused_rows(const double (&C)[2][NT][2], double fy, int kq,
                                           double (&Rh)[RowCfg<DEG>::QMAX], double (&Rl)[RowCfg<DEG>::QMAX],
                                           double isc = 0.0) {
    constexpr int QMAX = RowCfg<DEG>::QMAX;
    const unsigned smask = kq == 0 ? bsf_start_mask(DEG, 0)
                           : kq == 1 ? bsf_start_mask(DEG, 1)
                           : kq == 2 ? bsf_start_mask(DEG, 2) : bsf_start_mask(DEG, 3);
    const unsigned vmask = kq == 0 ? bsf_valid_mask(DEG, 0)
                           : kq == 1 ? bsf_valid_mask(DEG, 1)
                           : kq == 2 ? bsf_valid_mask(DEG, 2) : bsf_valid_mask(DEG, 3);
#pragma unroll
    for (int q = 0; q < QMAX; ++q) Rh[q] = Rl[q] = 0.0;
    // slot 0 starts a row on every lane that has rows (bsf_start_mask): no
    // Horner step, the row value is the slot itself
    const bool any = vmask & 1u;
    double rh = any ? C[0][0][0] : 0.0, rl = any ? C[1][0][0] : 0.0;
    if constexpr (NORM) {
        const dd e0 = two_sum(rh, rl * isc);
        rh = e0.hi;
        rl = e0.lo;
    }
    int q = any ? 0 : -1;
#pragma unroll
    for (int k = 1; k < 2 * NT; ++k) {
        const bool start = (smask >> k) & 1, valid = (vmask >> k) & 1;
        // (A, B) = (exact integer limb, remainder limb) is already an exact,
        // unnormalised double-double of E (|B| <= 2^-kbits |A| scale): the
        // compensated Horner step takes it as is
        const dd e = NORM ? two_sum(C[0][k >> 1][k & 1], C[1][k >> 1][k & 1] * isc)
                          : dd{C[0][k >> 1][k & 1], C[1][k >> 1][k & 1]};
        double nh = rh, nl = rl;
        comp_step(nh, nl, fy, e.hi, e.lo);
        if (start) {
#pragma unroll
            for (int qq = 0; qq < QMAX; ++qq)
                if (qq == q) {
                    Rh[qq] = rh;
                    Rl[qq] = rl;
                }
            ++q;
        }
        rh = start ? e.hi : (valid ? nh : rh);
        rl = start ? e.lo : (valid ? nl : rl);
    }
#pragma unroll
    for (int qq = 0; qq < QMAX; ++qq)
        if (qq == q) {
            Rh[qq] = rh;
            Rl[qq] = rl;
        }
}

// Horner scheme in phi_x over the rows, gathered from the quad's lanes.
template <int DEG, int I>
__device__ __forceinline__ void fused_xhorner(const double (&Rh)[RowCfg<DEG>::QMAX],
                                              const double (&Rl)[RowCfg<DEG>::QMAX], double fx, double &ah,
                                              double &al) {
    constexpr int SRC = bsf_row_lane(DEG, I), Q = bsf_row_q(DEG, I);
    const int src = (threadIdx.x & 28) | SRC;
    const double h = __shfl_sync(0xffffffffu, Rh[Q], src), l = __shfl_sync(0xffffffffu, Rl[Q], src);
    if constexpr (I == DEG) {
        ah = h;
        al = l;
    } else {
        comp_step(ah, al, fx, h, l);
    }
    if constexpr (I > 0) fused_xhorner<DEG, I - 1>(Rh, Rl, fx, ah, al);
}

// x-Horner of m-tile kq for four m-tiles: every row is shuffled for all four
// m-tiles and each lane keeps its own (compile-time row / slot indices)
template <int DEG, int I>
__device__ __forceinline__ void fused_xhorner4(const double (&Rh)[4][RowCfg<DEG>::QMAX],
                                               const double (&Rl)[4][RowCfg<DEG>::QMAX], int kq, double fx,
                                               double &ah, double &al) {
    constexpr int SRC = bsf_row_lane(DEG, I), Q = bsf_row_q(DEG, I);
    const int src = (threadIdx.x & 28) | SRC;
    double h = 0.0, l = 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const double ht = __shfl_sync(0xffffffffu, Rh[t][Q], src);
        const double lt = __shfl_sync(0xffffffffu, Rl[t][Q], src);
        h = kq == t ? ht : h;
        l = kq == t ? lt : l;
    }
    if constexpr (I == DEG) {
        ah = h;
        al = l;
    } else {
        comp_step(ah, al, fx, h, l);
    }
    if constexpr (I > 0) fused_xhorner4<DEG, I - 1>(Rh, Rl, kq, fx, ah, al);
}

// Contraction of one group of GS = 8 MT items sharing a key, on the FP64
// tensor cores: for every item (M), window slot (K) and monomial (N)
//   E_mu = sum_s G1_s n_{s,mu}  (exact)   and   sum_s G0_s n_{s,mu},
// the two limbs as separate accumulators; then F = sum_mu E_mu phi^mu straight
// from the accumulator fragments (rows per lane in phi_y, then phi_x across
// the quad), compensated.  Lane l feeds and receives item l/4 + 8t of m-tile
// t; (bxt, byt) are that item's tap base; (fxo, fyo) the fractional offset of
// the lane's own item (shuffled to the quads for the epilogue).
// u8 input: every running-sum level is an integer below 255 x the product of
// the line lengths so far (a line of step (sx, sy) has at most NY/sy + 1
// points, a row NX); a zero-scale variant plane (1 - T_s)^R G at most 2^R
// times that.  When this stays below 2^kbits the planes are their own exact
// split (G1 = G, G0 = 0): no scaling pass, and a single MMA limb.
__device__ __forceinline__ double u8_plane_bound(int basis, int R, int NX, int NY) {
    double bound = 255.0;
    for (int rep = 0; rep < R; ++rep)
        for (int lv = 0; lv < 4; ++lv) {
            const int sy = c_scan_order[basis][lv][1];
            bound *= sy == 0 ? (double)NX : (double)(NY / sy + 1);
        }
    return bound;
}

// Operand sources of fused_group: the A operand (two limbs) at a window point.
// PlaneSrc: a super-tile halo plane already split into (G1, G0) (phase 3).
struct PlaneSrc {
    static constexpr bool NORM = false;
    const double2 *__restrict__ G;
    int NX, NY;
    __device__ __forceinline__ double2 operator()(int lx, int ly, int &flags) const {
        return load_split(G, NX, NY, lx, ly, flags);
    }
};
// GlobSrc: the global int64 running sums of bsf_preintegrate_exact (u8 input;
// the plan checked that no sum reaches 2^62), read at domain point (lx, ly):
// zero above the domain (no image there), a zero-scale variant by its exact
// lattice difference G(q) - G(q - s) (order 1, R5), split exactly
// into G1 = v >> k and G0 = v & (2^k - 1): both limbs are integers below
// 2^kbits, so both contractions are exact (global mode).
struct GlobSrc {
    static constexpr bool NORM = true;
    const long long *__restrict__ G;
    int GW, GH, k;
    int sdx, sdy;  // lattice step of the dropped direction (variant planes), else (0, 0)
    bool var;
    __device__ __forceinline__ long long at(int lx, int ly, int &flags) const {
        const bool inside = lx >= 0 && lx < GW && ly >= 0 && ly < GH;
        flags |= (ly >= 0 && !inside) ? FLAG_RANGE : 0;
        const long long v = __ldg(G + (inside ? (size_t)ly * GW + lx : 0));
        return inside ? v : 0ll;
    }
    __device__ __forceinline__ double2 operator()(int lx, int ly, int &flags) const {
        long long v = at(lx, ly, flags);
        if (var) v -= at(lx - sdx, ly - sdy, flags);
        return make_double2((double)(v >> k), (double)(v & ((1ll << k) - 1)));
    }
};

template <int DEG, int MT, int LIMBS = 2, class Src = PlaneSrc>
__device__ __forceinline__ void fused_group(const Src &src, const int (&bxt)[MT],
                                            const int (&byt)[MT], double fxo, double fyo,
                                            const int2 *__restrict__ offs, const double *__restrict__ num, int nmonp,
                                            int n4, double (&Fh)[MT], double (&Fl)[MT], int &flags,
                                            double isc = 0.0) {
    constexpr int NT = DegCfg<DEG>::NT;
    const int lane = threadIdx.x & 31, kq = lane & 3, gq = lane >> 2;
    double C[MT][2][NT][2];
#pragma unroll
    for (int t = 0; t < MT; ++t)
#pragma unroll
        for (int L = 0; L < 2; ++L)
#pragma unroll
            for (int j = 0; j < NT; ++j) C[t][L][j][0] = C[t][L][j][1] = 0.0;
    // Software pipeline over k-steps of 4 window slots, unrolled by two with
    // ping-pong operand sets (A for even steps, B for odd): while one step's
    // MMAs issue, the other set is loaded for the next step, and the window
    // offsets one step further ahead.  No loaded value crosses the loop edge
    // through a register copy.
    const int nsteps = n4 >> 2;
    const double *cs = num + kq * nmonp + gq;
    const int cstep = 4 * nmonp;
    double2 aA[MT], aB[MT];
    double bA[NT], bB[NT];
    int2 dA = __ldg(offs + kq), dB = make_int2(0, 0);
#pragma unroll
    for (int t = 0; t < MT; ++t) aA[t] = src(bxt[t] + dA.x, byt[t] + dA.y, flags);
#pragma unroll
    for (int j = 0; j < NT; ++j) bA[j] = __ldg(cs + 8 * j);
    if (nsteps > 1) dB = __ldg(offs + 4 + kq);
    for (int st = 0; st < nsteps; st += 2) {
        if (st + 1 < nsteps) {
#pragma unroll
            for (int t = 0; t < MT; ++t) aB[t] = src(bxt[t] + dB.x, byt[t] + dB.y, flags);
#pragma unroll
            for (int j = 0; j < NT; ++j) bB[j] = __ldg(cs + (size_t)(st + 1) * cstep + 8 * j);
        }
        if (st + 2 < nsteps) dA = __ldg(offs + 4 * (st + 2) + kq);
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int t = 0; t < MT; ++t) {
                dmma(C[t][0][j], aA[t].x, bA[j]);  // exact: integers below 2^53
                if constexpr (LIMBS == 2) dmma(C[t][1][j], aA[t].y, bA[j]);  // LIMBS 1: the G0 limb is zero
            }
        if (st + 1 >= nsteps) break;
        if (st + 2 < nsteps) {
#pragma unroll
            for (int t = 0; t < MT; ++t) aA[t] = src(bxt[t] + dA.x, byt[t] + dA.y, flags);
#pragma unroll
            for (int j = 0; j < NT; ++j) bA[j] = __ldg(cs + (size_t)(st + 2) * cstep + 8 * j);
        }
        if (st + 3 < nsteps) dB = __ldg(offs + 4 * (st + 3) + kq);
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int t = 0; t < MT; ++t) {
                dmma(C[t][0][j], aB[t].x, bB[j]);
                if constexpr (LIMBS == 2) dmma(C[t][1][j], aB[t].y, bB[j]);
            }
    }
#ifdef BSF_DBG_NO_EPI
    // diagnostics build only (timing of the MMA loop without the polynomial
    // epilogue; results are wrong): keep every accumulator live
    {
        double s0 = fxo + fyo;
#pragma unroll
        for (int t = 0; t < MT; ++t)
#pragma unroll
            for (int L = 0; L < 2; ++L)
#pragma unroll
                for (int j = 0; j < NT; ++j) s0 += C[t][L][j][0] + C[t][L][j][1];
#pragma unroll
        for (int t = 0; t < MT; ++t) Fh[t] = Fl[t] = s0;
        return;
    }
#endif
    if constexpr (MT == 4) {
        // rows of all four m-tiles on their owner lanes; then lane kq of each
        // quad runs the x-Horner of m-tile kq only (one x-Horner per lane
        // instead of four): the result for item gq + 8 kq stays on lane (gq, kq)
        constexpr int QMAX = RowCfg<DEG>::QMAX;
        double Rh[MT][QMAX], Rl[MT][QMAX];
#pragma unroll
        for (int t = 0; t < MT; ++t) {
            const double fyq = __shfl_sync(0xffffffffu, fyo, gq + 8 * t);
            fused_rows<DEG, NT, Src::NORM>(C[t], fyq, kq, Rh[t], Rl[t], isc);
        }
        const double fxm = __shfl_sync(0xffffffffu, fxo, gq + 8 * kq);
        double ah = 0.0, al = 0.0;
        fused_xhorner4<DEG, DEG>(Rh, Rl, kq, fxm, ah, al);
        const dd F = fast_two_sum(ah, al);
        Fh[0] = F.hi;  // this lane's item: gq + 8 kq
        Fl[0] = F.lo;
    } else {
#pragma unroll
        for (int t = 0; t < MT; ++t) {
            // fractional offset of this m-tile's item, from the lane that set it up
            const double fxq = __shfl_sync(0xffffffffu, fxo, gq + 8 * t);
            const double fyq = __shfl_sync(0xffffffffu, fyo, gq + 8 * t);
            double Rh[RowCfg<DEG>::QMAX], Rl[RowCfg<DEG>::QMAX];
            fused_rows<DEG, NT, Src::NORM>(C[t], fyq, kq, Rh, Rl, isc);
            double ah, al;
            fused_xhorner<DEG, DEG>(Rh, Rl, fxq, ah, al);
            const dd F = fast_two_sum(ah, al);
            Fh[t] = F.hi;
            Fl[t] = F.lo;
        }
    }
}

// ---------------------------------------------------------------------------
// Pre-integration of one halo plane by a wavefront row sweep (a5).
//
// The levels with s_y >= 1 obey v_l(x, y) = v_{l-1}(x, y) + v_l(x - s_x, y - s_y)
// (zero state outside the domain).  At step tau level l (1-based) processes
// row tau - l + 1: it needs its own rows y - 1, y - 2 and row y of level l - 1,
// all written in earlier steps, so every level advances together with one
// barrier per step, each level keeping its last three rows in a shared-memory
// ring.  The Theta basis' horizontal levels (1, 0) are prefix sums along the
// rows and are taken first, all R of them in one pass per row (thread per
// row) -- on the truncated tile domain the order of the levels only changes
// the sums by functions the mesh annihilates (R18/R20).  The plane G receives
// the horizontal sums (Theta), then the final level of the sweep, row by row.
// Returns false (nothing done) when the ring does not fit in `ring_bytes`.
// ---------------------------------------------------------------------------
// Order >= 3: three G limbs split on the fly from the double-double planes,
// G = 2^e (G1 + 2^-k G2 + 2^-k G0), G1, G2 integers below 2^k (k = kbits),
// |G0| <= 1/2: G1 and G2 are contracted exactly, only G0 carries rounding, so
// the contraction error is 2^-k smaller than with two limbs (the (D/a)^{4r}
// conditioning of r = 3 needs it).  With split numerators (NSPLIT 2) the two
// exact limbs each meet n1 and n0.  The N dimension is taken in passes of NP
// n-tiles (bounded registers); the lock-step row Horner resumes across passes.
// I8 (plan option "i8_tc", PRE planes only): the exact part sum_s (G1 2^k + G2) n
// was formed on the tcgen05 tensor cores (i8_tile) and is read from shared
// memory (e12: this group's 8 items, row stride E12S, already scaled by 2^-k);
// only the rounded G0 limb is contracted here on DMMA.
constexpr int E12S = 72;  // E12 row stride (degree-10 tables: 9 n-tiles)
template <int DEG, int NSPLIT, int NP, int MT, bool PRE, bool I8 = false>
__device__ __forceinline__ void fused_group_g3(const double2 *__restrict__ G, int NX, int NY, const int (&bxt)[MT],
                                               const int (&byt)[MT], double fxo, double fyo,
                                               const int2 *__restrict__ offs, const float *__restrict__ numc,
                                               int nmonp, int n4, int shift, const double *__restrict__ G0,
                                               double sc_e, int kbits, double (&Fh)[MT], double (&Fl)[MT],
                                               int &flags, const double2 *e12 = nullptr) {
    constexpr int NT = DegCfg<DEG>::NT, NL = NSPLIT == 1 ? 3 : 5, QMAX = RowCfg<DEG>::QMAX;
    const int lane = threadIdx.x & 31, kq = lane & 3, gq = lane >> 2;
    // fractional offsets of this lane's items (gq + 8t), from the lanes that set them up
    double fxt[MT], fyt[MT];
#pragma unroll
    for (int t = 0; t < MT; ++t) {
        fxt[t] = __shfl_sync(0xffffffffu, fxo, gq + 8 * t);
        fyt[t] = __shfl_sync(0xffffffffu, fyo, gq + 8 * t);
    }
    const double S = ldexp(1.0, kbits), iS = ldexp(1.0, -kbits), ssh = ldexp(1.0, shift);
    const unsigned smask = kq == 0 ? bsf_start_mask(DEG, 0)
                           : kq == 1 ? bsf_start_mask(DEG, 1)
                           : kq == 2 ? bsf_start_mask(DEG, 2) : bsf_start_mask(DEG, 3);
    const unsigned vmask = kq == 0 ? bsf_valid_mask(DEG, 0)
                           : kq == 1 ? bsf_valid_mask(DEG, 1)
                           : kq == 2 ? bsf_valid_mask(DEG, 2) : bsf_valid_mask(DEG, 3);
    double Rh[MT][QMAX], Rl[MT][QMAX], rh[MT], rl[MT];
    int q = -1;  // the row counter is the same for every m-tile (same lane, same slots)
#pragma unroll
    for (int t = 0; t < MT; ++t) {
        rh[t] = rl[t] = 0.0;
#pragma unroll
        for (int qq = 0; qq < QMAX; ++qq) Rh[t][qq] = Rl[t][qq] = 0.0;
    }
    for (int j0 = 0; j0 < NT; j0 += NP) {
        double C[MT][NL][NP][2];
#pragma unroll
        for (int t = 0; t < MT; ++t)
#pragma unroll
            for (int L = 0; L < NL; ++L)
#pragma unroll
                for (int j = 0; j < NP; ++j) C[t][L][j][0] = C[t][L][j][1] = 0.0;
        for (int s0 = 0; s0 < n4; s0 += 4) {
            const int s = s0 + kq;
            const int2 d = __ldg(offs + s);
            double g1[MT], g2[MT], g0[MT];
#pragma unroll
            for (int t = 0; t < MT; ++t) {
                const int lx = bxt[t] + d.x, ly = byt[t] + d.y;
#ifdef BSF_CHECK_RANGE
                const bool inside = lx >= 0 && lx < NX && ly >= 0 && ly < NY;
                flags |= (ly >= 0 && !inside) ? FLAG_RANGE : 0;
#else
                const bool inside = true;  // fused_domain covers every window read
#endif
                // the order-3 halo planes are too large for L1 and are read from L2 anyway:
                // bypass L1 so that it keeps the region's coefficient table
                // (an L1 prefetch of the next step's sums evicted the table: +32 %)
                const size_t gi = inside ? (size_t)ly * NX + lx : 0;
                if constexpr (I8) {  // the exact limbs are in e12: only G0
                    g1[t] = g2[t] = 0.0;
                    g0[t] = inside ? __ldcg(G0 + gi) : 0.0;
                    continue;
                }
                const double2 g = __ldcg(G + gi);
                if constexpr (PRE) {  // (G1, G2) and G0 split once per plane
                    const double gz = __ldcg(G0 + gi);
                    g1[t] = inside ? g.x : 0.0;
                    g2[t] = inside ? g.y : 0.0;
                    g0[t] = inside ? gz : 0.0;
                } else {  // double-double plane, split on the fly (large domains)
                    g1[t] = g2[t] = g0[t] = 0.0;
                    if (inside) {
                        const double h = g.x * sc_e;  // exact (power of two)
                        g1[t] = rint(h);
                        const double r = (h - g1[t]) * S;  // exact: |h - g1| <= 1/2
                        g2[t] = rint(r);
                        g0[t] = (r - g2[t]) + g.y * sc_e * S;
                    }
                }
            }
            const size_t o = (size_t)s * nmonp + gq + 8 * j0;
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                if (j0 + j >= NT) break;
                // fp32 numerator tables (exact: all order-3 numerators are integers
                // below 2^24): half the bytes of the B loads, which L1 must hold
                double bA, bB = 0.0, bF = 0.0;
                if constexpr (NSPLIT == 1) {
                    bA = (double)__ldg(numc + o + 8 * j);
                } else {
                    const float2 v = __ldg(reinterpret_cast<const float2 *>(numc) + o + 8 * j);  // (n1, n0)
                    bA = (double)v.x;
                    bB = (double)v.y;
                    bF = fma(bA, ssh, bB);  // the full numerator n = n1 2^sh + n0, exact (|n| < 2^53)
                }
#pragma unroll
                for (int t = 0; t < MT; ++t) {
                    if constexpr (I8) {
                        dmma(C[t][2][j], g0[t], NSPLIT == 1 ? bA : bF);
                        continue;
                    }
                    dmma(C[t][0][j], g1[t], bA);  // exact
                    dmma(C[t][1][j], g2[t], bA);  // exact
                    if constexpr (NSPLIT == 1) {
                        dmma(C[t][2][j], g0[t], bA);
                    } else {
                        dmma(C[t][2][j], g0[t], bF);
                        dmma(C[t][3][j], g1[t], bB);  // exact
                        dmma(C[t][4][j], g2[t], bB);  // exact
                    }
                }
            }
        }
        // rows over this pass's slots (lock step, as fused_rows), every m-tile
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            if (j0 + j >= NT) break;
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                const int k = 2 * (j0 + j) + h2;
                const bool start = (smask >> k) & 1, valid = (vmask >> k) & 1;
#pragma unroll
                for (int t = 0; t < MT; ++t) {
                    dd e;
                    if constexpr (I8) {
                        const double2 x = e12[(gq + 8 * t) * E12S + 8 * (j0 + j) + 2 * kq + h2];
                        e = dd_add_d(dd{x.x, x.y}, C[t][2][j][h2] * iS);
                    } else if constexpr (NSPLIT == 1) {
                        e = dd_add_d(two_sum(C[t][0][j][h2], C[t][1][j][h2] * iS), C[t][2][j][h2] * iS);
                    } else {
                        const dd x = two_sum(C[t][0][j][h2] * ssh, C[t][3][j][h2]);
                        const dd y = two_sum(C[t][1][j][h2] * ssh, C[t][4][j][h2]);
                        e = dd_add_d(dd_add(x, {y.hi * iS, y.lo * iS}), C[t][2][j][h2] * iS);
                    }
                    double nh = rh[t], nl = rl[t];
                    comp_step(nh, nl, fyt[t], e.hi, e.lo);
                    if (start) {
#pragma unroll
                        for (int qq = 0; qq < QMAX; ++qq)
                            if (qq == q) {
                                Rh[t][qq] = rh[t];
                                Rl[t][qq] = rl[t];
                            }
                    }
                    rh[t] = start ? e.hi : (valid ? nh : rh[t]);
                    rl[t] = start ? e.lo : (valid ? nl : rl[t]);
                }
                if (start) ++q;
            }
        }
    }
#pragma unroll
    for (int t = 0; t < MT; ++t) {
#pragma unroll
        for (int qq = 0; qq < QMAX; ++qq)
            if (qq == q) {
                Rh[t][qq] = rh[t];
                Rl[t][qq] = rl[t];
            }
        double ah, al;
        fused_xhorner<DEG, DEG>(Rh[t], Rl[t], fxt[t], ah, al);
        const dd F = fast_two_sum(ah, al);
        Fh[t] = F.hi;
        Fl[t] = F.lo;
    }
}

template <int R, bool SAME_SIGN>
__device__ bool sweep_plane(double2 *__restrict__ G, int NX, int NY, int X0, int Y0, int basis, const TileArgs &a,
                            int img, double2 *ring, size_t ring_bytes) {
    const int tid = threadIdx.x;
    const int nh = basis == BASIS_THETA ? R : 0;  // horizontal levels, done first
    const int L = 4 * R - nh;                    // levels in the sweep
    // levels per pass: as many as the ring holds (large halo domains take
    // several passes, each reading the previous pass' last level from G)
    const int LC = min(L, (int)(ring_bytes / ((size_t)3 * NX * sizeof(double2))));
    if (LC < 1) return false;
    const size_t ipl = (size_t)a.H * a.W;
    auto fval = [&](int x, int y) -> double {
        int X = X0 + x, Y = Y0 + y;
        if (a.replicate) {  // BSF_BOUNDARY_REPLICATE: the nearest image pixel
            X = min(max(X, 0), a.W - 1);
            Y = min(max(Y, 0), a.H - 1);
        } else if (X < 0 || X >= a.W || Y < 0 || Y >= a.H) {
            return 0.0;
        }
        const size_t o = (size_t)img * ipl + (size_t)Y * a.W + X;
        return load_f(a, o);
    };
    // a u8 image makes every running sum non-negative: the cheaper same-sign
    // double-double addition is then exact to 3u^2 (float input may be signed;
    // scanning the domain for signs cost more than it saved on config 2)
    auto add = [&](dd u, dd v) -> dd {
        if constexpr (SAME_SIGN)
            return dd_add_same_sign(u, v);
        else
            return dd_add(u, v);
    };
    // u8 input: the running sums are integers, and a level whose values stay
    // below 2^53 (255 x the product of the line lengths so far) is exact in
    // plain fp64 -- one DADD instead of a double-double addition.  Bit k of
    // exact_h / exact_v: horizontal level k / sweep level k is exact.
    unsigned exact_h = 0u, exact_v = 0u;
    if (a.in_u8) {
        double bound = 255.0;
        int k = 0;
        for (int j = 0; j < nh; ++j, ++k) {
            bound *= NX;
            if (bound < 0x1p53) exact_h |= 1u << j;
        }
        k = 0;
        for (int rep = 0; rep < R; ++rep)
            for (int lv = 0; lv < 4; ++lv) {
                const int sy = c_scan_order[basis][lv][1];
                if (sy == 0) continue;
                bound *= (double)(NY / sy + 1);
                if (bound < 0x1p53) exact_v |= 1u << k;
                ++k;
            }
    }
    if (nh && exact_h == (1u << nh) - 1u) {
        // every horizontal level exact in fp64: one warp per row, 32-column
        // chunks, a warp-shuffle inclusive scan per level and chunk
        const int lane = tid & 31, wid = tid >> 5;
        for (int y = wid; y < NY; y += FT / 32) {
            double carry[R];
#pragma unroll
            for (int k = 0; k < R; ++k) carry[k] = 0.0;
            for (int x0 = 0; x0 < NX; x0 += 32) {
                const int x = x0 + lane;
                double v = x < NX ? fval(x, y) : 0.0;
#pragma unroll
                for (int k = 0; k < R; ++k) {
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const double t = __shfl_up_sync(0xffffffffu, v, o);
                        if (lane >= o) v += t;
                    }
                    v += carry[k];  // exact: integers below 2^53
                    carry[k] = __shfl_sync(0xffffffffu, v, 31);
                }
                if (x < NX) G[(size_t)y * NX + x] = make_double2(v, 0.0);
            }
        }
        __syncthreads();
    } else if (nh) {
        for (int y = tid; y < NY; y += FT) {
            dd acc[R];
#pragma unroll
            for (int k = 0; k < R; ++k) acc[k] = {0.0, 0.0};
            for (int x = 0; x < NX; ++x) {
                acc[0] = (exact_h & 1u) ? dd{acc[0].hi + fval(x, y), 0.0} : dd_add_d(acc[0], fval(x, y));
#pragma unroll
                for (int k = 1; k < R; ++k)
                    acc[k] = ((exact_h >> k) & 1u) ? dd{acc[k].hi + acc[k - 1].hi, 0.0} : add(acc[k], acc[k - 1]);
                G[(size_t)y * NX + x] = make_double2(acc[R - 1].hi, acc[R - 1].lo);
            }
        }
        __syncthreads();
    }
    // level steps of the sweep, in scan order with the horizontal levels removed,
    // packed 4 bits per level in one register word (sx + 2 in bits 0-2, sy - 1
    // in bit 3): no local-memory array in the inner loop
    unsigned long long steps = 0ull;
    {
        int k = 0;
        for (int rep = 0; rep < R; ++rep)
            for (int lv = 0; lv < 4; ++lv) {
                const int sx = c_scan_order[basis][lv][0], sy = c_scan_order[basis][lv][1];
                if (sy == 0) continue;
                steps |= (unsigned long long)((sx + 2) | ((sy - 1) << 3)) << (4 * k);
                ++k;
            }
    }
    if (a.in_u8 && exact_v == (1u << L) - 1u) {
        // every level exact in fp64 (u8 input, moderate domain): the same sweep
        // on a ring of plain doubles -- half the shared-memory traffic, no
        // double-double arithmetic; G receives (value, 0)
        double *rd = reinterpret_cast<double *>(ring);
        const int LD = min(L, (int)(ring_bytes / ((size_t)3 * NX * sizeof(double))));
        for (int lb = 0; lb < L; lb += LD) {
            const int Lp = min(LD, L - lb);
            const unsigned long long pst = steps >> (4 * lb);
            const int work = Lp * NX;
            const int l0 = tid / NX, x0 = tid - l0 * NX, dl = FT / NX, dx = FT - dl * NX;
            for (int tau = 0; tau < NY + Lp - 1; ++tau) {
                int l = l0, x = x0;
                int ym = (tau - l0) % 3;
                if (ym < 0) ym += 3;
                for (int i = tid; i < work; i += FT) {
                    const int y = tau - l;
                    if (y >= 0 && y < NY) {
                        const unsigned st4 = (unsigned)(pst >> (4 * l)) & 15u;
                        const int sx = (int)(st4 & 7u) - 2, sy = (int)(st4 >> 3) + 1;
                        double below;
                        if (l == 0)
                            below = (nh || lb > 0) ? G[y * NX + x].x : fval(x, y);
                        else
                            below = rd[((l - 1) * 3 + ym) * NX + x];
                        const int yp = y - sy, xp = x - sx;
                        if (yp >= 0 && xp >= 0 && xp < NX) {
                            const int ypm = ym >= sy ? ym - sy : ym - sy + 3;
                            below += rd[(l * 3 + ypm) * NX + xp];  // exact: integers below 2^53
                        }
                        rd[(l * 3 + ym) * NX + x] = below;
                        if (l == Lp - 1) G[y * NX + x] = make_double2(below, 0.0);
                    }
                    l += dl;
                    ym -= dl % 3;
                    if (ym < 0) ym += 3;
                    x += dx;
                    if (x >= NX) {
                        x -= NX;
                        ++l;
                        ym = ym == 0 ? 2 : ym - 1;
                    }
                }
                __syncthreads();
            }
        }
        return true;
    }
    for (int lb = 0; lb < L; lb += LC) {
        const int Lp = min(LC, L - lb);  // levels lb .. lb + Lp - 1 in this pass
        const unsigned long long pst = steps >> (4 * lb);
        // flat (level, x) work list over the CTA; (l, x) advanced incrementally;
        // ring rows rotate mod 3: row y of level l lives in slot (l, y mod 3)
        const int work = Lp * NX;
        const int l0 = tid / NX, x0 = tid - l0 * NX, dl = FT / NX, dx = FT - dl * NX;
        for (int tau = 0; tau < NY + Lp - 1; ++tau) {
            int l = l0, x = x0;
            int ym = (tau - l0) % 3;  // y mod 3 for y = tau - l (>= 0 when used)
            if (ym < 0) ym += 3;
            for (int i = tid; i < work; i += FT) {
                const int y = tau - l;  // level lb + l processes row tau - l
                if (y >= 0 && y < NY) {
                    const unsigned st4 = (unsigned)(pst >> (4 * l)) & 15u;
                    const int sx = (int)(st4 & 7u) - 2, sy = (int)(st4 >> 3) + 1;
                    dd below;
                    if (l == 0) {
                        if (nh || lb > 0) {  // horizontal sums, or the previous pass' last level
                            const double2 t = G[y * NX + x];
                            below = {t.x, t.y};
                        } else {
                            below = {fval(x, y), 0.0};
                        }
                    } else {
                        const double2 t = ring[((l - 1) * 3 + ym) * NX + x];
                        below = {t.x, t.y};
                    }
                    const int yp = y - sy, xp = x - sx;
                    if (yp >= 0 && xp >= 0 && xp < NX) {
                        const int ypm = ym >= sy ? ym - sy : ym - sy + 3;
                        const double2 t = ring[(l * 3 + ypm) * NX + xp];
                        below = ((exact_v >> (lb + l)) & 1u) ? dd{below.hi + t.x, 0.0} : add(below, {t.x, t.y});
                    }
                    const double2 v = make_double2(below.hi, below.lo);
                    ring[(l * 3 + ym) * NX + x] = v;
                    if (l == Lp - 1) G[y * NX + x] = v;
                }
                l += dl;
                ym -= dl % 3;
                if (ym < 0) ym += 3;
                x += dx;
                if (x >= NX) {
                    x -= NX;
                    ++l;
                    ym = ym == 0 ? 2 : ym - 1;
                }
            }
            __syncthreads();
        }
    }
    return true;
}

// GLOBAL (order 1, u8 input): no per-super-tile pre-integration -- the taps
// read the paper's single global pre-integration (Alg. 3
// step 2), the exact int64 running sums of bsf_preintegrate_exact, through
// GlobSrc; phases 2-3 are skipped and both contraction limbs are exact.
template <int R, bool SPLIT, bool GLOBAL = false, bool I8 = false>
__global__ void __launch_bounds__(FT, 1) fused_kernel(TileArgs a, const LutBasis *__restrict__ luts) {
    constexpr int NTAP = FusedCfg<R>::NTAP, P = FusedCfg<R>::P, ITEMS = P * NTAP;
    constexpr int MT = FusedCfg<R>::MT, GS = 8 * MT;
    extern __shared__ __align__(16) unsigned char smem[];
    double2 *s_F = a.fbuf + (size_t)blockIdx.x * ITEMS;  // global, L2-resident (see fused_items)
    double *s_scl = a.sbuf + (size_t)blockIdx.x * FUSED_NQ_MAX * FT * 5;  // per-pixel scales of the super-tile
    double *s_ap = reinterpret_cast<double *>(smem);
    double2 *s_tv = reinterpret_cast<double2 *>(s_ap + FT * 4);  // [pixel][5]: s_k a'_k (k < 4), centre
    uint16_t *s_key = reinterpret_cast<uint16_t *>(s_tv + FT * 5);
    uint16_t *s_sorted = s_key + ITEMS;
    int *s_hist = reinterpret_cast<int *>(s_sorted + ITEMS + GS * NKEY);  // [warp][key]
    int *s_info = s_hist + (FT / 32) * NKEY;
    __shared__ int s_item, s_ex[2], s_ey[2], s_vmask[2], s_bad, s_npad, s_any, s_nfb, s_quad;
    __shared__ int s_one[NPLANE];  // plane is its own exact split (u8, order 1): single-limb MMA
    __shared__ short s_fb[FT];
    __shared__ int s_dom[2][4];
    __shared__ long long s_poff[NPLANE];
    __shared__ int s_pe[NPLANE];
    __shared__ unsigned long long s_pmax[NPLANE];
    __shared__ ClsTables s_cls;
    __shared__ unsigned long long s_stats[8];  // per-CTA statistics, flushed once per super-tile

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 8) s_stats[tid] = 0ull;
    if (tid < 2) {
        const LutBasis &L = luts[tid];
        for (int k = 0; k < 4; ++k) {
            s_cls.normal[tid][k] = L.normal[k];
            s_cls.kmin[tid][k] = L.kmin[k];
            s_cls.radix[tid][k] = L.radix[k];
        }
        for (int i = 0; i < 81; ++i) s_cls.table[tid][i] = L.table[i];
    }
    // order 3, i8 route: 512 TMEM columns (accumulator classes 0..447, the A
    // slices 448..503) and the two mbarriers of i8_tile
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_i8bar[2];
    uint32_t i8_pa = 0, i8_pm = 0;  // mbarrier phases (every thread tracks them)
    if constexpr (I8) {
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_i8bar[0]))
                         : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_i8bar[1]))
                         : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(&s_tmem))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    __syncthreads();
    if constexpr (I8) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // optional phase timing (TileArgs::prof, diagnostics only): thread 0 adds
    // the SM cycles spent in each phase
    long long ph_t = clock64(), t_item = ph_t;
#define FUSED_PHASE(k)                                        \
    if (a.prof && tid == 0) {                                 \
        const long long t_ = clock64();                       \
        atomicAdd(a.prof + (k), (unsigned long long)(t_ - ph_t)); \
        ph_t = t_;                                            \
    }
    double2 *scr = a.scratch + (size_t)blockIdx.x * NPLANE * a.cap;
    double *scr0 = R >= 3 ? a.scratch0 + (size_t)blockIdx.x * NPLANE * a.cap : nullptr;  // G0 planes (order 3)
    // super-tile of ST x ST pixels = SQ x SQ sub-tiles of TILE x TILE (ST = 32 or 64, per plan)
    const int ST = a.stile, SQ = ST / TILE, NQ = SQ * SQ;
    // super-tile rows of the output window (all rows unless a row strip)
    const int sty0 = a.oy0 / ST;
    const int nstx = (a.W + ST - 1) / ST, nsty = (min(a.H, a.oy0 + out_rows(a)) + ST - 1) / ST - sty0;
    const int stiles_per_img = nstx * nsty;
    // work units: points, super-tiles, or in split mode the unit count the
    // order kernel wrote (quadrant units included)
    int nitems = a.pts ? a.npts : a.tiles ? a.ntiles : stiles_per_img * a.nimg;
    if constexpr (SPLIT) nitems = (int)__ldcg(a.order_hist + 2 * SCHED_NBIN);
    const size_t ipl = (size_t)a.H * a.W;

    for (;;) {
        if (tid == 0) {
            s_item = atomicAdd(a.counter, 1);
            // split mode: >= 0 when the unit is only this quadrant of the super-tile
            if constexpr (SPLIT) s_quad = s_item < nitems ? (__ldcg(a.order + s_item) & 7) - 1 : -1;
            s_ex[0] = s_ex[1] = s_ey[0] = s_ey[1] = 0;
            s_vmask[0] = s_vmask[1] = 0;
            s_bad = 0;
        }
        if (tid < NPLANE) s_pmax[tid] = 0ull;
        if (tid == 0) s_nfb = 0;
        __syncthreads();
        if (s_item >= nitems) break;
        const int unit = s_item;  // hand-out index (diagnostics are keyed by it: unique in split mode too)
        int item = a.tiles ? a.tiles[s_item] : (a.order && !a.pts ? a.order[s_item] : s_item);
        if constexpr (SPLIT) item >>= 3;  // unit code: super-tile << 3 | quadrant
        // sub-tile q of the super-tile belongs to this unit (always, unless split mode)
        auto qin = [&](int q) {
            if constexpr (!SPLIT) return true;
            const int qd = s_quad;
            return qd < 0 || ((2 * (q % SQ) >= SQ) == (qd & 1) && (2 * (q / SQ) >= SQ) == (qd >> 1));
        };
        if (a.prof && tid == 0) ph_t = t_item = clock64();
        // super-tile origin (X0s, Y0s): the running sums are anchored on its
        // halo domain; its four TILE x TILE sub-tiles are gathered in turn
        int img, X0s, Y0s, want = -1, qwant = -1;
        if (a.pts) {
            img = a.pts[3 * item];
            const int px = a.pts[3 * item + 1], py = a.pts[3 * item + 2];
            X0s = px & ~(ST - 1);
            Y0s = py & ~(ST - 1);
            qwant = (px - X0s) / TILE + SQ * ((py - Y0s) / TILE);
            want = (px & (TILE - 1)) + TILE * (py & (TILE - 1));
        } else {
            img = item / stiles_per_img;
            const int rem = item % stiles_per_img;
            X0s = (rem % nstx) * ST;
            Y0s = (sty0 + rem / nstx) * ST;
        }

        if (a.cov_mode == COV_ISO && !(a.sigma2[img / a.channels] > 0.0)) {
            // Algorithm 1 with sigma_b = 0: the isotropic pass is the identity
            for (int q = 0; q < NQ; ++q) {
                const int x = X0s + TILE * (q % SQ) + (tid % TILE), y = Y0s + TILE * (q / SQ) + tid / TILE;
                const bool mine = a.pts ? (q == qwant && tid == want) : (x < a.W && out_row(a, y) && qin(q));
                if (mine) {
                    const double v = load_f(a, (size_t)img * ipl + (size_t)y * a.W + x);
                    const long long oidx = a.pts ? item : out_index(a, img, x, y);
                    if (a.out_f32 && !a.pts)
                        ((float *)a.out)[oidx] = (float)v;
                    else
                        ((double *)a.out)[oidx] = v;
                }
            }
            __syncthreads();
            continue;
        }
        // ---- 1. reach of every pixel of the super-tile (a1-a4) -------------------
#pragma unroll 1
        for (int q = 0; q < NQ; ++q) {
            const int x = X0s + TILE * (q % SQ) + (tid % TILE), y = Y0s + TILE * (q / SQ) + tid / TILE;
            double *sb = s_scl + ((size_t)q * FT + tid) * 5;  // this pixel's scales, reused by its sub-tile
            if (x < a.W && out_row(a, y) && qin(q)) {
                PixelScales ps;
                double sx, sy, th;
                load_cov(a, img, x, y, sx, sy, th);
                pixel_scales(sx, sy, th, a.policy, a.clamp, R, ps);
#pragma unroll
                for (int k = 0; k < 4; ++k) sb[k] = ps.ap[k];
                sb[4] = (double)(ps.basis | ((ps.drop + 1) << 1) | (ps.clamped ? 32 : 0) | (ps.flags << 8));
                if (!(ps.flags & (FLAG_INFEASIBLE | FLAG_TWO_ZERO))) {
                    double ex = 0.0, ey = 0.0;
                    for (int k = 0; k < 4; ++k) {
                        ex += ps.ap[k] * abs(c_steps[ps.basis][k][0]);
                        ey += ps.ap[k] * c_steps[ps.basis][k][1];
                    }
                    atomicMax(&s_ex[ps.basis], (int)ceil(0.5 * R * ex));
                    atomicMax(&s_ey[ps.basis], (int)ceil(0.5 * R * ey));
                    atomicOr(&s_vmask[ps.basis], 1 << (ps.drop + 1));
                }
            }
        }
        __syncthreads();
        FUSED_PHASE(0);

        if constexpr (GLOBAL) {
            // the global running sums: domain x in [-P, W+P), y in [0, H+Pb)
            if (tid < 2) {
                s_dom[tid][0] = -a.gP;
                s_dom[tid][1] = 0;
                s_dom[tid][2] = a.gGW;
                s_dom[tid][3] = a.gGH;
            }
            if (tid < NPLANE) {
                const int b = tid / NVAR, v = tid % NVAR;
                s_pe[tid] = a.gshift[b];
                s_one[tid] = 0;
                s_poff[tid] = ((s_vmask[b] >> v) & 1) ? 0 : -1;
            }
            __syncthreads();
            FUSED_PHASE(2);
        } else {
        // ---- 2. pre-integration planes ------------------------------------------
        if (tid == 0) {
            int np = 0;
            for (int b = 0; b < 2; ++b) {
                TileDomain d;
                if constexpr (SPLIT) {  // a quadrant unit: its own 32 x 32 anchoring
                    const int qd = s_quad, hs = qd < 0 ? 0 : ST / 2;
                    d = fused_domain(luts[b], R, X0s + hs * (qd & 1), Y0s + hs * (qd >> 1), s_ex[b], s_ey[b],
                                     qd < 0 ? ST : hs);
                } else {
                    d = fused_domain(luts[b], R, X0s, Y0s, s_ex[b], s_ey[b], ST);
                }
                s_dom[b][0] = d.X0;
                s_dom[b][1] = d.Y0;
                s_dom[b][2] = d.NX;
                s_dom[b][3] = d.NY;
                // each plane is preceded by -wymin zero rows: window reads above
                // the domain (zero state) need no bounds check
                const int pad = -luts[b].wymin;
                for (int v = 0; v < NVAR; ++v) {
                    bool need = (s_vmask[b] >> v) & 1;
                    if (v == 0 && s_vmask[b]) need = true;  // the base plane feeds the variants
                    s_poff[b * NVAR + v] = need ? (long long)(np++) * a.cap + (long long)pad * d.NX : -1;
                }
                if (s_vmask[b] && (long long)d.NX * (d.NY + pad) > a.cap) s_bad = 1;
            }
        }
        __syncthreads();
        if (s_bad) {
            // domain exceeds the plan's capacity: NaN for every pixel (cannot
            // happen when max_sigma bounds the covariance field)
            for (int q = 0; q < NQ; ++q) {
                const int x = X0s + TILE * (q % SQ) + (tid % TILE), y = Y0s + TILE * (q / SQ) + tid / TILE;
                const bool mine = a.pts ? (q == qwant && tid == want) : (x < a.W && out_row(a, y) && qin(q));
                if (mine) {
                    const long long oidx = a.pts ? item : out_index(a, img, x, y);
                    if (a.out_f32 && !a.pts)
                        ((float *)a.out)[oidx] = __int_as_float(0x7fc00000);
                    else
                        ((double *)a.out)[oidx] = __longlong_as_double(0x7ff8000000000000LL);
                    if (a.stats) atomicOr(a.stats + 4, (unsigned long long)FLAG_RANGE);
                }
            }
            __syncthreads();
            continue;
        }
        for (int pi = 0; pi < NPLANE; ++pi) {
            const int b = pi / NVAR;
            if (s_poff[pi] < 0) continue;
            const int n = -luts[b].wymin * s_dom[b][2];
            double2 *P0 = scr + s_poff[pi] - n;
            for (int i = tid; i < n; i += FT) P0[i] = make_double2(0.0, 0.0);
            if constexpr (R >= 3) {
                double *Q0 = scr0 + s_poff[pi] - n;
                for (int i = tid; i < n; i += FT) Q0[i] = 0.0;
            }
        }
        for (int b = 0; b < 2; ++b) {
            if (!s_vmask[b]) continue;
            const int X0 = s_dom[b][0], Y0 = s_dom[b][1], NX = s_dom[b][2], NY = s_dom[b][3];
            double2 *G = scr + s_poff[b * NVAR];
            const int n = NX * NY;
            // wavefront sweep with its ring in the (idle) dynamic shared memory;
            // level-by-level scans when the ring does not fit
            const bool swept = a.in_u8 ? sweep_plane<R, true>(G, NX, NY, X0, Y0, b, a, img,
                                                                reinterpret_cast<double2 *>(smem), fused_smem_bytes<R>())
                                       : sweep_plane<R, false>(G, NX, NY, X0, Y0, b, a, img,
                                                                 reinterpret_cast<double2 *>(smem), fused_smem_bytes<R>());
            if (!swept) {
                for (int i = tid; i < n; i += FT) {
                    int X = X0 + i % NX, Y = Y0 + i / NX;
                    double v = 0.0;
                    if (a.replicate) {
                        X = min(max(X, 0), a.W - 1);
                        Y = min(max(Y, 0), a.H - 1);
                    }
                    if (X >= 0 && X < a.W && Y >= 0 && Y < a.H) {
                        const size_t o = (size_t)img * ipl + (size_t)Y * a.W + X;
                        v = load_f(a, o);
                    }
                    G[i] = make_double2(v, 0.0);
                }
                __syncthreads();
                for (int rep = 0; rep < R; ++rep)
                    for (int lv = 0; lv < 4; ++lv) {
                        tile_scan_level(G, NX, NY, c_scan_order[b][lv][0], c_scan_order[b][lv][1]);
                        __syncthreads();
                    }
            }
            __syncthreads();
            FUSED_PHASE(11);  // diagnostics: sweep of basis b
            // zero-scale variants: G' = (1 - T_{s_k})^R G, exact lattice difference (R5);
            // integer planes below 2^53 (u8 input) take plain fp64 arithmetic
            const bool exact_plane =
                a.in_u8 && u8_plane_bound(b, R, NX, NY) * (double)(1 << R) < 0x1p53;
            for (int v = 1; v < NVAR; ++v) {
                if (!((s_vmask[b] >> v) & 1)) continue;
                const int sx = c_steps[b][v - 1][0], sy = c_steps[b][v - 1][1];
                double2 *D = scr + s_poff[b * NVAR + v];
                if (exact_plane) {
                    for (int Y = 0; Y < NY; ++Y)
                        for (int X = tid; X < NX; X += FT) {
                            double acc = 0.0;
#pragma unroll
                            for (int m = 0; m <= R; ++m) {
                                const int yy = Y - m * sy, xx = X - m * sx;
                                if (yy < 0 || xx < 0 || xx >= NX) continue;
                                acc += (double)(binomR<R>(m) * ((m & 1) ? -1 : 1)) * G[yy * NX + xx].x;
                            }
                            D[Y * NX + X] = make_double2(acc, 0.0);
                        }
                    continue;
                }
                for (int i = tid; i < n; i += FT) {
                    const int X = i % NX, Y = i / NX;
                    dd acc = {0.0, 0.0};
#pragma unroll
                    for (int m = 0; m <= R; ++m) {
                        const int yy = Y - m * sy, xx = X - m * sx;
                        if (yy < 0 || xx < 0 || xx >= NX) continue;
                        const double2 t = G[(size_t)yy * NX + xx];
                        const int cb = binomR<R>(m) * ((m & 1) ? -1 : 1);
                        acc = dd_add(acc, dd_mul_d({t.x, t.y}, (double)cb));
                    }
                    D[i] = make_double2(acc.hi, acc.lo);
                }
            }
        }
        __syncthreads();
        FUSED_PHASE(12);  // diagnostics: zero-scale variant planes (remainder of phase 1)

        // ---- 3. exact split G = 2^e (G1 + G0) of every plane that is read --------
        if (tid < NPLANE) {
            const int b = tid / NVAR, v = tid % NVAR;
            bool one = false;
            if constexpr (R == 1) {
                const double bnd = u8_plane_bound(b, R, s_dom[b][2], s_dom[b][3]) * (v ? (double)(1 << R) : 1.0);
                one = a.in_u8 && bnd < ldexp(1.0, min(53, luts[b].var[v].kbits));
            }
            s_one[tid] = one;
        }
        __syncthreads();
        for (int pi = 0; pi < NPLANE; ++pi) {
            const int b = pi / NVAR, v = pi % NVAR;
            if (!((s_vmask[b] >> v) & 1) || s_one[pi]) continue;
            const double2 *G = scr + s_poff[pi];
            const int n = s_dom[b][2] * s_dom[b][3];
            double m = 0.0;
            for (int i = tid; i < n; i += FT) m = fmax(m, fabs(G[i].x));
            for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) atomicMax(&s_pmax[pi], (unsigned long long)__double_as_longlong(m));
        }
        __syncthreads();
        if (tid < NPLANE) {
            const double m = __longlong_as_double((long long)s_pmax[tid]);
            const int b = tid / NVAR, v = tid % NVAR;
            s_pe[tid] = (m > 0.0 && !s_one[tid]) ? ilogb(m) + 1 - luts[b].var[v].kbits : 0;
        }
        __syncthreads();
        if constexpr (R >= 3) {
            // three limbs G = 2^e (G1 + 2^-k G2 + 2^-k G0) (fused_group_g3): (G1, G2)
            // in place of the double-double value, G0 in its own plane
            for (int pi = 0; pi < NPLANE; ++pi) {
                const int b = pi / NVAR, v = pi % NVAR;
                if (!((s_vmask[b] >> v) & 1)) continue;
                const int n = s_dom[b][2] * s_dom[b][3];
                if (n > G3_PRESPLIT_MAX) continue;  // large domain: split on the fly
                double2 *G = scr + s_poff[pi];
                double *G0p = scr0 + s_poff[pi];
                const double sc = ldexp(1.0, -s_pe[pi]), S = ldexp(1.0, luts[b].var[v].kbits);
                for (int i = tid; i < n; i += FT) {
                    const double2 g = G[i];
                    const double h = g.x * sc;  // exact (power of two)
                    const double g1 = rint(h);
                    const double r = (h - g1) * S;  // exact: |h - g1| <= 1/2
                    const double g2 = rint(r);
                    G[i] = make_double2(g1, g2);
                    G0p[i] = (r - g2) + g.y * sc * S;
                }
            }
        }
        for (int pi = 0; pi < NPLANE; ++pi) {
            if constexpr (R >= 3) break;  // order >= 3: above
            const int b = pi / NVAR, v = pi % NVAR;
            if (!((s_vmask[b] >> v) & 1) || s_one[pi]) continue;  // s_one: already (G, 0)
            double2 *G = scr + s_poff[pi];
            const int n = s_dom[b][2] * s_dom[b][3];
            const double sc = ldexp(1.0, -s_pe[pi]);
            for (int i = tid; i < n; i += FT) {
                const double2 g = G[i];
                const double h = g.x * sc;      // exact (power of two)
                const double g1 = rint(h);      // |g1| <= 2^kbits
                G[i] = make_double2(g1, (h - g1) + g.y * sc);  // h - g1 exact
            }
        }
        __syncthreads();
        FUSED_PHASE(2);

        }  // !GLOBAL

        // ---- sub-tiles: per-pixel scales, then 4-5 ------------------------------
#pragma unroll 1
        for (int q = 0; q < NQ; ++q) {
        if ((a.pts && q != qwant) || !qin(q)) continue;
        const int x0 = X0s + TILE * (q % SQ), y0 = Y0s + TILE * (q / SQ);
        {
            const int x = x0 + (tid % TILE), y = y0 + tid / TILE;
            PixelScales ps;
            ps.flags = 0;
            ps.basis = 0;
            ps.drop = -1;
            ps.clamped = 0;
            ps.ap[0] = ps.ap[1] = ps.ap[2] = ps.ap[3] = 0.0;
            const bool valid = x < a.W && out_row(a, y);
            if (valid) {  // the scales solved in the reach pass (same thread, same pixel)
                const double *sb = s_scl + ((size_t)q * FT + tid) * 5;
#pragma unroll
                for (int k = 0; k < 4; ++k) ps.ap[k] = sb[k];
                const int w = (int)sb[4];
                ps.basis = w & 1;
                ps.drop = ((w >> 1) & 7) - 1;
                ps.clamped = (w >> 5) & 1;
                ps.flags = w >> 8;
            }
            const bool live = valid && !(ps.flags & (FLAG_INFEASIBLE | FLAG_TWO_ZERO));
            s_info[tid] = ps.basis | ((ps.drop + 1) << 1) | (live ? 16 : 0) | (ps.clamped ? 32 : 0) | (ps.flags << 8);
#pragma unroll
            for (int k = 0; k < 4; ++k) s_ap[tid * 4 + k] = ps.ap[k];
            // tap geometry: v_k = s_k a'_k and the centre sum_{k != drop} (R/2) v_k,
            // so tap j has D = centre - sum_k j_k v_k (all exact on the 2^-41 grid, R17)
            double cx = 0.0, cy = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double vx = c_steps[ps.basis][k][0] * ps.ap[k], vy = c_steps[ps.basis][k][1] * ps.ap[k];
                s_tv[tid * 5 + k] = make_double2(vx, vy);
                if (k != ps.drop) {
                    cx += (0.5 * R) * vx;
                    cy += (0.5 * R) * vy;
                }
            }
            s_tv[tid * 5 + 4] = make_double2(cx, cy);
        }
        __syncthreads();
        // ---- 4-5. taps bucketed by key, gather, per-pixel sums -------------------
        // Items are numbered tap-major, i = t * P + p (p the pixel within the
        // chunk), and bucketed by a STABLE counting sort, so a 16-lane group
        // holds the same tap of neighbouring pixels: their G reads are adjacent.
        constexpr int WPR = ((ITEMS + FT / 32 - 1) / (FT / 32) + 31) & ~31;  // items per warp range
        for (int c0 = 0; c0 < FT; c0 += P) {
            if (tid == 0) s_any = 0;
            __syncthreads();
            if (tid >= c0 && tid < c0 + P && info_live(s_info[tid]) && (!a.pts || tid == want)) s_any = 1;
            for (int k = tid; k < (FT / 32) * NKEY; k += FT) s_hist[k] = 0;
            __syncthreads();
            if (!s_any) continue;  // uniform
            FUSED_PHASE(8);
            // keys of all items (item i = t P + pixel): each thread keeps one
            // pixel's geometry in registers and walks its taps (t0, t0 + FT/P,
            // ...); the tap loop is unrolled so several chains overlap ...
            static_assert(FT % P == 0 || P % FT == 0, "chunk and block sizes must nest");
            constexpr int TSTEP = FT >= P ? FT / P : 1;
            if constexpr (TSTEP == 1 && R <= 2) {
                // one pixel per thread, its taps in order: the tap positions
                // D_t = centre - sum_k j_k v_k and the knot-line coordinates
                // U_m = n_m . D_t are walked incrementally (odometer over the
                // digits j_k, fully unrolled: every step is known at compile
                // time); all values are exact (R17: the 2^-41 grid, |n_m| small),
                // so floor(n_m . phi) = floor(U_m) - n_m . floor(D) equals the
                // direct classification of cls_region bit for bit
#pragma unroll 1
                for (int pl = tid % P; pl < P; pl += FT) {
                    const int p = c0 + pl;
                    const int w = s_info[p];
                    const int var = info_var(w);
                    const int ntap = var ? NTAP / (R + 1) : NTAP;
                    const bool live = info_live(w) && (!a.pts || p == want);
                    const int b = info_basis(w);
                    const int drop = var - 1;
                    // digit i's direction: the i-th non-dropped k
                    double2 dv[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int k = (drop >= 0 && i >= drop) ? min(i + 1, 3) : i;
                        dv[i] = s_tv[5 * p + k];
                    }
                    const double2 cen = s_tv[5 * p + 4];
                    int nx[4], ny[4], km[4], rx[4];
                    double U[4], cu[4][4];
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        nx[m] = s_cls.normal[b][m].x;
                        ny[m] = s_cls.normal[b][m].y;
                        km[m] = s_cls.kmin[b][m];
                        rx[m] = s_cls.radix[b][m];
                        U[m] = nx[m] * cen.x + ny[m] * cen.y;
#pragma unroll
                        for (int i = 0; i < 4; ++i) cu[i][m] = nx[m] * dv[i].x + ny[m] * dv[i].y;
                    }
                    double Dx = cen.x, Dy = cen.y;
#pragma unroll
                    for (int t = 0; t < NTAP; ++t) {
                        uint16_t key = NOKEY;
                        if (live && t < ntap) {
                            const double flx = floor(Dx), fly = floor(Dy);
                            const int ix = (int)flx, iy = (int)fly;
                            int idx = 0, mul = 1;
                            bool in = true;
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                const int f = (int)floor(U[m]) - (nx[m] * ix + ny[m] * iy) - km[m];
                                in = in && f >= 0 && f < rx[m];
                                idx += f * mul;
                                mul *= rx[m];
                            }
                            int reg = in ? s_cls.table[b][idx] : -1;
                            if (reg < 0) reg = cls_region(s_cls, b, Dx - flx, Dy - fly);  // knot lines
                            key = (uint16_t)((b * NVAR + var) * MAX_REG + reg);
                        }
                        s_key[t * P + pl] = key;
                        if (t + 1 < NTAP) {
                            // odometer step t -> t + 1: digits at R wrap to 0, the next one increments
                            int tt = t;
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                if (tt % (R + 1) < R) {
                                    Dx -= dv[i].x;
                                    Dy -= dv[i].y;
#pragma unroll
                                    for (int m = 0; m < 4; ++m) U[m] -= cu[i][m];
                                    break;
                                }
                                Dx += R * dv[i].x;
                                Dy += R * dv[i].y;
#pragma unroll
                                for (int m = 0; m < 4; ++m) U[m] += R * cu[i][m];
                                tt /= (R + 1);
                            }
                        }
                    }
                }
            } else {
#pragma unroll 1
                for (int pl = tid % P; pl < P; pl += (FT >= P ? P : FT)) {
                    const int p = c0 + pl;
                    const int w = s_info[p];
                    const int var = info_var(w);
                    const int ntap = var ? NTAP / (R + 1) : NTAP;
                    const bool live = info_live(w) && (!a.pts || p == want);
                    const int b = info_basis(w);
                    double2 tv[5];
#pragma unroll
                    for (int k = 0; k < 5; ++k) tv[k] = s_tv[5 * p + k];
#pragma unroll 4
                    for (int t = (FT >= P ? tid / P : 0); t < NTAP; t += TSTEP) {
                        uint16_t key = NOKEY;
                        if (live && t < ntap) {
                            double Dx, Dy;
                            fused_tap_v<R>(tv, var - 1, t, Dx, Dy);
                            const int reg = cls_region(s_cls, b, Dx - floor(Dx), Dy - floor(Dy));
                            key = (uint16_t)((b * NVAR + var) * MAX_REG + reg);
                        }
                        s_key[t * P + pl] = key;
                    }
                }
            }
            __syncthreads();
            // ... then per-warp histograms (warp w owns items [w*WPR, (w+1)*WPR))
            for (int base = warp * WPR; base < min(ITEMS, (warp + 1) * WPR); base += 32) {
                const int i = base + lane;
                const uint16_t key = i < ITEMS ? s_key[i] : NOKEY;
                const unsigned m = __match_any_sync(0xffffffffu, key);
                if (key != NOKEY && lane == __ffs(m) - 1) s_hist[warp * NKEY + key] += __popc(m);
                __syncwarp();
            }
            __syncthreads();
            FUSED_PHASE(9);
            // bucket starts (each bucket padded to a multiple of GS) and per-warp offsets
            if (warp == 0) {
                constexpr int PER = NKEY / 32;
                int loc = 0;
#pragma unroll
                for (int q = 0; q < PER; ++q) {
                    int tot = 0;
#pragma unroll
                    for (int w = 0; w < FT / 32; ++w) tot += s_hist[w * NKEY + lane * PER + q];
                    loc += (tot + GS - 1) / GS * GS;
                }
                int inc = loc;
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += t;
                }
                int run = inc - loc;
#pragma unroll
                for (int q = 0; q < PER; ++q) {
                    const int k = lane * PER + q;
                    int o = run;
#pragma unroll
                    for (int w = 0; w < FT / 32; ++w) {
                        const int h = s_hist[w * NKEY + k];
                        s_hist[w * NKEY + k] = o;
                        o += h;
                    }
                    run += (o - run + GS - 1) / GS * GS;
                }
                if (lane == 31) s_npad = inc;
            }
            __syncthreads();
            FUSED_PHASE(10);
            const int npad = s_npad;
            for (int i = tid; i < npad; i += FT) s_sorted[i] = NOKEY;
            __syncthreads();
            for (int base = warp * WPR; base < min(ITEMS, (warp + 1) * WPR); base += 32) {
                const int i = base + lane;
                const uint16_t key = i < ITEMS ? s_key[i] : NOKEY;
                const unsigned m = __match_any_sync(0xffffffffu, key);
                const int rank = __popc(m & ((1u << lane) - 1u));
                if (key != NOKEY) s_sorted[s_hist[warp * NKEY + key] + rank] = (uint16_t)i;
                __syncwarp();
                if (key != NOKEY && lane == __ffs(m) - 1) s_hist[warp * NKEY + key] += __popc(m);
                __syncwarp();
            }
            __syncthreads();
            FUSED_PHASE(3);
            // gather: groups of GS items sharing one key, one warp per group,
            // contraction on the FP64 tensor cores, polynomial from the fragments
            if constexpr (I8 && R == 3) {
#include "bsf_i8_gather.cuh"
            } else {
                const int ngroups = npad / GS;
                int flags = 0;
                for (int g = warp; g < ngroups; g += FT / 32) {
                    const int i0 = s_sorted[g * GS];
                    const int key = s_key[i0];
                    const int b = key / (NVAR * MAX_REG), var = (key / MAX_REG) % NVAR, reg = key % MAX_REG;
                    int idx = lane < GS ? s_sorted[g * GS + lane] : NOKEY;
                    const bool real = idx != NOKEY;
                    if (!real) idx = i0;  // dummy lanes repeat the group's first item
                    const int p = c0 + idx % P, t = idx / P;
                    double Dx, Dy;
                    fused_tap_v<R>(s_tv + 5 * p, var - 1, t, Dx, Dy);
                    const double flx = floor(Dx), fly = floor(Dy);
                    const int bx = x0 + (p % TILE) + (int)flx - s_dom[b][0];
                    const int by = y0 + p / TILE + (int)fly - s_dom[b][1];
                    const double fx = Dx - flx, fy = Dy - fly;
                    int bxt[MT], byt[MT];
#pragma unroll
                    for (int q = 0; q < MT; ++q) {
                        const int src = (lane >> 2) + 8 * q;
                        bxt[q] = __shfl_sync(0xffffffffu, bx, src);
                        byt[q] = __shfl_sync(0xffffffffu, by, src);
                    }
                    const double2 *G = scr + s_poff[b * NVAR + var];
                    const LutVar &V = luts[b].var[var];
                    const int n4 = (__ldg(V.counts + reg) + 3) & ~3;
                    const int NX = s_dom[b][2], NY = s_dom[b][3];
                    const int2 *offs = V.offs4 + (size_t)reg * V.nslot4;
                    const double *num = V.num + (size_t)reg * V.nslot4 * V.nmonp;
                    double Fh[MT], Fl[MT];
                    if (a.stats) {  // algorithmic work: window x monomials per real item
                        const unsigned nreal = __popc(__ballot_sync(0xffffffffu, real));
                        if (lane == 0)
                            atomicAdd(&s_stats[6], (unsigned long long)nreal * __ldg(V.counts + reg) *
                                                       (var == 0 ? DegCfg<4 * R - 2>::NMON : DegCfg<3 * R - 2>::NMON));
                    }
                    if (a.prof) {  // diagnostics: group fill, executed (padded) MMA MACs per limb
                        const unsigned nreal = __popc(__ballot_sync(0xffffffffu, real));
                        if (lane == 0) {
                            atomicAdd(a.prof + 13, (unsigned long long)GS * n4 * V.nmonp);
                            atomicAdd(a.prof + 14, (unsigned long long)nreal);
                            atomicAdd(a.prof + 15, (unsigned long long)GS);
                        }
                    }
                    long long tq0 = 0;
                    if (a.prof && lane == 0) tq0 = clock64();
                    if constexpr (R >= 3) {
                        // three G limbs from the double-double plane (MT = 1)
                        const size_t ro = (size_t)reg * V.nslot4 * V.nmonp;
                        const double *G0 = scr0 + s_poff[b * NVAR + var];
                        const double sce = ldexp(1.0, -s_pe[b * NVAR + var]);
                        const bool pre = NX * NY <= G3_PRESPLIT_MAX;
                        if (V.nsplit == 2) {
                            const float *nc = V.num32 + 2 * ro;  // (n1, n0) pairs
                            if (var == 0)
                                (pre ? (fused_group_g3<4 * R - 2, 2, BSF_G3_NP2, MT, true>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                             V.nmonp, n4, V.shift, G0, sce, V.kbits, Fh,
                                                                             Fl, flags)) : (fused_group_g3<4 * R - 2, 2, BSF_G3_NP2, MT, false>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                             V.nmonp, n4, V.shift, G0, sce, V.kbits, Fh,
                                                                             Fl, flags)));
                            else
                                (pre ? (fused_group_g3<3 * R - 2, 2, BSF_G3_NP2, MT, true>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                             V.nmonp, n4, V.shift, G0, sce, V.kbits, Fh,
                                                                             Fl, flags)) : (fused_group_g3<3 * R - 2, 2, BSF_G3_NP2, MT, false>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                             V.nmonp, n4, V.shift, G0, sce, V.kbits, Fh,
                                                                             Fl, flags)));
                        } else {
                            const float *nc = V.num32 + ro;
                            if (var == 0)
                                (pre ? (fused_group_g3<4 * R - 2, 1, BSF_G3_NP1, MT, true>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                             V.nmonp, n4, 0, G0, sce, V.kbits, Fh, Fl,
                                                                             flags)) : (fused_group_g3<4 * R - 2, 1, BSF_G3_NP1, MT, false>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                             V.nmonp, n4, 0, G0, sce, V.kbits, Fh, Fl,
                                                                             flags)));
                            else
                                (pre ? (fused_group_g3<3 * R - 2, 1, BSF_G3_NP1, MT, true>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                             V.nmonp, n4, 0, G0, sce, V.kbits, Fh, Fl,
                                                                             flags)) : (fused_group_g3<3 * R - 2, 1, BSF_G3_NP1, MT, false>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                             V.nmonp, n4, 0, G0, sce, V.kbits, Fh, Fl,
                                                                             flags)));
                        }
                    } else if (GLOBAL) {
                        const int k = s_pe[b * NVAR + var];
                        const GlobSrc gs{a.gglob[b] + (size_t)img * a.gGH * a.gGW, a.gGW, a.gGH, k,
                                         var ? c_steps[b][var - 1][0] : 0, var ? c_steps[b][var - 1][1] : 0, var != 0};
                        const double isc = ldexp(1.0, -k);
                        if (var == 0)
                            fused_group<4 * R - 2, MT, 2, GlobSrc>(gs, bxt, byt, fx, fy, offs, num, V.nmonp, n4, Fh, Fl,
                                                                   flags, isc);
                        else
                            fused_group<3 * R - 2, MT, 2, GlobSrc>(gs, bxt, byt, fx, fy, offs, num, V.nmonp, n4, Fh, Fl,
                                                                   flags, isc);
                    } else if (R == 1 && s_one[b * NVAR + var]) {
                        const PlaneSrc ps{G, NX, NY};
                        if (var == 0)
                            fused_group<4 * R - 2, MT, 1>(ps, bxt, byt, fx, fy, offs, num, V.nmonp, n4, Fh, Fl, flags);
                        else
                            fused_group<3 * R - 2, MT, 1>(ps, bxt, byt, fx, fy, offs, num, V.nmonp, n4, Fh, Fl, flags);
                    } else if (var == 0) {
                        fused_group<4 * R - 2, MT>(PlaneSrc{G, NX, NY}, bxt, byt, fx, fy, offs, num, V.nmonp, n4, Fh,
                                                   Fl, flags);
                    } else {
                        fused_group<3 * R - 2, MT>(PlaneSrc{G, NX, NY}, bxt, byt, fx, fy, offs, num, V.nmonp, n4, Fh,
                                                   Fl, flags);
                    }
                    if constexpr (MT == 4 && R < 3) {  // lane (g, k) holds item g + 8k's result
                        const int src = (lane >> 2) + 8 * (lane & 3);
                        const int iq = __shfl_sync(0xffffffffu, idx, src);
                        const bool rq = __shfl_sync(0xffffffffu, (int)real, src) != 0;
                        if (rq) s_F[iq] = make_double2(Fh[0], Fl[0]);
                    } else {
#pragma unroll
                        for (int q = 0; q < MT; ++q) {  // item lane/4 + 8q's result, from its quad's lane 0
                            const int src = (lane >> 2) + 8 * q;
                            const int iq = __shfl_sync(0xffffffffu, idx, src);
                            const bool rq = __shfl_sync(0xffffffffu, (int)real, src) != 0;
                            if ((lane & 3) == 0 && rq) s_F[iq] = make_double2(Fh[q], Fl[q]);
                        }
                    }
                    if (a.prof && lane == 0) {
                        const unsigned long long dt = clock64() - tq0;
                        atomicAdd(a.prof + 6, dt);
                        if (var == 0) atomicAdd(a.prof + 7, dt);
                    }
                }
                if (flags) atomicOr(&s_stats[4], (unsigned long long)flags);
            }
            __syncthreads();
            FUSED_PHASE(4);
            // per-pixel signed accumulation and normalisation (a7): TPP threads per
            // pixel sum interleaved taps in double-double, combined by shuffles
            {
                constexpr int TPP = FT / P;
                const int pl = tid / TPP, sub = tid % TPP;
                const int p = c0 + pl;
                const int w = s_info[p];
                const int b = info_basis(w), var = info_var(w);
                dd S = {0.0, 0.0};
                double sumCF = 0.0;  // sum_j |c_j F_j| (for the summation rounding term)
                if (info_live(w)) {
                    // compensated summation (TwoProd + TwoSum on the heads, all
                    // small terms in one fp64 accumulator), two interleaved
                    // accumulators for instruction-level parallelism
                    const int ntap = var ? NTAP / (R + 1) : NTAP;
                    double h0 = 0.0, e0 = 0.0, h1 = 0.0, e1 = 0.0;
                    int t = sub;
                    for (; t + TPP < ntap; t += 2 * TPP) {
                        const double2 F0 = s_F[t * P + pl], F1 = s_F[(t + TPP) * P + pl];
                        const double c0 = (double)tap_coef<R>(t, var - 1), c1 = (double)tap_coef<R>(t + TPP, var - 1);
                        const dd p0 = two_prod(c0, F0.x), p1 = two_prod(c1, F1.x);
                        const dd s0 = two_sum(h0, p0.hi), s1 = two_sum(h1, p1.hi);
                        h0 = s0.hi;
                        h1 = s1.hi;
                        e0 += s0.lo + (p0.lo + c0 * F0.y);
                        e1 += s1.lo + (p1.lo + c1 * F1.y);
                        sumCF += fabs(p0.hi) + fabs(p1.hi);
                    }
                    if (t < ntap) {
                        const double2 F0 = s_F[t * P + pl];
                        const double c0 = (double)tap_coef<R>(t, var - 1);
                        const dd p0 = two_prod(c0, F0.x);
                        const dd s0 = two_sum(h0, p0.hi);
                        h0 = s0.hi;
                        e0 += s0.lo + (p0.lo + c0 * F0.y);
                        sumCF += fabs(p0.hi);
                    }
                    S = dd_add(two_sum(h0, e0), two_sum(h1, e1));
                }
#pragma unroll
                for (int o = 1; o < TPP; o <<= 1) {
                    const dd T = {__shfl_xor_sync(0xffffffffu, S.hi, o), __shfl_xor_sync(0xffffffffu, S.lo, o)};
                    S = dd_add(S, T);
                    sumCF += __shfl_xor_sync(0xffffffffu, sumCF, o);
                }
                const int x = x0 + (p % TILE), y = y0 + p / TILE;
                const bool valid = x < a.W && out_row(a, y);
                const bool mine = sub == 0 && (a.pts ? (p == want) : valid);
                if (mine) {
                    double res = __longlong_as_double(0x7ff8000000000000LL);
                    double erel = 0.0;
                    if (info_live(w)) {
                        double norm = 1.0;
                        for (int k = 0; k < 4; ++k) {
                            if (k == var - 1) continue;
                            const double ia = 1.0 / s_ap[4 * p + k];
                            for (int i = 0; i < R; ++i) norm *= ia;
                        }
                        const double Sd = dd_to_d(S);
                        res = ldexp(Sd, s_pe[b * NVAR + var]) * norm / luts[b].var[var].L;
                        // a-posteriori bound of the split contraction:
                        // |S^ - S| <= sum_j |c_j| bnd + (2 ntap + 8) u^2 sum_j |c_j F_j|, sum_j |c_j| = 2^(R ns)
                        const int ns = var ? 3 : 4;
                        // (three limbs: 2^-kbits tighter; global int64 sums: both limbs exact)
                        const double lb = GLOBAL ? 0.0
                                          : R >= 3 ? ldexp(luts[b].var[var].bnd, -luts[b].var[var].kbits)
                                                   : luts[b].var[var].bnd;
                        const double err = ldexp(lb, R * ns) + 2.5e-30 * (NTAP / 81.0 + 1.0) * sumCF;
                        erel = err / fabs(Sd);
                        if (!(erel <= a.split_tol)) {  // NaN-safe: recompute in double-double
                            const int k = atomicAdd(&s_nfb, 1);
                            s_fb[k] = (short)p;
                        }
                    }
                    const long long oidx = a.pts ? item : out_index(a, img, x, y);
                    if (a.aux) {
                        double *ax = a.aux + BSF_AUX * oidx;
                        ax[0] = b;
                        ax[1] = var - 1;
                        ax[2] = (w >> 5) & 1;
                        ax[3] = w >> 8;
                        for (int k = 0; k < 4; ++k) ax[4 + k] = s_ap[4 * p + k];
                        ax[8] = 0.0;
                        ax[9] = erel;
                        ax[10] = ax[11] = 0.0;
                    }
                    if (a.out_f32 && !a.pts)
                        ((float *)a.out)[oidx] = (float)res;
                    else
                        ((double *)a.out)[oidx] = res;
                    {
                        atomicAdd(&s_stats[0], 1ull);
                        if ((w >> 5) & 1) atomicAdd(&s_stats[1], 1ull);
                        if (var) atomicAdd(&s_stats[2], 1ull);
                        if (b == BASIS_THETA_PRIME) atomicAdd(&s_stats[3], 1ull);
                        if (w >> 8) atomicOr(&s_stats[4], (unsigned long long)(w >> 8));
                    }
                }
            }
            __syncthreads();
            // double-double fallback for the pixels whose bound exceeds
            // TileArgs::split_tol: one warp per pixel (mesh_warp) on the base
            // plane, read back exactly from its split limbs
            for (int i = warp; i < s_nfb; i += FT / 32) {
                const int p = s_fb[i];
                const int w = s_info[p];
                PixelScales ps;
                ps.basis = info_basis(w);
                ps.drop = info_var(w) - 1;
                ps.flags = 0;
                ps.clamped = (w >> 5) & 1;
#pragma unroll
                for (int k = 0; k < 4; ++k) ps.ap[k] = s_ap[4 * p + k];
                const int b = ps.basis;
                // the base plane as left by phase 3: split limbs (G1, G0) for r <= 2;
                // at order 3 (G1, G2) plus the G0 plane when it was pre-split, else
                // still the double-double running sums
                const bool pre3 = R >= 3 && s_dom[b][2] * s_dom[b][3] <= G3_PRESPLIT_MAX;
                const double sc = ((R < 3 || pre3) && (s_vmask[b] & 1)) ? ldexp(1.0, s_pe[b * NVAR]) : 0.0;
                GView gv = {scr + s_poff[b * NVAR], s_dom[b][0], s_dom[b][1], s_dom[b][2], s_dom[b][3], sc};
                if constexpr (GLOBAL) {  // exact int64 global sums
                    gv.g = nullptr;
                    gv.sc = 0.0;
                    gv.gi = a.gglob[b] + (size_t)img * a.gGH * a.gGW;
                }
                if (pre3) {
                    gv.g0 = scr0 + s_poff[b * NVAR];
                    gv.sk = ldexp(1.0, -luts[b].var[0].kbits);
                }
                const int x = x0 + (p % TILE), y = y0 + p / TILE;
                int fl = 0;
                const double res = mesh_warp<R>(gv, luts[b], ps, x, y, &fl);
                fl = __reduce_or_sync(0xffffffffu, fl);
                if (lane == 0) {
                    const long long oidx = a.pts ? item : out_index(a, img, x, y);
                    if (a.out_f32 && !a.pts)
                        ((float *)a.out)[oidx] = (float)res;
                    else
                        ((double *)a.out)[oidx] = res;
                    if (a.aux) a.aux[BSF_AUX * oidx + 8] = 1.0;
                    {
                        atomicAdd(&s_stats[5], 1ull);
                        if (fl) atomicOr(&s_stats[4], (unsigned long long)fl);
                    }
                }
            }
            __syncthreads();
            if (tid == 0) s_nfb = 0;
            __syncthreads();
            FUSED_PHASE(5);

        }
        }  // sub-tiles
        __syncthreads();
        if (a.prof && tid == 0 && unit < BSF_PROF_ITEMS) {
            // per-item work (bsf_debug_item_cycles): interpolation MACs, fallback pixels,
            // halo domain points of the bases in use, planes
            unsigned long long halo = 0, planes = 0;
            for (int b = 0; b < 2; ++b)
                if (s_vmask[b]) halo += (unsigned long long)s_dom[b][2] * s_dom[b][3];
            for (int pi = 0; pi < NPLANE; ++pi) planes += s_poff[pi] >= 0;
            a.prof[BSF_PROF_WORK + 4 * unit] = s_stats[6];
            a.prof[BSF_PROF_WORK + 4 * unit + 1] = s_stats[5];
            a.prof[BSF_PROF_WORK + 4 * unit + 2] = halo;
            a.prof[BSF_PROF_WORK + 4 * unit + 3] = planes;
        }
        if (tid < 8 && a.stats && s_stats[tid]) {
            if (tid == 4)
                atomicOr(a.stats + 4, s_stats[4]);
            else
                atomicAdd(a.stats + tid, s_stats[tid]);
            s_stats[tid] = 0ull;
        }
        if (a.prof && tid == 0) {
            // per-item and per-CTA busy cycles (bsf_debug_item_cycles)
            const unsigned long long dt = (unsigned long long)(clock64() - t_item);
            if (unit < BSF_PROF_ITEMS) a.prof[16 + unit] = dt;
            if (blockIdx.x < BSF_PROF_CTAS) atomicAdd(a.prof + 16 + BSF_PROF_ITEMS + blockIdx.x, dt);
        }
    }
    if constexpr (I8) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
    }
}

// ---------------------------------------------------------------------------
// Algorithm 1 step 1 (Eq. (9) at PAPER.md:276-280): per
// covariance field b, sigma_b^2 = 1/2 min_p of the bound (9),
//   1/2 (C11 + C22 - (1/e_B(phi)) sqrt((C11 - C22)^2 + 4 C12^2)),
// e_B the elongation bound (as (rho-1)/(rho+1)) of the basis the pixel uses,
// C the (clamped) covariance the pixel is filtered with (R21).
// ---------------------------------------------------------------------------
__global__ void alg1_bound_kernel(const float *__restrict__ cov, int W, int H, int policy, int clamp, int layout,
                                  unsigned long long *__restrict__ minbits) {
    const size_t ipl = (size_t)H * W;
    const int b = blockIdx.y;
    double m = INFINITY;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < ipl; i += (size_t)gridDim.x * blockDim.x) {
        const float *cv = cov + (size_t)b * 3 * ipl + i;
        double sx = cv[0], sy = cv[ipl], th = cv[2 * ipl];
        if (layout == BSF_COV_C11_C12_C22) cov_from_c(sx, sy, th, sx, sy, th);
        double phi = th, maj = sx, mn = sy;
        if (sx < sy) {
            phi = th + M_PI / 2;
            maj = sy;
            mn = sx;
        }
        phi = fmod(phi, M_PI);
        if (phi < 0) phi += M_PI;
        double eT, eP;
        bounds_e(phi, &eT, &eP);
        int basis = policy;
        if (policy == BASIS_DUAL) basis = (sx == sy) ? BASIS_THETA : (eP > eT ? BASIS_THETA_PRIME : BASIS_THETA);
        const double eb = basis == BASIS_THETA ? eT : eP;
        double l1 = maj * maj, l2 = mn * mn;
        if (clamp && eb < 1.0 && sx != sy) {  // the clamp of pixel_scales (R9)
            const double rb = (1.0 + eb) / (1.0 - eb), rho = l1 / l2;
            if (rho > 0.95 * rb) {
                const double lim = 0.95 * rb, T = l1 + l2, e = (lim - 1.0) / (lim + 1.0);
                l1 = 0.5 * T * (1.0 + e);
                l2 = 0.5 * T * (1.0 - e);
            }
        }
        const double bound = 0.5 * (l1 + l2 - (l1 - l2) / fmin(eb, 1.0));
        m = fmin(m, bound);
    }
    for (int o = 16; o; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMin(minbits + b, (unsigned long long)__double_as_longlong(fmax(m, 0.0)));
}

__global__ void alg1_finish_kernel(const unsigned long long *__restrict__ minbits, int batch, double *sigma2) {
    const int b = threadIdx.x;
    if (b < batch) sigma2[b] = 0.5 * __longlong_as_double((long long)minbits[b]);  // half the bound
}

cudaError_t launch_alg1_sigma2(const float *cov, int batch, int W, int H, int policy, int clamp, int layout,
                               double *sigma2, cudaStream_t st, long long *nl) {
    // sigma2 holds 2 * batch doubles: [0, batch) results, [batch, 2 batch) min bits
    unsigned long long *bits = reinterpret_cast<unsigned long long *>(sigma2 + batch);
    cudaError_t e = cudaMemsetAsync(bits, 0x7f, batch * sizeof(unsigned long long), st);  // a large positive double
    if (e != cudaSuccess) return e;
    const int blocks = (int)((size_t)H * W / 256 + 1 < 1184 ? (size_t)H * W / 256 + 1 : 1184);
    alg1_bound_kernel<<<dim3(blocks, batch), 256, 0, st>>>(cov, W, H, policy, clamp, layout, bits);
    alg1_finish_kernel<<<1, 1024, 0, st>>>(bits, batch, sigma2);
    *nl += 2;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Work order of the persistent kernel: the super-tiles' interpolation work
// varies several-fold (variants and bases per pixel; profiles/README.md v13),
// so a raster hand-out leaves the CTAs that draw the last heavy tiles running
// alone.  fused_cost_kernel estimates each super-tile's work from 64 sampled
// pixels (their scales as in the reach pass): the interpolation MACs (taps x
// mean window slots x monomials of the table each pixel uses) plus the
// pre-integration (halo points x planes, weighted), and bins it on a log
// scale (four bins per octave); fused_order_kernel lists the super-tiles heaviest bin
// first (within a bin in any order).  The order changes nothing but which CTA
// computes a super-tile and when: each super-tile's arithmetic is the same.
// ---------------------------------------------------------------------------
// MAC-equivalents of one halo-plane point of the pre-integration (sweep and
// split), fitted on the measured per-super-tile cycles (tools/item_balance.py:
// cycles ~ a MACs + b halo-points x planes; b/a ~ 10 at r = 1, 140-180 at r = 2;
// at r = 3 the MACs alone explain 98 %)
template <int R>
__device__ __forceinline__ float sched_halo_weight() {
    return R == 1 ? 10.f : R == 2 ? 160.f : 0.f;  // (order 1 keeps raster order, launch_fused_impl)
}

// Split mode (64 x 64 super-tiles at order 2, u8 plans): a super-tile whose
// conditioning proxy (64 + 2E) / sigma_min exceeds SCHED_SPLIT_COND -- small
// scales next to a large reach, where the 64 x 64 anchoring sends pixels to the
// double-double fallback (profiles/README.md, tools/stile_risk.py: hundreds to
// thousands per super-tile once sigma_min < 1) -- is handed out as its four
// 32 x 32 quadrants, each anchored on its own halo.  Units are written to the
// bin array with stride S = 4: slot 4i + q = quadrant q of super-tile i (bin |
// 128), or slot 4i = the whole super-tile; unused slots hold 255.
constexpr float SCHED_SPLIT_COND = 160.f;

template <int R>
__global__ void __launch_bounds__(256) fused_cost_kernel(TileArgs a, const LutBasis *__restrict__ luts, int nitems,
                                                         int S) {
    constexpr int NTAP = FusedCfg<R>::NTAP;
    const int lane = threadIdx.x & 31, item = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (item >= nitems) return;
    const int ST = a.stile, nstx = (a.W + ST - 1) / ST, sty0 = a.oy0 / ST;
    const int spi = nstx * ((min(a.H, a.oy0 + out_rows(a)) + ST - 1) / ST - sty0);
    const int img = item / spi, rem = item % spi, X0s = (rem % nstx) * ST, Y0s = (sty0 + rem / nstx) * ST;
    const int step = ST / 8;
    float acc = 0.f, smin = 3.0e38f;
    int ex[2] = {0, 0}, ey[2] = {0, 0}, vm[2] = {0, 0};
    if (!(a.cov_mode == COV_ISO && !(a.sigma2[img / a.channels] > 0.0))) {
        for (int s = lane; s < 64; s += 32) {
            const int x = X0s + (s & 7) * step + step / 2, y = Y0s + (s >> 3) * step + step / 2;
            if (x < a.W && out_row(a, y)) {
                double sx, sy, th;
                load_cov(a, img, x, y, sx, sy, th);
                smin = fminf(smin, (float)fmin(sx, sy));
                PixelScales ps;
                pixel_scales(sx, sy, th, a.policy, a.clamp, R, ps);
                if (!(ps.flags & (FLAG_INFEASIBLE | FLAG_TWO_ZERO))) {
                    const LutVar &V = luts[ps.basis].var[ps.drop + 1];
                    acc += (float)(ps.drop >= 0 ? NTAP / (R + 1) : NTAP) * V.mean_count * (float)V.nmon;
                    double rx = 0.0, ry = 0.0;  // the reach, as in the kernel's reach pass
                    for (int k = 0; k < 4; ++k) {
                        rx += ps.ap[k] * abs(c_steps[ps.basis][k][0]);
                        ry += ps.ap[k] * c_steps[ps.basis][k][1];
                    }
                    ex[ps.basis] = max(ex[ps.basis], (int)ceil(0.5 * R * rx));
                    ey[ps.basis] = max(ey[ps.basis], (int)ceil(0.5 * R * ry));
                    vm[ps.basis] |= 1 << (ps.drop + 1);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        smin = fminf(smin, __shfl_xor_sync(0xffffffffu, smin, o));
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            ex[b] = max(ex[b], __shfl_xor_sync(0xffffffffu, ex[b], o));
            ey[b] = max(ey[b], __shfl_xor_sync(0xffffffffu, ey[b], o));
            vm[b] |= __shfl_xor_sync(0xffffffffu, vm[b], o);
        }
    }
    if (lane == 0) {
        float cost = acc * (float)(ST * ST) / 64.f;  // sampled MACs scaled to the super-tile
        for (int b = 0; b < 2; ++b)
            if (vm[b]) {
                const TileDomain d = fused_domain(luts[b], R, X0s, Y0s, ex[b], ey[b], ST);
                cost += sched_halo_weight<R>() * (float)d.NX * (float)d.NY * (float)__popc(vm[b] | 1);
            }
        const int E = max(max(ex[0], ex[1]), max(ey[0], ey[1]));
        const bool split = S == 4 && (float)(ST + 2 * E) > SCHED_SPLIT_COND * smin;
        if (!split) {
            // bins stop at SCHED_NBIN - 2: a split unit is stored as bin | 128,
            // which must never equal the unused-slot sentinel 255
            const int b = cost >= 1.f ? min(SCHED_NBIN - 2, 1 + (int)(4.f * __log2f(cost))) : 0;
            a.order_bin[(size_t)S * item] = (unsigned char)b;
            atomicAdd(a.order_hist + b, 1u);
            for (int q = 1; q < S; ++q) a.order_bin[(size_t)S * item + q] = 255;
        } else {
            const float c4 = 0.25f * cost;
            const int b = c4 >= 1.f ? min(SCHED_NBIN - 2, 1 + (int)(4.f * __log2f(c4))) : 0;
            for (int q = 0; q < 4; ++q) {
                const bool in = X0s + (ST / 2) * (q & 1) < a.W && Y0s + (ST / 2) * (q >> 1) < a.H;
                a.order_bin[(size_t)4 * item + q] = in ? (unsigned char)(b | 128) : 255;
                if (in) atomicAdd(a.order_hist + b, 1u);
            }
        }
    }
}

__global__ void __launch_bounds__(256) fused_order_kernel(TileArgs a, int nslots, int S) {
    static_assert(SCHED_NBIN == 128, "four bins per lane");
    __shared__ unsigned base[SCHED_NBIN];
    if (threadIdx.x < 32) {
        // exclusive scan over the bins in descending order: lane l owns bins
        // 127 - 4l ... 124 - 4l
        const int lane = threadIdx.x;
        unsigned h[4], t = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) t += (h[k] = a.order_hist[SCHED_NBIN - 1 - 4 * lane - k]);
        unsigned inc = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        unsigned run = inc - t;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            base[SCHED_NBIN - 1 - 4 * lane - k] = run;
            run += h[k];
        }
        // the number of units, for the fused kernel's loop bound
        if (blockIdx.x == 0 && lane == 31) a.order_hist[2 * SCHED_NBIN] = inc;
    }
    __syncthreads();
    // unit code: the super-tile (S = 1), or super-tile << 3 | (0 whole, 1 + q
    // quadrant q) in split mode
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nslots; i += gridDim.x * blockDim.x) {
        const int v = a.order_bin[i];
        if (v == 255) continue;
        const int b = v & 127;
        const int code = S == 1 ? i : ((i / S) << 3) | ((v & 128) ? 1 + i % S : 0);
        a.order[base[b] + atomicAdd(a.order_hist + SCHED_NBIN + b, 1u)] = code;
    }
}

template <int R, bool SPLIT = false, bool GLOBAL = false, bool I8 = false>
static cudaError_t launch_fused_r(const TileArgs &a, int slots, cudaStream_t st, const LutBasis *luts) {
    constexpr size_t sm = I8 ? i8_smem_off<R>() + I8_SMEM : fused_smem_bytes<R>();
    static std::atomic<unsigned long long> attr{0ull};
    cudaError_t e = set_smem_attr(fused_kernel<R, SPLIT, GLOBAL, I8>, (int)sm, attr);
    if (e != cudaSuccess) return e;
    fused_kernel<R, SPLIT, GLOBAL, I8><<<slots, FT, sm, st>>>(a, luts);
    return cudaGetLastError();
}

size_t fused_fbuf_items(int order) {
    switch (order) {
        case 1: return fused_items<1>();
        case 2: return fused_items<2>();
        case 3: return fused_items<3>();
        case 4: return fused_items<4>();
    }
    return 0;
}

int fused_slots() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

cudaError_t launch_fused_impl(const TileArgs &a, int order, int slots, cudaStream_t st, const LutBasis *luts,
                              long long *nl) {
    cudaError_t e = cudaMemsetAsync(a.counter, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    TileArgs b = a;
    const int oh = a.oH ? a.oH : a.H, sty0 = a.oy0 / a.stile;
    const long long nitems = (long long)((a.W + a.stile - 1) / a.stile) *
                             ((std::min(a.H, a.oy0 + oh) + a.stile - 1) / a.stile - sty0) * a.nimg;
    // split mode (see fused_cost_kernel): 64 x 64 super-tiles at order 2 run the
    // scheduling kernels at any item count
    const int S = (a.stile == 64 && order == 2) ? 4 : 1;
    if ((a.gglob[0] || a.gglob[1]) && order != 1) return cudaErrorInvalidValue;  // global mode: order 1 only
    if (a.order && !a.pts && !a.tiles && order >= 2 && (S == 4 || nitems >= 2 * (long long)slots) &&
        nitems * S <= a.order_cap) {
        // largest-first work order (see fused_cost_kernel); at order 1 the
        // balance it gains (3.7 -> 1.2 % on config 3) is lost to the halo reads
        // of raster neighbours no longer sharing L2, so raster order stays
        if ((e = cudaMemsetAsync(a.order_hist, 0, (2 * SCHED_NBIN + 1) * sizeof(unsigned), st)) != cudaSuccess)
            return e;
        const int nb = (int)((nitems + 7) / 8);
        switch (order) {
            case 1: fused_cost_kernel<1><<<nb, 256, 0, st>>>(a, luts, (int)nitems, S); break;
            case 2: fused_cost_kernel<2><<<nb, 256, 0, st>>>(a, luts, (int)nitems, S); break;
            case 3: fused_cost_kernel<3><<<nb, 256, 0, st>>>(a, luts, (int)nitems, S); break;
            case 4: fused_cost_kernel<4><<<nb, 256, 0, st>>>(a, luts, (int)nitems, S); break;
            default: return cudaErrorInvalidValue;
        }
        fused_order_kernel<<<(int)std::min<long long>((nitems * S + 255) / 256, 4 * (long long)slots), 256, 0, st>>>(
            a, (int)(nitems * S), S);
        *nl += 2;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    } else {
        b.order = nullptr;
    }
    switch (order) {
        case 1: e = (b.gglob[0] || b.gglob[1]) ? launch_fused_r<1, false, true>(b, slots, st, luts) : launch_fused_r<1>(b, slots, st, luts); break;
        case 2:  // split mode only in its own instantiation (register allocation of the other plans untouched)
            e = b.order && S == 4 ? launch_fused_r<2, true>(b, slots, st, luts) : launch_fused_r<2>(b, slots, st, luts);
            break;
        case 3: e = b.i8 ? launch_fused_r<3, false, false, true>(b, slots, st, luts) : launch_fused_r<3>(b, slots, st, luts); break;
        case 4: e = launch_fused_r<4>(b, slots, st, luts); break;
        default: return cudaErrorInvalidValue;
    }
    ++*nl;
    return e;
}
