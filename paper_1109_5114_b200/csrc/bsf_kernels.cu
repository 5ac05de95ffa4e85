// Hot-path kernels for sm_100a.
//
//  * fill      f -> g (zero-padded domain)                       [HBM]
//  * scan      one running-sum level along a lattice step s      [HBM]
//              (Alg. 3 step 2)
//  * gather    per pixel: decode, Alg. 2 basis choice, clamp, scale solve,
//              (r+1)^4-tap mesh (Table 1 / Eq. 10) with the Eq. (11)
//              interpolation, signed accumulation, normalisation   [FP64 ALU]
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cuda.h>  // CUtensorMap (types only; cuTensorMapEncodeTiled through cudaGetDriverEntryPoint)

#include <mutex>
#include <type_traits>

#include "bsf_dd.cuh"
#include "bsf_internal.h"
#include "bsf_pixel.cuh"

namespace bsf {

// ---------------------------------------------------------------------------
// lattice steps; scan level order Theta (1,0),(1,1),(0,1),(-1,1), Theta' the
// Alg. 3 order (a)-(d) = (1,2),(2,1),(-1,2),(-2,1)
// ---------------------------------------------------------------------------
__constant__ int c_steps[2][4][2] = {{{1, 0}, {1, 1}, {0, 1}, {-1, 1}}, {{2, 1}, {1, 2}, {-1, 2}, {-2, 1}}};
static const int h_scan_order[2][4][2] = {{{1, 0}, {1, 1}, {0, 1}, {-1, 1}}, {{1, 2}, {2, 1}, {-1, 2}, {-2, 1}}};
__constant__ int c_scan_order[2][4][2] = {{{1, 0}, {1, 1}, {0, 1}, {-1, 1}}, {{1, 2}, {2, 1}, {-1, 2}, {-2, 1}}};

// ---------------------------------------------------------------------------
// element types for the scans
// ---------------------------------------------------------------------------
struct OpDD {
    typedef double2 T;
    __device__ static T zero() { return make_double2(0.0, 0.0); }
    __device__ static T add(T a, T b) {
        dd r = dd_add({a.x, a.y}, {b.x, b.y});
        return make_double2(r.hi, r.lo);
    }
    __device__ static T shfl_up(T v, int d) {
        return make_double2(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d));
    }
    __device__ static T shfl_idx(T v, int l) {
        return make_double2(__shfl_sync(0xffffffffu, v.x, l), __shfl_sync(0xffffffffu, v.y, l));
    }
    __device__ static T shfl_xor(T v, int l) {
        return make_double2(__shfl_xor_sync(0xffffffffu, v.x, l), __shfl_xor_sync(0xffffffffu, v.y, l));
    }
};
struct OpU64 {
    typedef unsigned long long T;
    __device__ static T zero() { return 0ull; }
    __device__ static T add(T a, T b) { return a + b; }  // wraps mod 2^64
    __device__ static T shfl_up(T v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
    __device__ static T shfl_idx(T v, int l) { return __shfl_sync(0xffffffffu, v, l); }
    __device__ static T shfl_xor(T v, int l) { return __shfl_xor_sync(0xffffffffu, v, l); }
};

#include "bsf_scan.cuh"

// ---------------------------------------------------------------------------
// launchers of the global pre-integration (one kernel per level)
// ---------------------------------------------------------------------------
// per level: rows (sy = 0) or strips of 32 u-columns walked in blocks of 32
// rows, ND row blocks in flight (64 KB of shared memory per block)
// block shapes (measured on config 3, tools/time_preint.py): int64 8 warps x 16
// rows, 2 blocks in flight (64 KB); double-double 8 warps x 8 rows, 3 blocks (96 KB)
#ifndef BSF_SCAN_NW_I64
#define BSF_SCAN_NW_I64 8
#define BSF_SCAN_RPW_I64 16
#define BSF_SCAN_ND_I64 2
#endif
#ifndef BSF_SCAN_NW_DD
#define BSF_SCAN_NW_DD 8
#define BSF_SCAN_RPW_DD 8
#define BSF_SCAN_ND_DD 3
#endif
// TMA tensor map of a level input (3-D: x, y, image), box {TmaRow::BX, 1, 1};
// false when TMA's rules (16-byte aligned base and row pitch) do not hold
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    });
    return fn;
}

template <class In, class T>
static bool scan_tensor_map(CUtensorMap *map, const In *in, const Geometry &geo) {
    constexpr bool IMG = !std::is_same<In, T>::value;
    EncodeTiledFn fn = encode_tiled();
    if (!fn || ((uintptr_t)in & 15)) return false;
    const int xs = TmaRow<In>::XS;  // double-double: pairs of fp64
    const size_t es = TmaRow<In>::ES;
    const cuuint64_t X = (cuuint64_t)(IMG ? geo.W : geo.GW) * xs, Y = IMG ? geo.H : geo.GH;
    const cuuint64_t dims[3] = {X, Y, (cuuint64_t)geo.nimg};
    const cuuint64_t strides[2] = {X * es, X * es * Y};
    if (strides[0] % 16 || strides[0] >= (1ull << 40) || strides[1] >= (1ull << 40)) return false;
    const cuuint32_t box[3] = {(cuuint32_t)TmaRow<In>::BX, 1u, 1u}, estr[3] = {1u, 1u, 1u};
    const CUtensorMapDataType dt = std::is_same<In, uint8_t>::value   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                   : std::is_same<In, float>::value   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                   : sizeof(In) == 8                  ? CU_TENSOR_MAP_DATA_TYPE_INT64
                                                                      : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
    return fn(map, dt, 3, (void *)in, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

static std::atomic<int> g_scan_tma{1};
static int scan_use_tma() { return g_scan_tma.load(std::memory_order_relaxed); }
void set_scan_tma(int on) { g_scan_tma.store(on ? 1 : 0, std::memory_order_relaxed); }

template <class Op, class In, int SX, int SY>
static cudaError_t scan_strips(const In *in, typename Op::T *g, const Geometry &geo, const typename Op::T *carry,
                               cudaStream_t st) {
    constexpr bool DD = sizeof(typename Op::T) == 16;
    constexpr int NW = DD ? BSF_SCAN_NW_DD : BSF_SCAN_NW_I64, RPW = DD ? BSF_SCAN_RPW_DD : BSF_SCAN_RPW_I64,
                  ND = DD ? BSF_SCAN_ND_DD : BSF_SCAN_ND_I64;
    const int span = abs(SX) * ((geo.GH - 1) / SY);
    const int U0 = SX > 0 ? -span : 0, NS = (geo.GW + span + 31) / 32;
    const unsigned grid = (unsigned)((long long)geo.nimg * NS);
    CUtensorMap map;
    if (scan_use_tma() && scan_tensor_map<In, typename Op::T>(&map, in, geo)) {
        // rows streamed by TMA (bulk tensor copies completing on mbarriers)
        constexpr int SMEM = ND * NW * RPW * tma_row_bytes<In>() + 128;  // + alignment slack
        static std::atomic<unsigned long long> attr{0ull};
        cudaError_t e = set_smem_attr(scan_strip_tma_kernel<Op, In, SX, SY, NW, RPW, ND>, SMEM, attr);
        if (e != cudaSuccess) return e;
        scan_strip_tma_kernel<Op, In, SX, SY, NW, RPW, ND><<<grid, 32 * NW, SMEM, st>>>(map, g, geo, U0, NS, carry);
        return cudaGetLastError();
    }
    constexpr int SMEM = ND * NW * RPW * 32 * (int)sizeof(typename Op::T);
    static std::atomic<unsigned long long> attr{0ull};
    cudaError_t e = set_smem_attr(scan_strip_kernel<Op, In, SX, SY, NW, RPW, ND>, SMEM, attr);
    if (e != cudaSuccess) return e;
    scan_strip_kernel<Op, In, SX, SY, NW, RPW, ND><<<grid, 32 * NW, SMEM, st>>>(in, g, geo, U0, NS, carry);
    return cudaGetLastError();
}

template <class Op, class In>
static cudaError_t scan_level(const In *in, typename Op::T *g, const Geometry &geo, int sx, int sy,
                              const typename Op::T *carry, cudaStream_t st) {
    if (sy == 0) {
        constexpr int EPL = sizeof(typename Op::T) == 16 ? 4 : 8, WPC = 8;
        const long long rows = (long long)geo.nimg * geo.GH;
        scan_row_kernel<Op, In, EPL, WPC><<<(unsigned)((rows + WPC - 1) / WPC), 32 * WPC, 0, st>>>(in, g, geo);
        return cudaGetLastError();
    }
    // the seven lattice steps of the two bases (c_scan_order)
    if (sy == 1 && sx == 1) return scan_strips<Op, In, 1, 1>(in, g, geo, carry, st);
    if (sy == 1 && sx == 0) return scan_strips<Op, In, 0, 1>(in, g, geo, carry, st);
    if (sy == 1 && sx == -1) return scan_strips<Op, In, -1, 1>(in, g, geo, carry, st);
    if (sy == 2 && sx == 1) return scan_strips<Op, In, 1, 2>(in, g, geo, carry, st);
    if (sy == 1 && sx == 2) return scan_strips<Op, In, 2, 1>(in, g, geo, carry, st);
    if (sy == 2 && sx == -1) return scan_strips<Op, In, -1, 2>(in, g, geo, carry, st);
    if (sy == 1 && sx == -2) return scan_strips<Op, In, -2, 1>(in, g, geo, carry, st);
    return cudaErrorInvalidValue;
}

template <class Op, class In>
static cudaError_t scan_basis(const In *f, typename Op::T *g, const Geometry &geo, int basis, int order,
                              cudaStream_t st, long long *nl) {
    for (int rep = 0; rep < order; ++rep)
        for (int lv = 0; lv < 4; ++lv) {
            const int sx = h_scan_order[basis][lv][0], sy = h_scan_order[basis][lv][1];
            cudaError_t e = (rep == 0 && lv == 0) ? scan_level<Op, In>(f, g, geo, sx, sy, nullptr, st)
                                                  : scan_level<Op, typename Op::T>(g, g, geo, sx, sy, nullptr, st);
            ++*nl;
            if (e != cudaSuccess) return e;
        }
    return cudaSuccess;
}

cudaError_t launch_preint_dd(const void *f, int u8, double2 *g, const Geometry &geo, int basis, int order,
                             cudaStream_t st, long long *nl) {
    if (u8) return scan_basis<OpDD, uint8_t>((const uint8_t *)f, g, geo, basis, order, st, nl);
    return scan_basis<OpDD, float>((const float *)f, g, geo, basis, order, st, nl);
}

cudaError_t launch_preint_i64(const uint8_t *f, unsigned long long *g, const Geometry &geo, int basis, int order,
                              cudaStream_t st, long long *nl) {
    return scan_basis<OpU64, uint8_t>(f, g, geo, basis, order, st, nl);
}

void scan_step(int basis, int level, int *sx, int *sy) {
    *sx = h_scan_order[basis][level % 4][0];
    *sy = h_scan_order[basis][level % 4][1];
}

cudaError_t launch_scan_level(const void *f, int u8, void *g, int exact, const Geometry &geo, int basis, int level,
                              const void *carry, cudaStream_t st) {
    int sx, sy;
    scan_step(basis, level, &sx, &sy);
    if (exact) {
        typedef unsigned long long T;
        if (level == 0) return scan_level<OpU64, uint8_t>((const uint8_t *)f, (T *)g, geo, sx, sy, (const T *)carry, st);
        return scan_level<OpU64, T>((const T *)g, (T *)g, geo, sx, sy, (const T *)carry, st);
    }
    if (level == 0) {
        if (u8) return scan_level<OpDD, uint8_t>((const uint8_t *)f, (double2 *)g, geo, sx, sy, (const double2 *)carry, st);
        return scan_level<OpDD, float>((const float *)f, (double2 *)g, geo, sx, sy, (const double2 *)carry, st);
    }
    return scan_level<OpDD, double2>((const double2 *)g, (double2 *)g, geo, sx, sy, (const double2 *)carry, st);
}

// ---------------------------------------------------------------------------
// DC renormalisation (R12): out / (filter of the
// image indicator), the indicator being an image of ones in the input type
// ---------------------------------------------------------------------------
__global__ void fill_ones_kernel(void *f, int u8, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        if (u8)
            ((uint8_t *)f)[i] = 1;
        else
            ((float *)f)[i] = 1.0f;
    }
}

__global__ void normalize_kernel(void *out, int out_f32, const double *__restrict__ den, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        if (out_f32)
            ((float *)out)[i] = (float)((double)((float *)out)[i] / den[i]);
        else
            ((double *)out)[i] /= den[i];
    }
}

cudaError_t launch_fill_ones(void *f, int u8, size_t n, cudaStream_t st, long long *nl) {
    fill_ones_kernel<<<148 * 8, 256, 0, st>>>(f, u8, n);
    ++*nl;
    return cudaGetLastError();
}

cudaError_t launch_normalize(void *out, int out_f32, const double *den, size_t n, cudaStream_t st, long long *nl) {
    normalize_kernel<<<148 * 8, 256, 0, st>>>(out, out_f32, den, n);
    ++*nl;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Gather
// ---------------------------------------------------------------------------

__device__ __forceinline__ int binom_small(int n, int k) {
    int r = 1;
    for (int i = 0; i < k; ++i) r = r * (n - i) / (i + 1);
    return r;
}

__device__ __forceinline__ int region_key_index(const LutBasis &L, double x, double y) {
    int idx = 0, mul = 1;
    for (int k = 0; k < 4; ++k) {
        int f = (int)floor(L.normal[k].x * x + L.normal[k].y * y) - L.kmin[k];
        if (f < 0 || f >= L.radix[k]) return -1;
        idx += f * mul;
        mul *= L.radix[k];
    }
    return L.table[idx];
}

__device__ __forceinline__ int classify(const LutBasis &L, double x, double y) {
    const double one_m = 1.0 - 1.1102230246251565e-16;
    x = fmin(fmax(x, 0.0), one_m);
    y = fmin(fmax(y, 0.0), one_m);
    int r = region_key_index(L, x, y);
    if (r >= 0) return r;
    // exactly on knot lines: any adjacent region gives the same value (M is
    // continuous), so step into one.
    const double e = 1e-12;
    const double dx[4] = {e, -e, 0.7 * e, -0.3 * e};
    const double dy[4] = {0.37 * e, 0.61 * e, -e, -0.77 * e};
    for (int i = 0; i < 4; ++i) {
        r = region_key_index(L, fmin(fmax(x + dx[i], 0.0), one_m), fmin(fmax(y + dy[i], 0.0), one_m));
        if (r >= 0) return r;
    }
    return 0;
}

// ---------------------------------------------------------------------------
// Interpolation weights M(phi - d): polynomials in phi (exact doubles, R17)
// with double-double coefficients.
// ---------------------------------------------------------------------------

// plain fp64 2D Horner (BSF_PREC_FP64)
__device__ __forceinline__ double horner2_d(const double2 *__restrict__ c, int deg, double x, double y) {
    int idx = 0;
    double ax = 0.0;
    for (int i = deg; i >= 0; --i) {
        double2 c0 = __ldg(c + idx++);
        double ay = c0.x + c0.y;
        for (int j = deg - i - 1; j >= 0; --j) {
            double2 cj = __ldg(c + idx++);
            ay = fma(ay, y, cj.x + cj.y);
        }
        ax = (i == deg) ? ay : fma(ax, x, ay);
    }
    return ax;
}

// One compensated Horner step (Graillat-Langlois-Louvet): value (h + l) <-
// (h + l) * x + (ch + cl), with the rounding errors of h*x and of the sum
// carried in l.  11 fp64 instructions; result accurate to ~u^2 * cond.
__device__ __forceinline__ void comp_step(double &h, double &l, double x, double ch, double cl) {
    double p = __dmul_rn(h, x);
    double pe = __fma_rn(h, x, -p);
    double s = __dadd_rn(p, ch);
    double bb = __dadd_rn(s, -p);
    double se = __dadd_rn(__dadd_rn(p, -__dadd_rn(s, -bb)), __dadd_rn(ch, -bb));
    l = __fma_rn(l, x, __dadd_rn(__dadd_rn(pe, se), cl));
    h = s;
}

// compensated 2D Horner with double-double coefficients at an exact point;
// NW independent polynomials (window points) are evaluated in lock-step so the
// serial dependency chain of each is interleaved with the others (ILP).
template <int NW>
__device__ __forceinline__ void horner2_comp_n(const double2 *__restrict__ c, int nmon, int deg, double x, double y,
                                               double *wh, double *wl) {
    double ah[NW], al[NW];
    int idx = 0;
    for (int i = deg; i >= 0; --i) {
        double sh[NW], sl[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            double2 c0 = __ldg(c + w * nmon + idx);
            sh[w] = c0.x;
            sl[w] = c0.y;
        }
        ++idx;
        for (int j = deg - i - 1; j >= 0; --j) {
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                double2 cj = __ldg(c + w * nmon + idx);
                comp_step(sh[w], sl[w], y, cj.x, cj.y);
            }
            ++idx;
        }
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            if (i == deg) {
                ah[w] = sh[w];
                al[w] = sl[w];
            } else {
                comp_step(ah[w], al[w], x, sh[w], sl[w]);
            }
        }
    }
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        wh[w] = ah[w];
        wl[w] = al[w];
    }
}

// Where the running sums are read from: the global domain (bsf_filter) or a
// tile's local domain (tile path).  Points above Y0 are zero (no image above);
// other points outside the stored domain are a margin violation.
struct GView {
    const double2 *g;
    int X0, Y0, NX, NY;
    double sc;  // 0: double-double {hi, lo}; else split limbs (G1, G0) of G = sc (G1 + G0) (bsf_fused.cuh)
    const double *g0 = nullptr;  // order 3: g holds (G1, G2) and g0 the third limb, G = sc (G1 + sk (G2 + G0))
    double sk = 0.0;
    const long long *gi = nullptr;  // exact int64 global sums (fused global mode): read as exact double-doubles
};

__device__ __forceinline__ double2 load_g2(const GView &v, int qx, int qy, int *flags) {
    int ly = qy - v.Y0, lx = qx - v.X0;
    if (ly < 0) return make_double2(0.0, 0.0);  // above the rows that hold any image
    if (lx < 0 || lx >= v.NX || ly >= v.NY) {
        *flags |= FLAG_RANGE;
        return make_double2(0.0, 0.0);
    }
    const size_t i = (size_t)ly * v.NX + lx;
    if (v.gi) {  // |value| < 2^62: hi = fl(value), the remainder is exact
        const long long q = __ldg(v.gi + i);
        const double hi = (double)q;
        return make_double2(hi, (double)(q - (long long)hi));
    }
    const double2 t = v.g[i];  // plain load: tile scratch is written in-kernel
    if (v.sc == 0.0) return t;
    if (v.g0) {  // three limbs: every product below is an exact power-of-two scaling
        const dd e = dd_add_d(two_sum(t.x * v.sc, t.y * v.sc * v.sk), v.g0[i] * v.sc * v.sk);
        return make_double2(e.hi, e.lo);
    }
    const dd e = two_sum(t.x * v.sc, t.y * v.sc);  // exact: power-of-two scaling of both limbs
    return make_double2(e.hi, e.lo);
}

// G' = (1 - T_{s_drop})^R G  (exact lattice difference, R5), double-double
template <int R>
__device__ __forceinline__ double2 load_gp(const GView &v, int qx, int qy, int drop, int2 sdrop, int *flags) {
    if (drop < 0) return load_g2(v, qx, qy, flags);
    dd G = {0.0, 0.0};
#pragma unroll
    for (int i = 0; i <= R; ++i) {
        double2 t = load_g2(v, qx - i * sdrop.x, qy - i * sdrop.y, flags);
        int cb = binom_small(R, i) * ((i & 1) ? -1 : 1);
        G = dd_add(G, dd_mul_d({t.x, t.y}, (double)cb));
    }
    return make_double2(G.hi, G.lo);
}

// F(b + phi) = sum_d G'(b + d) M(phi - d)   (Eq. 11, r-fold, R4/R5)
// Double-double: weights by compensated Horner, products by TwoProd, the
// large partial sum by TwoSum, all small terms in one fp64 accumulator.
template <int R, bool DD>
__device__ __forceinline__ dd interp(const GView &gv, const LutBasis &L, const LutVar &V, int bx, int by, double fx,
                                     double fy, int drop, int2 sdrop, int *flags, double *sumG) {
    int reg = classify(L, fx, fy);
    int n = __ldg(V.counts + reg);
    const int2 *offs = V.offs + reg * V.nmax;
    const double2 *cf = V.coef + (size_t)reg * V.nmax * V.nmon;
    double Fh = 0.0, Fl = 0.0;
    // F += G * w with w = wh + wl: TwoProd for G.hi * wh, TwoSum into Fh, all
    // small terms (product error, sum error, G.hi*wl, G.lo*wh) into Fl.
    auto accum = [&](double2 G, double wh, double wl) {
        double p = __dmul_rn(G.x, wh);
        double pe = __fma_rn(G.x, wh, -p);
        double t = __dadd_rn(Fh, p);
        double bb = __dadd_rn(t, -Fh);
        double te = __dadd_rn(__dadd_rn(Fh, -__dadd_rn(t, -bb)), __dadd_rn(p, -bb));
        Fh = t;
        Fl = __fma_rn(G.x, wl, __fma_rn(G.y, wh, __dadd_rn(Fl, __dadd_rn(te, pe))));
    };
    int s = 0;
    if (DD) {
        for (; s + 2 <= n; s += 2) {
            int2 d0 = __ldg(offs + s), d1 = __ldg(offs + s + 1);
            double2 G0 = load_gp<R>(gv, bx + d0.x, by + d0.y, drop, sdrop, flags);
            double2 G1 = load_gp<R>(gv, bx + d1.x, by + d1.y, drop, sdrop, flags);
            double wh[2], wl[2];
            horner2_comp_n<2>(cf + (size_t)s * V.nmon, V.nmon, V.deg, fx, fy, wh, wl);
            accum(G0, wh[0], wl[0]);
            accum(G1, wh[1], wl[1]);
        }
    }
    for (; s < n; ++s) {
        int2 d = __ldg(offs + s);
        double2 G = load_gp<R>(gv, bx + d.x, by + d.y, drop, sdrop, flags);
        if (DD) {
            double wh, wl;
            horner2_comp_n<1>(cf + (size_t)s * V.nmon, V.nmon, V.deg, fx, fy, &wh, &wl);
            accum(G, wh, wl);
        } else {
            double w = horner2_d(cf + (size_t)s * V.nmon, V.deg, fx, fy);
            double g = G.x + G.y;
            Fh = fma(g, w, Fh);
            *sumG += fabs(g);
        }
    }
    return fast_two_sum(Fh, Fl);
}

// out(p) = prod_k (1/a'_k)^R sum_j c_j F(p + sum_k (R/2 - j_k) a'_k s_k)
// a'_k lies on the 2^-40 grid (R17), so each displacement and their sum are
// exact doubles: the tap's lattice base b and fractional offset phi are exact.
#ifdef BSF_TAP_DUMP
__device__ double *g_tap_dump;
#endif
// err (fp64 path only): a-posteriori estimate of |computed - exact| / |result|
// (BSF_PREC_AUTO).
template <int R, bool DD>
__device__ double mesh(const GView &gv, const LutBasis &L, const PixelScales &ps, int x, int y, int *flags,
                       double *err = nullptr, double *ratios = nullptr) {
    int dirs[4];
    int ns = 0;
    for (int k = 0; k < 4; ++k)
        if (k != ps.drop) dirs[ns++] = k;
    const LutVar &V = L.var[ps.drop + 1];
    int2 sdrop = make_int2(0, 0);
    if (ps.drop >= 0) sdrop = make_int2(c_steps[ps.basis][ps.drop][0], c_steps[ps.basis][ps.drop][1]);
    int ntap = 1;
    for (int q = 0; q < ns; ++q) ntap *= (R + 1);
    dd acc = {0.0, 0.0};
    double sumCG = 0.0, sumCF = 0.0;
    for (int t = 0; t < ntap; ++t) {
        int tt = t, coef = 1;
        double Dx = 0.0, Dy = 0.0;
        for (int q = 0; q < ns; ++q) {
            int j = tt % (R + 1);
            tt /= (R + 1);
            coef *= binom_small(R, j) * ((j & 1) ? -1 : 1);
            int k = dirs[q];
            double m = 0.5 * R - j;  // half-integer
            Dx += (m * c_steps[ps.basis][k][0]) * ps.ap[k];  // exact (R17)
            Dy += (m * c_steps[ps.basis][k][1]) * ps.ap[k];
        }
        double flx = floor(Dx), fly = floor(Dy);
        double fx = Dx - flx, fy = Dy - fly;  // exact
        double sumG = 0.0;
        dd F = interp<R, DD>(gv, L, V, x + (int)flx, y + (int)fly, fx, fy, ps.drop, sdrop, flags, &sumG);
        if (!DD) {
            sumCG += abs(coef) * sumG;
            sumCF += fabs(coef * F.hi);
        }
#ifdef BSF_TAP_DUMP
        if (g_tap_dump && x == 0 && y == 23) {
            double *o = g_tap_dump + 8 * t;
            o[0] = x + flx; o[1] = y + fly; o[2] = fx; o[3] = 0; o[4] = fy; o[5] = 0; o[6] = F.hi; o[7] = F.lo;
        }
#endif
        acc = dd_add(acc, dd_mul_d(F, (double)coef));
    }
    double norm = 1.0;
    for (int q = 0; q < ns; ++q) {
        double ia = 1.0 / ps.ap[dirs[q]];
        for (int i = 0; i < R; ++i) norm *= ia;
    }
    double S = dd_to_d(acc);
    if (!DD && err) {
        // error estimate 4 u sum_j |c_j| sum_d |G_d| / |S|.  Calibrated on
        // 200k config-2 pixels against double-double (profiles/
        // r01_auto_calibration.md): the true fp64 error never exceeded
        // 0.12 u sum|c||G| / |S|, so this estimate carries >= 30x headroom.
        const double u = 1.1102230246251565e-16;
        *err = 4.0 * u * sumCG / fabs(S);
    }
    if (!DD && ratios) {
        ratios[0] = sumCF / fabs(S);
        ratios[1] = sumCG / fabs(S);
    }
    return S * norm;
}

// Warp-cooperative double-double mesh (the exact split path's fallback,
// bsf_fused.cuh): the lanes share the taps of ONE pixel, each interpolates its
// taps in double-double, and the signed sum is reduced by shuffles.  All 32
// lanes must call it with the same arguments; every lane returns the result.
template <int R>
__device__ double mesh_warp(const GView &gv, const LutBasis &L, const PixelScales &ps, int x, int y, int *flags) {
    const int lane = threadIdx.x & 31;
    int dirs[4];
    int ns = 0;
    for (int k = 0; k < 4; ++k)
        if (k != ps.drop) dirs[ns++] = k;
    const LutVar &V = L.var[ps.drop + 1];
    int2 sdrop = make_int2(0, 0);
    if (ps.drop >= 0) sdrop = make_int2(c_steps[ps.basis][ps.drop][0], c_steps[ps.basis][ps.drop][1]);
    int ntap = 1;
    for (int q = 0; q < ns; ++q) ntap *= (R + 1);
    dd acc = {0.0, 0.0};
    for (int t = lane; t < ntap; t += 32) {
        int tt = t, coef = 1;
        double Dx = 0.0, Dy = 0.0;
        for (int q = 0; q < ns; ++q) {
            const int j = tt % (R + 1);
            tt /= (R + 1);
            coef *= binom_small(R, j) * ((j & 1) ? -1 : 1);
            const int k = dirs[q];
            const double m = 0.5 * R - j;
            Dx += (m * c_steps[ps.basis][k][0]) * ps.ap[k];  // exact (R17)
            Dy += (m * c_steps[ps.basis][k][1]) * ps.ap[k];
        }
        const double flx = floor(Dx), fly = floor(Dy);
        double sumG = 0.0;
        const dd F = interp<R, true>(gv, L, V, x + (int)flx, y + (int)fly, Dx - flx, Dy - fly, ps.drop, sdrop, flags,
                                     &sumG);
        acc = dd_add(acc, dd_mul_d(F, (double)coef));
    }
    for (int o = 16; o; o >>= 1) {
        const dd T = {__shfl_xor_sync(0xffffffffu, acc.hi, o), __shfl_xor_sync(0xffffffffu, acc.lo, o)};
        acc = dd_add(acc, T);
    }
    double norm = 1.0;
    for (int q = 0; q < ns; ++q) {
        const double ia = 1.0 / ps.ap[dirs[q]];
        for (int i = 0; i < R; ++i) norm *= ia;
    }
    return dd_to_d(acc) * norm;
}

// BSF_PREC_AUTO: fp64 first; recompute in double-double when the estimate
// exceeds 1e-9 (the fp64 results kept were within 1.6e-11 in calibration).
template <int R>
__device__ __forceinline__ double mesh_auto(const GView &gv, const LutBasis &L, const PixelScales &ps, int x, int y,
                                            int *flags, int *used_dd, double *ratios = nullptr) {
    double err = 1.0;
    double v = mesh<R, false>(gv, L, ps, x, y, flags, &err, ratios);
    *used_dd = !(err <= 1e-9);
    if (*used_dd) v = mesh<R, true>(gv, L, ps, x, y, flags);
    return v;
}

__device__ __forceinline__ void warp_count(unsigned long long *ctr, bool pred) {
    unsigned m = __activemask();
    unsigned b = __ballot_sync(m, pred);
    int leader = __ffs(m) - 1;
    if ((int)(threadIdx.x & 31) == leader && b) atomicAdd(ctr, (unsigned long long)__popc(b));
}

template <int R, int MODE>
#ifndef BSF_GATHER_MINB
#define BSF_GATHER_MINB 6
#endif
__global__ void __launch_bounds__(128, BSF_GATHER_MINB) gather_kernel(GatherArgs a, const LutBasis *__restrict__ luts) {
    int img, x, y;
    long long oidx;
    if (a.pts) {
        int idx = blockIdx.x * 128 + threadIdx.x;
        if (idx >= a.npts) return;
        img = a.pts[3 * idx];
        x = a.pts[3 * idx + 1];
        y = a.pts[3 * idx + 2];
        oidx = idx;
    } else {
        x = blockIdx.x * 16 + (threadIdx.x & 15);
        y = blockIdx.y * 8 + (threadIdx.x >> 4);
        img = blockIdx.z;
        if (x >= a.geo.W || y >= a.geo.H) return;
        oidx = ((long long)img * a.geo.H + y) * a.geo.W + x;
    }
    const Geometry &geo = a.geo;
    size_t plane = (size_t)geo.H * geo.W;
    int bc = img / a.channels;
    const float *cv = a.cov + (size_t)bc * 3 * plane + (size_t)y * geo.W + x;
    PixelScales ps;
    double sx = __ldg(cv), sy = __ldg(cv + plane), th = __ldg(cv + 2 * plane);
    if (a.cov_layout == BSF_COV_C11_C12_C22) cov_from_c(sx, sy, th, sx, sy, th);
    pixel_scales(sx, sy, th, a.policy, a.clamp, R, ps);
    double res;
    int flags = ps.flags;
    int used_dd = MODE == BSF_PREC_DD;
    double ratios[2] = {0.0, 0.0};
    if (flags & (FLAG_INFEASIBLE | FLAG_TWO_ZERO)) {
        res = __longlong_as_double(0x7ff8000000000000LL);
    } else {
        int slot = geo.nbases == 2 ? ps.basis : 0;
        GView gv = {a.g + ((size_t)slot * geo.nimg + img) * geo.GH * geo.GW, -geo.P, 0, geo.GW, geo.GH, 0.0};
        if (MODE == BSF_PREC_AUTO)
            res = mesh_auto<R>(gv, luts[ps.basis], ps, x, y, &flags, &used_dd, ratios);
        else
            res = mesh<R, MODE == BSF_PREC_DD>(gv, luts[ps.basis], ps, x, y, &flags, nullptr, ratios);
    }
    if (a.aux) {
        double *ax = a.aux + BSF_AUX * oidx;
        ax[0] = ps.basis;
        ax[1] = ps.drop;
        ax[2] = ps.clamped;
        ax[3] = flags;
        for (int k = 0; k < 4; ++k) ax[4 + k] = ps.ap[k];
        ax[8] = used_dd;
        ax[9] = ratios[0];
        ax[10] = ratios[1];
        ax[11] = 0.0;
    }
    if (a.out_f32)
        ((float *)a.out)[oidx] = (float)res;
    else
        ((double *)a.out)[oidx] = res;
    if (a.stats) {
        warp_count(a.stats + 0, true);
        warp_count(a.stats + 1, ps.clamped != 0);
        warp_count(a.stats + 2, ps.drop >= 0);
        warp_count(a.stats + 3, ps.basis == BASIS_THETA_PRIME);
        warp_count(a.stats + 5, used_dd != 0);
        if (flags) atomicOr(a.stats + 4, (unsigned long long)flags);
    }
}


// ---------------------------------------------------------------------------
// Tile-anchored fused path.
//
// Restarting the running sums at zero on a window that contains the kernel
// supports of a tile's pixels (plus the windows of their taps) leaves the
// filter output unchanged (the output only depends on f inside the supports,
// and truncating the sum domain adds only functions constant along a sum
// direction, which the mesh annihilates: SURVEY F9, R18).  It bounds
// the sums' magnitude by the tile's own reach (conditioning) and
// keeps the sums in an L2-resident per-CTA scratch instead of an HBM image.
// ---------------------------------------------------------------------------
struct TileDomain {
    int X0, Y0, NX, NY;
};

__device__ __forceinline__ TileDomain tile_domain(const LutBasis &L, int R, int x0, int y0, int EX, int EY) {
    TileDomain d;
    d.X0 = x0 - EX + L.wxmin - 2 * R - 1;  // zero-scale lattice difference reaches back R|s_x| <= 2R
    int X1 = x0 + TILE - 1 + EX + L.wxmax + 2 * R + 1;
    d.Y0 = y0 - EY;                        // no kernel support above: zero state
    int Y1 = y0 + TILE - 1 + EY + L.wymax + 1;
    d.NX = X1 - d.X0 + 1;
    d.NY = Y1 - d.Y0 + 1;
    return d;
}

// one running-sum level along (sx, sy) on the NX x NY local domain; threads own lines
__device__ __forceinline__ void tile_scan_level(double2 *__restrict__ G, int NX, int NY, int sx, int sy) {
    int nlines = sy == 0 ? NY : sy * NX + abs(sx) * (NY - sy);
    for (int l = threadIdx.x; l < nlines; l += blockDim.x) {
        int xs, ys;
        if (sy == 0) {
            xs = 0;
            ys = l;
        } else if (l < sy * NX) {
            xs = l % NX;
            ys = l / NX;
        } else {
            int q = l - sy * NX, as = abs(sx);
            ys = sy + q / as;
            xs = sx > 0 ? q % as : NX - 1 - q % as;
        }
        dd acc = {0.0, 0.0};
        for (int xx = xs, yy = ys; xx >= 0 && xx < NX && yy < NY; xx += sx, yy += sy) {
            double2 v = G[(size_t)yy * NX + xx];
            acc = dd_add(acc, {v.x, v.y});
            G[(size_t)yy * NX + xx] = make_double2(acc.hi, acc.lo);
        }
    }
}

template <int R, int MODE>
#ifndef BSF_TILE_MINB
#define BSF_TILE_MINB 3
#endif
__global__ void __launch_bounds__(256, BSF_TILE_MINB) tile_kernel(TileArgs a, const LutBasis *__restrict__ luts) {
    __shared__ int s_item, s_ex[2], s_ey[2], s_used, s_bad;
    const int tid = threadIdx.x;
    double2 *scr = a.scratch + (size_t)blockIdx.x * 2 * a.cap;
    const int tiles_per_img = a.ntx * a.nty;
    const int nitems = a.pts ? a.npts : a.tiles ? a.ntiles : tiles_per_img * a.nimg;
    for (;;) {
        if (tid == 0) {
            s_item = atomicAdd(a.counter, 1);
            s_ex[0] = s_ex[1] = s_ey[0] = s_ey[1] = 0;
            s_used = 0;
            s_bad = 0;
        }
        __syncthreads();
        if (s_item >= nitems) break;
        const int item = a.tiles ? a.tiles[s_item] : s_item;
        int img, x0, y0, want = -1;
        if (a.pts) {
            img = a.pts[3 * item];
            int px = a.pts[3 * item + 1], py = a.pts[3 * item + 2];
            x0 = px & ~(TILE - 1);
            y0 = py & ~(TILE - 1);
            want = (px - x0) + TILE * (py - y0);
        } else {
            img = item / tiles_per_img;
            int rem = item % tiles_per_img;
            x0 = (rem % a.ntx) * TILE;
            y0 = (rem / a.ntx) * TILE;
        }
        const int x = x0 + (tid % TILE), y = y0 + tid / TILE;
        const bool valid = x < a.W && y < a.H;
        PixelScales ps;
        ps.flags = 0;
        ps.basis = 0;
        ps.drop = -1;
        ps.clamped = 0;
        if (valid) {
            size_t plane = (size_t)a.H * a.W;
            const float *cv = a.cov + (size_t)(img / a.channels) * 3 * plane + (size_t)y * a.W + x;
            double sx = __ldg(cv), sy = __ldg(cv + plane), th = __ldg(cv + 2 * plane);
            if (a.cov_layout == BSF_COV_C11_C12_C22) cov_from_c(sx, sy, th, sx, sy, th);
            pixel_scales(sx, sy, th, a.policy, a.clamp, R, ps);
        }
        const bool live = valid && !(ps.flags & (FLAG_INFEASIBLE | FLAG_TWO_ZERO));
        if (live) {
            double ex = 0.0, ey = 0.0;
            for (int k = 0; k < 4; ++k) {
                ex += ps.ap[k] * abs(c_steps[ps.basis][k][0]);
                ey += ps.ap[k] * c_steps[ps.basis][k][1];
            }
            atomicMax(&s_ex[ps.basis], (int)ceil(0.5 * R * ex));
            atomicMax(&s_ey[ps.basis], (int)ceil(0.5 * R * ey));
            atomicOr(&s_used, 1 << ps.basis);
        }
        __syncthreads();
        const int used = s_used;
        const size_t ipl = (size_t)a.H * a.W;
        for (int b = 0; b < 2; ++b) {
            if (!(used & (1 << b))) continue;
            TileDomain d = tile_domain(luts[b], R, x0, y0, s_ex[b], s_ey[b]);
            if ((long long)d.NX * d.NY > a.cap) {
                if (tid == 0) s_bad = 1;
                continue;
            }
            double2 *G = scr + (size_t)b * a.cap;
            const int n = d.NX * d.NY;
            for (int i = tid; i < n; i += blockDim.x) {
                int X = d.X0 + i % d.NX, Y = d.Y0 + i / d.NX;
                double v = 0.0;
                if (X >= 0 && X < a.W && Y >= 0 && Y < a.H) {
                    size_t o = (size_t)img * ipl + (size_t)Y * a.W + X;
                    v = a.in_u8 ? (double)((const uint8_t *)a.f)[o] : (double)((const float *)a.f)[o];
                }
                G[i] = make_double2(v, 0.0);
            }
            __syncthreads();
            for (int rep = 0; rep < R; ++rep)
                for (int lv = 0; lv < 4; ++lv) {
                    tile_scan_level(G, d.NX, d.NY, c_scan_order[b][lv][0], c_scan_order[b][lv][1]);
                    __syncthreads();
                }
        }
        __syncthreads();
        int flags = ps.flags | (s_bad ? FLAG_RANGE : 0);
        const bool mine = a.pts ? (tid == want) : valid;
        double res = __longlong_as_double(0x7ff8000000000000LL);
        int used_dd = MODE == BSF_PREC_DD;
        double ratios[2] = {0.0, 0.0};
        if (mine && live && !s_bad) {
            TileDomain d = tile_domain(luts[ps.basis], R, x0, y0, s_ex[ps.basis], s_ey[ps.basis]);
            GView gv = {scr + (size_t)ps.basis * a.cap, d.X0, d.Y0, d.NX, d.NY, 0.0};
            if (MODE == BSF_PREC_AUTO) {
                double err = 1.0;
                res = mesh<R, false>(gv, luts[ps.basis], ps, x, y, &flags, &err, ratios);
                used_dd = !(err <= 1e-9);
            } else {
                res = mesh<R, MODE == BSF_PREC_DD>(gv, luts[ps.basis], ps, x, y, &flags, nullptr, ratios);
            }
        }
        if (MODE == BSF_PREC_AUTO) {
            // recompute the rejected pixels in double-double, packed densely
            // onto the first threads so warps do not run it with idle lanes
            __shared__ int s_nrej;
            __shared__ short s_rej[256];
            __shared__ PixelScales s_ps[256];
            __shared__ double s_res[256];
            __shared__ int s_flags[256];
            if (tid == 0) s_nrej = 0;
            __syncthreads();
            if (used_dd && mine && live && !s_bad) {
                int k = atomicAdd(&s_nrej, 1);
                s_rej[k] = (short)tid;
                s_ps[tid] = ps;
            }
            __syncthreads();
            if (tid < s_nrej) {
                int src = s_rej[tid];
                PixelScales q = s_ps[src];
                int qx = x0 + (src % TILE), qy = y0 + src / TILE, qf = 0;
                TileDomain d = tile_domain(luts[q.basis], R, x0, y0, s_ex[q.basis], s_ey[q.basis]);
                GView gv = {scr + (size_t)q.basis * a.cap, d.X0, d.Y0, d.NX, d.NY, 0.0};
                s_res[src] = mesh<R, true>(gv, luts[q.basis], q, qx, qy, &qf);
                s_flags[src] = qf;
            }
            __syncthreads();
            if (used_dd && mine && live && !s_bad) {
                res = s_res[tid];
                flags |= s_flags[tid];
            }
        }
        if (mine) {
            long long oidx = a.pts ? item : (long long)img * ipl + (size_t)y * a.W + x;
            if (a.aux) {
                double *ax = a.aux + BSF_AUX * oidx;
                ax[0] = ps.basis;
                ax[1] = ps.drop;
                ax[2] = ps.clamped;
                ax[3] = flags;
                for (int k = 0; k < 4; ++k) ax[4 + k] = ps.ap[k];
                ax[8] = used_dd;
                ax[9] = ratios[0];
                ax[10] = ratios[1];
                ax[11] = 0.0;
            }
            if (a.out_f32 && !a.pts)
                ((float *)a.out)[oidx] = (float)res;
            else
                ((double *)a.out)[oidx] = res;
            if (a.stats) {
                atomicAdd(a.stats + 0, 1ull);
                if (ps.clamped) atomicAdd(a.stats + 1, 1ull);
                if (ps.drop >= 0) atomicAdd(a.stats + 2, 1ull);
                if (ps.basis == BASIS_THETA_PRIME) atomicAdd(a.stats + 3, 1ull);
                if (used_dd) atomicAdd(a.stats + 5, 1ull);
                if (flags) atomicOr(a.stats + 4, (unsigned long long)flags);
            }
        }
        __syncthreads();
    }
}

size_t tile_capacity(int order, float max_sigma, const LutBasis *L, int basis_mask, int tile) {
    int E = (int)ceil((double)max_sigma * sqrt(24.0 * order)) + 1;  // (r/2) sum_k a'_k |s_k| bound
    size_t cap = 0;
    for (int b = 0; b < 2; ++b) {
        if (!(basis_mask & (1 << b))) continue;
        size_t nx = tile + 2 * E + (L[b].wxmax - L[b].wxmin) + 4 * order + 4;
        size_t ny = tile + 2 * E + L[b].wymax - L[b].wymin + 2;
        cap = nx * ny > cap ? nx * ny : cap;
    }
    return cap;
}

int tile_slots() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return BSF_TILE_MINB * sms;
}

template <int R>
static void launch_tile_r(const TileArgs &a, int prec, int slots, cudaStream_t st, const LutBasis *luts) {
    if (prec == BSF_PREC_DD)
        tile_kernel<R, BSF_PREC_DD><<<slots, 256, 0, st>>>(a, luts);
    else if (prec == BSF_PREC_AUTO)
        tile_kernel<R, BSF_PREC_AUTO><<<slots, 256, 0, st>>>(a, luts);
    else
        tile_kernel<R, BSF_PREC_FP64><<<slots, 256, 0, st>>>(a, luts);
}

cudaError_t launch_tile_impl(const TileArgs &a, int order, int prec, int slots, cudaStream_t st,
                             const LutBasis *luts, long long *nl) {
    const cudaError_t e = cudaMemsetAsync(a.counter, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    switch (order) {
        case 1: launch_tile_r<1>(a, prec, slots, st, luts); break;
        case 2: launch_tile_r<2>(a, prec, slots, st, luts); break;
        case 3: launch_tile_r<3>(a, prec, slots, st, luts); break;
        case 4: launch_tile_r<4>(a, prec, slots, st, luts); break;
        default: return cudaErrorInvalidValue;
    }
    ++*nl;
    return cudaGetLastError();
}

template <int R>
static void launch_r(const GatherArgs &a, int prec, cudaStream_t st, const LutBasis *luts) {
    dim3 grid, block(128);
    if (a.pts)
        grid = dim3((a.npts + 127) / 128, 1, 1);
    else
        grid = dim3((a.geo.W + 15) / 16, (a.geo.H + 7) / 8, a.geo.nimg);
    if (prec == BSF_PREC_DD)
        gather_kernel<R, BSF_PREC_DD><<<grid, block, 0, st>>>(a, luts);
    else if (prec == BSF_PREC_AUTO)
        gather_kernel<R, BSF_PREC_AUTO><<<grid, block, 0, st>>>(a, luts);
    else
        gather_kernel<R, BSF_PREC_FP64><<<grid, block, 0, st>>>(a, luts);
}

#include "bsf_fused.cuh"
#include "bsf_gx1.cuh"

#ifdef BSF_TAP_DUMP
extern "C" void bsf_debug_set_dump(double *p) { cudaMemcpyToSymbol(g_tap_dump, &p, sizeof p); }
#endif
cudaError_t launch_gather_impl(const GatherArgs &a, int order, int prec, cudaStream_t st, const LutBasis *luts,
                               long long *nl) {
    switch (order) {
        case 1: launch_r<1>(a, prec, st, luts); break;
        case 2: launch_r<2>(a, prec, st, luts); break;
        case 3: launch_r<3>(a, prec, st, luts); break;
        case 4: launch_r<4>(a, prec, st, luts); break;
        default: return cudaErrorInvalidValue;
    }
    ++*nl;
    return cudaGetLastError();
}

}  // namespace bsf
