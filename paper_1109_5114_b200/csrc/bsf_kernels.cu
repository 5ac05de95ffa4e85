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
};
struct OpU64 {
    typedef unsigned long long T;
    __device__ static T zero() { return 0ull; }
    __device__ static T add(T a, T b) { return a + b; }  // wraps mod 2^64
    __device__ static T shfl_up(T v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
};

// ---------------------------------------------------------------------------
// fill: g = 0 on the domain, g[y][x+P] = f[y][x] on the image
// ---------------------------------------------------------------------------
template <class Op, class In>
__global__ void fill_kernel(const In *__restrict__ f, typename Op::T *__restrict__ g, Geometry geo, int ncopy) {
    long long n = (long long)geo.GH * geo.GW;
    int img = blockIdx.y;
    const In *fi = f + (size_t)img * geo.H * geo.W;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        int y = (int)(i / geo.GW), xg = (int)(i % geo.GW);
        int x = xg - geo.P;
        typename Op::T v = Op::zero();
        if (y < geo.H && x >= 0 && x < geo.W) {
            if constexpr (sizeof(typename Op::T) == 16)
                v = make_double2((double)fi[(size_t)y * geo.W + x], 0.0);
            else
                v = (typename Op::T)fi[(size_t)y * geo.W + x];
        }
        for (int b = 0; b < ncopy; ++b) g[((size_t)b * geo.nimg + img) * n + i] = v;
    }
}

// ---------------------------------------------------------------------------
// Horizontal level s = (1, 0): one CTA per (row, image); tiles of 256 with a
// warp-shuffle block scan and a running carry.
// ---------------------------------------------------------------------------
template <class Op>
__global__ void __launch_bounds__(256) scan_rows_kernel(typename Op::T *__restrict__ g, int GW, size_t img_stride) {
    typedef typename Op::T T;
    __shared__ T warp_tot[8];
    __shared__ T carry_s;
    T *row = g + blockIdx.y * img_stride + (size_t)blockIdx.x * GW;
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T carry = Op::zero();
    for (int base = 0; base < GW; base += 256) {
        int x = base + threadIdx.x;
        T v = x < GW ? row[x] : Op::zero();
        // inclusive warp scan
        for (int d = 1; d < 32; d <<= 1) {
            T o = Op::shfl_up(v, d);
            if (lane >= d) v = Op::add(v, o);
        }
        if (lane == 31) warp_tot[wid] = v;
        __syncthreads();
        T pre = carry;
        for (int w = 0; w < wid; ++w) pre = Op::add(pre, warp_tot[w]);
        v = Op::add(pre, v);
        if (x < GW) row[x] = v;
        if (threadIdx.x == 255) carry_s = v;
        __syncthreads();
        carry = carry_s;
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Levels with s_y >= 1: lines q0 + j s.  Rows are cut into chunks of RC rows;
// a line meets chunk c in one segment.  Three passes:
//   partial: per (chunk, phase, line) segment sum          (reads level input)
//   carry:   per line, exclusive scan over chunks          (tiny)
//   apply:   per segment, inclusive scan + carry, in place (reads + writes)
// Lines are indexed at the chunk's first row of their phase by i = x + Xpad,
// i in [0, NL); a line moves by delta = sx*RC/sy columns per chunk.
// Points outside the domain are zero state (truncated domain, R3).
// ---------------------------------------------------------------------------
constexpr int RC = 32;

struct ScanShape {
    int sx, sy, Xpad, NL, NC, delta;
};

static ScanShape scan_shape(const Geometry &geo, int sx, int sy) {
    ScanShape s;
    s.sx = sx;
    s.sy = sy;
    s.Xpad = abs(sx) * ((RC + sy - 1) / sy);
    s.NL = geo.GW + 2 * s.Xpad;
    s.NC = (geo.GH + RC - 1) / RC;
    s.delta = sx * (RC / sy);
    return s;
}

template <class Op>
__global__ void scan_partial_kernel(const typename Op::T *__restrict__ g, Geometry geo, ScanShape sh,
                                    typename Op::T *__restrict__ partial) {
    typedef typename Op::T T;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= sh.NL) return;
    int c = blockIdx.y / sh.sy, ph = blockIdx.y % sh.sy, img = blockIdx.z;
    const T *gi = g + (size_t)img * geo.GH * geo.GW;
    int y = c * RC + ph, x = i - sh.Xpad;
    int yend = min((c + 1) * RC, geo.GH);
    T acc = Op::zero();
    for (; y < yend; y += sh.sy, x += sh.sx)
        if (x >= 0 && x < geo.GW) acc = Op::add(acc, gi[(size_t)y * geo.GW + x]);
    partial[(((size_t)img * sh.NC + c) * sh.sy + ph) * sh.NL + i] = acc;
}

template <class Op>
__global__ void scan_carry_kernel(const typename Op::T *__restrict__ partial, typename Op::T *__restrict__ carry,
                                  ScanShape sh, int i0lo, int nlines) {
    typedef typename Op::T T;
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nlines * sh.sy) return;
    int img = blockIdx.y;
    int ph = t % sh.sy, i0 = i0lo + t / sh.sy;
    size_t base = (size_t)img * sh.NC * sh.sy * sh.NL;
    T run = Op::zero();
    for (int c = 0; c < sh.NC; ++c) {
        int ic = i0 + c * sh.delta;
        if (ic >= 0 && ic < sh.NL) {
            size_t o = base + ((size_t)c * sh.sy + ph) * sh.NL + ic;
            carry[o] = run;
            run = Op::add(run, partial[o]);
        }
    }
}

template <class Op>
__global__ void scan_apply_kernel(typename Op::T *__restrict__ g, Geometry geo, ScanShape sh,
                                  const typename Op::T *__restrict__ carry) {
    typedef typename Op::T T;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= sh.NL) return;
    int c = blockIdx.y / sh.sy, ph = blockIdx.y % sh.sy, img = blockIdx.z;
    T *gi = g + (size_t)img * geo.GH * geo.GW;
    int y = c * RC + ph, x = i - sh.Xpad;
    int yend = min((c + 1) * RC, geo.GH);
    T acc = carry[(((size_t)img * sh.NC + c) * sh.sy + ph) * sh.NL + i];
    for (; y < yend; y += sh.sy, x += sh.sx)
        if (x >= 0 && x < geo.GW) {
            size_t o = (size_t)y * geo.GW + x;
            acc = Op::add(acc, gi[o]);
            gi[o] = acc;
        }
}

size_t scan_workspace_bytes(const Geometry &geo) {
    ScanShape s = scan_shape(geo, 2, 1);  // widest NL, most chunks per phase
    size_t per = (size_t)s.NC * 2 * (geo.GW + 4 * RC);
    return 2 * per * 16 * (size_t)geo.nimg;
}

template <class Op>
static cudaError_t scan_levels(typename Op::T *g, const Geometry &geo, int basis, int order, void *ws,
                               size_t ws_bytes, cudaStream_t st, long long *nl) {
    typedef typename Op::T T;
    if (ws_bytes < scan_workspace_bytes(geo)) return cudaErrorInvalidValue;
    size_t half = ws_bytes / 2;
    T *partial = (T *)ws;
    T *carry = (T *)((char *)ws + half);
    size_t img_stride = (size_t)geo.GH * geo.GW;
    for (int rep = 0; rep < order; ++rep) {
        for (int lv = 0; lv < 4; ++lv) {
            int sx = h_scan_order[basis][lv][0], sy = h_scan_order[basis][lv][1];
            if (sy == 0) {
                scan_rows_kernel<Op><<<dim3(geo.GH, geo.nimg), 256, 0, st>>>(g, geo.GW, img_stride);
                ++*nl;
                continue;
            }
            ScanShape sh = scan_shape(geo, sx, sy);
            dim3 grid((sh.NL + 127) / 128, sh.NC * sh.sy, geo.nimg);
            scan_partial_kernel<Op><<<grid, 128, 0, st>>>(g, geo, sh, partial);
            int span = (sh.NC - 1) * abs(sh.delta);
            int i0lo = sh.delta > 0 ? -span : 0;
            int nlines = sh.NL + span;
            scan_carry_kernel<Op><<<dim3((nlines * sh.sy + 127) / 128, geo.nimg), 128, 0, st>>>(partial, carry, sh,
                                                                                                  i0lo, nlines);
            scan_apply_kernel<Op><<<grid, 128, 0, st>>>(g, geo, sh, carry);
            *nl += 3;
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_fill_dd(const void *f, int u8, double2 *g, const Geometry &geo, int ncopy, cudaStream_t st,
                           long long *nl) {
    long long n = (long long)geo.GH * geo.GW;
    int blocks = (int)min((n + 255) / 256, 148LL * 8);
    dim3 grid(blocks, geo.nimg);
    if (u8)
        fill_kernel<OpDD, uint8_t><<<grid, 256, 0, st>>>((const uint8_t *)f, g, geo, ncopy);
    else
        fill_kernel<OpDD, float><<<grid, 256, 0, st>>>((const float *)f, g, geo, ncopy);
    ++*nl;
    return cudaGetLastError();
}

cudaError_t launch_fill_i64(const uint8_t *f, unsigned long long *g, const Geometry &geo, int ncopy,
                            cudaStream_t st, long long *nl) {
    long long n = (long long)geo.GH * geo.GW;
    int blocks = (int)min((n + 255) / 256, 148LL * 8);
    fill_kernel<OpU64, uint8_t><<<dim3(blocks, geo.nimg), 256, 0, st>>>(f, g, geo, ncopy);
    ++*nl;
    return cudaGetLastError();
}

cudaError_t launch_scan_dd(double2 *g, const Geometry &geo, int basis, int order, void *ws, size_t ws_bytes,
                           cudaStream_t st, long long *nl) {
    return scan_levels<OpDD>(g, geo, basis, order, ws, ws_bytes, st, nl);
}

cudaError_t launch_scan_i64(unsigned long long *g, const Geometry &geo, int basis, int order, void *ws,
                            size_t ws_bytes, cudaStream_t st, long long *nl) {
    return scan_levels<OpU64>(g, geo, basis, order, ws, ws_bytes, st, nl);
}

// ---------------------------------------------------------------------------
// Gather
// ---------------------------------------------------------------------------

// arithmetic policies: double-double or plain fp64
struct ArDD {
    typedef dd V;
    __device__ static V zero() { return {0.0, 0.0}; }
    __device__ static V from(double2 c) { return {c.x, c.y}; }
    __device__ static V fma(V a, V b, V c) { return dd_fma(a, b, c); }
    __device__ static V add(V a, V b) { return dd_add(a, b); }
    __device__ static V mul(V a, V b) { return dd_mul(a, b); }
    __device__ static V muli(V a, int k) { return dd_mul_d(a, (double)k); }
    __device__ static double to_d(V a) { return dd_to_d(a); }
};
struct ArD {
    typedef double V;
    __device__ static V zero() { return 0.0; }
    __device__ static V from(double2 c) { return c.x + c.y; }
    __device__ static V fma(V a, V b, V c) { return ::fma(a, b, c); }
    __device__ static V add(V a, V b) { return a + b; }
    __device__ static V mul(V a, V b) { return a * b; }
    __device__ static V muli(V a, int k) { return a * (double)k; }
    __device__ static double to_d(V a) { return a; }
};

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

template <class Ar>
__device__ __forceinline__ typename Ar::V horner2(const double2 *__restrict__ c, int deg, typename Ar::V px,
                                                  typename Ar::V py) {
    typedef typename Ar::V V;
    int idx = 0;
    V ax = Ar::zero();
    for (int i = deg; i >= 0; --i) {
        V ay = Ar::from(__ldg(c + idx++));
        for (int j = deg - i - 1; j >= 0; --j) ay = Ar::fma(ay, py, Ar::from(__ldg(c + idx++)));
        ax = (i == deg) ? ay : Ar::fma(ax, px, ay);
    }
    return ax;
}

template <class Ar>
__device__ __forceinline__ typename Ar::V load_g(const double2 *__restrict__ g, const Geometry &geo, int qx, int qy,
                                                 int *flags) {
    if (qy < 0) return Ar::zero();  // above the image every running sum is zero
    int gx = qx + geo.P;
    if (gx < 0 || gx >= geo.GW || qy >= geo.GH) {
        *flags |= FLAG_RANGE;
        return Ar::zero();
    }
    return Ar::from(__ldg(g + (size_t)qy * geo.GW + gx));
}

// F(Y) = sum_d G'(floor(Y) + d) M(frac(Y) - d)   (Eq. 11, r-fold, R4/R5)
template <int R, class Ar>
__device__ __forceinline__ typename Ar::V interp(const double2 *__restrict__ g, const Geometry &geo,
                                                 const LutBasis &L, const LutVar &V, dd Yx, dd Yy, int drop,
                                                 int2 sdrop, int *flags) {
    typedef typename Ar::V Val;
    dd fx, fy;
    int bx = (int)dd_floor(Yx, &fx);
    int by = (int)dd_floor(Yy, &fy);
    int reg = classify(L, fx.hi, fy.hi);
    double2 c = L.centre[reg];
    Val px, py;
    if constexpr (sizeof(Val) == 16) {
        px = dd_add_d(fx, -c.x);
        py = dd_add_d(fy, -c.y);
    } else {
        px = (fx.hi - c.x) + fx.lo;
        py = (fy.hi - c.y) + fy.lo;
    }
    int n = __ldg(V.counts + reg);
    const int2 *offs = V.offs + reg * V.nmax;
    const double2 *cf = V.coef + (size_t)reg * V.nmax * V.nmon;
    Val F = Ar::zero();
    for (int s = 0; s < n; ++s) {
        int2 d = __ldg(offs + s);
        int qx = bx + d.x, qy = by + d.y;
        Val G;
        if (drop < 0) {
            G = load_g<Ar>(g, geo, qx, qy, flags);
        } else {
            // G' = (1 - T_{s_drop})^R G  (exact lattice difference, R5)
            G = Ar::zero();
#pragma unroll
            for (int i = 0; i <= R; ++i) {
                Val t = load_g<Ar>(g, geo, qx - i * sdrop.x, qy - i * sdrop.y, flags);
                int cb = binom_small(R, i) * ((i & 1) ? -1 : 1);
                G = Ar::add(G, Ar::muli(t, cb));
            }
        }
        Val w = horner2<Ar>(cf + (size_t)s * V.nmon, V.deg, px, py);
        F = Ar::fma(G, w, F);
    }
    return F;
}

// out(p) = prod_k (1/a'_k)^R sum_j c_j F(p + sum_k (R/2 - j_k) a'_k s_k)
#ifdef BSF_TAP_DUMP
__device__ double *g_tap_dump;
#endif
template <int R, class Ar>
__device__ double mesh(const double2 *__restrict__ g, const Geometry &geo, const LutBasis &L, const PixelScales &ps,
                       int x, int y, int *flags) {
    typedef typename Ar::V Val;
    int dirs[4];
    int ns = 0;
    for (int k = 0; k < 4; ++k)
        if (k != ps.drop) dirs[ns++] = k;
    const LutVar &V = L.var[ps.drop + 1];
    int2 sdrop = make_int2(0, 0);
    if (ps.drop >= 0) sdrop = make_int2(c_steps[ps.basis][ps.drop][0], c_steps[ps.basis][ps.drop][1]);
    int ntap = 1;
    for (int q = 0; q < ns; ++q) ntap *= (R + 1);
    Val acc = Ar::zero();
    for (int t = 0; t < ntap; ++t) {
        int tt = t, coef = 1;
        dd Yx = dd_make((double)x), Yy = dd_make((double)y);
        for (int q = 0; q < ns; ++q) {
            int j = tt % (R + 1);
            tt /= (R + 1);
            coef *= binom_small(R, j) * ((j & 1) ? -1 : 1);
            int k = dirs[q];
            double m = 0.5 * R - j;  // half-integer: m * s exact
            Yx = dd_add(Yx, two_prod(m * c_steps[ps.basis][k][0], ps.ap[k]));
            Yy = dd_add(Yy, two_prod(m * c_steps[ps.basis][k][1], ps.ap[k]));
        }
        Val F = interp<R, Ar>(g, geo, L, V, Yx, Yy, ps.drop, sdrop, flags);
#ifdef BSF_TAP_DUMP
        if (g_tap_dump && x == 0 && y == 23) {
            double *o = g_tap_dump + 8 * t;
            dd fx, fy;
            o[0] = dd_floor(Yx, &fx);
            o[1] = dd_floor(Yy, &fy);
            o[2] = fx.hi; o[3] = fx.lo; o[4] = fy.hi; o[5] = fy.lo;
            if constexpr (sizeof(Val) == 16) { o[6] = F.hi; o[7] = F.lo; } else { o[6] = F; o[7] = 0; }
        }
#endif
        acc = Ar::add(acc, Ar::muli(F, coef));
    }
    double norm = 1.0;
    for (int q = 0; q < ns; ++q) {
        double ia = 1.0 / ps.ap[dirs[q]];
        for (int i = 0; i < R; ++i) norm *= ia;
    }
    return Ar::to_d(acc) * norm;
}

__device__ __forceinline__ void warp_count(unsigned long long *ctr, bool pred) {
    unsigned m = __activemask();
    unsigned b = __ballot_sync(m, pred);
    int leader = __ffs(m) - 1;
    if ((int)(threadIdx.x & 31) == leader && b) atomicAdd(ctr, (unsigned long long)__popc(b));
}

template <int R, class Ar>
__global__ void __launch_bounds__(128) gather_kernel(GatherArgs a, const LutBasis *__restrict__ luts) {
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
    pixel_scales(__ldg(cv), __ldg(cv + plane), __ldg(cv + 2 * plane), a.policy, a.clamp, R, ps);
    double res;
    int flags = ps.flags;
    if (flags & (FLAG_INFEASIBLE | FLAG_TWO_ZERO)) {
        res = __longlong_as_double(0x7ff8000000000000LL);
    } else {
        int slot = geo.nbases == 2 ? ps.basis : 0;
        const double2 *g = a.g + ((size_t)slot * geo.nimg + img) * geo.GH * geo.GW;
        res = mesh<R, Ar>(g, geo, luts[ps.basis], ps, x, y, &flags);
    }
    if (a.aux) {
        double *ax = a.aux + 8 * oidx;
        ax[0] = ps.basis;
        ax[1] = ps.drop;
        ax[2] = ps.clamped;
        ax[3] = flags;
        for (int k = 0; k < 4; ++k) ax[4 + k] = ps.ap[k];
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
        if (flags) atomicOr(a.stats + 4, (unsigned long long)flags);
    }
}

template <int R>
static void launch_r(const GatherArgs &a, int prec, cudaStream_t st, const LutBasis *luts) {
    dim3 grid, block(128);
    if (a.pts)
        grid = dim3((a.npts + 127) / 128, 1, 1);
    else
        grid = dim3((a.geo.W + 15) / 16, (a.geo.H + 7) / 8, a.geo.nimg);
    if (prec == BSF_PREC_DD)
        gather_kernel<R, ArDD><<<grid, block, 0, st>>>(a, luts);
    else
        gather_kernel<R, ArD><<<grid, block, 0, st>>>(a, luts);
}

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
