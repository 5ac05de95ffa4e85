// Internal declarations shared by bsf_api.cu and bsf_kernels.cu.
#pragma once
#include <atomic>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bsf.h"

namespace bsf {

constexpr int MAX_REG = 32;
constexpr int BSF_AUX = 12;  // doubles of per-point diagnostics
// device-side condition flags (also in bsf_pixel.cuh)
enum { FLAG_RANGE_H = 1, FLAG_INFEASIBLE_H = 2, FLAG_TWO_ZERO_H = 4, FLAG_SOLVER_H = 8 };
constexpr int NVAR = 5;  // full kernel + one per dropped direction

// Column layout of the integer tables for the FP64 MMA contraction
// (bsf_fused.cuh).  The N dimension (monomials phi_x^i phi_y^j, degree <= deg)
// is padded to 8 bsf_nt(deg) columns; lane l of a warp holds accumulator
// columns 8 j + 2 (l % 4) + {0, 1}.  Each polynomial row i (the DEG - i + 1
// monomials of x-power i) is given whole to one lane of the quad, at
// consecutive slots k (column 8 (k / 2) + 2 lane + k % 2), highest y power
// first, so that lane can run the row's Horner scheme in phi_y on its own
// registers.  Partition of the row lengths 1..deg+1 over the 4 lanes:
__host__ __device__ constexpr int bsf_nt(int deg) {
    return deg == 1 ? 1 : deg == 2 ? 2 : deg == 4 ? 3 : deg == 6 ? 4 : deg == 7 ? 5 : deg == 10 ? 9 : deg == 14 ? 15 : -1;
}
__host__ __device__ constexpr int bsf_part(int deg, int lane, int k) {  // k-th row length of a lane, 0 = end
    const int t1[4][3] = {{2, 0, 0}, {1, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    const int t2[4][3] = {{3, 1, 0}, {2, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    const int t4[4][3] = {{5, 1, 0}, {4, 2, 0}, {3, 0, 0}, {0, 0, 0}};
    const int t6[4][3] = {{7, 1, 0}, {6, 2, 0}, {5, 3, 0}, {4, 0, 0}};
    const int t7[4][3] = {{8, 2, 0}, {7, 3, 0}, {6, 4, 0}, {5, 1, 0}};
    const int t10[4][5] = {{11, 7, 0, 0, 0}, {10, 8, 0, 0, 0}, {9, 6, 3, 0, 0}, {5, 4, 2, 1, 0}};
    const int t14[4][7] = {{15, 14, 1, 0, 0, 0, 0}, {13, 12, 5, 0, 0, 0, 0}, {11, 10, 9, 0, 0, 0, 0}, {8, 7, 6, 4, 3, 2, 0}};
    return deg == 1 ? (k < 3 ? t1[lane][k] : 0)
         : deg == 2 ? (k < 3 ? t2[lane][k] : 0)
         : deg == 4 ? (k < 3 ? t4[lane][k] : 0)
         : deg == 6 ? (k < 3 ? t6[lane][k] : 0)
         : deg == 7 ? (k < 3 ? t7[lane][k] : 0)
         : deg == 10 ? (k < 5 ? t10[lane][k] : 0)
         : deg == 14 ? (k < 7 ? t14[lane][k] : 0) : 0;
}
__host__ __device__ constexpr int bsf_row_lane(int deg, int i) {  // lane holding row i
    for (int l = 0; l < 4; ++l)
        for (int k = 0; bsf_part(deg, l, k); ++k)
            if (bsf_part(deg, l, k) == deg - i + 1) return l;
    return -1;
}
__host__ __device__ constexpr int bsf_row_slot(int deg, int i) {  // first slot of row i in its lane
    const int l = bsf_row_lane(deg, i);
    int s = 0;
    for (int k = 0; bsf_part(deg, l, k); ++k) {
        if (bsf_part(deg, l, k) == deg - i + 1) return s;
        s += bsf_part(deg, l, k);
    }
    return -1;
}
__host__ __device__ constexpr int bsf_row_q(int deg, int i) {  // position of row i in its lane's list
    const int l = bsf_row_lane(deg, i);
    for (int k = 0; bsf_part(deg, l, k); ++k)
        if (bsf_part(deg, l, k) == deg - i + 1) return k;
    return -1;
}
__host__ __device__ constexpr int bsf_lane_rows(int deg, int lane) {
    int k = 0;
    while (bsf_part(deg, lane, k)) ++k;
    return k;
}
// slot masks of a lane: bit k set if slot k starts a row / belongs to a row
__host__ __device__ constexpr unsigned bsf_start_mask(int deg, int lane) {
    unsigned m = 0;
    int s = 0;
    for (int k = 0; bsf_part(deg, lane, k); ++k) {
        m |= 1u << s;
        s += bsf_part(deg, lane, k);
    }
    return m;
}
__host__ __device__ constexpr unsigned bsf_valid_mask(int deg, int lane) {
    int s = 0;
    for (int k = 0; bsf_part(deg, lane, k); ++k) s += bsf_part(deg, lane, k);
    return s >= 32 ? 0xffffffffu : ((1u << s) - 1u);
}
// accumulator column of monomial phi_x^i phi_y^j
__host__ __device__ constexpr int bsf_mono_col(int deg, int i, int j) {
    return 8 * ((bsf_row_slot(deg, i) + deg - i - j) >> 1) + 2 * bsf_row_lane(deg, i) +
           ((bsf_row_slot(deg, i) + deg - i - j) & 1);
}

// One interpolation table (basis, order, variant) in device memory.
struct LutVar {
    int deg, nmon, nmax;
    const int2 *offs;      // [nreg][nmax]
    const int *counts;     // [nreg]
    const double2 *coef;   // [nreg][nmax][nmon] double-double (n / L)
    const double *num;     // [nreg][nslot4][nmonp] integer numerators n (exact doubles), zero padded
    const int2 *offs4;     // [nreg][nslot4] window offsets, padded with (0, 0)
    int nmonp;             // 8 bsf_nt(deg) columns (FP64 MMA n-tiles), bsf_mono_col layout
    int nslot4;            // nmax rounded up to 4 (FP64 MMA k-steps)
    int kbits;             // |G1| <= 2^kbits keeps sum_s G1 * n (or n1, n0) exact in fp64
    int nsplit;            // 1: num = n; 2: numerators split n = n1 2^shift + n0 (num = n1, num2 = n0, numf = n)
    int shift;
    const double *num2;    // [nreg][nslot4][nmonp] n0 (nsplit 2)
    const double *numf;    // [nreg][nslot4][nmonp] n (nsplit 2: the G0 limb's operand)
    const float *num32;    // order >= 3, when exact in fp32: [nreg][nslot4][nmonp] n (nsplit 1) or
                           // interleaved (n1, n0) pairs (nsplit 2) -- half the bytes of the MMA's B loads
    const signed char *n8; // order 1 (global-mode gather, bsf_gx1.cuh): [nreg][nmax][8] numerators n as int8
                           // (monomials in gen_lut order, zero padded); null when some |n| > 127
    const uint8_t *i8tab;  // order 3: numerator byte slices, UMMA canonical layout (bsf_api.cu), or null
    int i8na, i8nchunk;    // slices (the top one signed), 32-slot chunks per region
    float mean_count;      // window slots averaged over the regions (work-item cost estimate)
    double nabs;           // max over (region, monomial) of sum_s |n| (order 1: the gather's limb widths)
    double bnd;            // bound on |F - F^| (units 2^e) of the split contraction: gamma_{n+1} 0.5 max_reg sum_s,mu |n|
    double L;              // common denominator
};

struct LutBasis {
    int nreg;
    int2 normal[4];        // knot-line normals n_k = perp(s_k)
    int kmin[4];           // min floor(n_k . phi) over the unit cell
    int radix[4];
    signed char table[81]; // mixed-radix key -> region (or -1)
    double2 centre[MAX_REG];
    int wxmin, wxmax, wymin, wymax;  // window offset extents over all variants
    double hornerB;                  // max over all weights of sum_mu |c_mu| (Horner bound on [0,1]^2)
    LutVar var[NVAR];
};

struct Geometry {
    int W, H, P, Pb, GW, GH;
    int nimg;     // batch * channels
    int nbases;
};

struct GatherArgs {
    Geometry geo;
    int policy;   // BSF_THETA / BSF_THETA_PRIME / BSF_DUAL
    int clamp;
    int channels;
    int out_f32;
    const double2 *g;       // [nbases][nimg][GH][GW]
    const float *cov;       // [batch][3][H][W]
    void *out;              // [nimg][H][W]
    const int *pts;         // optional (img, x, y) triples
    int npts;
    double *aux;            // optional per-point diagnostics [8 * npts]
    unsigned long long *stats;  // [6]: pixels, clamped, zero, theta', flags(or), double-double
    int cov_layout;             // BSF_COV_SIGMA_THETA / BSF_COV_C11_C12_C22
};

// Tile-anchored fused path: per 16x16 output tile, local running sums on the
// tile's halo (zero state), then the gather from them.
struct TileArgs {
    int W, H, nimg, channels;
    int policy, clamp, out_f32, in_u8;
    int in_f64;             // input image is float64 (Algorithm 1's second pass)
    int cov_mode;           // COV_PLANES, COV_ISO (sigma_b^2 I), COV_SUB (C - sigma_b^2 I)
    const double *sigma2;   // [batch] sigma_b^2 of Algorithm 1 (COV_ISO / COV_SUB)
    double sigma2_scale;    // multiplies sigma2 (1 for Algorithm 1; the split shares of bsf_run_split)
    const void *f;          // [nimg][H][W]
    const float *cov;       // [batch][3][H][W]
    void *out;              // [nimg][H][W] (or float64[npts] with pts)
    const int *pts;         // optional (img, x, y) triples
    int npts;
    double *aux;            // optional per-point diagnostics
    double2 *scratch;       // [slots][2][cap]
    long long cap;          // points per basis per slot
    int *counter;           // work counter (zeroed before launch)
    int ntx, nty;
    unsigned long long *stats;
    unsigned long long *prof;  // optional [8] phase cycles (bsf_debug_phase_cycles)
    double split_tol;          // relative bound above which a pixel is recomputed in double-double
    double2 *fbuf;             // fused path: per-CTA tap values [slots][fused_items<R>()]
    int stile;                 // fused path: super-tile side (32 or 64)
    int replicate;             // fused path: f outside the image = nearest image pixel
    double *sbuf;              // fused path: per-CTA per-pixel scales [slots][FUSED_NQ_MAX][FT][5]
    double *scratch0;          // fused path, order >= 3: the rounded limb G0 of every plane, [slots][NPLANE][cap]
    // fused path work order (optional): order[i] = super-tile handed out i-th,
    // largest estimated work first (fused_cost_kernel / fused_order_kernel)
    int *order;
    unsigned char *order_bin;  // [items] cost bin of each super-tile
    unsigned *order_hist;      // [2][SCHED_NBIN] bin counts, scatter cursors, then the unit count
    long long order_cap;       // units (bin slots) the order buffers hold
    // global mode (order 1, u8): taps read the exact int64 global running sums
    // [nbases][nimg][gGH][gGW] (bsf_preintegrate_exact layout), limb shift per basis
    // output row window (row strips, bsf_plan_desc.nranks > 1): only image rows
    // [oy0, oy0 + oH) of the f block are filtered (oy0 a multiple of the
    // super-tile side); cov and out hold those rows only.  oH = 0: all rows.
    int oy0, oH;
    int cov_layout;             // BSF_COV_SIGMA_THETA / BSF_COV_C11_C12_C22
    const int *tiles;           // optional list of anchoring-tile indices to compute (bsf_run_tiles);
    int ntiles;                 // index = (img * tiles_y + ty) * tiles_x + tx in units of the plan's tile side
    const long long *gglob[2];  // per basis id (null: basis not in the plan / not global mode): the
                                // bsf_preintegrate_exact sums [nimg][gGH][gGW] of that basis
    int gP, gGW, gGH;
    int gGHv;                   // order-1 gather: domain rows already pre-integrated (bsf_run_host's banded
                                // scans; gGH otherwise): a pixel reading below is flagged FLAG_RANGE
    int gshift[2];
    int gvw[2];                 // order-1 gather, per basis id: limb width w of the two-limb contraction
                                // of zero-scale variant differences (0: three 21-bit limbs)
    int gdp4a;                  // order-1 gather: byte-plane dp4a contraction (bsf_gx1.cuh gx1_tap_dp)
    int i8;                     // order 3: exact limbs on tcgen05 kind::i8 (bsf_fused.cuh i8_tile)
};
constexpr int SCHED_NBIN = 128;
// Opt a kernel into more than 48 KB of dynamic shared memory, once per device
// (the attribute belongs to the device's context; plans may live on several
// devices of one process).  `done` is the caller's per-kernel flag array.
template <class K>
inline cudaError_t set_smem_attr(K kernel, int bytes, std::atomic<unsigned long long> &done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

constexpr int TILE = 16;
constexpr int FUSED_NQ_MAX = 16;  // sub-tiles per super-tile (64 x 64)
// diagnostics buffer (TileArgs::prof): 16 phase counters, then the busy cycles
// of the first BSF_PROF_ITEMS work items, then those of the first BSF_PROF_CTAS CTAs
constexpr int BSF_PROF_ITEMS = 8192, BSF_PROF_CTAS = 1024;
constexpr int BSF_PROF_WORK = 16 + BSF_PROF_ITEMS + BSF_PROF_CTAS;  // then 4 work figures per item
constexpr int BSF_PROF_WORDS = BSF_PROF_WORK + 4 * BSF_PROF_ITEMS;
enum { COV_PLANES = 0, COV_ISO = 1, COV_SUB = 2 };
cudaError_t launch_alg1_sigma2(const float *cov, int batch, int W, int H, int policy, int clamp, int layout,
                               double *sigma2, cudaStream_t st, long long *nlaunch);
size_t tile_capacity(int order, float max_sigma, const LutBasis *host_luts, int basis_mask, int tile);
int tile_slots();
cudaError_t launch_tile_impl(const TileArgs &a, int order, int precision, int slots, cudaStream_t st,
                             const LutBasis *luts_dev, long long *nlaunch);

// exact split contraction path (bsf_fused.cuh): one persistent CTA per SM,
// NPLANE_MAX planes of `cap` points per slot
constexpr int NPLANE_MAX = 10;
constexpr int KBITS_MIN = 20;
constexpr double BSF_SPLIT_TOL_DEFAULT = 5e-10;  // half the fp64 parity tolerance; see TileArgs::split_tol
#ifndef BSF_STILE64_REACH
#define BSF_STILE64_REACH 64.0  // reach above which the order-1 fused path uses 64 x 64 super-tiles
#endif
int fused_slots();
size_t fused_fbuf_items(int order);
cudaError_t launch_fused_impl(const TileArgs &a, int order, int slots, cudaStream_t st, const LutBasis *luts_dev,
                              long long *nlaunch);
// global-mode gather at order 1 (bsf_gx1.cuh): one thread per pixel, exact int32-limb contraction
constexpr int GX1_SLOTS_H = 2048, GX1_MAXREG_H = 32;
cudaError_t launch_gx1(const TileArgs &a, cudaStream_t st, const LutBasis *luts_dev, long long *nlaunch);

// launchers (bsf_kernels.cu)
// global pre-integration: one single-pass kernel per level (bsf_scan.cuh)
cudaError_t launch_preint_dd(const void *f, int u8, double2 *g, const Geometry &geo, int basis, int order,
                             cudaStream_t st, long long *nlaunch);
cudaError_t launch_preint_i64(const uint8_t *f, unsigned long long *g, const Geometry &geo, int basis, int order,
                              cudaStream_t st, long long *nlaunch);
// one level (level 0 reads f) of one basis, optionally continuing the running
// sums from the sy domain rows above (carry, [nimg][sy][GW]; null = zero state)
cudaError_t launch_scan_level(const void *f, int u8, void *g, int exact, const Geometry &geo, int basis, int level,
                              const void *carry, cudaStream_t st);
void scan_step(int basis, int level, int *sx, int *sy);
void set_scan_tma(int on);  // diagnostics: 0 = the cp.async strip kernel instead of the TMA-fed one
cudaError_t launch_fill_ones(void *f, int u8, size_t n, cudaStream_t st, long long *nlaunch);
cudaError_t launch_normalize(void *out, int out_f32, const double *den, size_t n, cudaStream_t st,
                             long long *nlaunch);
cudaError_t launch_gather_impl(const GatherArgs &a, int order, int precision, cudaStream_t st,
                               const LutBasis *luts_dev, long long *nlaunch);

}  // namespace bsf
