// Internal declarations shared by bsf_api.cu and bsf_kernels.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bsf.h"

namespace bsf {

constexpr int MAX_REG = 32;
constexpr int BSF_AUX = 12;  // doubles of per-point diagnostics
// device-side condition flags (also in bsf_pixel.cuh)
enum { FLAG_RANGE_H = 1, FLAG_INFEASIBLE_H = 2, FLAG_TWO_ZERO_H = 4, FLAG_SOLVER_H = 8 };
constexpr int NVAR = 5;  // full kernel + one per dropped direction

// One interpolation table (basis, order, variant) in device memory.
struct LutVar {
    int deg, nmon, nmax;
    const int2 *offs;      // [nreg][nmax]
    const int *counts;     // [nreg]
    const double2 *coef;   // [nreg][nmax][nmon] double-double (n / L)
    const double *num;     // [nreg][nslot4][nmonp] integer numerators n (exact doubles), zero padded
    const int2 *offs4;     // [nreg][nslot4] window offsets, padded with (0, 0)
    int nmonp;             // nmon rounded up to 8 (FP64 MMA n-tiles)
    int nslot4;            // nmax rounded up to 4 (FP64 MMA k-steps)
    int kbits;             // |G1| <= 2^kbits keeps sum_s G1 * n exact in fp64
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
};

// Tile-anchored fused path: per 16x16 output tile, local running sums on the
// tile's halo (zero state), then the gather from them.
struct TileArgs {
    int W, H, nimg, channels;
    int policy, clamp, out_f32, in_u8;
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
};
constexpr int TILE = 16;
size_t tile_capacity(int order, float max_sigma, const LutBasis *host_luts, int basis_mask, int tile);
int tile_slots();
cudaError_t launch_tile_impl(const TileArgs &a, int order, int precision, int slots, cudaStream_t st,
                             const LutBasis *luts_dev, long long *nlaunch);

// exact split contraction path (bsf_fused.cuh): one persistent CTA per SM,
// NPLANE_MAX planes of `cap` points per slot
constexpr int NPLANE_MAX = 10;
constexpr int KBITS_MIN = 20;  // tables whose exact limb would be narrower use the double-double tile kernel
int fused_slots();
cudaError_t launch_fused_impl(const TileArgs &a, int order, int slots, cudaStream_t st, const LutBasis *luts_dev,
                              long long *nlaunch);

// launchers (bsf_kernels.cu)
cudaError_t launch_fill_dd(const void *f, int u8, double2 *g, const Geometry &geo, int nbasis_copy,
                           cudaStream_t st, long long *nlaunch);
cudaError_t launch_fill_i64(const uint8_t *f, unsigned long long *g, const Geometry &geo, int nbasis_copy,
                            cudaStream_t st, long long *nlaunch);
cudaError_t launch_scan_dd(double2 *g, const Geometry &geo, int basis, int order, void *ws, size_t ws_bytes,
                           cudaStream_t st, long long *nlaunch);
cudaError_t launch_scan_i64(unsigned long long *g, const Geometry &geo, int basis, int order, void *ws,
                            size_t ws_bytes, cudaStream_t st, long long *nlaunch);
size_t scan_workspace_bytes(const Geometry &geo);
cudaError_t launch_gather_impl(const GatherArgs &a, int order, int precision, cudaStream_t st,
                               const LutBasis *luts_dev, long long *nlaunch);

}  // namespace bsf
