/*
 * bsf.h -- C ABI of the B200-native O(1) space-variant box-spline filter.
 *
 * Method: Chaudhury & Sanyal, "Improvements on 'Fast space-variant elliptical
 * filtering using box splines'" (arXiv 1109.5114), cited PAPER.md:<line>.
 *
 *   out(p) = sum_q f(q) beta^{(r)}_{a(p)}(p - q)
 *
 * computed by pre-integration (running sums along the four grid directions of
 * the box spline, each repeated r times; Alg. 3
 * step 2 PAPER.md:395-399) followed by a per-pixel local finite difference
 * (the (r+1)^4-tap mesh of Table 1, shifts of Eq. (10),
 * PAPER.md:339-342) whose taps are read from the running sums with the
 * interpolation of Eq. (11).  Where the running sums start
 * is the plan's anchoring (bsf_anchor): the paper's ONE global
 * pre-integration of the image (exact int64 at order 1 on u8 images, the
 * "global mode"; double-double otherwise), or sums restarted per output
 * super-tile on its halo (the same filter up to rounding, R18) at
 * orders where exact global sums would overflow.
 * The per-pixel scales a(p) come from the pixel's covariance (sigma_x,
 * sigma_y, theta) by the minimum-kurtosis rule on
 * C(p)/r (Prop. 1); basis Theta, Theta' or the per-pixel
 * dual choice of Algorithm 2.  DESIGN.md lists every
 * reading taken where the paper is silent.
 *
 * Conventions
 *  - Images are row-major, x fastest; the paper's (m, n) is (x, y).
 *  - All buffers are owned by the caller (device buffers from PyTorch unless a
 *    function says "host").  The library never frees caller memory.  The plan
 *    owns its workspace and its interpolation tables.
 *  - Every call that takes a stream is asynchronous on that stream
 *    (cudaStream_t passed as void*; NULL = legacy default stream).  Argument
 *    errors are returned synchronously; device-side conditions (margin
 *    violation, infeasible covariance with clamp = 0) raise flags read by
 *    bsf_get_stats(), which synchronises the stream.
 *  - Thread safety: a plan may be used by one host thread at a time, and its
 *    calls must be ordered (one stream, or streams the caller serialises):
 *    the plan's workspace (halo planes, tap and scale buffers, work counter)
 *    is shared by its launches.  Use one plan per concurrent stream.
 */
#ifndef BSF_H
#define BSF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bsf_plan_s *bsf_plan_t;

typedef enum {
    BSF_OK = 0,
    BSF_EINVAL = 1,      /* bad argument or descriptor field                  */
    BSF_ENOMEM = 2,      /* device or host allocation failed                  */
    BSF_ECUDA = 3,       /* CUDA runtime error (see bsf_last_error())          */
    BSF_EINFEASIBLE = 4, /* covariance outside the basis' elongation bound    */
    BSF_ERANGE = 5,      /* kernel reach exceeds the plan margins             */
    BSF_ENCCL = 6,       /* collective/transport error                        */
    BSF_EUNSUPPORTED = 7 /* valid request not implemented by this build       */
} bsf_status;

typedef enum { BSF_U8 = 0, BSF_F32 = 1, BSF_F64 = 2, BSF_I64 = 3, BSF_DD = 4 } bsf_dtype;

typedef enum {
    BSF_THETA = 0,       /* {0, 45, 90, 135} deg, steps (1,0),(1,1),(0,1),(-1,1) */
    BSF_THETA_PRIME = 1, /* {26.6, 63.4, 116.6, 153.4} deg, steps (2,1),(1,2),(-1,2),(-2,1) */
    BSF_DUAL = 2         /* Algorithm 2: per-pixel choice of the basis with the larger bound */
} bsf_basis;

typedef enum {
    BSF_PREC_FP64 = 0,   /* fp64 taps and weights: fast, ill-conditioned for large images */
    BSF_PREC_DD = 1,     /* double-double taps, weights and accumulation                                      */
    BSF_PREC_AUTO = 2    /* fp64 with an a-posteriori error bound; pixels whose bound exceeds 1e-11 are        */
                         /* recomputed in double-double                                */
} bsf_precision;

typedef enum {
    BSF_ANCHOR_GLOBAL = 0, /* the paper's single pre-integration of the whole image.
                            * u8 input at order 1 with every running sum below 2^62 ("global mode",
                            * bsf_geometry.global_mode = 1): exact int64 sums (bsf_preintegrate_exact)
                            * gathered by gx1_kernel with an exact int32-limb contraction (DESIGN.md
                            * §6.3; the fused kernel's DMMA groups as bsf_debug_option global_kernel 0).
                            * Otherwise double-double sums (bsf_preintegrate) + the per-pixel
                            * double-double gather (bsf_filter), whose rounding grows with the image
                            * size                                                      */
    BSF_ANCHOR_TILE = 1,   /* fused: running sums restarted per 32x32 (16x16 on small images, 64x64
                            * at order 1-2 with a large reach) output super-tile on its halo domain
                            * (R18, R20)                                                     */
    BSF_ANCHOR_AUTO = 2    /* global mode when the plan qualifies, else BSF_ANCHOR_TILE              */
} bsf_anchor;

typedef enum {
    BSF_BOUNDARY_ZERO = 0,     /* f = 0 outside the image (the paper's running sums, R1)  */
    BSF_BOUNDARY_REPLICATE = 1 /* f(q) = f(nearest image pixel) outside;    */
                               /* fused path only (BSF_ANCHOR_TILE, order <= 3)                   */
} bsf_boundary;

typedef enum {
    BSF_COV_SIGMA_THETA = 0, /* planes (sigma_x, sigma_y, theta): C = R(theta) diag(sx^2, sy^2) R(theta)^T,
                              * theta the angle of the sigma_x axis from the x axis (R14) */
    BSF_COV_C11_C12_C22 = 1  /* planes (C11, C12, C22) of the target covariance;
                              * decoded in fp64 to the same (sigma_x >= sigma_y, theta) form     */
} bsf_cov_layout;

typedef struct {
    int width, height;   /* image size W, H (pixels); with nranks > 1 the WHOLE image's size   */
    int batch;           /* number of covariance fields (independent images / frames)         */
    int channels;        /* images per covariance field (e.g. 3 for RGB); image b*C+c uses    */
                         /* covariance field b                                                */
    bsf_dtype in_dtype;  /* BSF_U8 or BSF_F32                                                 */
    bsf_dtype out_dtype; /* BSF_F64 or BSF_F32                                                */
    int order;           /* r >= 1: each direction repeated r times (north star)              */
    bsf_basis basis;
    float max_sigma;     /* upper bound of sigma_x, sigma_y over the covariance field         */
    int margin_x;        /* P: domain columns [-P, W+P); 0 = derive from max_sigma            */
    int margin_y;        /* Pb: domain rows [0, H+Pb); 0 = derive from max_sigma; -1 = none:
                          * the plan is a row strip of a larger domain (multi-GPU GLOBAL
                          * mode, bsf_scan_level), only pre-integration calls are valid   */
    int clamp;           /* 1: rho <- min(rho, 0.95 rho_B(phi)) at fixed trace/orientation    */
                         /* 0: infeasible pixels give NaN and raise BSF_EINFEASIBLE            */
    bsf_precision precision;
    int device;          /* CUDA device ordinal                                               */
    bsf_anchor anchor;   /* how bsf_run anchors the running sums                              */
    bsf_boundary boundary; /* image extension outside [0, W) x [0, H)                         */
    int super_tile;      /* BSF_ANCHOR_TILE anchoring unit: 0 = automatic (16 for images of
                          * fewer than 148 32x32 tiles, 64 at order 1 with a large reach, else
                          * 32), or 16 / 32 / 64.  Row strips that must reproduce a one-GPU
                          * run bit for bit pass the full image's geometry.super_tile      */
    bsf_cov_layout cov_layout; /* meaning of the three covariance planes                      */
    /* Multi-GPU: one image sharded by row strips over nranks
     * processes, one GPU each.  nranks = 1: single GPU (rank, nccl_id unused).
     * nranks > 1: the plan covers this rank's strip (bsf_strip_rows; rows given
     * by geometry.row0 / row_count), and
     *  - bsf_run (tile path) filters the strip: it needs the input rows within
     *    geometry.halo of the strip, which the library exchanges with the
     *    neighbouring ranks (ncclSend / ncclRecv on the call's stream) when the
     *    plan has a communicator (nccl_id != NULL); f_dev then holds the
     *    strip's own rows [row0, row0 + row_count).  Without a communicator
     *    (nccl_id == NULL: the caller assembles the halo, e.g. through
     *    torch.distributed) f_dev holds the block rows [block_row0,
     *    block_row0 + block_rows).  cov_dev and out_dev always hold the strip's
     *    own rows.  Only the own rows are computed; the result is bit-identical
     *    to a one-GPU run (same anchoring super-tiles).
     *  - bsf_preintegrate_exact computes the strip's rows of the paper's single
     *    global pre-integration (GLOBAL mode): domain rows [g_row0, g_row0 +
     *    g_rows) (the last rank also holds the bottom margin), scan carries
     *    passed down the rank chain after every level with a vertical step
     *    (needs the communicator); bit-identical to the one-GPU sums.
     * Plans with nranks > 1 are created collectively (ncclCommInitRank). */
    int rank, nranks;
    const void *nccl_id; /* 128-byte unique id from bsf_get_unique_id on rank 0, the same bytes on
                          * every rank (broadcast by the caller); NULL: no communicator      */
} bsf_plan_desc;

typedef struct {
    int margin_x, margin_y;  /* P, Pb actually used                                          */
    int g_width, g_height;   /* W + 2P, H + Pb                                                */
    int nbases;              /* running-sum sets per image: 2 for BSF_DUAL, else 1             */
    size_t g_bytes;          /* bytes of the pre-integrated buffer bsf_preintegrate writes    */
    size_t g_exact_bytes;    /* bytes of the bit-exact int64 buffer (u8 input only, else 0)   */
    int super_tile;          /* BSF_ANCHOR_TILE: side of the super-tiles the running sums are
                              * anchored on (16, 32 or 64); row strips that must reproduce a
                              * one-GPU run align to it and use it in their plans           */
    int global_mode;         /* 1: bsf_run gathers from exact int64 global sums (BSF_ANCHOR_GLOBAL /
                              * BSF_ANCHOR_AUTO, u8 input, order 1, sums below 2^62)        */
    int tile_unit;           /* side of the tiles bsf_run_tiles indexes (the anchoring unit of the tile
                              * path: super_tile, or 16 for the double-double tile kernel); 0 in
                              * global mode                                                 */
    /* row strips (nranks > 1; else the whole image): */
    int row0, row_count;     /* the image rows this rank filters                              */
    int block_row0, block_rows; /* the input rows the filter reads (own rows + halo)          */
    int halo;                /* halo rows (a multiple of super_tile)                          */
    int g_row0, g_rows;      /* GLOBAL mode: this rank's domain rows of the global sums       */
} bsf_geometry;

/* Partition of H image rows into nranks row strips aligned to `unit` rows
 * (super-tiles; the strips hold whole units, balanced, in rank order) and the
 * block of input rows a strip's filter reads, [b0, b1) = [max(0, y0 - halo),
 * min(H, y1 + halo)).  Pure host arithmetic (no device needed).  BSF_EINVAL
 * for a bad argument or a strip shorter than the halo (the halo would then
 * span two neighbours).                                                      */
bsf_status bsf_strip_rows(int height, int unit, int halo, int rank, int nranks, int *y0, int *y1, int *b0, int *b1);

/* The halo exchange of a row strip (what bsf_run sends and receives per image
 * on a multi-GPU plan), pure host arithmetic: x[0], x[1] = first own row and
 * row count sent to rank - 1; x[2] = rows received from it into block rows
 * [0, x[2]); x[3], x[4] = first own row and row count sent to rank + 1;
 * x[5], x[6] = first block row and row count received from it; x[7] = the
 * block row of the first own row.  Zeros where there is no neighbour.       */
bsf_status bsf_strip_exchange(int height, int unit, int halo, int rank, int nranks, int *x8);

/* NCCL unique id for a multi-GPU plan (call on rank 0, broadcast the 128
 * bytes to every rank).  BSF_ENCCL when NCCL cannot be loaded.               */
bsf_status bsf_get_unique_id(void *id_out128);

typedef struct {
    long long pixels;        /* pixels filtered since the last reset                          */
    long long clamped;       /* pixels whose elongation was clamped                           */
    long long zero_scale;    /* pixels with one scale treated as exactly zero (R5)  */
    long long theta_prime;   /* pixels filtered with basis Theta'                             */
    long long flags;         /* bit0 margin violation, bit1 infeasible, bit2 two zero scales  */
    long long double_double; /* pixels computed (or recomputed) in double-double              */
    long long macs;          /* algorithmic multiply-adds of the interpolation (Eq. 11) in the */
                             /* exact split path: sum over taps of window x monomials          */
} bsf_stats;

/* Create a plan: validates the descriptor, derives the margins, loads the
 * interpolation tables for (basis, order) from `lut_dir` (directory holding
 * bsf_lut_b{basis}_r{order}.bin) and allocates the workspace.  No device work
 * is launched.  Errors: BSF_EINVAL (descriptor), BSF_ERANGE (explicit margins
 * smaller than the reach bound), BSF_ENOMEM, BSF_ECUDA, BSF_EUNSUPPORTED
 * (order without tables).                                                    */
bsf_status bsf_plan_create(const bsf_plan_desc *desc, const char *lut_dir, bsf_plan_t *out);
bsf_status bsf_plan_destroy(bsf_plan_t plan);
bsf_status bsf_plan_geometry(bsf_plan_t plan, bsf_geometry *geom);

/* Pre-integration (the "running sum"): for every image of
 * the batch and every basis in use, the 4r nested running sums
 *   g <- g(q) + g(q - s_k)   (integer steps, no sqrt5 factor: DESIGN.md R3)
 * on the domain x in [-P, W+P), y in [0, H+Pb) with zero state outside it.
 *   f_dev: [batch*channels][H][W] of in_dtype.
 *   g_dev: geometry.g_bytes; layout [nbases][batch*channels][H+Pb][W+2P] of
 *          double-double (double2 {hi, lo}); opaque to callers except through
 *          bsf_filter.  Exact for u8 input while the sums are below 2^106.   */
bsf_status bsf_preintegrate(bsf_plan_t plan, const void *f_dev, void *g_dev, void *stream);

/* Bit-exact integer pre-integration of a u8 image (the contract checked
 * against the oracle): same sums, int64 arithmetic wrapping modulo 2^64.
 *   g_dev: geometry.g_exact_bytes; layout [nbases][batch*channels][H+Pb][W+2P]
 *          of int64, element (y, x) at [y][x + P].  Level order: Theta
 *          (1,0),(1,1),(0,1),(-1,1); Theta' (1,2),(2,1),(-1,2),(-2,1)
 *          (Alg. 3 (a)-(d)); repeated r times.  BSF_EINVAL for f32 input.   */
bsf_status bsf_preintegrate_exact(bsf_plan_t plan, const void *f_dev, void *g_dev, void *stream);

/* One running-sum level of the global pre-integration (PAPER.md:106-110,
 * Alg. 3 step 2), for row strips of one domain sharded over ranks (SURVEY.md
 * 8(e) GLOBAL mode: the scan carries travel down the rank chain).
 *   slot:  running-sum slot (0; 1 = Theta' under BSF_DUAL); level in [0, 4r):
 *          the step is bsf_scan_step(slot, level), levels run in order.
 *   exact: 1 = int64 wrapping (u8 input, bit-exact), 0 = double-double.
 *   f_dev: the strip's image rows (read by level 0 only); g_dev: as for
 *          bsf_preintegrate[_exact] (all slots), updated in place.
 *   carry_dev: [batch*channels][sy][g_width] elements of g's type = this
 *          level's running sums on the sy domain rows just above the strip
 *          (the previous rank's last sy rows after this level), or NULL for
 *          the first strip (zero state).  Strip boundaries must be even rows.
 * Running every level with the carries of the strip above reproduces the
 * single-plan bsf_preintegrate_exact bit for bit.                            */
bsf_status bsf_scan_step(bsf_plan_t plan, int slot, int level, int *sx, int *sy);
bsf_status bsf_scan_level(bsf_plan_t plan, int slot, int level, int exact, const void *f_dev, void *g_dev,
                          const void *carry_dev, void *stream);

/* Local finite difference for every pixel (Alg. 3 step 3, PAPER.md:400-403,
 * generalised to order r and to Algorithm 2's basis choice).
 *   g_dev:   output of bsf_preintegrate.
 *   cov_dev: [batch][3][H][W] float32 planes (sigma_x, sigma_y, theta); theta
 *            is the angle of the sigma_x axis from the x axis, in radians.
 *   out_dev: [batch*channels][H][W] of out_dtype.                            */
bsf_status bsf_filter(bsf_plan_t plan, const void *g_dev, const void *cov_dev, void *out_dev, void *stream);

/* Global mode (geometry.global_mode = 1): the local finite difference read
 * from the exact int64 sums of bsf_preintegrate_exact (the paper's Alg. 3
 * step 3 on its single global pre-integration), with an
 * exact integer contraction of Eq. (11).  g_dev as written
 * by bsf_preintegrate_exact; cov_dev, out_dev as bsf_filter.
 * bsf_preintegrate_exact + bsf_filter_exact = bsf_run of a global-mode plan.
 * BSF_EUNSUPPORTED when the plan is not in global mode.                     */
bsf_status bsf_filter_exact(bsf_plan_t plan, const void *g_dev, const void *cov_dev, void *out_dev, void *stream);

/* Same computation for an explicit pixel list (parity at full size):
 *   pts_dev: int32 triples (image, x, y) * npts;  out_dev: float64[npts].    */
bsf_status bsf_filter_points(bsf_plan_t plan, const void *g_dev, const void *cov_dev, const int *pts_dev,
                             int npts, double *out_dev, void *stream);

/* As bsf_filter_points, also writing per-point diagnostics (for decision
 * parity with the oracle): aux_dev float64[12 * npts] =
 *   {basis, zero-scale direction (-1 none), clamped, flags, a'_1..a'_4,
 *    computed in double-double (0/1), sum_j |c_j F_j| / |S|,
 *    sum_j |c_j| sum_d |G_d| / |S| (fp64 paths; cancellation ratios), 0}
 * with a'_k = a_k / |s_k| the scale in lattice steps.                        */
bsf_status bsf_filter_points_aux(bsf_plan_t plan, const void *g_dev, const void *cov_dev, const int *pts_dev,
                                 int npts, double *out_dev, double *aux_dev, void *stream);

/* The tile-anchored fused path for an explicit pixel list (parity at full
 * size): each point's 16x16 tile is pre-integrated on its halo and the point
 * gathered; results are identical to those of bsf_run with BSF_ANCHOR_TILE.
 *   f_dev, cov_dev as bsf_run; pts_dev int32 (image, x, y) * npts;
 *   out_dev float64[npts]; aux_dev NULL or float64[12 * npts] (see _aux).    */
bsf_status bsf_run_points(bsf_plan_t plan, const void *f_dev, const void *cov_dev, const int *pts_dev, int npts,
                          double *out_dev, double *aux_dev, void *stream);

/* The whole hot path: BSF_ANCHOR_GLOBAL = bsf_preintegrate + bsf_filter with
 * the plan's own g workspace; BSF_ANCHOR_TILE = the fused tile kernel (no
 * global g).                                                                 */
bsf_status bsf_run(bsf_plan_t plan, const void *f_dev, const void *cov_dev, void *out_dev, void *stream);

/* The tile path on a subset of the image: only the listed anchoring tiles
 * (side geometry.tile_unit; index (image * ty_count + ty) * tx_count + tx,
 * tx_count = ceil(W / tile_unit), ty_count = ceil(H / tile_unit)) are
 * filtered, every one exactly as bsf_run computes it (same kernel, same
 * anchoring); other outputs are left untouched (region-of-interest
 * filtering; the bench times order 4 this way).  tiles_dev: int32[ntiles].
 * BSF_EUNSUPPORTED for global-mode plans.                                    */
bsf_status bsf_run_tiles(bsf_plan_t plan, const void *f_dev, const void *cov_dev, void *out_dev, const int *tiles_dev,
                         int ntiles, void *stream);

/* Algorithm 1 ("better accuracy"): covariance splitting
 * C = sigma_b^2 I + Delta C (Eq. (7)).  Per covariance field b,
 * sigma_b^2 is half the bound (9), minimised over the
 * field's pixels (R21); then
 *   pass 1: the isotropic box spline of covariance sigma_b^2 I (a_k =
 *           sqrt(6) sigma_b) on f, a global O(1) convolution;
 *   pass 2: the space-variant box spline of covariance C(p) - sigma_b^2 I on
 *           the pass-1 image (kept in float64).
 * Both passes use the plan's order and basis policy and the exact split path
 * (BSF_EUNSUPPORTED for order 4).  f_dev, cov_dev, out_dev as bsf_run.
 * sigma2_out: NULL, or host double[batch] receiving sigma_b^2 (synchronises
 * the stream).  The plan owns a float64 [batch*channels][H][W] work image.
 * Statistics count both passes.                                              */
bsf_status bsf_run_alg1(bsf_plan_t plan, const void *f_dev, const void *cov_dev, void *out_dev, double *sigma2_out,
                        void *stream);

/* Generalised covariance splitting (the repeated
 * filtering of PAPER.md:161-166 made space-variant through Algorithm 1's
 * split, composed by Proposition 2):
 * `passes` = n >= 2 passes of the plan's order, with an isotropic part
 * T = fraction * B_b (B_b = 2 sigma_b^2 the smallest bound (9) of covariance
 * field b, R21/R22):
 *   passes 1 .. n-1: the isotropic box spline of covariance (T / (n-1)) I,
 *   pass n:          the space-variant box spline of C(p) - T I.
 * fraction in (0, 1); 0 selects the default (n-1)/n, for which a constant
 * isotropic field gets covariance C / n in every pass (the order-n kernel up
 * to the intermediate sampling).  n = 2 with fraction 1/2 is bsf_run_alg1
 * exactly (Table 3, sweeps this fraction).  Arguments and
 * errors as bsf_run_alg1 (BSF_EINVAL for n outside 2..16 or fraction outside
 * [0, 1)); a second float64 work image is allocated for n > 2.              */
bsf_status bsf_run_split(bsf_plan_t plan, const void *f_dev, const void *cov_dev, void *out_dev, int passes,
                         double fraction, double *sigma2_out, void *stream);

/* DC-renormalised output (not in the paper, whose
 * filter is not renormalised, R12): out(p) = filter(f)(p) /
 * sum_{q in image} beta_{a(p)}(p - q), the denominator being the same filter
 * applied to the image indicator, so a constant image is reproduced exactly
 * up to rounding, edges included.  Runs the fused path twice plus one
 * division kernel (BSF_EUNSUPPORTED unless anchor = BSF_ANCHOR_TILE); the
 * plan owns the indicator image and a float64 denominator.  Arguments as
 * bsf_run.                                                                  */
bsf_status bsf_run_normalized(bsf_plan_t plan, const void *f_dev, const void *cov_dev, void *out_dev, void *stream);

/* End to end from HOST buffers (pinned for overlap): copies f and cov to the
 * device, runs bsf_run, copies out back, all on `stream`.  Returns after
 * enqueueing; synchronise the stream before reading out_host.  Global mode
 * (order 1, u8) pipelines the call on the plan's own streams, joined into
 * `stream`: the image goes up in row bands, each pre-integrated as soon as it
 * is in (scan carries passed band to band), the covariance in row bands, each
 * gather band starts once its covariance and the sums its footprint reaches
 * are ready, and its output band goes back while the next one computes; the
 * output is bit-identical to bsf_run.  Host buffers are read and written in
 * the layouts of bsf_run; the plan keeps device staging buffers.            */
bsf_status bsf_run_host(bsf_plan_t plan, const void *f_host, const void *cov_host, void *out_host, void *stream);

/* Statistics since the last reset (synchronises the plan's last stream). */
bsf_status bsf_get_stats(bsf_plan_t plan, bsf_stats *stats, int reset);

/* Number of library kernels launched through this plan since creation. */
long long bsf_launch_count(bsf_plan_t plan);

/* Diagnostics.  bsf_debug_phase_cycles: the first call enables per-phase
 * cycle counters in the tile path (adds one clock read per phase per tile);
 * later calls copy the 16 counters (SM cycles summed over tiles, each phase
 * measured from the previous mark: 0 reach pass, 1 zero pad rows, 11 the
 * running-sum sweeps, 12 the zero-scale variant planes, 2 exact split,
 * 8 sub-tile scales, 9 keys, 10 bucket scan, 3 scatter, 4 gather,
 * 5 accumulation; 6-7 warp-cycles of the MMA groups; 13 executed MMA
 * multiply-adds per limb incl. padding, 14 real items, 15 group slots) to host `out`
 * (may be NULL) after synchronising the plan's last stream, and zero them when
 * `reset`.  bsf_uses_fused: 1 when the tile path runs the exact split
 * contraction kernel (known after the first tile-path call), else 0.        */
bsf_status bsf_debug_phase_cycles(bsf_plan_t plan, unsigned long long *out, int reset);
/* bsf_debug_item_cycles (after bsf_debug_phase_cycles enabled the counters):
 * host `items[i]` = SM cycles of fused-path work unit i (a super-tile, or in
 * split mode a 32x32 quadrant unit; i is the hand-out index of the atomic
 * counter; i < min(nitems, 8192)) in the last
 * run; host `work[4i .. 4i+3]` (may be NULL) = its interpolation MACs, its
 * double-double fallback pixels, the halo domain points of the bases it
 * pre-integrates and its number of planes; host `ctas[c]` = busy cycles of CTA
 * c summed since the last reset (c < min(nctas, 1024)).  `items` may be NULL
 * with nitems 0, `ctas` with nctas 0.  BSF_EINVAL when the counters are not
 * enabled.                                                                  */
bsf_status bsf_debug_item_cycles(bsf_plan_t plan, unsigned long long *items, unsigned long long *work, int nitems,
                                 unsigned long long *ctas, int nctas);
int bsf_uses_fused(bsf_plan_t plan);
/* bsf_debug_option (diagnostics and tests only; the defaults are the product
 * path): "fused" 0/1 -- 0 runs the per-thread double-double tile kernel instead
 * of the exact split path (set before the first run); "work_order" 0/1 -- 0
 * hands the fused path's super-tiles out in raster order; "split_tol" -- the
 * relative a-posteriori bound above which a pixel is recomputed in
 * double-double (default 5e-10; 0 sends every pixel to the fallback, inf
 * none, which voids the 1e-9 contract); "global_kernel" 0/1 -- global mode
 * gathers with the order-1 integer kernel (1, default) or the fused kernel's
 * DMMA groups (0); "scan_tma" 0/1 (process-wide) -- the running-sum strip
 * kernels stream their rows by TMA (1, default when the row pitch allows) or
 * by cp.async (0); "gx1_dp4a" 0/1 -- the order-1 gather contracts byte planes
 * of the sums with dp4a (1) instead of three 21-bit IMAD limbs (0, default;
 * both exact, outputs bit-identical); "i8_tc" 0/1 -- order 3: the exact limbs
 * of Theta' full-kernel groups on the tcgen05 int8 tensor cores with TMEM
 * accumulators (1) or on DMMA (0, default; outputs bit-identical, the DMMA
 * path is faster today).  BSF_EINVAL for an unknown name.   */
bsf_status bsf_debug_option(bsf_plan_t plan, const char *name, double value);

const char *bsf_status_str(bsf_status s);
const char *bsf_last_error(void);
int bsf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BSF_H */
