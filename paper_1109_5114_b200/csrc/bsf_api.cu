// C-ABI of the library (include/bsf.h): plans, table loading, dispatch.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <algorithm>
#include <string.h>

#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>  // types only: the library is loaded at run time (dlopen), no link dependency

#include <mutex>

#include "bsf_internal.h"

using namespace bsf;

// ---------------------------------------------------------------------------
// NCCL, loaded on first use: the process' libnccl.so.2 (the one PyTorch
// already loaded when present, else the system's).  Used for the row-strip
// halo exchange and the GLOBAL-mode scan carries of multi-GPU plans.
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
    bool ok = false;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclGetErrorString) errStr = nullptr;
};
NcclApi &nccl_api() {
    static NcclApi n;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.getUniqueId = (decltype(n.getUniqueId))dlsym(h, "ncclGetUniqueId");
        n.commInitRank = (decltype(n.commInitRank))dlsym(h, "ncclCommInitRank");
        n.commDestroy = (decltype(n.commDestroy))dlsym(h, "ncclCommDestroy");
        n.send = (decltype(n.send))dlsym(h, "ncclSend");
        n.recv = (decltype(n.recv))dlsym(h, "ncclRecv");
        n.groupStart = (decltype(n.groupStart))dlsym(h, "ncclGroupStart");
        n.groupEnd = (decltype(n.groupEnd))dlsym(h, "ncclGroupEnd");
        n.errStr = (decltype(n.errStr))dlsym(h, "ncclGetErrorString");
        n.ok = n.getUniqueId && n.commInitRank && n.commDestroy && n.send && n.recv && n.groupStart && n.groupEnd &&
               n.errStr;
    });
    return n;
}
}  // namespace

static thread_local std::string g_last_error;

static bsf_status set_err(bsf_status s, const std::string &msg) {
    g_last_error = msg;
    return s;
}

#define NCCL_TRY(expr)                                                                        \
    do {                                                                                      \
        ncclResult_t r_ = (expr);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return set_err(BSF_ENCCL, std::string(#expr ": ") + nccl_api().errStr(r_));      \
    } while (0)

#define CUDA_TRY(expr)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return set_err(BSF_ECUDA, std::string(#expr ": ") + cudaGetErrorString(e_));      \
    } while (0)

#ifndef BSF_HOST_BANDS_T
#define BSF_HOST_BANDS_T 16
#endif
constexpr int BSF_HOST_BANDS = BSF_HOST_BANDS_T;  // bsf_run_host (global mode): row bands of the copy / compute pipeline
#ifndef BSF_SCAN_BANDS_T
#define BSF_SCAN_BANDS_T 4
#endif
constexpr int BSF_SCAN_BANDS = BSF_SCAN_BANDS_T;  // bsf_run_host (global mode): image row bands of the banded scans

struct bsf_plan_s {
    bsf_plan_desc d;
    Geometry geo;
    int bases[2];           // basis of each running-sum slot
    std::vector<void *> dev_allocs;
    LutBasis *luts_dev = nullptr;  // [2], indexed by basis id
    double2 *g_ws = nullptr;       // for bsf_run
    void *f_stage = nullptr, *cov_stage = nullptr, *out_stage = nullptr;
    unsigned long long *stats = nullptr;
    LutBasis host_luts[2];
    double2 *tile_scratch = nullptr;
    size_t tile_cap = 0;
    int tile_nslots = 0;
    int stile = 32;                // fused path: super-tile side
    bool fused = false;
    unsigned long long *prof = nullptr;  // phase cycles of the fused kernel (diagnostics)
    double2 *fbuf = nullptr;             // fused path: per-CTA tap values
    double *sbuf = nullptr;              // fused path: per-CTA per-pixel scales
    double *scratch0 = nullptr;          // fused path, order >= 3: rounded limb planes
    double *alg1_work = nullptr;         // Algorithm 1: float64 intermediate image
    double *alg1_work2 = nullptr;        // generalised splitting: second intermediate (ping-pong)
    void *ones = nullptr;                // DC renormalisation: image indicator (input type)
    double *norm_den = nullptr;          // DC renormalisation: filtered indicator
    double *alg1_sigma2 = nullptr;       // Algorithm 1: sigma_b^2 per covariance field (+ reduction bits)
    int *tile_counter = nullptr;
    int *sched_order = nullptr;          // fused path: work order of the super-tiles (largest first)
    unsigned char *sched_bin = nullptr;
    unsigned *sched_hist = nullptr;
    long long sched_cap = 0;
    long long nlaunch = 0;
    cudaStream_t last = nullptr;
    bool fused_ready = false;            // fused-path buffers (fbuf, sbuf, counter, order) allocated
    cudaStream_t s_in = nullptr, s_out = nullptr;  // bsf_run_host pipeline (global mode): copy streams
    cudaStream_t s_c2 = nullptr;                   // second compute stream (odd bands fill the even bands' tails)
    cudaEvent_t ev[2 * BSF_HOST_BANDS + 5] = {};
    cudaEvent_t ev_fb[BSF_SCAN_BANDS] = {};          // bsf_run_host: image band k is on the device
    cudaEvent_t ev_sb[2][BSF_SCAN_BANDS] = {};       // bsf_run_host: image band k of basis slot sl pre-integrated
    cudaStream_t s_scan[2] = {nullptr, nullptr};     // bsf_run_host: banded scans, one stream per basis slot
    unsigned long long *hcarry = nullptr;            // bsf_run_host banded scans: [2 parity][2 slots][levels][nimg][2][GW]
    // the two bases' running sums are independent: basis 1 runs on a side
    // stream forked from (and joined back into) the caller's stream
    cudaStream_t s_side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool scratch_ready = false;          // tile-anchored halo scratch allocated
    // global mode (order 1, u8 input): the exact int64 running
    // sums of the whole image, read by the fused kernel's taps
    bool global_ok = false;              // every sum of every basis stays below 2^62
    int gshift[2] = {0, 0};              // limb split G = 2^k G1 + G0 per basis
    int gvw[2] = {0, 0};                 // order-1 gather: two-limb width for the variants (TileArgs.gvw)
    int stile_global = 32;
    long long *gx_ws = nullptr;          // [nbases][nimg][GH][GW] int64
    // row strips (nranks > 1): own rows [y0, y1), block [b0, b1), halo; GLOBAL-mode
    // strip: image rows [gy0, gy1), domain rows [gy0, gy0 + g_rows)
    int y0 = 0, y1 = 0, b0 = 0, b1 = 0, halo = 0, gy0 = 0, gy1 = 0, g_rows = 0;
    ncclComm_t comm = nullptr;
    void *f_blk = nullptr;                // block image (library halo exchange)
    unsigned long long *carry = nullptr;  // scan carries [nimg][2][GW]
    // diagnostics options (bsf_debug_option); the defaults are the product path
    bool opt_fused = true;
    bool opt_order = true;
    int opt_global_kernel = 1;  // global mode: 1 the order-1 integer gather (bsf_gx1.cuh), 0 the fused kernel
    int opt_gx1_dp4a = 0;       // order-1 gather: 1 byte-plane dp4a contraction, 0 three 21-bit IMAD limbs
    int opt_i8_tc = 0;          // order 3: 1 the exact limbs on tcgen05 kind::i8 (bsf_fused.cuh i8_tile), 0 DMMA
    double opt_split_tol = BSF_SPLIT_TOL_DEFAULT;
};

// Select the plan's device for the duration of a call and restore the
// caller's current device afterwards (plans may live on any device).
struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

static bool global_exact(const bsf_plan_s *p);
static bool use_fused(const bsf_plan_s *p);
static size_t g_bytes(const bsf_plan_s *p) {
    return (size_t)p->geo.nbases * p->geo.nimg * p->geo.GH * p->geo.GW * sizeof(double2);
}

static int required_disp(float max_sigma, int order) {
    // |tap - p| <= (r/2) sum_k a_k <= sigma_max sqrt(24 r)
    return (int)ceil((double)max_sigma * sqrt(24.0 * order)) + 1;
}

// ---------------------------------------------------------------------------
// interpolation tables
// ---------------------------------------------------------------------------
static bsf_status load_lut(bsf_plan_s *p, const char *dir, int basis, LutBasis *out) {
    char path[4096];
    snprintf(path, sizeof path, "%s/bsf_lut_b%d_r%d.bin", dir ? dir : ".", basis, p->d.order);
    FILE *fh = fopen(path, "rb");
    if (!fh) return set_err(BSF_EUNSUPPORTED, std::string("missing interpolation table ") + path);
    std::vector<char> buf;
    fseek(fh, 0, SEEK_END);
    long n = ftell(fh);
    fseek(fh, 0, SEEK_SET);
    buf.resize(n);
    size_t got = fread(buf.data(), 1, n, fh);
    fclose(fh);
    if ((long)got != n) return set_err(BSF_EINVAL, "short read " + std::string(path));
    size_t off = 0;
    auto take = [&](void *dst, size_t sz) -> bool {
        if (off + sz > buf.size()) return false;
        memcpy(dst, buf.data() + off, sz);
        off += sz;
        return true;
    };
    uint32_t hdr[5], nreg;
    if (!take(hdr, sizeof hdr) || hdr[0] != 0x4C465342u || hdr[1] != 2u || (int)hdr[2] != basis ||
        (int)hdr[3] != p->d.order ||
        hdr[4] != NVAR || !take(&nreg, 4) || nreg > MAX_REG)
        return set_err(BSF_EINVAL, "bad table header " + std::string(path));
    memset(out, 0, sizeof *out);
    out->nreg = nreg;
    out->wxmin = out->wymin = 1 << 30;
    out->wxmax = out->wymax = -(1 << 30);
    for (int k = 0; k < 4; ++k) {
        int nv[2];
        take(nv, 8);
        out->normal[k] = make_int2(nv[0], nv[1]);
    }
    std::vector<int> keys(4 * nreg);
    for (uint32_t r = 0; r < nreg; ++r) {
        take(&keys[4 * r], 16);
        double c[2];
        take(c, 16);
        out->centre[r] = make_double2(c[0], c[1]);
        if (c[0] != 0.0 || c[1] != 0.0)  // the gather evaluates at phi itself (R17)
            return set_err(BSF_EINVAL, "table expanded around a non-zero centre (regenerate): " + std::string(path));
    }
    int kmax[4];
    for (int k = 0; k < 4; ++k) {
        out->kmin[k] = 1 << 30;
        kmax[k] = -(1 << 30);
        for (uint32_t r = 0; r < nreg; ++r) {
            out->kmin[k] = keys[4 * r + k] < out->kmin[k] ? keys[4 * r + k] : out->kmin[k];
            kmax[k] = keys[4 * r + k] > kmax[k] ? keys[4 * r + k] : kmax[k];
        }
        out->radix[k] = kmax[k] - out->kmin[k] + 1;
    }
    if (out->radix[0] * out->radix[1] * out->radix[2] * out->radix[3] > 81)
        return set_err(BSF_EINVAL, "region key space too large");
    memset(out->table, -1, sizeof out->table);
    for (uint32_t r = 0; r < nreg; ++r) {
        int idx = 0, mul = 1;
        for (int k = 0; k < 4; ++k) {
            idx += (keys[4 * r + k] - out->kmin[k]) * mul;
            mul *= out->radix[k];
        }
        out->table[idx] = (signed char)r;
    }
    for (int v = 0; v < NVAR; ++v) {
        int hv[4];
        if (!take(hv, 16)) return set_err(BSF_EINVAL, "truncated table");
        LutVar &V = out->var[v];
        V.deg = hv[1];
        V.nmon = hv[2];
        V.nmax = hv[3];
        uint64_t Lden;
        if (!take(&Lden, 8) || Lden >= (1ull << 53)) return set_err(BSF_EINVAL, "bad denominator");
        const bool exact = Lden != 0;  // 0: double-double pairs, no integer form (no fused path)
        const double L = exact ? (double)Lden : 1.0;
        std::vector<int> counts(nreg);
        std::vector<int2> offs((size_t)nreg * V.nmax, make_int2(0, 0));
        std::vector<double> num((size_t)nreg * V.nmax * V.nmon, 0.0);
        std::vector<double2> coef(num.size());
        double csum = 0.0;
        for (uint32_t r = 0; r < nreg; ++r) {
            take(&counts[r], 4);
            csum += counts[r];
            for (int s = 0; s < V.nmax; ++s) {
                int o[2];
                take(o, 8);
                offs[(size_t)r * V.nmax + s] = make_int2(o[0], o[1]);
                const size_t at = ((size_t)r * V.nmax + s) * V.nmon;
                if (!(exact ? take(&num[at], 8 * (size_t)V.nmon) : take(&coef[at], 16 * (size_t)V.nmon)))
                    return set_err(BSF_EINVAL, "truncated table");
            }
        }
        // double-double coefficients n / L, correctly rounded: hi = fl(n/L);
        // n - hi*L is exact in one fma (it is a multiple of ulp(hi) below L*ulp(hi)),
        // lo = fl((n - hi*L)/L).
        if (exact)
            for (size_t i = 0; i < num.size(); ++i) {
                double hi = num[i] / L;
                double rem = fma(-hi, L, num[i]);
                coef[i] = make_double2(hi, rem / L);
            }
        // integer table for the exact split contraction (bsf_fused.cuh, FP64
        // tensor-core fragments): per region nslot4 = nmax rounded up to 4 window
        // slots, per slot nmonp = nmon rounded up to 8 monomials (zero padded),
        // monomials in the gen_lut order; offsets padded alike with (0, 0).
        if (bsf_nt(V.deg) < 0) return set_err(BSF_EUNSUPPORTED, "no MMA column layout for this table degree");
        V.nmonp = 8 * bsf_nt(V.deg);
        V.nslot4 = (V.nmax + 3) & ~3;
        std::vector<int> col(V.nmon);
        {
            int m = 0;
            for (int i = V.deg; i >= 0; --i)  // gen_lut order: x-major, i and j descending
                for (int j = V.deg - i; j >= 0; --j) col[m++] = bsf_mono_col(V.deg, i, j);
        }
        std::vector<double> nump((size_t)nreg * V.nslot4 * V.nmonp, 0.0);
        std::vector<int2> offs4((size_t)nreg * V.nslot4, make_int2(0, 0));
        for (uint32_t r = 0; r < nreg; ++r)
            for (int sl = 0; sl < V.nmax; ++sl) {
                offs4[(size_t)r * V.nslot4 + sl] = offs[(size_t)r * V.nmax + sl];
                for (int m = 0; m < V.nmon; ++m)
                    nump[((size_t)r * V.nslot4 + sl) * V.nmonp + col[m]] = num[((size_t)r * V.nmax + sl) * V.nmon + m];
            }
        double colmax = 0.0;  // max over (region, monomial) of sum_s |n|
        for (uint32_t r = 0; r < nreg; ++r)
            for (int m = 0; m < V.nmon; ++m) {
                double cs = 0.0;
                for (int s = 0; s < V.nmax; ++s) cs += fabs(num[((size_t)r * V.nmax + s) * V.nmon + m]);
                colmax = cs > colmax ? cs : colmax;
            }
        // a-posteriori bound of the G0 limb (bsf_fused.cuh): |F^ - F| <= gamma_{n+1} 0.5 sum_s,mu |n_s,mu|
        {
            double worst = 0.0;
            for (uint32_t r = 0; r < nreg; ++r) {
                double t = 0.0;
                for (int sl = 0; sl < V.nmax; ++sl)
                    for (int m = 0; m < V.nmon; ++m) t += fabs(num[((size_t)r * V.nmax + sl) * V.nmon + m]);
                worst = t > worst ? t : worst;
            }
            const double u = 1.1102230246251565e-16, nn = V.nslot4 + 1;
            V.bnd = (nn * u / (1.0 - nn * u)) * 0.5 * worst;
        }
        // sums of G1 * n stay exact while |G1| sum|n| <= 2^53
        int cm = 0;
        while (ldexp(1.0, cm) < colmax) ++cm;
        V.kbits = exact ? 53 - cm : 0;  // no integer form: the fused path is unavailable
        V.L = L;
        V.mean_count = nreg ? (float)(csum / nreg) : 0.f;
        V.nsplit = 1;
        V.shift = 0;
        V.num2 = V.numf = nullptr;
        std::vector<double> num1s, num0s;
        if (exact && V.kbits < KBITS_MIN) {
            // split the numerators n = n1 2^sh + n0 (|n0| <= 2^(sh-1)) so that both
            // column sums, and with them the exact limb, stay wide
            const int sh = (int)ceil(0.5 * log2(2.0 * colmax / V.nslot4));
            num1s.assign(nump.size(), 0.0);
            num0s.assign(nump.size(), 0.0);
            double c1 = 0.0, c0 = 0.0;
            const double scale = ldexp(1.0, sh);
            for (size_t i = 0; i < nump.size(); ++i) {
                const double n1 = rint(nump[i] / scale);
                num1s[i] = n1;
                num0s[i] = nump[i] - n1 * scale;  // exact: |n| < 2^53
            }
            for (uint32_t r = 0; r < nreg; ++r)
                for (int m = 0; m < V.nmonp; ++m) {
                    double s1 = 0.0, s0 = 0.0;
                    for (int sl = 0; sl < V.nslot4; ++sl) {
                        const size_t i = ((size_t)r * V.nslot4 + sl) * V.nmonp + m;
                        s1 += fabs(num1s[i]);
                        s0 += fabs(num0s[i]);
                    }
                    c1 = s1 > c1 ? s1 : c1;
                    c0 = s0 > c0 ? s0 : c0;
                }
            const double cmax = c1 > c0 ? c1 : c0;
            int cs = 0;
            while (ldexp(1.0, cs) < cmax) ++cs;
            V.kbits = 53 - cs;
            V.nsplit = 2;
            V.shift = sh;
        }
        void *d_counts, *d_offs, *d_coef, *d_num, *d_offs4;
        CUDA_TRY(cudaMalloc(&d_offs4, offs4.size() * sizeof(int2)));
        p->dev_allocs.push_back(d_offs4);
        CUDA_TRY(cudaMemcpy(d_offs4, offs4.data(), offs4.size() * sizeof(int2), cudaMemcpyHostToDevice));
        V.offs4 = (const int2 *)d_offs4;
        CUDA_TRY(cudaMalloc(&d_counts, counts.size() * sizeof(int)));
        p->dev_allocs.push_back(d_counts);
        CUDA_TRY(cudaMalloc(&d_offs, offs.size() * sizeof(int2)));
        p->dev_allocs.push_back(d_offs);
        CUDA_TRY(cudaMalloc(&d_coef, coef.size() * sizeof(double2)));
        p->dev_allocs.push_back(d_coef);
        CUDA_TRY(cudaMalloc(&d_num, nump.size() * sizeof(double)));
        p->dev_allocs.push_back(d_num);
        CUDA_TRY(cudaMemcpy(d_counts, counts.data(), counts.size() * sizeof(int), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(d_offs, offs.data(), offs.size() * sizeof(int2), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(d_coef, coef.data(), coef.size() * sizeof(double2), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(d_num, nump.data(), nump.size() * sizeof(double), cudaMemcpyHostToDevice));
        V.num = (const double *)d_num;
        if (V.nsplit == 2) {
            void *d1, *d0;
            CUDA_TRY(cudaMalloc(&d1, num1s.size() * sizeof(double)));
            p->dev_allocs.push_back(d1);
            CUDA_TRY(cudaMalloc(&d0, num0s.size() * sizeof(double)));
            p->dev_allocs.push_back(d0);
            CUDA_TRY(cudaMemcpy(d1, num1s.data(), num1s.size() * sizeof(double), cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(d0, num0s.data(), num0s.size() * sizeof(double), cudaMemcpyHostToDevice));
            V.numf = V.num;             // full numerators: the G0 limb
            V.num = (const double *)d1;  // n1 with G1 (exact)
            V.num2 = (const double *)d0; // n0 with G1 (exact)
        }
        // order 1: int8 numerators for the global-mode gather (bsf_gx1.cuh)
        V.n8 = nullptr;
        V.nabs = 0.0;
        if (exact) {
            for (uint32_t r = 0; r < nreg; ++r)
                for (int m = 0; m < V.nmon; ++m) {
                    double sa = 0.0;
                    for (int s2 = 0; s2 < V.nmax; ++s2) sa += fabs(num[((size_t)r * V.nmax + s2) * V.nmon + m]);
                    V.nabs = sa > V.nabs ? sa : V.nabs;
                }
        }
        if (exact && p->d.order == 1 && V.nmon <= 8) {
            std::vector<signed char> n8((size_t)nreg * V.nmax * 8, 0);
            bool fits = true;
            for (size_t i = 0; i < (size_t)nreg * V.nmax; ++i)
                for (int m = 0; m < V.nmon; ++m) {
                    const double v = num[i * V.nmon + m];
                    // int8, and the gather's int32 limb sums: 2^21 |n| nmax < 2^31
                    fits = fits && fabs(v) <= 127.0 && ldexp(fabs(v) * V.nmax, 21) < 0x1p31;
                    n8[i * 8 + m] = (signed char)v;
                }
            if (fits) {
                void *d8;
                CUDA_TRY(cudaMalloc(&d8, n8.size()));
                p->dev_allocs.push_back(d8);
                CUDA_TRY(cudaMemcpy(d8, n8.data(), n8.size(), cudaMemcpyHostToDevice));
                V.n8 = (const signed char *)d8;
            }
        }
        // order 3, tcgen05 kind::i8 route (plan option "i8_tc", bsf_fused.cuh
        // i8_tile): the integer numerators as byte slices in the UMMA canonical
        // K-major layout, [region][32-slot chunk][slice][128 rows = table
        // columns][32 slots] (row r, slot k at (r / 8) 256 + (k / 16) 128 +
        // (r % 8) 16 + k % 16), slices A_0.. unsigned and the top one signed
        V.i8tab = nullptr;
        V.i8na = 0;
        V.i8nchunk = 0;
        // (the tile's window values G1 2^k + G2 are below 2^(2k+1): int64, 8 byte
        // slices, for kbits <= 31; tables with wider limbs keep the DMMA path)
        if (exact && p->d.order == 3 && V.nmonp <= 128 && V.kbits <= 31) {
            double nmax_abs = 0.0;
            for (double v : nump) nmax_abs = std::max(nmax_abs, fabs(v));
            int na = 1;
            while (na < 7 && !(nmax_abs < ldexp(1.0, 8 * na - 1))) ++na;
            if (nmax_abs < ldexp(1.0, 8 * na - 1)) {
                const int nch = (V.nslot4 + 31) / 32;
                std::vector<uint8_t> t8((size_t)nreg * nch * na * 4096, 0);
                for (uint32_t r = 0; r < nreg; ++r)
                    for (int ch = 0; ch < nch; ++ch)
                        for (int k = 0; k < 32; ++k) {
                            const int sl = ch * 32 + k;
                            if (sl >= V.nslot4) continue;
                            for (int m = 0; m < V.nmonp; ++m) {
                                const long long v = (long long)nump[((size_t)r * V.nslot4 + sl) * V.nmonp + m];
                                const int off = (m >> 3) * 256 + (k >> 4) * 128 + (m & 7) * 16 + (k & 15);
                                for (int a = 0; a < na; ++a)
                                    t8[(((size_t)r * nch + ch) * na + a) * 4096 + off] =
                                        (uint8_t)((unsigned long long)v >> (8 * a));
                            }
                        }
                void *d8;
                CUDA_TRY(cudaMalloc(&d8, t8.size()));
                p->dev_allocs.push_back(d8);
                CUDA_TRY(cudaMemcpy(d8, t8.data(), t8.size(), cudaMemcpyHostToDevice));
                V.i8tab = (const uint8_t *)d8;
                V.i8na = na;
                V.i8nchunk = nch;
            }
        }
        // order >= 3: the B operand tables in fp32 when every value is exact there
        // (|n| <= 2^24 integers; all order-3 tables qualify)
        V.num32 = nullptr;
        if (exact && p->d.order >= 3) {
            std::vector<float> c32;
            bool ok = true;
            auto put = [&](double v) {
                const float f = (float)v;
                ok = ok && (double)f == v;
                c32.push_back(f);
            };
            if (V.nsplit == 1) {
                for (double v : nump) put(v);
            } else {
                for (size_t i = 0; i < num1s.size(); ++i) {
                    put(num1s[i]);
                    put(num0s[i]);
                }
            }
            if (ok) {
                void *d32;
                CUDA_TRY(cudaMalloc(&d32, c32.size() * sizeof(float)));
                p->dev_allocs.push_back(d32);
                CUDA_TRY(cudaMemcpy(d32, c32.data(), c32.size() * sizeof(float), cudaMemcpyHostToDevice));
                V.num32 = (const float *)d32;
            }
        }
        for (uint32_t r = 0; r < nreg; ++r)
            for (int s2 = 0; s2 < counts[r]; ++s2) {
                double sb = 0.0;
                for (int m = 0; m < V.nmon; ++m) sb += fabs(coef[((size_t)r * V.nmax + s2) * V.nmon + m].x);
                out->hornerB = sb > out->hornerB ? sb : out->hornerB;
                int2 o = offs[(size_t)r * V.nmax + s2];
                out->wxmin = o.x < out->wxmin ? o.x : out->wxmin;
                out->wxmax = o.x > out->wxmax ? o.x : out->wxmax;
                out->wymin = o.y < out->wymin ? o.y : out->wymin;
                out->wymax = o.y > out->wymax ? o.y : out->wymax;
            }
        V.counts = (const int *)d_counts;
        V.offs = (const int2 *)d_offs;
        V.coef = (const double2 *)d_coef;
    }
    return BSF_OK;
}

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
extern "C" bsf_status bsf_plan_create(const bsf_plan_desc *desc, const char *lut_dir, bsf_plan_t *out) {
    if (!desc || !out) return set_err(BSF_EINVAL, "null argument");
    *out = nullptr;
    const bsf_plan_desc &d = *desc;
    if (d.width < 1 || d.height < 1 || d.batch < 1 || d.channels < 1)
        return set_err(BSF_EINVAL, "image size, batch and channels must be >= 1");
    if (d.in_dtype != BSF_U8 && d.in_dtype != BSF_F32) return set_err(BSF_EINVAL, "in_dtype must be U8 or F32");
    if (d.out_dtype != BSF_F64 && d.out_dtype != BSF_F32) return set_err(BSF_EINVAL, "out_dtype must be F64 or F32");
    if (d.order < 1 || d.order > 4) return set_err(BSF_EINVAL, "order must be 1..4");
    if (d.basis < BSF_THETA || d.basis > BSF_DUAL) return set_err(BSF_EINVAL, "bad basis");
    if (!(d.max_sigma > 0) || !isfinite(d.max_sigma)) return set_err(BSF_EINVAL, "max_sigma must be > 0");
    if (d.precision != BSF_PREC_FP64 && d.precision != BSF_PREC_DD && d.precision != BSF_PREC_AUTO)
        return set_err(BSF_EINVAL, "bad precision");
    if (d.margin_x < 0 || d.margin_y < -1) return set_err(BSF_EINVAL, "negative margin");
    if (d.anchor != BSF_ANCHOR_GLOBAL && d.anchor != BSF_ANCHOR_TILE && d.anchor != BSF_ANCHOR_AUTO)
        return set_err(BSF_EINVAL, "bad anchor");
    if (d.boundary != BSF_BOUNDARY_ZERO && d.boundary != BSF_BOUNDARY_REPLICATE)
        return set_err(BSF_EINVAL, "bad boundary");
    if (d.super_tile != 0 && d.super_tile != 16 && d.super_tile != 32 && d.super_tile != 64)
        return set_err(BSF_EINVAL, "super_tile must be 0, 16, 32 or 64");
    if (d.cov_layout != BSF_COV_SIGMA_THETA && d.cov_layout != BSF_COV_C11_C12_C22)
        return set_err(BSF_EINVAL, "bad cov_layout");
    if (d.nranks < 1 || d.rank < 0 || d.rank >= d.nranks) return set_err(BSF_EINVAL, "bad rank / nranks");
    int disp = required_disp(d.max_sigma, d.order);
    int needP = disp + 3 * d.order + 2, needPb = disp + 2;
    if ((d.margin_x && d.margin_x < needP) || (d.margin_y > 0 && d.margin_y < needPb))
        return set_err(BSF_ERANGE, "margins smaller than the kernel reach (need P >= " + std::to_string(needP) +
                                       ", Pb >= " + std::to_string(needPb) + ")");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (d.device < 0 || d.device >= ndev) return set_err(BSF_EINVAL, "device ordinal out of range");
    DevGuard guard(d.device);
    bsf_plan_s *p = new bsf_plan_s();
    p->d = d;
    Geometry &g = p->geo;
    g.W = d.width;
    g.H = d.height;
    g.P = d.margin_x ? d.margin_x : needP;
    g.Pb = d.margin_y > 0 ? d.margin_y : (d.margin_y == 0 ? needPb : 0);  // -1: row strip, no bottom margin
    g.GW = g.W + 2 * g.P;
    g.GH = g.H + g.Pb;
    g.nimg = d.batch * d.channels;
    // super-tile of the fused path: the halo domain per super-tile grows with
    // the reach E = max_sigma sqrt(24 r); 64 x 64 super-tiles amortise it over
    // 4x the pixels once E is large: order 1 (config 3: +33 %) and order 2
    // with u8 input (config 3: +20 %, 0.03 % of the pixels to the fallback).
    // Otherwise the larger domains push pixels to the double-double fallback
    // (config 2, f32, r = 2: 85k pixels, 16x slower; u8 r = 3: 3x slower);
    // the passes of bsf_run_split run 32 x 32 at order 2 for that reason.
    {
        const double E = (double)d.max_sigma * sqrt(24.0 * d.order);
        const bool big = d.order == 1 || (d.order == 2 && d.in_dtype == BSF_U8);
        p->stile = (big && E > BSF_STILE64_REACH) ? 64 : 32;
        // small images: 16 x 16 super-tiles when 32 x 32 ones would leave most
        // SMs idle (config 1: 16 super-tiles for 148 SMs)
        const long long n32 = (long long)((d.width + 31) / 32) * ((d.height + 31) / 32) * d.batch * d.channels;
        if (p->stile == 32 && n32 < 148) p->stile = 16;
        if (d.super_tile) p->stile = d.super_tile;
    }
    g.nbases = d.basis == BSF_DUAL ? 2 : 1;
    p->bases[0] = d.basis == BSF_DUAL ? BSF_THETA : d.basis;
    p->bases[1] = BSF_THETA_PRIME;
    {
        const long long n32 = (long long)((d.width + 31) / 32) * ((d.height + 31) / 32) * d.batch * d.channels;
        p->stile_global = n32 < 148 ? 16 : 32;
    }
    LutBasis host[2];
    memset(host, 0, sizeof host);
    for (int b = 0; b < 2; ++b) {
        bool used = d.basis == BSF_DUAL || d.basis == b;
        if (!used) continue;
        bsf_status s = load_lut(p, lut_dir, b, &host[b]);
        if (s != BSF_OK) {
            bsf_plan_destroy(p);
            return s;
        }
    }
    auto dmalloc = [&](void **ptr, size_t n) -> cudaError_t {
        cudaError_t e = cudaMalloc(ptr, n);
        if (e == cudaSuccess) p->dev_allocs.push_back(*ptr);
        return e;
    };
    memcpy(p->host_luts, host, sizeof host);
    if (dmalloc((void **)&p->luts_dev, sizeof host) != cudaSuccess ||
        cudaMemcpy(p->luts_dev, host, sizeof host, cudaMemcpyHostToDevice) != cudaSuccess) {
        bsf_plan_destroy(p);
        return set_err(BSF_ENOMEM, "table upload failed");
    }
    if (dmalloc((void **)&p->stats, 8 * sizeof(unsigned long long)) != cudaSuccess) {
        bsf_plan_destroy(p);
        return set_err(BSF_ENOMEM, "workspace allocation failed");
    }
    cudaMemset(p->stats, 0, 8 * sizeof(unsigned long long));
    // global mode eligibility (u8, order 1, zero extension, full-domain plan):
    // every running sum is an integer of at most 255 x the product of the line
    // lengths of its levels (a row holds GW points, a line of step (sx, sy)
    // at most GH/sy + 1), a zero-scale variant difference at most twice that;
    // it must stay below 2^62 (int64, no wrap), and the limb split
    // G = 2^k G1 + G0 keeps |G1|, G0 below 2^kbits of every table in use
    if (d.in_dtype == BSF_U8 && d.order == 1 && d.boundary == BSF_BOUNDARY_ZERO && d.margin_y != -1) {
        bool ok = true;
        for (int b = 0; b < 2; ++b) {
            if (!(d.basis == BSF_DUAL || d.basis == b)) continue;
            static const int sy_order[2][4] = {{0, 1, 1, 1}, {2, 1, 2, 1}};
            double bound = 255.0 * 2.0;
            for (int lv = 0; lv < 4; ++lv)
                bound *= sy_order[b][lv] == 0 ? (double)g.GW : (double)(g.GH / sy_order[b][lv] + 1);
            int bits = 0;
            while (ldexp(1.0, bits) <= bound) ++bits;
            int kb = 64;
            for (int v = 0; v < NVAR; ++v) kb = std::min(kb, host[b].var[v].kbits);
            const int k = std::max(1, bits - kb);
            if (bits > 62 || k > kb) ok = false;
            p->gshift[b] = k;
            // the order-1 gather's zero-scale variants: G(q) - G(q - s_k) is the
            // three-level sum without direction k, at most 255 x the product of
            // the other three line lengths; with sum_s |n| <= nabs the
            // contraction fits two w-bit limbs in int32 when nabs 2^w < 2^31 and
            // the sum stays below 2^2w, and E_mu (below 2^53) is exact in fp64
            double lmin = 1e300, nv = 0.0;
            for (int lv = 0; lv < 4; ++lv)
                lmin = std::min(lmin, sy_order[b][lv] == 0 ? (double)g.GW : (double)(g.GH / sy_order[b][lv] + 1));
            for (int v = 1; v < NVAR; ++v) nv = std::max(nv, host[b].var[v].nabs);
            const double bvar = bound / 2.0 / lmin;
            int w = 0;
            while (w < 30 && ldexp(nv, w + 1) < 0x1p31) ++w;
            p->gvw[b] = (nv > 0.0 && bvar < ldexp(1.0, 2 * w) && bvar * nv < 0x1p53) ? w : 0;
        }
        // the order-1 gather stages every table in use in shared memory
        int slots = 0;
        for (int b = 0; b < 2; ++b) {
            if (!(d.basis == BSF_DUAL || d.basis == b)) continue;
            if (host[b].nreg > GX1_MAXREG_H) ok = false;
            for (int v = 0; v < NVAR; ++v) {
                slots += host[b].nreg * ((host[b].var[v].nmax + 3) & ~3);
                if (!host[b].var[v].n8) ok = false;
            }
        }
        p->global_ok = ok && slots <= GX1_SLOTS_H;
    }
    // row strips: own rows aligned to the super-tile, a halo
    // covering a super-tile's halo domain (tap reach + interpolation window),
    // and the GLOBAL-mode strip aligned to 32 rows (even: Theta' steps sy = 2)
    if (d.nranks > 1) {
        p->global_ok = false;  // global mode needs the whole image's sums on one GPU
        const int disp = required_disp(d.max_sigma, d.order);
        p->halo = p->stile * ((disp + 6 * d.order + 4 + p->stile - 1) / p->stile);
        bsf_status s = bsf_strip_rows(d.height, p->stile, p->halo, d.rank, d.nranks, &p->y0, &p->y1, &p->b0, &p->b1);
        if (s != BSF_OK) {
            bsf_plan_destroy(p);
            return s;
        }
        int gb0, gb1;
        s = bsf_strip_rows(d.height, 32, 0, d.rank, d.nranks, &p->gy0, &p->gy1, &gb0, &gb1);
        if (s != BSF_OK) {
            bsf_plan_destroy(p);
            return s;
        }
        p->g_rows = (p->gy1 - p->gy0) + (d.rank == d.nranks - 1 ? g.Pb : 0);
        if (d.nccl_id) {
            NcclApi &nc = nccl_api();
            if (!nc.ok) {
                bsf_plan_destroy(p);
                return set_err(BSF_ENCCL, "libnccl.so.2 could not be loaded");
            }
            ncclUniqueId id;
            memcpy(&id, d.nccl_id, sizeof id);
            const ncclResult_t r = nc.commInitRank(&p->comm, d.nranks, id, d.rank);
            if (r != ncclSuccess) {
                p->comm = nullptr;
                bsf_plan_destroy(p);
                return set_err(BSF_ENCCL, std::string("ncclCommInitRank: ") + nc.errStr(r));
            }
        }
    } else {
        p->y0 = p->gy0 = 0;
        p->y1 = p->gy1 = p->b1 = d.height;
        p->g_rows = g.GH;
    }
    *out = p;
    return BSF_OK;
}

extern "C" bsf_status bsf_strip_rows(int H, int unit, int halo, int rank, int nranks, int *y0, int *y1, int *b0,
                                     int *b1) {
    if (!y0 || !y1 || !b0 || !b1) return set_err(BSF_EINVAL, "null argument");
    if (H < 1 || unit < 1 || halo < 0 || nranks < 1 || rank < 0 || rank >= nranks)
        return set_err(BSF_EINVAL, "bad strip arguments");
    const long long n = (H + unit - 1) / unit, base = n / nranks, extra = n % nranks;
    const long long t0 = rank * base + std::min<long long>(rank, extra);
    const long long t1 = t0 + base + (rank < extra ? 1 : 0);
    *y0 = (int)std::min<long long>(H, t0 * unit);
    *y1 = (int)std::min<long long>(H, t1 * unit);
    *b0 = std::max(0, *y0 - halo);
    *b1 = std::min(H, *y1 + halo);
    if (*y1 <= *y0) return set_err(BSF_EINVAL, "empty row strip (more ranks than row units)");
    // the neighbours' halos must come from this strip alone
    // (rank - 1's bottom halo is my first rows, rank + 1's top halo my last rows)
    if ((rank > 0 && *y1 - *y0 < std::min(halo, H - *y0)) || (rank < nranks - 1 && *y1 - *y0 < std::min(halo, *y1)))
        return set_err(BSF_EINVAL, "row strip shorter than the halo (" + std::to_string(*y1 - *y0) + " < " +
                                       std::to_string(halo) + " rows): use fewer ranks");
    return BSF_OK;
}

extern "C" bsf_status bsf_strip_exchange(int H, int unit, int halo, int rank, int nranks, int *x) {
    if (!x) return set_err(BSF_EINVAL, "null argument");
    int y0, y1, b0, b1;
    bsf_status s = bsf_strip_rows(H, unit, halo, rank, nranks, &y0, &y1, &b0, &b1);
    if (s != BSF_OK) return s;
    const int own = y1 - y0, top = y0 - b0, bot = b1 - y1;
    for (int i = 0; i < 8; ++i) x[i] = 0;
    if (rank > 0) {
        x[0] = 0;                                // rank - 1's bottom halo = my first rows
        x[1] = std::min(std::min(halo, H - y0), own);
        x[2] = top;                              // my block rows [0, top) = rank - 1's last rows
    }
    if (rank < nranks - 1) {
        const int dn = std::min(std::min(halo, y1), own);  // rank + 1's top halo = my last rows
        x[3] = own - dn;
        x[4] = dn;
        x[5] = top + own;                        // my block rows [top + own, top + own + bot)
        x[6] = bot;
    }
    x[7] = top;                                  // block row of my first own row
    return BSF_OK;
}

extern "C" bsf_status bsf_get_unique_id(void *id_out) {
    if (!id_out) return set_err(BSF_EINVAL, "null argument");
    NcclApi &nc = nccl_api();
    if (!nc.ok) return set_err(BSF_ENCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    NCCL_TRY(nc.getUniqueId(&id));
    memcpy(id_out, &id, sizeof id);
    return BSF_OK;
}

extern "C" bsf_status bsf_plan_destroy(bsf_plan_t p) {
    if (!p) return BSF_OK;
    DevGuard guard(p->d.device);
    if (p->comm) nccl_api().commDestroy(p->comm);
    if (p->s_in) {
        cudaStreamSynchronize(p->s_in);
        cudaStreamSynchronize(p->s_out);
        cudaStreamSynchronize(p->s_c2);
        cudaStreamDestroy(p->s_in);
        cudaStreamDestroy(p->s_out);
        cudaStreamDestroy(p->s_c2);
        for (cudaStream_t q : p->s_scan)
            if (q) {
                cudaStreamSynchronize(q);
                cudaStreamDestroy(q);
            }
        for (cudaEvent_t e : p->ev)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : p->ev_fb)
            if (e) cudaEventDestroy(e);
        for (auto &row : p->ev_sb)
            for (cudaEvent_t e : row)
                if (e) cudaEventDestroy(e);
    }
    if (p->s_side) {
        cudaStreamSynchronize(p->s_side);
        cudaStreamDestroy(p->s_side);
        cudaEventDestroy(p->ev_fork);
        cudaEventDestroy(p->ev_join);
    }
    for (void *q : p->dev_allocs) cudaFree(q);
    delete p;
    return BSF_OK;
}

extern "C" bsf_status bsf_plan_geometry(bsf_plan_t p, bsf_geometry *geom) {
    if (!p || !geom) return set_err(BSF_EINVAL, "null argument");
    geom->margin_x = p->geo.P;
    geom->margin_y = p->geo.Pb;
    geom->g_width = p->geo.GW;
    geom->g_height = p->geo.GH;
    geom->nbases = p->geo.nbases;
    geom->g_bytes = g_bytes(p);
    geom->g_exact_bytes = p->d.in_dtype == BSF_U8 ? g_bytes(p) / 2 : 0;
    geom->super_tile = p->stile;
    geom->global_mode = global_exact(p) ? 1 : 0;
    geom->tile_unit = global_exact(p) ? 0 : (use_fused(p) ? p->stile : TILE);
    geom->row0 = p->y0;
    geom->row_count = p->y1 - p->y0;
    geom->block_row0 = p->b0;
    geom->block_rows = p->b1 - p->b0;
    geom->halo = p->halo;
    geom->g_row0 = p->gy0;
    geom->g_rows = p->g_rows;
    if (p->d.nranks > 1) {  // the strip's share of the GLOBAL-mode sums
        geom->g_height = p->g_rows;
        geom->g_bytes = (size_t)geom->nbases * p->geo.nimg * p->g_rows * p->geo.GW * sizeof(double2);
        geom->g_exact_bytes = p->d.in_dtype == BSF_U8 ? geom->g_bytes / 2 : 0;
    }
    return BSF_OK;
}

// The pre-integration of every basis of the plan (launch(slot, stream) runs
// one basis' 4r levels): with two bases, basis 1 runs concurrently on the
// plan's side stream (its levels' grids are ~1 CTA per SM each: two bases in
// flight fill the GPU), forked from and joined back into `st` by events, so
// the caller sees one stream (CUDA-graph capture included).
template <class F>
static bsf_status preint_bases(bsf_plan_s *p, cudaStream_t st, F launch) {
    if (p->geo.nbases == 2 && !p->s_side) {
        if (cudaStreamCreateWithFlags(&p->s_side, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming) != cudaSuccess) {
            p->s_side = nullptr;
            return set_err(BSF_ECUDA, "side stream for the second basis");
        }
    }
    if (p->geo.nbases == 2) {
        CUDA_TRY(cudaEventRecord(p->ev_fork, st));
        CUDA_TRY(cudaStreamWaitEvent(p->s_side, p->ev_fork, 0));
        CUDA_TRY(launch(1, p->s_side));
        CUDA_TRY(launch(0, st));
        CUDA_TRY(cudaEventRecord(p->ev_join, p->s_side));
        CUDA_TRY(cudaStreamWaitEvent(st, p->ev_join, 0));
        return BSF_OK;
    }
    for (int s = 0; s < p->geo.nbases; ++s) CUDA_TRY(launch(s, st));
    return BSF_OK;
}

extern "C" bsf_status bsf_preintegrate(bsf_plan_t p, const void *f, void *g, void *stream) {
    if (!p || !f || !g) return set_err(BSF_EINVAL, "null argument");
    DevGuard guard(p->d.device);
    if (p->d.nranks > 1) return set_err(BSF_EUNSUPPORTED, "multi-GPU plans: bsf_run and bsf_preintegrate_exact only");
    if (p->d.boundary != BSF_BOUNDARY_ZERO) return set_err(BSF_EUNSUPPORTED, "replicate boundary: fused path only");
    cudaStream_t st = (cudaStream_t)stream;
    p->last = st;
    double2 *gd = (double2 *)g;
    size_t slot = (size_t)p->geo.nimg * p->geo.GH * p->geo.GW;
    return preint_bases(p, st, [&](int s, cudaStream_t ss) {
        return launch_preint_dd(f, p->d.in_dtype == BSF_U8, gd + s * slot, p->geo, p->bases[s], p->d.order, ss,
                                &p->nlaunch);
    });
}

// GLOBAL mode over row strips (Alg. 3 step 2):
// this rank holds image rows [gy0, gy1) and domain rows [gy0, gy0 + g_rows) of
// the single global pre-integration.  Before every level with a vertical step
// it receives the level's sums on the sy domain rows just above the strip
// (the scan carry) from rank - 1, runs the level from them, and sends its own
// last sy rows of the level to rank + 1.  The ranks form a chain (no cycle);
// the result is the one-GPU bsf_preintegrate_exact, bit for bit.
static bsf_status preintegrate_exact_strip(bsf_plan_s *p, const uint8_t *f, unsigned long long *g, cudaStream_t st) {
    if (!p->comm) return set_err(BSF_EINVAL, "multi-GPU GLOBAL-mode pre-integration needs the plan's communicator");
    NcclApi &nc = nccl_api();
    Geometry gs = p->geo;
    gs.H = p->gy1 - p->gy0;
    gs.Pb = p->d.rank == p->d.nranks - 1 ? p->geo.Pb : 0;
    gs.GH = gs.H + gs.Pb;
    const size_t GW = gs.GW, nimg = gs.nimg, slot = nimg * gs.GH * GW;
    if (!p->carry) {
        void *q;
        if (cudaMalloc(&q, nimg * 2 * GW * sizeof(unsigned long long)) != cudaSuccess)
            return set_err(BSF_ENOMEM, "scan carry buffer");
        p->dev_allocs.push_back(q);
        p->carry = (unsigned long long *)q;
    }
    const bool first = p->d.rank == 0, last = p->d.rank == p->d.nranks - 1;
    for (int sl = 0; sl < gs.nbases; ++sl) {
        unsigned long long *gsl = g + sl * slot;
        for (int lv = 0; lv < 4 * p->d.order; ++lv) {
            int sx, sy;
            scan_step(p->bases[sl], lv, &sx, &sy);
            if (sy > 0 && !first) {
                NCCL_TRY(nc.groupStart());
                for (size_t i = 0; i < nimg; ++i)
                    NCCL_TRY(nc.recv(p->carry + i * sy * GW, sy * GW, ncclUint64, p->d.rank - 1, p->comm, st));
                NCCL_TRY(nc.groupEnd());
            }
            CUDA_TRY(launch_scan_level(f, 1, gsl, 1, gs, p->bases[sl], lv, (sy > 0 && !first) ? p->carry : nullptr,
                                       st));
            ++p->nlaunch;
            if (sy > 0 && !last) {
                NCCL_TRY(nc.groupStart());
                for (size_t i = 0; i < nimg; ++i)
                    NCCL_TRY(nc.send(gsl + (i * gs.GH + gs.GH - sy) * GW, sy * GW, ncclUint64, p->d.rank + 1, p->comm,
                                     st));
                NCCL_TRY(nc.groupEnd());
            }
        }
    }
    return BSF_OK;
}

extern "C" bsf_status bsf_preintegrate_exact(bsf_plan_t p, const void *f, void *g, void *stream) {
    if (!p || !f || !g) return set_err(BSF_EINVAL, "null argument");
    DevGuard guard(p->d.device);
    if (p->d.boundary != BSF_BOUNDARY_ZERO) return set_err(BSF_EUNSUPPORTED, "replicate boundary: fused path only");
    if (p->d.in_dtype != BSF_U8) return set_err(BSF_EINVAL, "exact pre-integration needs u8 input");
    cudaStream_t st = (cudaStream_t)stream;
    p->last = st;
    unsigned long long *gd = (unsigned long long *)g;
    if (p->d.nranks > 1) return preintegrate_exact_strip(p, (const uint8_t *)f, gd, st);
    size_t slot = (size_t)p->geo.nimg * p->geo.GH * p->geo.GW;
    return preint_bases(p, st, [&](int s, cudaStream_t ss) {
        return launch_preint_i64((const uint8_t *)f, gd + s * slot, p->geo, p->bases[s], p->d.order, ss, &p->nlaunch);
    });
}

extern "C" bsf_status bsf_scan_step(bsf_plan_t p, int slot, int level, int *sx, int *sy) {
    if (!p || !sx || !sy) return set_err(BSF_EINVAL, "null argument");
    if (slot < 0 || slot >= p->geo.nbases || level < 0 || level >= 4 * p->d.order)
        return set_err(BSF_EINVAL, "slot or level out of range");
    scan_step(p->bases[slot], level, sx, sy);
    return BSF_OK;
}

extern "C" bsf_status bsf_scan_level(bsf_plan_t p, int slot, int level, int exact, const void *f, void *g,
                                     const void *carry, void *stream) {
    if (!p || !g || (level == 0 && !f)) return set_err(BSF_EINVAL, "null argument");
    DevGuard guard(p->d.device);
    if (p->d.nranks > 1) return set_err(BSF_EUNSUPPORTED, "multi-GPU plans: bsf_run and bsf_preintegrate_exact only");
    if (p->d.boundary != BSF_BOUNDARY_ZERO) return set_err(BSF_EUNSUPPORTED, "replicate boundary: fused path only");
    if (slot < 0 || slot >= p->geo.nbases || level < 0 || level >= 4 * p->d.order)
        return set_err(BSF_EINVAL, "slot or level out of range");
    if (exact && p->d.in_dtype != BSF_U8) return set_err(BSF_EINVAL, "exact pre-integration needs u8 input");
    cudaStream_t st = (cudaStream_t)stream;
    p->last = st;
    const size_t slot_bytes = (size_t)p->geo.nimg * p->geo.GH * p->geo.GW * (exact ? 8 : 16);
    CUDA_TRY(launch_scan_level(f, p->d.in_dtype == BSF_U8, (char *)g + slot * slot_bytes, exact, p->geo,
                               p->bases[slot], level, carry, st));
    ++p->nlaunch;
    return BSF_OK;
}

static GatherArgs gather_args(bsf_plan_s *p, const void *g, const void *cov, void *out) {
    GatherArgs a;
    memset(&a, 0, sizeof a);
    a.geo = p->geo;
    a.policy = p->d.basis;
    a.clamp = p->d.clamp;
    a.channels = p->d.channels;
    a.out_f32 = p->d.out_dtype == BSF_F32;
    a.g = (const double2 *)g;
    a.cov = (const float *)cov;
    a.out = out;
    a.stats = p->stats;
    a.cov_layout = p->d.cov_layout;
    return a;
}

extern "C" bsf_status bsf_filter(bsf_plan_t p, const void *g, const void *cov, void *out, void *stream) {
    if (!p || !g || !cov || !out) return set_err(BSF_EINVAL, "null argument");
    DevGuard guard(p->d.device);
    if (p->d.nranks > 1) return set_err(BSF_EUNSUPPORTED, "multi-GPU plans: bsf_run and bsf_preintegrate_exact only");
    if (p->d.margin_y == -1) return set_err(BSF_EINVAL, "row-strip plan (margin_y = -1): pre-integration only");
    cudaStream_t st = (cudaStream_t)stream;
    p->last = st;
    GatherArgs a = gather_args(p, g, cov, out);
    CUDA_TRY(launch_gather_impl(a, p->d.order, p->d.precision, st, p->luts_dev, &p->nlaunch));
    return BSF_OK;
}

extern "C" bsf_status bsf_filter_points(bsf_plan_t p, const void *g, const void *cov, const int *pts, int npts,
                                        double *out, void *stream) {
    return bsf_filter_points_aux(p, g, cov, pts, npts, out, nullptr, stream);
}

extern "C" bsf_status bsf_filter_points_aux(bsf_plan_t p, const void *g, const void *cov, const int *pts, int npts,
                                            double *out, double *aux, void *stream) {
    if (!p || !g || !cov || !out || (!pts && npts)) return set_err(BSF_EINVAL, "null argument");
    DevGuard guard(p->d.device);
    if (p->d.nranks > 1) return set_err(BSF_EUNSUPPORTED, "multi-GPU plans: bsf_run and bsf_preintegrate_exact only");
    if (p->d.margin_y == -1) return set_err(BSF_EINVAL, "row-strip plan (margin_y = -1): pre-integration only");
    if (npts < 0) return set_err(BSF_EINVAL, "npts < 0");
    if (npts == 0) return BSF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    p->last = st;
    GatherArgs a = gather_args(p, g, cov, out);
    a.out_f32 = 0;
    a.pts = pts;
    a.npts = npts;
    a.aux = aux;
    CUDA_TRY(launch_gather_impl(a, p->d.order, p->d.precision, st, p->luts_dev, &p->nlaunch));
    return BSF_OK;
}

// The exact split contraction (bsf_fused.cuh) serves the tile path whenever
// every table in use keeps an exact limb of >= KBITS_MIN bits; otherwise (and
// for BSF_PREC_FP64, or the diagnostics option "fused" = 0) the per-thread
// double-double tile kernel runs.
static bool use_fused(const bsf_plan_s *p) {
    if (p->d.precision == BSF_PREC_FP64 || p->d.order > 3) return false;
    if (!p->opt_fused) return false;
    for (int b = 0; b < 2; ++b) {
        if (!(p->d.basis == BSF_DUAL || p->d.basis == b)) continue;
        for (int v = 0; v < NVAR; ++v) {
            if (p->host_luts[b].var[v].kbits < KBITS_MIN) return false;
            if (p->d.order >= 3 && !p->host_luts[b].var[v].num32) return false;  // fp32-exact B tables
        }
    }
    return true;
}

// Workspace of the tile path (fused or double-double tile kernel).  The halo
// scratch (`scratch`) is only needed by tile-anchored runs; global-mode runs
// use the fused buffers alone.  Each group is marked ready only once all of its
// allocations succeeded, so a failed call can be retried.
static bsf_status ensure_tile_ws(bsf_plan_s *p, bool scratch = true) {
    if (p->fused_ready && (p->scratch_ready || !scratch)) return BSF_OK;
    int mask = p->d.basis == BSF_DUAL ? 3 : (1 << p->d.basis);
    p->fused = use_fused(p);
    p->tile_cap = tile_capacity(p->d.order, p->d.max_sigma, p->host_luts, mask, p->fused ? p->stile : TILE);
    p->tile_nslots = p->fused ? fused_slots() : tile_slots();
    void *q;
    if (scratch && !p->scratch_ready) {
        size_t bytes = (size_t)p->tile_nslots * (p->fused ? NPLANE_MAX : 2) * p->tile_cap * sizeof(double2);
        if (cudaMalloc(&q, bytes) != cudaSuccess) return set_err(BSF_ENOMEM, "tile scratch " + std::to_string(bytes));
        p->dev_allocs.push_back(q);
        p->tile_scratch = (double2 *)q;
        if (p->fused && p->d.order >= 3) {
            const size_t b0 = (size_t)p->tile_nslots * NPLANE_MAX * p->tile_cap * sizeof(double);
            if (cudaMalloc(&q, b0) != cudaSuccess) return set_err(BSF_ENOMEM, "limb scratch " + std::to_string(b0));
            p->dev_allocs.push_back(q);
            p->scratch0 = (double *)q;
        }
        p->scratch_ready = true;
    }
    if (p->fused_ready) return BSF_OK;
    if (p->fused) {
        const size_t fb = (size_t)p->tile_nslots * fused_fbuf_items(p->d.order) * sizeof(double2);
        if (cudaMalloc(&q, fb) != cudaSuccess) return set_err(BSF_ENOMEM, "tap buffer " + std::to_string(fb));
        p->dev_allocs.push_back(q);
        p->fbuf = (double2 *)q;
        const size_t sb = (size_t)p->tile_nslots * FUSED_NQ_MAX * 256 * 5 * sizeof(double);
        if (cudaMalloc(&q, sb) != cudaSuccess) return set_err(BSF_ENOMEM, "scale buffer " + std::to_string(sb));
        p->dev_allocs.push_back(q);
        p->sbuf = (double *)q;
    }
    if (cudaMalloc(&q, sizeof(int)) != cudaSuccess) return set_err(BSF_ENOMEM, "tile counter");
    p->dev_allocs.push_back(q);
    p->tile_counter = (int *)q;
    if (p->fused) {
        // largest-first work order of the super-tiles (launch_fused_impl)
        // units: super-tiles, or at 64 x 64 and order >= 2 up to four 32 x 32
        // quadrants each (split mode; also covers bsf_run_split's 32 x 32 passes)
        const int ts = p->stile;
        long long n = (long long)((p->geo.W + ts - 1) / ts) * ((p->geo.H + ts - 1) / ts) * p->geo.nimg;
        if (ts == 64 && p->d.order >= 2) n *= 4;
        const size_t hw = 2 * SCHED_NBIN + 4;  // bin counts, cursors, unit count (+ pad)
        const size_t ob = (size_t)n * (sizeof(int) + 1) + hw * sizeof(unsigned) + 16;
        if (cudaMalloc(&q, ob) != cudaSuccess) return set_err(BSF_ENOMEM, "work order " + std::to_string(ob));
        p->dev_allocs.push_back(q);
        p->sched_hist = (unsigned *)q;
        p->sched_order = (int *)((char *)q + hw * sizeof(unsigned));
        p->sched_bin = (unsigned char *)(p->sched_order + n);
        p->sched_cap = n;
    }
    p->fused_ready = true;
    return BSF_OK;
}

static TileArgs tile_args(bsf_plan_s *p, const void *f, const void *cov, void *out) {
    TileArgs a;
    memset(&a, 0, sizeof a);
    a.W = p->geo.W;
    a.H = p->geo.H;
    a.nimg = p->geo.nimg;
    a.channels = p->d.channels;
    a.policy = p->d.basis;
    a.clamp = p->d.clamp;
    a.out_f32 = p->d.out_dtype == BSF_F32;
    a.in_u8 = p->d.in_dtype == BSF_U8;
    a.f = f;
    a.cov = (const float *)cov;
    a.out = out;
    a.scratch = p->tile_scratch;
    a.cap = (long long)p->tile_cap;
    a.counter = p->tile_counter;
    a.ntx = (p->geo.W + TILE - 1) / TILE;
    a.nty = (p->geo.H + TILE - 1) / TILE;
    a.stats = p->stats;
    a.prof = p->prof;
    a.fbuf = p->fbuf;
    a.sbuf = p->sbuf;
    a.scratch0 = p->scratch0;
    a.stile = p->stile;
    a.replicate = p->d.boundary == BSF_BOUNDARY_REPLICATE;
    a.sigma2_scale = 1.0;
    // diagnostics option "work_order" = 0: hand the super-tiles out in raster order
    if (p->opt_order) {
        a.order = p->sched_order;
        a.order_bin = p->sched_bin;
        a.order_hist = p->sched_hist;
        a.order_cap = p->sched_cap;
    }
    a.split_tol = p->opt_split_tol;  // BSF_SPLIT_TOL_DEFAULT unless a diagnostics option changed it
    a.i8 = p->opt_i8_tc;
    a.cov_layout = p->d.cov_layout;
    return a;
}

static cudaError_t launch_tile(bsf_plan_s *p, const TileArgs &a, cudaStream_t st) {
    if (p->fused) return launch_fused_impl(a, p->d.order, p->tile_nslots, st, p->luts_dev, &p->nlaunch);
    if (a.replicate) return cudaErrorNotSupported;  // the double-double tile kernel is zero-extension only
    return launch_tile_impl(a, p->d.order, p->d.precision, p->tile_nslots, st, p->luts_dev, &p->nlaunch);
}

// Global mode: the paper's single global pre-integration as
// exact int64 running sums, gathered by the fused kernel with both limbs of
// the contraction exact.  Used by BSF_ANCHOR_GLOBAL and BSF_ANCHOR_AUTO when
// the plan qualifies (u8 input, order 1, sums below 2^62).
static bool global_exact(const bsf_plan_s *p) {
    return p->global_ok && p->d.anchor != BSF_ANCHOR_TILE && p->opt_fused && p->d.precision != BSF_PREC_FP64;
}

// gather of global mode from exact int64 sums g ([nbases][nimg][GH][GW], the
// bsf_preintegrate_exact layout): the order-1 integer kernel (bsf_gx1.cuh),
// or (diagnostics option global_kernel = 0) the fused kernel's global mode
static bsf_status filter_global(bsf_plan_s *p, const void *g, const void *cov, void *out, const int *pts, int npts,
                                double *aux, cudaStream_t st) {
    bsf_status s = ensure_tile_ws(p, false);
    if (s != BSF_OK) return s;
    if (!p->fused) return set_err(BSF_EUNSUPPORTED, "global mode needs the exact split path");
    p->last = st;
    const Geometry &geo = p->geo;
    const size_t slot = (size_t)geo.nimg * geo.GH * geo.GW;
    TileArgs a = tile_args(p, nullptr, cov, out);
    a.stile = p->stile_global;
    a.order = nullptr;  // order 1: raster hand-out
    a.gP = geo.P;
    a.gGW = geo.GW;
    a.gGH = geo.GH;
    a.gGHv = geo.GH;
    for (int sl = 0; sl < geo.nbases; ++sl) {  // slot sl of the int64 buffer holds basis bases[sl]
        a.gglob[p->bases[sl]] = (const long long *)g + sl * slot;
        a.gshift[p->bases[sl]] = p->gshift[p->bases[sl]];
        a.gvw[p->bases[sl]] = p->gvw[p->bases[sl]];
    }
    a.gdp4a = p->opt_gx1_dp4a;
    if (pts) {
        a.pts = pts;
        a.npts = npts;
        a.aux = aux;
        a.out_f32 = 0;
    }
    if (p->opt_global_kernel == 1)
        CUDA_TRY(launch_gx1(a, st, p->luts_dev, &p->nlaunch));
    else
        CUDA_TRY(launch_fused_impl(a, p->d.order, p->tile_nslots, st, p->luts_dev, &p->nlaunch));
    return BSF_OK;
}

// the order-1 gather on output rows [y0, y0 + h) only (cov and out hold those
// rows: [batch][3][h][W] and [nimg][h][W]); y0 a multiple of 32
static bsf_status filter_global_window(bsf_plan_s *p, const void *g, const void *cov, void *out, int y0, int h,
                                       int rows_ready, cudaStream_t st) {
    bsf_status s = ensure_tile_ws(p, false);
    if (s != BSF_OK) return s;
    const Geometry &geo = p->geo;
    const size_t slot = (size_t)geo.nimg * geo.GH * geo.GW;
    TileArgs a = tile_args(p, nullptr, cov, out);
    a.order = nullptr;
    a.gP = geo.P;
    a.gGW = geo.GW;
    a.gGH = geo.GH;
    a.gGHv = rows_ready;
    a.oy0 = y0;
    a.oH = h;
    for (int sl = 0; sl < geo.nbases; ++sl) {
        a.gglob[p->bases[sl]] = (const long long *)g + sl * slot;
        a.gshift[p->bases[sl]] = p->gshift[p->bases[sl]];
        a.gvw[p->bases[sl]] = p->gvw[p->bases[sl]];
    }
    a.gdp4a = p->opt_gx1_dp4a;
    CUDA_TRY(launch_gx1(a, st, p->luts_dev, &p->nlaunch));
    return BSF_OK;
}

static bsf_status run_global(bsf_plan_s *p, const void *f, const void *cov, void *out, const int *pts, int npts,
                             double *aux, cudaStream_t st) {
    if (!p->gx_ws) {
        void *q;
        const size_t bytes = g_bytes(p) / 2;  // int64 elements
        if (cudaMalloc(&q, bytes) != cudaSuccess) return set_err(BSF_ENOMEM, "global int64 sums " + std::to_string(bytes));
        p->dev_allocs.push_back(q);
        p->gx_ws = (long long *)q;
    }
    p->last = st;
    const size_t slot = (size_t)p->geo.nimg * p->geo.GH * p->geo.GW;
    const bsf_status e = preint_bases(p, st, [&](int b, cudaStream_t ss) {
        return launch_preint_i64((const uint8_t *)f, (unsigned long long *)p->gx_ws + b * slot, p->geo, p->bases[b],
                                 p->d.order, ss, &p->nlaunch);
    });
    if (e != BSF_OK) return e;
    return filter_global(p, p->gx_ws, cov, out, pts, npts, aux, st);
}

extern "C" bsf_status bsf_filter_exact(bsf_plan_t p, const void *g, const void *cov, void *out, void *stream) {
    if (!p || !g || !cov || !out) return set_err(BSF_EINVAL, "null argument");
    if (p->d.margin_y == -1) return set_err(BSF_EINVAL, "row-strip plan (margin_y = -1): pre-integration only");
    DevGuard guard(p->d.device);
    if (p->d.nranks > 1) return set_err(BSF_EUNSUPPORTED, "multi-GPU plans: bsf_run and bsf_preintegrate_exact only");
    if (!global_exact(p)) return set_err(BSF_EUNSUPPORTED, "bsf_filter_exact: the plan is not in global mode");
    return filter_global(p, g, cov, out, nullptr, 0, nullptr, (cudaStream_t)stream);
}

extern "C" bsf_status bsf_run_points(bsf_plan_t p, const void *f, const void *cov, const int *pts, int npts,
                                     double *out, double *aux, void *stream) {
    if (!p || !f || !cov || !out || (!pts && npts)) return set_err(BSF_EINVAL, "null argument");
    if (p->d.margin_y == -1) return set_err(BSF_EINVAL, "row-strip plan (margin_y = -1): pre-integration only");
    if (npts < 0) return set_err(BSF_EINVAL, "npts < 0");
    if (npts == 0) return BSF_OK;
    DevGuard guard(p->d.device);
    if (p->d.nranks > 1) return set_err(BSF_EUNSUPPORTED, "multi-GPU plans: bsf_run and bsf_preintegrate_exact only");
    if (global_exact(p)) return run_global(p, f, cov, out, pts, npts, aux, (cudaStream_t)stream);
    bsf_status s = ensure_tile_ws(p);
    if (s != BSF_OK) return s;
    if (p->d.boundary != BSF_BOUNDARY_ZERO && !p->fused)
        return set_err(BSF_EUNSUPPORTED, "replicate boundary: fused path only (order <= 3)");
    cudaStream_t st = (cudaStream_t)stream;
    p->last = st;
    TileArgs a = tile_args(p, f, cov, out);
    a.pts = pts;
    a.npts = npts;
    a.aux = aux;
    a.out_f32 = 0;
    CUDA_TRY(launch_tile(p, a, st));
    return BSF_OK;
}

extern "C" bsf_status bsf_run_tiles(bsf_plan_t p, const void *f, const void *cov, void *out, const int *tiles,
                                    int ntiles, void *stream) {
    if (!p || !f || !cov || !out || (!tiles && ntiles)) return set_err(BSF_EINVAL, "null argument");
    if (p->d.margin_y == -1) return set_err(BSF_EINVAL, "row-strip plan (margin_y = -1): pre-integration only");
    if (ntiles < 0) return set_err(BSF_EINVAL, "ntiles < 0");
    DevGuard guard(p->d.device);
    if (p->d.nranks > 1) return set_err(BSF_EUNSUPPORTED, "multi-GPU plans: bsf_run and bsf_preintegrate_exact only");
    if (global_exact(p)) return set_err(BSF_EUNSUPPORTED, "bsf_run_tiles: global-mode plans have no anchoring tiles");
    if (ntiles == 0) return BSF_OK;
    bsf_status s = ensure_tile_ws(p);
    if (s != BSF_OK) return s;
    if (p->d.boundary != BSF_BOUNDARY_ZERO && !p->fused)
        return set_err(BSF_EUNSUPPORTED, "replicate boundary: fused path only (order <= 3)");
    cudaStream_t st = (cudaStream_t)stream;
    p->last = st;
    TileArgs a = tile_args(p, f, cov, out);
    a.tiles = tiles;
    a.ntiles = ntiles;
    CUDA_TRY(launch_tile(p, a, st));
    return BSF_OK;
}

// Row strip of a multi-GPU plan (include/bsf.h, bsf_plan_desc): the block of
// input rows [b0, b1) is assembled from this rank's rows and the neighbours'
// halo rows (ncclSend / ncclRecv, one group per call) unless the caller passed
// the block itself (no communicator); then the fused kernel filters the own
// rows [y0, y1) only, anchored on the full image's super-tiles.
static bsf_status run_strip(bsf_plan_s *p, const void *f, const void *cov, void *out, cudaStream_t st) {
    if (p->d.anchor == BSF_ANCHOR_GLOBAL) return set_err(BSF_EUNSUPPORTED, "row strips run the tile path");
    bsf_status s = ensure_tile_ws(p);
    if (s != BSF_OK) return s;
    if (!p->fused) return set_err(BSF_EUNSUPPORTED, "row strips need the exact split path (order <= 3)");
    p->last = st;
    const int W = p->geo.W, nimg = p->geo.nimg;
    const int own = p->y1 - p->y0, blk = p->b1 - p->b0, top = p->y0 - p->b0;
    const size_t es = p->d.in_dtype == BSF_U8 ? 1 : 4;
    const void *fb = f;
    if (p->comm) {
        if (!p->f_blk) {
            void *q;
            if (cudaMalloc(&q, (size_t)nimg * blk * W * es) != cudaSuccess) return set_err(BSF_ENOMEM, "strip block");
            p->dev_allocs.push_back(q);
            p->f_blk = q;
        }
        char *B = (char *)p->f_blk;
        const char *F = (const char *)f;
        const size_t row = (size_t)W * es;
        for (int i = 0; i < nimg; ++i)
            CUDA_TRY(cudaMemcpyAsync(B + ((size_t)i * blk + top) * row, F + (size_t)i * own * row, (size_t)own * row,
                                     cudaMemcpyDeviceToDevice, st));
        int x[8];
        bsf_status xs = bsf_strip_exchange(p->geo.H, p->stile, p->halo, p->d.rank, p->d.nranks, x);
        if (xs != BSF_OK) return xs;
        NcclApi &nc = nccl_api();
        const ncclDataType_t dt = p->d.in_dtype == BSF_U8 ? ncclUint8 : ncclFloat32;
        NCCL_TRY(nc.groupStart());
        for (int i = 0; i < nimg; ++i) {
            const char *Fi = F + (size_t)i * own * row;
            char *Bi = B + (size_t)i * blk * row;
            if (p->d.rank > 0) {  // my first rows to rank - 1, block rows [0, top) from it
                NCCL_TRY(nc.send(Fi + (size_t)x[0] * row, (size_t)x[1] * W, dt, p->d.rank - 1, p->comm, st));
                NCCL_TRY(nc.recv(Bi, (size_t)x[2] * W, dt, p->d.rank - 1, p->comm, st));
            }
            if (p->d.rank < p->d.nranks - 1) {  // my last rows to rank + 1, block rows [top + own, blk) from it
                NCCL_TRY(nc.send(Fi + (size_t)x[3] * row, (size_t)x[4] * W, dt, p->d.rank + 1, p->comm, st));
                NCCL_TRY(nc.recv(Bi + (size_t)x[5] * row, (size_t)x[6] * W, dt, p->d.rank + 1, p->comm, st));
            }
        }
        NCCL_TRY(nc.groupEnd());
        fb = p->f_blk;
    }
    TileArgs a = tile_args(p, fb, cov, out);
    a.H = blk;
    a.oy0 = top;
    a.oH = own;
    CUDA_TRY(launch_tile(p, a, st));
    return BSF_OK;
}

extern "C" bsf_status bsf_run(bsf_plan_t p, const void *f, const void *cov, void *out, void *stream) {
    if (!p) return set_err(BSF_EINVAL, "null plan");
    if (p->d.margin_y == -1) return set_err(BSF_EINVAL, "row-strip plan (margin_y = -1): pre-integration only");
    DevGuard guard(p->d.device);
    if (global_exact(p)) {
        if (!f || !cov || !out) return set_err(BSF_EINVAL, "null argument");
        return run_global(p, f, cov, out, nullptr, 0, nullptr, (cudaStream_t)stream);
    }
    if (p->d.nranks > 1) {
        if (!f || !cov || !out) return set_err(BSF_EINVAL, "null argument");
        return run_strip(p, f, cov, out, (cudaStream_t)stream);
    }
    if (p->d.anchor != BSF_ANCHOR_GLOBAL) {  // BSF_ANCHOR_TILE, or AUTO without global mode
        if (!f || !cov || !out) return set_err(BSF_EINVAL, "null argument");
        bsf_status s = ensure_tile_ws(p);
        if (s != BSF_OK) return s;
        if (p->d.boundary != BSF_BOUNDARY_ZERO && !p->fused)
            return set_err(BSF_EUNSUPPORTED, "replicate boundary: fused path only (order <= 3)");
        cudaStream_t st = (cudaStream_t)stream;
        p->last = st;
        TileArgs a = tile_args(p, f, cov, out);
        CUDA_TRY(launch_tile(p, a, st));
        return BSF_OK;
    }
    if (!p->g_ws) {
        void *q;
        if (cudaMalloc(&q, g_bytes(p)) != cudaSuccess) return set_err(BSF_ENOMEM, "g workspace");
        p->dev_allocs.push_back(q);
        p->g_ws = (double2 *)q;
    }
    bsf_status s = bsf_preintegrate(p, f, p->g_ws, stream);
    if (s != BSF_OK) return s;
    return bsf_filter(p, p->g_ws, cov, out, stream);
}

extern "C" bsf_status bsf_run_normalized(bsf_plan_t p, const void *f, const void *cov, void *out, void *stream) {
    if (!p || !f || !cov || !out) return set_err(BSF_EINVAL, "null argument");
    DevGuard guard(p->d.device);
    if (p->d.nranks > 1) return set_err(BSF_EUNSUPPORTED, "multi-GPU plans: bsf_run and bsf_preintegrate_exact only");
    if (p->d.margin_y == -1) return set_err(BSF_EINVAL, "row-strip plan (margin_y = -1): pre-integration only");
    if (p->d.anchor != BSF_ANCHOR_TILE) return set_err(BSF_EUNSUPPORTED, "DC renormalisation runs with BSF_ANCHOR_TILE");
    bsf_status s = ensure_tile_ws(p);
    if (s != BSF_OK) return s;
    if (p->d.boundary != BSF_BOUNDARY_ZERO && !p->fused)
        return set_err(BSF_EUNSUPPORTED, "replicate boundary: fused path only (order <= 3)");
    const Geometry &g = p->geo;
    const size_t n = (size_t)g.nimg * g.H * g.W;
    cudaStream_t st = (cudaStream_t)stream;
    p->last = st;
    if (!p->ones) {
        void *q;
        if (cudaMalloc(&q, n * (p->d.in_dtype == BSF_U8 ? 1 : 4)) != cudaSuccess)
            return set_err(BSF_ENOMEM, "indicator image");
        p->dev_allocs.push_back(q);
        p->ones = q;
        if (cudaMalloc(&q, n * sizeof(double)) != cudaSuccess) return set_err(BSF_ENOMEM, "normaliser");
        p->dev_allocs.push_back(q);
        p->norm_den = (double *)q;
        CUDA_TRY(launch_fill_ones(p->ones, p->d.in_dtype == BSF_U8, n, st, &p->nlaunch));
    }
    TileArgs a = tile_args(p, f, cov, out);
    CUDA_TRY(launch_tile(p, a, st));
    TileArgs b = tile_args(p, p->ones, cov, p->norm_den);  // sum_q beta(p - q) over the image
    b.out_f32 = 0;
    CUDA_TRY(launch_tile(p, b, st));
    CUDA_TRY(launch_normalize(out, p->d.out_dtype == BSF_F32, p->norm_den, n, st, &p->nlaunch));
    return BSF_OK;
}

static bsf_status ensure_alg1_ws(bsf_plan_s *p, bool two) {
    const Geometry &g = p->geo;
    const size_t img_bytes = (size_t)g.nimg * g.H * g.W * sizeof(double);
    void *q;
    if (!p->alg1_work) {
        if (cudaMalloc(&q, img_bytes) != cudaSuccess) return set_err(BSF_ENOMEM, "Algorithm 1 work image");
        p->dev_allocs.push_back(q);
        p->alg1_work = (double *)q;
        if (cudaMalloc(&q, 2 * (size_t)p->d.batch * sizeof(double)) != cudaSuccess)
            return set_err(BSF_ENOMEM, "Algorithm 1 sigma");
        p->dev_allocs.push_back(q);
        p->alg1_sigma2 = (double *)q;
    }
    if (two && !p->alg1_work2) {
        if (cudaMalloc(&q, img_bytes) != cudaSuccess) return set_err(BSF_ENOMEM, "splitting work image");
        p->dev_allocs.push_back(q);
        p->alg1_work2 = (double *)q;
    }
    return BSF_OK;
}

extern "C" bsf_status bsf_run_split(bsf_plan_t p, const void *f, const void *cov, void *out, int passes,
                                    double fraction, double *sigma2_out, void *stream) {
    if (!p || !f || !cov || !out) return set_err(BSF_EINVAL, "null argument");
    DevGuard guard(p->d.device);
    if (p->d.nranks > 1) return set_err(BSF_EUNSUPPORTED, "multi-GPU plans: bsf_run and bsf_preintegrate_exact only");
    if (p->d.margin_y == -1) return set_err(BSF_EINVAL, "row-strip plan (margin_y = -1): pre-integration only");
    if (passes < 2 || passes > 16) return set_err(BSF_EINVAL, "passes must be 2..16");
    if (!(fraction < 1.0) || fraction < 0.0 || fraction != fraction)
        return set_err(BSF_EINVAL, "fraction must be in [0, 1) (0: the default (n - 1) / n)");
    bsf_status s = ensure_tile_ws(p);
    if (s != BSF_OK) return s;
    if (!p->fused) return set_err(BSF_EUNSUPPORTED, "covariance splitting runs on the exact split path (order <= 3)");
    s = ensure_alg1_ws(p, passes > 2);
    if (s != BSF_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    p->last = st;
    // sigma_b^2 = half the smallest bound (9) of the field (R21): the bound is 2 sigma_b^2
    CUDA_TRY(launch_alg1_sigma2((const float *)cov, p->d.batch, p->geo.W, p->geo.H, p->d.basis, p->d.clamp,
                                p->d.cov_layout, p->alg1_sigma2, st, &p->nlaunch));
    // the isotropic part T = phi B (B = 2 sigma_b^2 the bound, phi = fraction,
    // default (n - 1) / n): passes - 1 isotropic passes of T / (n - 1) each,
    // ping-ponging through float64 work images, then the space-variant
    // residual C - T I (R22; n = 2, phi = 1/2 is Algorithm 1)
    const double n = passes;
    const double phi = fraction > 0.0 ? fraction : (n - 1.0) / n;
    const void *src = f;
    bool src_f64 = false;
    double *bufs[2] = {p->alg1_work, p->alg1_work2};
    for (int i = 0; i < passes - 1; ++i) {
        double *dst = bufs[i & 1];
        TileArgs a = tile_args(p, src, cov, dst);
        a.out_f32 = 0;
        if (src_f64) {
            a.in_u8 = 0;
            a.in_f64 = 1;
        }
        // 64 x 64 anchoring at order 2 only for the plain u8 run: the small
        // isotropic scales of these passes (and float64 input) send every pixel
        // of a 64 x 64 domain to the fallback (config 3: 16.8M of 16.8M)
        if (p->d.order >= 2) a.stile = std::min(a.stile, 32);
        a.cov_mode = COV_ISO;
        a.sigma2 = p->alg1_sigma2;
        a.sigma2_scale = 2.0 * phi / (n - 1.0);
        CUDA_TRY(launch_tile(p, a, st));
        src = dst;
        src_f64 = true;
    }
    TileArgs a = tile_args(p, src, cov, out);
    a.in_u8 = 0;
    a.in_f64 = 1;
    if (p->d.order >= 2) a.stile = std::min(a.stile, 32);
    a.cov_mode = COV_SUB;
    a.sigma2 = p->alg1_sigma2;
    a.sigma2_scale = 2.0 * phi;
    CUDA_TRY(launch_tile(p, a, st));
    if (sigma2_out) {
        CUDA_TRY(cudaStreamSynchronize(st));
        CUDA_TRY(cudaMemcpy(sigma2_out, p->alg1_sigma2, p->d.batch * sizeof(double), cudaMemcpyDeviceToHost));
    }
    return BSF_OK;
}

extern "C" bsf_status bsf_run_alg1(bsf_plan_t p, const void *f, const void *cov, void *out, double *sigma2_out,
                                   void *stream) {
    return bsf_run_split(p, f, cov, out, 2, 0.5, sigma2_out, stream);
}

// Global mode from host buffers: the copies overlap the compute.  The image
// goes first (the pre-integration needs all of it), then the covariance in
// row bands on a copy-in stream while the scans run; the gather runs band by
// band as each band's covariance lands (its output row window), and each
// finished band of the output goes back on a copy-out stream (the H2D and
// D2H engines work in parallel).  The caller's stream waits for the last copy.
// The single global pre-integration of bsf_run_host's staged image in row
// bands (Alg. 3 step 2): band k of every image is scanned
// once its rows are on the device (event ev_fb[k]), level by level, each level
// with a vertical step starting from the level's last s_y rows of band k - 1
// (the scan carry, copied out right after that level ran: the levels run in
// place).  The same arithmetic as preintegrate_exact_strip's rank chain, so
// the sums equal bsf_preintegrate_exact's bit for bit.  Each basis runs on its
// own scan stream and records ev_sb[slot][k] after band k: a gather band waits
// only for the scan bands its footprint reaches.
// bsf_run_host's staged images (u8, global mode) start on 16-byte boundaries:
// the scans read image i's band through its own base pointer, and the u8 row
// loads assume a 4-byte aligned base
static size_t host_f_pitch(const Geometry &g) { return ((size_t)g.H * g.W + 15) / 16 * 16; }

static bsf_status banded_scans_basis(bsf_plan_s *p, int sl, int k, int srows, int nsb, cudaStream_t ss) {
    const Geometry &g = p->geo;
    const int nlev = 4 * p->d.order;
    const size_t GW = g.GW, rowset = (size_t)g.nimg * 2 * GW;  // one level's carry: [nimg][2][GW]
    unsigned long long *gsl = (unsigned long long *)p->gx_ws + sl * (size_t)g.nimg * g.GH * GW;
    const int y0 = k * srows;
    const bool last = k == nsb - 1;
    Geometry gs = g;
    gs.nimg = 1;
    gs.H = std::min(srows, g.H - y0);
    gs.Pb = last ? g.Pb : 0;
    gs.GH = gs.H + gs.Pb;
    CUDA_TRY(cudaStreamWaitEvent(ss, p->ev_fb[k], 0));
    for (int lv = 0; lv < nlev; ++lv) {
        int sx, sy;
        scan_step(p->bases[sl], lv, &sx, &sy);
        unsigned long long *cin = p->hcarry + (((size_t)((k + 1) & 1) * 2 + sl) * nlev + lv) * rowset;
        unsigned long long *cout = p->hcarry + (((size_t)(k & 1) * 2 + sl) * nlev + lv) * rowset;
        for (int i = 0; i < g.nimg; ++i) {
            const uint8_t *fi = (const uint8_t *)p->f_stage + (size_t)i * host_f_pitch(g) + (size_t)y0 * g.W;
            unsigned long long *gi = gsl + ((size_t)i * g.GH + y0) * GW;
            CUDA_TRY(launch_scan_level(fi, 1, gi, 1, gs, p->bases[sl], lv,
                                       (sy > 0 && k > 0) ? cin + (size_t)i * 2 * GW : nullptr, ss));
            ++p->nlaunch;
            if (sy > 0 && !last)  // this band's last sy rows of the level: the next band's carry
                CUDA_TRY(cudaMemcpyAsync(cout + (size_t)i * 2 * GW, gi + (size_t)(gs.GH - sy) * GW,
                                         (size_t)sy * GW * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, ss));
        }
    }
    CUDA_TRY(cudaEventRecord(p->ev_sb[sl][k], ss));
    return BSF_OK;
}

static bsf_status run_host_global(bsf_plan_s *p, const void *f_host, const void *cov_host, void *out_host,
                                  cudaStream_t st) {
    const Geometry &g = p->geo;
    const int nb = BSF_HOST_BANDS;
    if (!p->s_in) {
        CUDA_TRY(cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&p->s_c2, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) CUDA_TRY(cudaStreamCreateWithFlags(&p->s_scan[i], cudaStreamNonBlocking));
        for (int i = 0; i < 2 * BSF_HOST_BANDS + 5; ++i)
            CUDA_TRY(cudaEventCreateWithFlags(&p->ev[i], cudaEventDisableTiming));
        for (int i = 0; i < BSF_SCAN_BANDS; ++i) {
            CUDA_TRY(cudaEventCreateWithFlags(&p->ev_fb[i], cudaEventDisableTiming));
            for (int sl = 0; sl < 2; ++sl) CUDA_TRY(cudaEventCreateWithFlags(&p->ev_sb[sl][i], cudaEventDisableTiming));
        }
    }
    cudaEvent_t ev_start = p->ev[0], ev_end = p->ev[2], ev_c2 = p->ev[4];
    cudaEvent_t *ev_cov = p->ev + 5, *ev_band = p->ev + 5 + BSF_HOST_BANDS;
    p->last = st;
    const size_t plane = (size_t)g.H * g.W, oes = p->d.out_dtype == BSF_F32 ? 4 : 8;
    if (!p->gx_ws) {
        void *q;
        const size_t bytes = g_bytes(p) / 2;
        if (cudaMalloc(&q, bytes) != cudaSuccess) return set_err(BSF_ENOMEM, "global int64 sums " + std::to_string(bytes));
        p->dev_allocs.push_back(q);
        p->gx_ws = (long long *)q;
    }
    if (!p->hcarry) {
        const size_t n = 2 * 2 * (size_t)(4 * p->d.order) * g.nimg * 2 * g.GW;
        void *q;
        if (cudaMalloc(&q, n * sizeof(unsigned long long)) != cudaSuccess)
            return set_err(BSF_ENOMEM, "banded scan carries");
        p->dev_allocs.push_back(q);
        p->hcarry = (unsigned long long *)q;
    }
    // gather bands of whole tiles (rows multiple of 32); image (scan) bands of
    // whole gather bands
    const int rows = ((g.H + nb - 1) / nb + 31) / 32 * 32;
    const int per = std::max(1, ((g.H + BSF_SCAN_BANDS - 1) / BSF_SCAN_BANDS + rows - 1) / rows);
    const int srows = per * rows;
    const int nsb = (g.H + srows - 1) / srows;
    CUDA_TRY(cudaEventRecord(ev_start, st));  // earlier work on the caller's stream comes first
    CUDA_TRY(cudaStreamWaitEvent(p->s_in, ev_start, 0));
    for (int sl = 0; sl < g.nbases; ++sl) CUDA_TRY(cudaStreamWaitEvent(p->s_scan[sl], ev_start, 0));
    // copy-in order: image band k, then the covariance bands of its rows; each
    // image band is scanned as soon as it is in (both bases concurrently)
    int band = 0;
    for (int k = 0; k < nsb; ++k) {
        const int y0 = k * srows, h = std::min(srows, g.H - y0);
        for (int i = 0; i < g.nimg; ++i)
            CUDA_TRY(cudaMemcpyAsync((char *)p->f_stage + (size_t)i * host_f_pitch(g) + (size_t)y0 * g.W,
                                     (const char *)f_host + (size_t)i * plane + (size_t)y0 * g.W, (size_t)h * g.W,
                                     cudaMemcpyHostToDevice, p->s_in));
        CUDA_TRY(cudaEventRecord(p->ev_fb[k], p->s_in));
        for (int sl = 0; sl < g.nbases; ++sl) {
            const bsf_status e = banded_scans_basis(p, sl, k, srows, nsb, p->s_scan[sl]);
            if (e != BSF_OK) return e;
        }
        for (int yb = y0; yb < y0 + h; yb += rows, ++band) {
            const int hb = std::min(rows, g.H - yb);
            // the band's covariance as planes [batch][3][hb][W], stored contiguously at
            // float offset batch 3 yb W of cov_stage (the bands tile the buffer)
            float *cb = (float *)p->cov_stage + (size_t)p->d.batch * 3 * (size_t)yb * g.W;
            for (int b = 0; b < p->d.batch; ++b)
                for (int c = 0; c < 3; ++c)
                    CUDA_TRY(cudaMemcpyAsync(cb + ((size_t)b * 3 + c) * (size_t)hb * g.W,
                                             (const float *)cov_host + ((size_t)b * 3 + c) * plane + (size_t)yb * g.W,
                                             (size_t)hb * g.W * sizeof(float), cudaMemcpyHostToDevice, p->s_in));
            CUDA_TRY(cudaEventRecord(ev_cov[band], p->s_in));
        }
    }
    // the gather band by band on two alternating streams, each band after its
    // covariance and the scan bands its footprint reaches (every read of a
    // pixel of rows [yb, yb + hb) lies above domain row yb + hb - 1 + Pb)
    CUDA_TRY(cudaStreamWaitEvent(p->s_c2, ev_start, 0));
    band = 0;
    for (int yb = 0; yb < g.H; yb += rows, ++band) {
        const int hb = std::min(rows, g.H - yb);
        cudaStream_t sc = (band & 1) ? p->s_c2 : st;  // alternate: a band's blocks fill the previous band's tail
        const int kneed = std::min(nsb - 1, (yb + hb - 1 + g.Pb) / srows);
        CUDA_TRY(cudaStreamWaitEvent(sc, ev_cov[band], 0));
        for (int sl = 0; sl < g.nbases; ++sl) CUDA_TRY(cudaStreamWaitEvent(sc, p->ev_sb[sl][kneed], 0));
        const size_t obase = (size_t)g.nimg * (size_t)yb * g.W;  // band output: [nimg][hb][W] at nimg yb W
        // domain rows pre-integrated once scan band kneed is done (the last band holds the bottom margin)
        const int ready = kneed == nsb - 1 ? g.GH : (kneed + 1) * srows;
        bsf_status s = filter_global_window(p, p->gx_ws, (const float *)p->cov_stage + (size_t)p->d.batch * 3 * yb * g.W,
                                            (char *)p->out_stage + obase * oes, yb, hb, ready, sc);
        if (s != BSF_OK) return s;
        CUDA_TRY(cudaEventRecord(ev_band[band], sc));
        CUDA_TRY(cudaStreamWaitEvent(p->s_out, ev_band[band], 0));
        for (int i = 0; i < g.nimg; ++i)
            CUDA_TRY(cudaMemcpyAsync((char *)out_host + ((size_t)i * plane + (size_t)yb * g.W) * oes,
                                     (char *)p->out_stage + (obase + (size_t)i * hb * g.W) * oes, (size_t)hb * g.W * oes,
                                     cudaMemcpyDeviceToHost, p->s_out));
    }
    CUDA_TRY(cudaEventRecord(ev_c2, p->s_c2));
    CUDA_TRY(cudaStreamWaitEvent(st, ev_c2, 0));
    for (int sl = 0; sl < g.nbases; ++sl) CUDA_TRY(cudaStreamWaitEvent(st, p->ev_sb[sl][nsb - 1], 0));
    CUDA_TRY(cudaEventRecord(ev_end, p->s_out));
    CUDA_TRY(cudaStreamWaitEvent(st, ev_end, 0));
    return BSF_OK;
}

extern "C" bsf_status bsf_run_host(bsf_plan_t p, const void *f_host, const void *cov_host, void *out_host,
                                   void *stream) {
    if (!p || !f_host || !cov_host || !out_host) return set_err(BSF_EINVAL, "null argument");
    DevGuard guard(p->d.device);
    if (p->d.nranks > 1) return set_err(BSF_EUNSUPPORTED, "multi-GPU plans: bsf_run and bsf_preintegrate_exact only");
    if (p->d.margin_y == -1) return set_err(BSF_EINVAL, "row-strip plan (margin_y = -1): pre-integration only");
    const Geometry &g = p->geo;
    size_t fb = (size_t)g.nimg * g.H * g.W * (p->d.in_dtype == BSF_U8 ? 1 : 4);
    if (p->d.in_dtype == BSF_U8) fb = std::max(fb, (size_t)g.nimg * host_f_pitch(g));  // global mode's staging pitch
    size_t cb = (size_t)p->d.batch * 3 * g.H * g.W * 4;
    size_t ob = (size_t)g.nimg * g.H * g.W * (p->d.out_dtype == BSF_F32 ? 4 : 8);
    if (!p->f_stage) {
        void *a, *b, *c;
        if (cudaMalloc(&a, fb) != cudaSuccess || cudaMalloc(&b, cb) != cudaSuccess || cudaMalloc(&c, ob) != cudaSuccess)
            return set_err(BSF_ENOMEM, "staging buffers");
        p->dev_allocs.push_back(a);
        p->dev_allocs.push_back(b);
        p->dev_allocs.push_back(c);
        p->f_stage = a;
        p->cov_stage = b;
        p->out_stage = c;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (global_exact(p)) return run_host_global(p, f_host, cov_host, out_host, st);
    CUDA_TRY(cudaMemcpyAsync(p->f_stage, f_host, fb, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(p->cov_stage, cov_host, cb, cudaMemcpyHostToDevice, st));
    bsf_status s = bsf_run(p, p->f_stage, p->cov_stage, p->out_stage, stream);
    if (s != BSF_OK) return s;
    CUDA_TRY(cudaMemcpyAsync(out_host, p->out_stage, ob, cudaMemcpyDeviceToHost, st));
    return BSF_OK;
}

extern "C" bsf_status bsf_get_stats(bsf_plan_t p, bsf_stats *s, int reset) {
    if (!p || !s) return set_err(BSF_EINVAL, "null argument");
    DevGuard guard(p->d.device);
    CUDA_TRY(cudaStreamSynchronize(p->last));
    unsigned long long h[8];
    CUDA_TRY(cudaMemcpy(h, p->stats, sizeof h, cudaMemcpyDeviceToHost));
    s->pixels = (long long)h[0];
    s->clamped = (long long)h[1];
    s->zero_scale = (long long)h[2];
    s->theta_prime = (long long)h[3];
    s->flags = (long long)h[4];
    s->double_double = (long long)h[5];
    s->macs = (long long)h[6];
    if (reset) CUDA_TRY(cudaMemset(p->stats, 0, sizeof h));
    if (s->flags & FLAG_RANGE_H) return set_err(BSF_ERANGE, "a tap window left the pre-integration domain");
    if (s->flags & FLAG_INFEASIBLE_H) return set_err(BSF_EINFEASIBLE, "covariance outside the elongation bound");
    return BSF_OK;
}

extern "C" long long bsf_launch_count(bsf_plan_t p) { return p ? p->nlaunch : 0; }

extern "C" bsf_status bsf_debug_phase_cycles(bsf_plan_t p, unsigned long long *out, int reset) {
    if (!p) return set_err(BSF_EINVAL, "null plan");
    DevGuard guard(p->d.device);
    if (!p->prof) {
        void *q;
        CUDA_TRY(cudaMalloc(&q, BSF_PROF_WORDS * sizeof(unsigned long long)));
        p->dev_allocs.push_back(q);
        p->prof = (unsigned long long *)q;
        CUDA_TRY(cudaMemset(q, 0, BSF_PROF_WORDS * sizeof(unsigned long long)));
    }
    if (out) {
        CUDA_TRY(cudaStreamSynchronize(p->last));
        CUDA_TRY(cudaMemcpy(out, p->prof, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    }
    if (reset) CUDA_TRY(cudaMemset(p->prof, 0, BSF_PROF_WORDS * sizeof(unsigned long long)));
    return BSF_OK;
}

extern "C" bsf_status bsf_debug_item_cycles(bsf_plan_t p, unsigned long long *items, unsigned long long *work,
                                            int nitems, unsigned long long *ctas, int nctas) {
    if (!p) return set_err(BSF_EINVAL, "null plan");
    DevGuard guard(p->d.device);
    if (!p->prof) return set_err(BSF_EINVAL, "enable the counters with bsf_debug_phase_cycles first");
    if (nitems < 0 || nctas < 0 || (nitems && !items) || (nctas && !ctas))
        return set_err(BSF_EINVAL, "bad output buffers");
    CUDA_TRY(cudaStreamSynchronize(p->last));
    if (nitems)
        CUDA_TRY(cudaMemcpy(items, p->prof + 16, (size_t)std::min(nitems, BSF_PROF_ITEMS) * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost));
    if (nitems && work)
        CUDA_TRY(cudaMemcpy(work, p->prof + BSF_PROF_WORK,
                            4 * (size_t)std::min(nitems, BSF_PROF_ITEMS) * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost));
    if (nctas)
        CUDA_TRY(cudaMemcpy(ctas, p->prof + 16 + BSF_PROF_ITEMS,
                            (size_t)std::min(nctas, BSF_PROF_CTAS) * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost));
    return BSF_OK;
}

extern "C" int bsf_uses_fused(bsf_plan_t p) { return p && p->fused ? 1 : 0; }

extern "C" bsf_status bsf_debug_option(bsf_plan_t p, const char *name, double value) {
    if (!p || !name) return set_err(BSF_EINVAL, "null argument");
    const std::string n(name);
    if (n == "fused") {
        if (p->fused_ready || p->scratch_ready) return set_err(BSF_EINVAL, "option 'fused' must be set before the first run");
        p->opt_fused = value != 0.0;
    } else if (n == "work_order") {
        p->opt_order = value != 0.0;
    } else if (n == "scan_tma") {  // process-wide: the scans' row streaming (TMA or cp.async)
        set_scan_tma(value != 0.0);
    } else if (n == "global_kernel") {
        p->opt_global_kernel = value != 0.0 ? 1 : 0;
    } else if (n == "i8_tc") {
        p->opt_i8_tc = value != 0.0 ? 1 : 0;
    } else if (n == "gx1_dp4a") {
        p->opt_gx1_dp4a = value != 0.0 ? 1 : 0;
    } else if (n == "split_tol") {
        if (!(value >= 0.0)) return set_err(BSF_EINVAL, "split_tol must be >= 0");
        p->opt_split_tol = value;
    } else {
        return set_err(BSF_EINVAL, "unknown option " + n);
    }
    return BSF_OK;
}

extern "C" const char *bsf_status_str(bsf_status s) {
    switch (s) {
        case BSF_OK: return "ok";
        case BSF_EINVAL: return "invalid argument";
        case BSF_ENOMEM: return "out of memory";
        case BSF_ECUDA: return "CUDA error";
        case BSF_EINFEASIBLE: return "infeasible covariance";
        case BSF_ERANGE: return "kernel reach exceeds plan margins";
        case BSF_ENCCL: return "communication error";
        case BSF_EUNSUPPORTED: return "unsupported";
    }
    return "unknown status";
}

extern "C" const char *bsf_last_error(void) { return g_last_error.c_str(); }
extern "C" int bsf_version(void) { return 100; }
