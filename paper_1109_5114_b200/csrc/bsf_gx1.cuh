// Global-mode gather at order 1: the paper's Algorithm 3 step
// 3 read from the single global pre-integration
// held as exact int64 running sums
// (bsf_preintegrate_exact), one thread per pixel, with an EXACT integer
// contraction of Eq. (11):
//
//   E_mu = sum_s G'(b + o_s) n_{s,mu}        (integers; G' = G or its zero-
//                                             scale lattice difference, R5)
//   F    = (1/L) sum_mu E_mu phi_x^i phi_y^j (double-double Horner)
//   out  = prod_k a'_k^{-1} sum_j c_j F_j    (double-double signed sum)
//
// At order 1 every table numerator n is a small integer (|n| < 2^5, L <= 2^6,
// lut/gen_lut.py) and every sum |G'| < 2^62 (the plan checks it), so the
// running sum is split into three 21-bit limbs G' = 2^42 v2 + 2^21 v1 + v0 and
// each limb is contracted in int32 (|v| n summed over <= 24 window slots stays
// below 2^31): one IMAD per limb and coefficient, no rounding at all before
// the polynomial in phi.  The only rounding is in the double-double Horner and
// signed sum (relative ~u^2 x the cancellation), bounded a posteriori; pixels
// over the bound are recomputed by the double-double per-pixel mesh (never
// observed).
//
// Included by bsf_kernels.cu after bsf_fused.cuh (uses pixel_scales,
// ClsTables / cls_region, comp_step, mesh<>, warp_count).

#ifndef GX1_BLOCK_T
#define GX1_BLOCK_T 256
#endif
constexpr int GX1_BLOCK = GX1_BLOCK_T;   // threads per block
#ifndef GX1_TH_T
#define GX1_TH_T 32
#endif
constexpr int GX1_TW = 32, GX1_TH = GX1_TH_T;  // pixel tile
constexpr int GX1_TILE = GX1_TW * GX1_TH, GX1_PPT = GX1_TILE / GX1_BLOCK;
constexpr size_t GX1_DYN_SMEM = (size_t)GX1_TILE * (4 * sizeof(double) + sizeof(int) + sizeof(short));
extern __shared__ __align__(16) unsigned char gx1_dyn[];
constexpr int GX1_MAXREG = 32;
constexpr int GX1_SLOTS = 2048;          // window slots of all order-1 tables, padded to 4 (Theta 96, Theta' 1800)

// order-1 tables of one (basis, variant) in shared memory
struct Gx1Var {
    int nmax4, base;  // slots per region (padded to 4), first slot of region 0 in the flat arrays
    double invL;
};

struct Gx1Smem {
    ClsTables cls;
    double2 nrm[2][4];                        // the knot-line normals as doubles (no per-tap conversions)
    Gx1Var var[2][NVAR];
    unsigned char cnt[2][NVAR][GX1_MAXREG];   // window slots of the region
    int4 ext[2];                              // window offset extents (wxmin, wxmax, wymin, wymax) per basis
    int vw[2];                                // TileArgs.gvw: two-limb width of the variants (0: three limbs)
    // per (basis, variant, region, slot), flat: the window offset as a linear
    // byte offset 8 (dy GW + dx) into the running sums, and the numerators n_mu
    // (monomials in gen_lut order, int8, padded to 8 bytes); padding slots
    // have offset 0 and zero numerators
    alignas(16) int off[GX1_SLOTS];     // groups of four slots are read as one 16-byte word
    alignas(16) uint2 num[GX1_SLOTS];
};

template <int K>
__device__ __forceinline__ int gx1_byte(unsigned w) {  // signed byte K of w: one PRMT
    // prmt selector nibbles: byte K, then three copies of its sign (K | 8)
    // (PTX prmt default mode; __byte_perm ignores the nibbles' sign bit)
    int r;
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(w), "n"(K | ((8 | K) << 4) | ((8 | K) << 8) | ((8 | K) << 12)));
    return r;
}

// One tap: F(b + phi) for the region's window, exact integer contraction then
// double-double Horner.  NMON = 6 (degree 2, full kernel) or 3 (degree 1,
// zero-scale variant: G' = G(q) - G(q - s_drop), exact).  Gt points at the
// running sum of the tap's lattice base; the pixel's reach was checked against
// the domain (and the buffer has zero rows above it), so no read is bounds
// checked.  Slots go in groups of four with all loads of a group issued before
// its multiply-adds.
// NL = 2 (zero-scale variants where the plan proved it safe, TileArgs.gvw):
// two limbs G' = 2^w v1 + v0, and E_mu (below 2^53) exact as one double.
template <int NMON, bool TOP, int NL = 3>
__device__ __forceinline__ dd gx1_tap(const Gx1Smem &S, const long long *__restrict__ Gt, int b, int v, int reg,
                                      double fx, double fy, int sdl, int row0, int GW, int w = 21) {
    int acc[NL][NMON];
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
        for (int m = 0; m < NMON; ++m) acc[l][m] = 0;
    const int n4 = (S.cnt[b][v][reg] + 3) & ~3;
    const int row = S.var[b][v].base + reg * S.var[b][v].nmax4;
    const int *off = S.off + row;  // byte offsets (8 x element offsets): one 64-bit add per load address
    const char *Gb = reinterpret_cast<const char *>(Gt);
    const char *Gv = reinterpret_cast<const char *>(Gt - sdl);  // the variant's lattice-shifted reads
    const uint2 *num = S.num + row;
    for (int s0 = 0; s0 < n4; s0 += 4) {
        long long g[4];
        // rows start on multiples of four slots: one 16-byte shared load for
        // the group's four offsets, two for its numerators
        const int4 ob4 = *reinterpret_cast<const int4 *>(off + s0);
        const uint4 nwa = *reinterpret_cast<const uint4 *>(num + s0);
        const uint4 nwb = *reinterpret_cast<const uint4 *>(num + s0 + 2);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int ob = i == 0 ? ob4.x : i == 1 ? ob4.y : i == 2 ? ob4.z : ob4.w;
            const long long *p0 = reinterpret_cast<const long long *>(Gb + ob);
            const long long *p1 = reinterpret_cast<const long long *>(Gv + ob);
            if constexpr (TOP) {
                // the tap's window reaches above the domain: zero state there
                // (row of a read = row0 + floor((o + GW/2) / GW), GW > 2 |dx|)
                const int o = ob >> 3;
                const int ry = row0 + (o + (GW >> 1) + 16 * GW) / GW - 16;
                const int ryv = ry - (sdl + (GW >> 1) + 16 * GW) / GW + 16;
                g[i] = ry >= 0 ? __ldg(p0) : 0ll;
                if (NMON == 3) g[i] -= ryv >= 0 ? __ldg(p1) : 0ll;
            } else {
                g[i] = __ldg(p0);
                if (NMON == 3) g[i] -= __ldg(p1);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint2 nw = i == 0 ? make_uint2(nwa.x, nwa.y) : i == 1 ? make_uint2(nwa.z, nwa.w)
                             : i == 2 ? make_uint2(nwb.x, nwb.y) : make_uint2(nwb.z, nwb.w);
            int vl[NL];
            if constexpr (NL == 3) {
                vl[0] = (int)(g[i] & 0x1FFFFF);
                vl[1] = (int)((g[i] >> 21) & 0x1FFFFF);
                vl[NL - 1] = (int)(g[i] >> 42);
            } else {
                vl[0] = (int)(g[i] & ((1ll << w) - 1));
                vl[NL - 1] = (int)(g[i] >> w);
            }
            int cm[6];  // the monomials' numerators, sign-extended (gen_lut order)
            cm[0] = gx1_byte<0>(nw.x);
            cm[1] = gx1_byte<1>(nw.x);
            cm[2] = gx1_byte<2>(nw.x);
            cm[3] = gx1_byte<3>(nw.x);
            cm[4] = gx1_byte<0>(nw.y);
            cm[5] = gx1_byte<1>(nw.y);
#pragma unroll
            for (int m = 0; m < NMON; ++m) {
                const int c = cm[m];
#pragma unroll
                for (int l = 0; l < NL; ++l) acc[l][m] += vl[l] * c;
            }
        }
    }
    // E_mu = 2^21 (2^21 acc2 + acc1) + acc0 as an exact double-double: the
    // bracket is an integer below 2^53 (exact in fp64, times 2^21 exact), and
    // TwoSum is error-free
    dd E[NMON];
#pragma unroll
    for (int m = 0; m < NMON; ++m) {
        if constexpr (NL == 3) {
            const long long hi = ((long long)acc[NL - 1][m] << 21) + acc[1][m];
            E[m] = two_sum((double)hi * 0x1p21, (double)acc[0][m]);
        } else {  // an integer below 2^53: exact (the scaling by 2^w is exact)
            E[m].hi = fma((double)acc[NL - 1][m], (double)(1ll << w), (double)acc[0][m]);
            E[m].lo = 0.0;
        }
    }
    // Horner: rows i (x power) in phi_y, then phi_x; monomial order (i, j):
    // i = deg..0, j = deg - i..0 (lut/gen_lut.py)
    double h, l;
    if constexpr (NMON == 6) {  // (2,0) | (1,1) (1,0) | (0,2) (0,1) (0,0)
        double r1h = E[1].hi, r1l = E[1].lo;
        comp_step(r1h, r1l, fy, E[2].hi, E[2].lo);
        double r0h = E[3].hi, r0l = E[3].lo;
        comp_step(r0h, r0l, fy, E[4].hi, E[4].lo);
        comp_step(r0h, r0l, fy, E[5].hi, E[5].lo);
        h = E[0].hi;
        l = E[0].lo;
        comp_step(h, l, fx, r1h, r1l);
        comp_step(h, l, fx, r0h, r0l);
    } else {  // (1,0) | (0,1) (0,0)
        double r0h = E[1].hi, r0l = E[1].lo;
        comp_step(r0h, r0l, fy, E[2].hi, E[2].lo);
        h = E[0].hi;
        l = E[0].lo;
        comp_step(h, l, fx, r0h, r0l);
    }
    return fast_two_sum(h, l);
}

// The same exact contraction on byte planes with the 4-way int8 dot product
// (IDP.4A): G' = sum_j 2^{8j} B_j with B_0..B_6 unsigned bytes and B_7 the
// signed top byte (two's complement), so
//   E_mu = sum_j 2^{8j} sum_s B_j(G'_s) n_{s,mu},
// and one dp4a takes four window slots of one plane against the four slots'
// numerators of one monomial.  The numerators are staged TRANSPOSED per group
// of four slots (word mu of a group = the four slots' n_mu as int8), so no
// sign extension is needed; the four values' bytes are transposed into eight
// plane words by 16 PRMTs.  Per plane and monomial |sum| <= 255 sum_s |n| <
// 2^18, so the pair p = acc_j + 2^8 acc_{j+1} fits int32 and
// E = 2^32 (p45 + 2^16 p67) + (p01 + 2^16 p23) is exact as a double-double
// (both brackets are integers below 2^53).
__device__ __forceinline__ int gx1_dp4a_us(unsigned a, unsigned b, int c) {  // unsigned a bytes x signed b bytes
    int d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ int gx1_dp4a_ss(unsigned a, unsigned b, int c) {  // signed x signed (top plane)
    int d;
    asm("dp4a.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

template <int NMON, bool TOP>
__device__ __forceinline__ dd gx1_tap_dp(const Gx1Smem &S, const long long *__restrict__ Gt, int b, int v, int reg,
                                         double fx, double fy, int sdl, int row0, int GW) {
    int acc[8][NMON];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int m = 0; m < NMON; ++m) acc[j][m] = 0;
    const int n4 = (S.cnt[b][v][reg] + 3) & ~3;
    const int row = S.var[b][v].base + reg * S.var[b][v].nmax4;
    const int *off = S.off + row;
    const char *Gb = reinterpret_cast<const char *>(Gt);
    const char *Gv = reinterpret_cast<const char *>(Gt - sdl);
    const uint2 *num = S.num + row;  // transposed per group of four slots (gx1_kernel staging)
    for (int s0 = 0; s0 < n4; s0 += 4) {
        long long g[4];
        const int4 ob4 = *reinterpret_cast<const int4 *>(off + s0);
        const uint4 nwa = *reinterpret_cast<const uint4 *>(num + s0);
        uint4 nwb = make_uint4(0u, 0u, 0u, 0u);
        if constexpr (NMON > 4) nwb = *reinterpret_cast<const uint4 *>(num + s0 + 2);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int ob = i == 0 ? ob4.x : i == 1 ? ob4.y : i == 2 ? ob4.z : ob4.w;
            const long long *p0 = reinterpret_cast<const long long *>(Gb + ob);
            const long long *p1 = reinterpret_cast<const long long *>(Gv + ob);
            if constexpr (TOP) {
                const int o = ob >> 3;
                const int ry = row0 + (o + (GW >> 1) + 16 * GW) / GW - 16;
                const int ryv = ry - (sdl + (GW >> 1) + 16 * GW) / GW + 16;
                g[i] = ry >= 0 ? __ldg(p0) : 0ll;
                if (NMON == 3) g[i] -= ryv >= 0 ? __ldg(p1) : 0ll;
            } else {
                g[i] = __ldg(p0);
                if (NMON == 3) g[i] -= __ldg(p1);
            }
        }
        // byte transpose: plane j = byte j of the four values
        unsigned pl[8];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const unsigned w0 = (unsigned)((unsigned long long)g[0] >> (32 * h));
            const unsigned w1 = (unsigned)((unsigned long long)g[1] >> (32 * h));
            const unsigned w2 = (unsigned)((unsigned long long)g[2] >> (32 * h));
            const unsigned w3 = (unsigned)((unsigned long long)g[3] >> (32 * h));
            const unsigned a01 = __byte_perm(w0, w1, 0x5140), a23 = __byte_perm(w2, w3, 0x5140);
            const unsigned b01 = __byte_perm(w0, w1, 0x7362), b23 = __byte_perm(w2, w3, 0x7362);
            pl[4 * h + 0] = __byte_perm(a01, a23, 0x5410);
            pl[4 * h + 1] = __byte_perm(a01, a23, 0x7632);
            pl[4 * h + 2] = __byte_perm(b01, b23, 0x5410);
            pl[4 * h + 3] = __byte_perm(b01, b23, 0x7632);
        }
        const unsigned nw[8] = {nwa.x, nwa.y, nwa.z, nwa.w, nwb.x, nwb.y, nwb.z, nwb.w};
#pragma unroll
        for (int m = 0; m < NMON; ++m) {
#pragma unroll
            for (int j = 0; j < 7; ++j) acc[j][m] = gx1_dp4a_us(pl[j], nw[m], acc[j][m]);
            acc[7][m] = gx1_dp4a_ss(pl[7], nw[m], acc[7][m]);
        }
    }
    dd E[NMON];
#pragma unroll
    for (int m = 0; m < NMON; ++m) {
        const int p01 = acc[0][m] + acc[1][m] * 256, p23 = acc[2][m] + acc[3][m] * 256;
        const int p45 = acc[4][m] + acc[5][m] * 256, p67 = acc[6][m] + acc[7][m] * 256;
        const double lo = fma((double)p23, 0x1p16, (double)p01);  // exact: integers below 2^53
        const double hi = fma((double)p67, 0x1p16, (double)p45);
        E[m] = two_sum(hi * 0x1p32, lo);
    }
    double h, l;
    if constexpr (NMON == 6) {  // (2,0) | (1,1) (1,0) | (0,2) (0,1) (0,0)
        double r1h = E[1].hi, r1l = E[1].lo;
        comp_step(r1h, r1l, fy, E[2].hi, E[2].lo);
        double r0h = E[3].hi, r0l = E[3].lo;
        comp_step(r0h, r0l, fy, E[4].hi, E[4].lo);
        comp_step(r0h, r0l, fy, E[5].hi, E[5].lo);
        h = E[0].hi;
        l = E[0].lo;
        comp_step(h, l, fx, r1h, r1l);
        comp_step(h, l, fx, r0h, r0l);
    } else {  // (1,0) | (0,1) (0,0)
        double r0h = E[1].hi, r0l = E[1].lo;
        comp_step(r0h, r0l, fy, E[2].hi, E[2].lo);
        h = E[0].hi;
        l = E[0].lo;
        comp_step(h, l, fx, r0h, r0l);
    }
    return fast_two_sum(h, l);
}

// The pixel's (r+1)^ns = 2^ns taps (Table 1, generalised to
// both bases; shift of Eq. (10) absorbed in the uncentred interpolant, DESIGN.md
// R3): D_j = sum_k (1/2 - j_k) a'_k s_k, sign (-1)^{sum j}.
template <int NMON, bool DP>
__device__ __forceinline__ double gx1_mesh(const Gx1Smem &S, const long long *__restrict__ G, int GW, int P,
                                           int b, int drop, const double *apm, int x, int y, double &erel,
                                           unsigned int &macs) {
    // apm: the pixel's scales a'_k in shared memory (read at each step, not
    // held in registers across the tap loop)
    const int v = drop + 1;
    const int ns = drop < 0 ? 4 : 3;
    auto dir = [&](int q) { return q + (drop >= 0 && q >= drop ? 1 : 0); };  // q-th direction in use
    // v_k = s_k a'_k and the centre sum_k v_k / 2 (exact on the 2^-41 grid, R17)
    double cx = 0.0, cy = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (q < ns) {
            const int k = dir(q);
            cx += 0.5 * (c_steps[b][k][0] * apm[k]);
            cy += 0.5 * (c_steps[b][k][1] * apm[k]);
        }
    }
    const int sdl = v ? c_steps[b][v - 1][1] * GW + c_steps[b][v - 1][0] : 0;
    const int wymin = S.ext[b].z;
    const int ntap = 1 << ns;
    double h0 = 0.0, e0 = 0.0, sumF = 0.0;
    // taps in Gray-code order: consecutive taps differ in one digit j_q, so
    // the displacement D moves by one exact step (R17: every value on the
    // 2^-41 grid) and phi = D - floor(D) is exact.  The region key
    // floor(n_m . phi) (cls_region's) is formed per tap from phi (exact:
    // |n_m| <= 2), the normals read from shared memory, so no per-line state
    // lives across the taps
    double Dx = cx, Dy = cy;
    int sgn = 1;
    for (int t = 0; t < ntap; ++t) {
        if (t > 0) {  // Gray step: digit q = ctz(t) flips to (gray(t) >> q) & 1
            const int q = __ffs(t) - 1;
            const bool on = ((t ^ (t >> 1)) >> q) & 1;
            const int k = dir(q);
            const double ak = apm[k];
            const double dx = c_steps[b][k][0] * ak, dy = c_steps[b][k][1] * ak;  // v_q, as at the centre
            Dx = on ? Dx - dx : Dx + dx;  // exact
            Dy = on ? Dy - dy : Dy + dy;
            sgn = -sgn;
        }
        const double flx = floor(Dx), fly = floor(Dy);
        const double fx = Dx - flx, fy = Dy - fly;  // exact
        const int ix = (int)flx, iy = (int)fly;
        int idx = 0, mul = 1;
        bool in = true;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const double2 nm = S.nrm[b][m];
            const int rxm = S.cls.radix[b][m];
            const int f = (int)floor(nm.x * fx + nm.y * fy) - S.cls.kmin[b][m];  // n_m . phi: exact
            in = in && f >= 0 && f < rxm;
            idx += f * mul;
            mul *= rxm;
        }
        int reg = in ? S.cls.table[b][idx] : -1;
        if (reg < 0) reg = cls_region(S.cls, b, fx, fy);  // exactly on a knot line
        const int by = y + iy;
        const long long *Gt = G + ((ptrdiff_t)by * GW + (x + ix + P));
        // windows that reach above row 0 read the zero state there (checked
        // loads); all other reads are inside the domain (reach checked)
        dd F;
        const int vw = NMON == 3 ? S.vw[b] : 0;
        // DP: byte-plane dp4a contraction on the transposed tables (full
        // taps, and variants without the two-limb form); see gx1_kernel staging
        if (DP && !(NMON == 3 && vw)) {
            if (by + wymin - 2 < 0)
                F = gx1_tap_dp<NMON, true>(S, Gt, b, v, reg, fx, fy, sdl, by, GW);
            else
                F = gx1_tap_dp<NMON, false>(S, Gt, b, v, reg, fx, fy, sdl, by, GW);
        } else if (by + wymin - 2 < 0)
            F = gx1_tap<NMON, true>(S, Gt, b, v, reg, fx, fy, sdl, by, GW);
        else if (NMON == 3 && vw)
            F = gx1_tap<NMON, false, 2>(S, Gt, b, v, reg, fx, fy, sdl, by, GW, vw);
        else
            F = gx1_tap<NMON, false>(S, Gt, b, v, reg, fx, fy, sdl, by, GW);
        macs += S.cnt[b][v][reg] * NMON;  // algorithmic: window x monomials
        // compensated signed sum: TwoSum on the heads, small terms in e0
        const double fh = sgn > 0 ? F.hi : -F.hi, fl = sgn > 0 ? F.lo : -F.lo;
        const dd s = two_sum(h0, fh);
        h0 = s.hi;
        e0 += s.lo + fl;
        sumF += fabs(F.hi);
    }
    const dd Ssum = fast_two_sum(h0, e0);
    double den = 1.0;  // prod_k a'_k over the directions in use (one division below)
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (q < ns) den *= apm[dir(q)];
    const double norm = S.var[b][v].invL / den;  // 1 / (L prod a'_k)
    const double Sd = dd_to_d(Ssum);
    // rounding of the Horner steps and of the sum: (2 ntap + 8) u^2 sum_j |F_j|
    erel = 2.5e-30 * (double)(2 * ntap + 8) * sumF / fabs(Sd);
    return Sd * norm;
}

// the double-double fallback, out of line (rarely taken: keeps the main
// path's register allocation small)
__device__ __noinline__ double gx1_fallback(const long long *G, int P, int GW, int GH, const LutBasis &L,
                                            const PixelScales &ps, int x, int y, int *flags) {
    GView gv = {nullptr, -P, 0, GW, GH, 0.0};
    gv.gi = G;
    return mesh<1, true>(gv, L, ps, x, y, flags);
}

#ifndef GX1_MINB
#define GX1_MINB 2
#endif
template <bool DP>
__global__ void __launch_bounds__(GX1_BLOCK, GX1_MINB) gx1_kernel(TileArgs a, const LutBasis *__restrict__ luts) {
    __shared__ Gx1Smem S;
    const int tid = threadIdx.x;
    // stage the classifier and the order-1 integer tables of both bases
    if (tid < 2) {
        const LutBasis &L = luts[tid];
        for (int k = 0; k < 4; ++k) {
            S.cls.normal[tid][k] = L.normal[k];
            S.nrm[tid][k] = make_double2(L.normal[k].x, L.normal[k].y);
            S.cls.kmin[tid][k] = L.kmin[k];
            S.cls.radix[tid][k] = L.radix[k];
        }
        for (int i = 0; i < 81; ++i) S.cls.table[tid][i] = L.table[i];
    }
    int base = 0;  // the host checked that the tables in use fit GX1_SLOTS / GX1_MAXREG
    for (int bv = 0; bv < 2 * NVAR; ++bv) {
        const int b = bv / NVAR, v = bv % NVAR;
        if (!a.gglob[b]) continue;  // basis not in the plan
        const LutVar &V = luts[b].var[v];
        const int nreg = luts[b].nreg;
        const int nmax4 = (V.nmax + 3) & ~3;
        if (tid == 0) S.var[b][v] = Gx1Var{nmax4, base, 1.0 / V.L};
        if (tid == 0 && v == 0) S.ext[b] = make_int4(luts[b].wxmin, luts[b].wxmax, luts[b].wymin, luts[b].wymax);
        if (tid == 0 && v == 0) S.vw[b] = a.gvw[b];
        for (int i = tid; i < nreg; i += GX1_BLOCK) S.cnt[b][v][i] = (unsigned char)__ldg(V.counts + i);
        for (int i = tid; i < nreg * nmax4; i += GX1_BLOCK) {
            const int r = i / nmax4, sl = i % nmax4;
            const bool real = sl < __ldg(V.counts + r);
            const int2 o = real ? __ldg(V.offs + r * V.nmax + sl) : make_int2(0, 0);
            S.off[base + i] = 8 * (o.y * a.gGW + o.x);  // bytes
            const uint2 nv = real ? __ldg(reinterpret_cast<const uint2 *>(V.n8) + r * V.nmax + sl) : make_uint2(0u, 0u);
            if (DP && (v == 0 || !a.gvw[b])) {
                // transposed per group of four slots (rows start on multiples
                // of four): byte 4 mu + (slot & 3) of the group holds n_mu
                unsigned char *g8 = reinterpret_cast<unsigned char *>(S.num + ((base + i) & ~3));
                const int q = (base + i) & 3;
#pragma unroll
                for (int m = 0; m < 8; ++m)
                    g8[4 * m + q] = (unsigned char)((m < 4 ? nv.x >> (8 * m) : nv.y >> (8 * (m - 4))) & 0xFFu);
            } else {
                S.num[base + i] = nv;
            }
        }
        base += nreg * nmax4;
    }
    __syncthreads();
    // tiles of the output row window (a band of rows, bsf_run_host's pipeline;
    // all rows when oH = 0); the window starts on a multiple of GX1_TH
    const int ty0 = a.oy0 / GX1_TH;
    const int ntx = (a.W + GX1_TW - 1) / GX1_TW, nty = (min(a.H, a.oy0 + out_rows(a)) + GX1_TH - 1) / GX1_TH - ty0;
    const long long nunits = a.pts ? ((long long)a.npts + GX1_TILE - 1) / GX1_TILE : (long long)ntx * nty * a.nimg;
    unsigned long long macs = 0;
    // per tile of GX1_TILE pixels: phase A solves every pixel's scales
    // (a1-a4, GX1_PPT pixels per thread); a counting sort orders the pixels
    // by class (basis, zero-scale variant), most expensive class first, dead
    // pixels last; in phase B the warps take groups of 32 consecutive sorted
    // pixels from a block counter, so a warp mostly runs ONE tap program (same
    // tap count, same tables: lanes of mixed classes would run both programs
    // one after the other) and the expensive groups are handed out first
    // (the block's warps finish together at the tile barrier)
    constexpr int NCLS = 2 * NVAR + 1, NPAIR = GX1_PPT * (GX1_BLOCK / 32);
    static_assert(NPAIR <= 32, "one lane per (round, warp) pair in the class scan");
    double(*s_ap)[4] = reinterpret_cast<double(*)[4]>(gx1_dyn);
    int *s_info = reinterpret_cast<int *>(s_ap + GX1_TILE);  // basis | (drop+1) << 1 | clamped << 4 | valid << 5 | flags << 8
    short *s_order = reinterpret_cast<short *>(s_info + GX1_TILE);
    __shared__ int s_pcnt[NPAIR][NCLS];  // class counts per (round, warp), then exclusive offsets
    __shared__ int s_next;
    const int lane = tid & 31, warp = tid >> 5;
    // static grid-stride over 32 x 32 pixel tiles in raster order: the blocks of
    // a wave read neighbouring rows of the running sums (L2 reuse of the taps)
    for (long long u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int img_t = a.pts ? 0 : (int)(u / ((long long)ntx * nty));
        const int rem_t = a.pts ? 0 : (int)(u % ((long long)ntx * nty));
        const int x0 = (rem_t % ntx) * GX1_TW, y0 = (ty0 + rem_t / ntx) * GX1_TH;
        if (tid == 0) s_next = 0;
        // ---- phase A: pixels tid + GX1_BLOCK k of the tile
#pragma unroll 1
        for (int k = 0; k < GX1_PPT; ++k) {
            const int e = tid + GX1_BLOCK * k;
            int img, x, y;
            bool valid;
            if (a.pts) {
                const long long i = u * GX1_TILE + e;
                valid = i < a.npts;
                img = valid ? a.pts[3 * i] : 0;
                x = valid ? a.pts[3 * i + 1] : 0;
                y = valid ? a.pts[3 * i + 2] : 0;
            } else {
                img = img_t;
                x = x0 + e % GX1_TW;
                y = y0 + e / GX1_TW;
                valid = x < a.W && out_row(a, y);
            }
            PixelScales ps;
            ps.flags = 0;
            ps.basis = 0;
            ps.drop = -1;
            ps.clamped = 0;
            ps.ap[0] = ps.ap[1] = ps.ap[2] = ps.ap[3] = 0.0;
            if (valid) {
                double sx, sy, th;
                load_cov(a, img, x, y, sx, sy, th);
                pixel_scales(sx, sy, th, a.policy, a.clamp, 1, ps);
            }
            const bool live = valid && !(ps.flags & (FLAG_INFEASIBLE | FLAG_TWO_ZERO));
#pragma unroll
            for (int q = 0; q < 4; ++q) s_ap[e][q] = ps.ap[q];
            s_info[e] = ps.basis | ((ps.drop + 1) << 1) | (ps.clamped << 4) | (valid ? 32 : 0) | (ps.flags << 8);
            // class rank, most expensive first: Theta' full, Theta full,
            // Theta' variants, Theta variants, dead
            const int cls = !live ? NCLS - 1
                                  : ps.drop < 0 ? (ps.basis == BASIS_THETA_PRIME ? 0 : 1)
                                                : 2 + (ps.basis == BASIS_THETA_PRIME ? 0 : 4) + ps.drop;
            const unsigned m = __match_any_sync(0xffffffffu, cls);
            const int pair = k * (GX1_BLOCK / 32) + warp;
            if (lane < NCLS) s_pcnt[pair][lane] = 0;
            __syncwarp();
            if (lane == __ffs(m) - 1) s_pcnt[pair][cls] = __popc(m);
            s_order[e] = (short)(cls | (__popc(m & ((1u << lane) - 1u)) << 4));  // class, rank in the warp
        }
        __syncthreads();
        // exclusive offsets: class bases (in class-rank order) + earlier pairs
        if (warp == 0) {
            int run = 0;
#pragma unroll 1
            for (int c = 0; c < NCLS; ++c) {
                const int v = lane < NPAIR ? s_pcnt[lane][c] : 0;
                int inc = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += t;
                }
                if (lane < NPAIR) s_pcnt[lane][c] = run + inc - v;
                run += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
        __syncthreads();
        short slot[GX1_PPT];
#pragma unroll
        for (int k = 0; k < GX1_PPT; ++k) {
            const int e = tid + GX1_BLOCK * k;
            const int w = s_order[e];
            slot[k] = (short)(s_pcnt[k * (GX1_BLOCK / 32) + warp][w & 15] + (w >> 4));
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < GX1_PPT; ++k) s_order[slot[k]] = (short)(tid + GX1_BLOCK * k);
        __syncthreads();
        // ---- phase B: groups of 32 sorted pixels from the block counter
        for (;;) {
            int grp = 0;
            if (lane == 0) grp = atomicAdd(&s_next, 1);
            grp = __shfl_sync(0xffffffffu, grp, 0);
            if (grp >= GX1_TILE / 32) break;
            const int p = s_order[32 * grp + lane];
            const int w = s_info[p];
            const bool valid = (w >> 5) & 1;
            // the scales stay in shared memory (s_ap[p]): re-read where used,
            // not held in registers across the tap loop
            const int basis = w & 1, drop = ((w >> 1) & 7) - 1;
            int img, x, y;
            long long oidx;
            if (a.pts) {
                const long long i = u * GX1_TILE + p;
                img = valid ? a.pts[3 * i] : 0;
                x = valid ? a.pts[3 * i + 1] : 0;
                y = valid ? a.pts[3 * i + 2] : 0;
                oidx = i;
            } else {
                img = img_t;
                x = x0 + p % GX1_TW;
                y = y0 + p / GX1_TW;
                oidx = out_index(a, img, x, y);
            }
            int flags = w >> 8;
            const bool live = valid && !(flags & (FLAG_INFEASIBLE | FLAG_TWO_ZERO));
            double res = __longlong_as_double(0x7ff8000000000000LL), erel = 0.0;
            bool used_dd = false;
            if (live) {
                // every read stays inside the domain when the pixel's reach is
                // within the plan's margins; else NaN and BSF_ERANGE (a
                // covariance above the plan's max_sigma)
                double rx = 0.0, ry = 0.0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    rx += s_ap[p][k] * abs(c_steps[basis][k][0]);
                    ry += s_ap[p][k] * c_steps[basis][k][1];
                }
                const int ex = (int)ceil(0.5 * rx) + 1, ey = (int)ceil(0.5 * ry) + 1;
                const int4 E = S.ext[basis];
                const bool in = x + a.gP - ex + E.x - 2 >= 0 && x + a.gP + ex + E.y + 2 < a.gGW &&
                                y + ey + E.w < a.gGHv;
                if (!in) {
                    flags |= FLAG_RANGE;
                } else {
                    const long long *G = a.gglob[basis] + (size_t)img * a.gGH * a.gGW;
                    unsigned int pm = 0;
                    res = drop < 0 ? gx1_mesh<6, DP>(S, G, a.gGW, a.gP, basis, drop, s_ap[p], x, y, erel, pm)
                                   : gx1_mesh<3, DP>(S, G, a.gGW, a.gP, basis, drop, s_ap[p], x, y, erel, pm);
                    macs += pm;
                    if (!(erel <= a.split_tol)) {  // NaN-safe: the double-double mesh on the same sums
                        PixelScales ps;
                        ps.basis = basis;
                        ps.drop = drop;
                        ps.clamped = (w >> 4) & 1;
                        ps.flags = w >> 8;
#pragma unroll
                        for (int q = 0; q < 4; ++q) ps.ap[q] = s_ap[p][q];
                        res = gx1_fallback(G, a.gP, a.gGW, a.gGH, luts[basis], ps, x, y, &flags);
                        used_dd = true;
                    }
                }
            }
            if (valid) {
                if (a.aux) {
                    double *ax = a.aux + BSF_AUX * oidx;
                    ax[0] = basis;
                    ax[1] = drop;
                    ax[2] = (w >> 4) & 1;
                    ax[3] = flags;
                    for (int k = 0; k < 4; ++k) ax[4 + k] = s_ap[p][k];
                    ax[8] = used_dd;
                    ax[9] = erel;
                    ax[10] = ax[11] = 0.0;
                }
                if (a.out_f32 && !a.pts)
                    ((float *)a.out)[oidx] = (float)res;
                else
                    ((double *)a.out)[oidx] = res;
            }
            if (a.stats) {
                warp_count(a.stats + 0, valid);
                warp_count(a.stats + 1, valid && ((w >> 4) & 1));
                warp_count(a.stats + 2, valid && drop >= 0);
                warp_count(a.stats + 3, valid && basis == BASIS_THETA_PRIME);
                warp_count(a.stats + 5, used_dd);
                if (valid && flags) atomicOr(a.stats + 4, (unsigned long long)flags);
            }
        }
        __syncthreads();  // s_ap / s_info / s_order / s_next are rewritten by the next tile
    }
    if (a.stats) {
        for (int o = 16; o; o >>= 1) macs += __shfl_xor_sync(0xffffffffu, macs, o);
        if ((tid & 31) == 0 && macs) atomicAdd(a.stats + 6, macs);
    }
}

int gx1_slots() {
    int dev = 0, sms = 148, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gx1_kernel<false>, GX1_BLOCK, GX1_DYN_SMEM) != cudaSuccess ||
        per < 1)
        per = 1;
    return sms * per;
}

cudaError_t launch_gx1(const TileArgs &a, cudaStream_t st, const LutBasis *luts, long long *nl) {
    static std::atomic<unsigned long long> attr[2] = {{0ull}, {0ull}};
    cudaError_t e = a.gdp4a ? set_smem_attr(gx1_kernel<true>, (int)GX1_DYN_SMEM, attr[1])
                            : set_smem_attr(gx1_kernel<false>, (int)GX1_DYN_SMEM, attr[0]);
    if (e != cudaSuccess) return e;
    static int slots = 0;
    if (!slots) slots = gx1_slots();
    if (a.gdp4a)
        gx1_kernel<true><<<slots, GX1_BLOCK, GX1_DYN_SMEM, st>>>(a, luts);
    else
        gx1_kernel<false><<<slots, GX1_BLOCK, GX1_DYN_SMEM, st>>>(a, luts);
    ++*nl;
    return cudaGetLastError();
}
