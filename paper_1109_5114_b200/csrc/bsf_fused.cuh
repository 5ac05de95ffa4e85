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

constexpr int FT = 256;                       // threads per CTA = pixels per tile
constexpr int NKEY = 2 * NVAR * MAX_REG;      // (basis, variant, region)
constexpr int NPLANE = 2 * NVAR;              // (basis, variant)
constexpr uint16_t NOKEY = 0xFFFF;

template <int R> struct FusedCfg;
template <> struct FusedCfg<1> { static constexpr int NTAP = 16, P = 256; };
template <> struct FusedCfg<2> { static constexpr int NTAP = 81, P = 64; };
template <> struct FusedCfg<3> { static constexpr int NTAP = 256, P = 16; };
template <> struct FusedCfg<4> { static constexpr int NTAP = 625, P = 8; };

template <int R>
constexpr size_t fused_smem_bytes() {
    constexpr size_t ITEMS = (size_t)FusedCfg<R>::P * FusedCfg<R>::NTAP;
    return ITEMS * 16 + FT * 4 * 8 + ITEMS * 2 + (ITEMS + 16 * NKEY) * 2 + 2 * NKEY * 4 + FT * 4;
}

// pixel info word: bit0 basis, bits1-3 variant (drop + 1), bit4 live, bit5 clamped, bits 8.. flags
__device__ __forceinline__ int info_basis(int w) { return w & 1; }
__device__ __forceinline__ int info_var(int w) { return (w >> 1) & 7; }
__device__ __forceinline__ bool info_live(int w) { return (w >> 4) & 1; }

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
        coef *= binom_small(R, j) * ((j & 1) ? -1 : 1);
        double m = 0.5 * R - j;
        Dx += (m * c_steps[basis][k][0]) * ap[k];
        Dy += (m * c_steps[basis][k][1]) * ap[k];
    }
}

// One chunk of rows [IHI .. ILO] of the contraction + compensated Horner.
template <int DEG, int IHI>
__device__ __forceinline__ void fused_chunk(const double2 *__restrict__ G, int NX, int NY, int bx, int by,
                                            const int2 *__restrict__ offs, const double *__restrict__ num, int nmonp,
                                            int n, double fx, double fy, double &ah, double &al, int &flags) {
    constexpr int ILO = bsf_chunk_lo(DEG, IHI);
    constexpr int NM = bsf_chunk_len(DEG, IHI);
    constexpr int NMP = (NM + 1) & ~1;
    constexpr int OFF = bsf_chunk_off(DEG, IHI);
    double A[NMP], B[NMP];
#pragma unroll
    for (int m = 0; m < NMP; ++m) {
        A[m] = 0.0;
        B[m] = 0.0;
    }
#pragma unroll 2
    for (int s = 0; s < n; ++s) {
        const int2 d = __ldg(offs + s);
        const int lx = bx + d.x, ly = by + d.y;
        double2 g = make_double2(0.0, 0.0);
        if (ly >= 0) {  // above the domain: zero state
            if (lx >= 0 && lx < NX && ly < NY)
                g = G[(size_t)ly * NX + lx];
            else
                flags |= FLAG_RANGE;
        }
        const double2 *c = reinterpret_cast<const double2 *>(num + (size_t)s * nmonp + OFF);
#pragma unroll
        for (int m = 0; m < NMP / 2; ++m) {
            const double2 cc = __ldg(c + m);
            A[2 * m] = fma(g.x, cc.x, A[2 * m]);  // exact: integers below 2^53
            B[2 * m] = fma(g.y, cc.x, B[2 * m]);
            A[2 * m + 1] = fma(g.x, cc.y, A[2 * m + 1]);
            B[2 * m + 1] = fma(g.y, cc.y, B[2 * m + 1]);
        }
    }
#pragma unroll
    for (int i = IHI; i >= ILO; --i) {
        const int base = bsf_row_start(DEG, i) - bsf_row_start(DEG, IHI);
        double rh = 0.0, rl = 0.0;
#pragma unroll
        for (int j = DEG - i; j >= 0; --j) {
            const int m = base + (DEG - i - j);
            const dd E = two_sum(A[m], B[m]);
            if (j == DEG - i) {
                rh = E.hi;
                rl = E.lo;
            } else {
                comp_step(rh, rl, fy, E.hi, E.lo);
            }
        }
        if (i == DEG) {
            ah = rh;
            al = rl;
        } else {
            comp_step(ah, al, fx, rh, rl);
        }
    }
    if constexpr (ILO > 0)
        fused_chunk<DEG, ILO - 1>(G, NX, NY, bx, by, offs, num, nmonp, n, fx, fy, ah, al, flags);
}

template <int DEG>
__device__ __forceinline__ void fused_item(const double2 *__restrict__ G, int NX, int NY, int bx, int by,
                                           const LutVar &V, int reg, double fx, double fy, double &Fh, double &Fl,
                                           int &flags) {
    const int n = __ldg(V.counts + reg);
    fused_chunk<DEG, DEG>(G, NX, NY, bx, by, V.offs + (size_t)reg * V.nmax, V.num + (size_t)reg * V.nmax * V.nmonp,
                          V.nmonp, n, fx, fy, Fh, Fl, flags);
}

template <int R>
__global__ void __launch_bounds__(FT, 1) fused_kernel(TileArgs a, const LutBasis *__restrict__ luts) {
    constexpr int NTAP = FusedCfg<R>::NTAP, P = FusedCfg<R>::P, ITEMS = P * NTAP;
    extern __shared__ __align__(16) unsigned char smem[];
    double2 *s_F = reinterpret_cast<double2 *>(smem);
    double *s_ap = reinterpret_cast<double *>(s_F + ITEMS);
    uint16_t *s_key = reinterpret_cast<uint16_t *>(s_ap + FT * 4);
    uint16_t *s_sorted = s_key + ITEMS;
    int *s_cnt = reinterpret_cast<int *>(s_sorted + ITEMS + 16 * NKEY);
    int *s_start = s_cnt + NKEY;
    int *s_info = s_start + NKEY;
    __shared__ int s_item, s_ex[2], s_ey[2], s_vmask[2], s_bad, s_npad, s_any;
    __shared__ int s_dom[2][4];
    __shared__ long long s_poff[NPLANE];
    __shared__ int s_pe[NPLANE];
    __shared__ unsigned long long s_pmax[NPLANE];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double2 *scr = a.scratch + (size_t)blockIdx.x * NPLANE * a.cap;
    const int tiles_per_img = a.ntx * a.nty;
    const int nitems = a.pts ? a.npts : tiles_per_img * a.nimg;
    const size_t ipl = (size_t)a.H * a.W;

    for (;;) {
        if (tid == 0) {
            s_item = atomicAdd(a.counter, 1);
            s_ex[0] = s_ex[1] = s_ey[0] = s_ey[1] = 0;
            s_vmask[0] = s_vmask[1] = 0;
            s_bad = 0;
        }
        if (tid < NPLANE) s_pmax[tid] = 0ull;
        __syncthreads();
        const int item = s_item;
        if (item >= nitems) break;
        int img, x0, y0, want = -1;
        if (a.pts) {
            img = a.pts[3 * item];
            const int px = a.pts[3 * item + 1], py = a.pts[3 * item + 2];
            x0 = px & ~(TILE - 1);
            y0 = py & ~(TILE - 1);
            want = (px - x0) + TILE * (py - y0);
        } else {
            img = item / tiles_per_img;
            const int rem = item % tiles_per_img;
            x0 = (rem % a.ntx) * TILE;
            y0 = (rem / a.ntx) * TILE;
        }

        // ---- 1. per-pixel scales ------------------------------------------------
        {
            const int x = x0 + (tid % TILE), y = y0 + tid / TILE;
            PixelScales ps;
            ps.flags = 0;
            ps.basis = 0;
            ps.drop = -1;
            ps.clamped = 0;
            ps.ap[0] = ps.ap[1] = ps.ap[2] = ps.ap[3] = 0.0;
            const bool valid = x < a.W && y < a.H;
            if (valid) {
                const float *cv = a.cov + (size_t)(img / a.channels) * 3 * ipl + (size_t)y * a.W + x;
                pixel_scales(__ldg(cv), __ldg(cv + ipl), __ldg(cv + 2 * ipl), a.policy, a.clamp, R, ps);
            }
            const bool live = valid && !(ps.flags & (FLAG_INFEASIBLE | FLAG_TWO_ZERO));
            const int var = ps.drop + 1;
            s_info[tid] = ps.basis | (var << 1) | (live ? 16 : 0) | (ps.clamped ? 32 : 0) | (ps.flags << 8);
#pragma unroll
            for (int k = 0; k < 4; ++k) s_ap[tid * 4 + k] = ps.ap[k];
            if (live) {
                double ex = 0.0, ey = 0.0;
                for (int k = 0; k < 4; ++k) {
                    ex += ps.ap[k] * abs(c_steps[ps.basis][k][0]);
                    ey += ps.ap[k] * c_steps[ps.basis][k][1];
                }
                atomicMax(&s_ex[ps.basis], (int)ceil(0.5 * R * ex));
                atomicMax(&s_ey[ps.basis], (int)ceil(0.5 * R * ey));
                atomicOr(&s_vmask[ps.basis], 1 << var);
            }
        }
        __syncthreads();

        // ---- 2. pre-integration planes ------------------------------------------
        if (tid == 0) {
            int np = 0;
            for (int b = 0; b < 2; ++b) {
                TileDomain d = tile_domain(luts[b], R, x0, y0, s_ex[b], s_ey[b]);
                s_dom[b][0] = d.X0;
                s_dom[b][1] = d.Y0;
                s_dom[b][2] = d.NX;
                s_dom[b][3] = d.NY;
                for (int v = 0; v < NVAR; ++v) {
                    bool need = (s_vmask[b] >> v) & 1;
                    if (v == 0 && s_vmask[b]) need = true;  // the base plane feeds the variants
                    s_poff[b * NVAR + v] = need ? (long long)(np++) * a.cap : -1;
                }
                if (s_vmask[b] && (long long)d.NX * d.NY > a.cap) s_bad = 1;
            }
        }
        __syncthreads();
        if (s_bad) {
            // domain exceeds the plan's capacity: flag every pixel (cannot happen
            // when max_sigma bounds the covariance field)
            const int x = x0 + (tid % TILE), y = y0 + tid / TILE;
            const bool mine = a.pts ? (tid == want) : (x < a.W && y < a.H);
            if (mine) {
                const long long oidx = a.pts ? item : (long long)img * ipl + (size_t)y * a.W + x;
                if (a.out_f32 && !a.pts)
                    ((float *)a.out)[oidx] = __int_as_float(0x7fc00000);
                else
                    ((double *)a.out)[oidx] = __longlong_as_double(0x7ff8000000000000LL);
                if (a.stats) atomicOr(a.stats + 4, (unsigned long long)FLAG_RANGE);
            }
            __syncthreads();
            continue;
        }
        for (int b = 0; b < 2; ++b) {
            if (!s_vmask[b]) continue;
            const int X0 = s_dom[b][0], Y0 = s_dom[b][1], NX = s_dom[b][2], NY = s_dom[b][3];
            double2 *G = scr + s_poff[b * NVAR];
            const int n = NX * NY;
            for (int i = tid; i < n; i += FT) {
                const int X = X0 + i % NX, Y = Y0 + i / NX;
                double v = 0.0;
                if (X >= 0 && X < a.W && Y >= 0 && Y < a.H) {
                    const size_t o = (size_t)img * ipl + (size_t)Y * a.W + X;
                    v = a.in_u8 ? (double)((const uint8_t *)a.f)[o] : (double)((const float *)a.f)[o];
                }
                G[i] = make_double2(v, 0.0);
            }
            __syncthreads();
            for (int rep = 0; rep < R; ++rep)
                for (int lv = 0; lv < 4; ++lv) {
                    tile_scan_level(G, NX, NY, c_scan_order[b][lv][0], c_scan_order[b][lv][1]);
                    __syncthreads();
                }
            // zero-scale variants: G' = (1 - T_{s_k})^R G, exact lattice difference (R5)
            for (int v = 1; v < NVAR; ++v) {
                if (!((s_vmask[b] >> v) & 1)) continue;
                const int sx = c_steps[b][v - 1][0], sy = c_steps[b][v - 1][1];
                double2 *D = scr + s_poff[b * NVAR + v];
                for (int i = tid; i < n; i += FT) {
                    const int X = i % NX, Y = i / NX;
                    dd acc = {0.0, 0.0};
#pragma unroll
                    for (int m = 0; m <= R; ++m) {
                        const int yy = Y - m * sy, xx = X - m * sx;
                        if (yy < 0 || xx < 0 || xx >= NX) continue;
                        const double2 t = G[(size_t)yy * NX + xx];
                        const int cb = binom_small(R, m) * ((m & 1) ? -1 : 1);
                        acc = dd_add(acc, dd_mul_d({t.x, t.y}, (double)cb));
                    }
                    D[i] = make_double2(acc.hi, acc.lo);
                }
            }
        }
        __syncthreads();

        // ---- 3. exact split G = 2^e (G1 + G0) of every plane that is read --------
        for (int pi = 0; pi < NPLANE; ++pi) {
            const int b = pi / NVAR, v = pi % NVAR;
            if (!((s_vmask[b] >> v) & 1)) continue;
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
            s_pe[tid] = m > 0.0 ? ilogb(m) + 1 - luts[b].var[v].kbits : 0;
        }
        __syncthreads();
        for (int pi = 0; pi < NPLANE; ++pi) {
            const int b = pi / NVAR, v = pi % NVAR;
            if (!((s_vmask[b] >> v) & 1)) continue;
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

        // ---- 4-5. taps bucketed by key, gather, per-pixel sums -------------------
        for (int c0 = 0; c0 < FT; c0 += P) {
            if (tid == 0) s_any = 0;
            __syncthreads();
            if (tid >= c0 && tid < c0 + P && info_live(s_info[tid]) && (!a.pts || tid == want)) s_any = 1;
            for (int k = tid; k < NKEY; k += FT) s_cnt[k] = 0;
            __syncthreads();
            if (!s_any) continue;  // uniform
            // keys
            for (int i = tid; i < ITEMS; i += FT) {
                const int p = c0 + i / NTAP, t = i % NTAP;
                const int w = s_info[p];
                uint16_t key = NOKEY;
                const int var = info_var(w);
                const int ntap = var ? NTAP / (R + 1) : NTAP;
                if (info_live(w) && (!a.pts || p == want) && t < ntap) {
                    const int b = info_basis(w);
                    double Dx, Dy;
                    int cf;
                    fused_tap<R>(s_ap + 4 * p, b, var - 1, t, Dx, Dy, cf);
                    const double fx = Dx - floor(Dx), fy = Dy - floor(Dy);
                    const int reg = classify(luts[b], fx, fy);
                    key = (uint16_t)((b * NVAR + var) * MAX_REG + reg);
                    atomicAdd(&s_cnt[key], 1);
                }
                s_key[i] = key;
            }
            __syncthreads();
            // bucket starts, each bucket padded to a multiple of 16 (warp 0)
            if (warp == 0) {
                constexpr int PER = NKEY / 32;
                int loc = 0;
#pragma unroll
                for (int q = 0; q < PER; ++q) loc += (s_cnt[lane * PER + q] + 15) & ~15;
                int inc = loc;
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += t;
                }
                int run = inc - loc;
#pragma unroll
                for (int q = 0; q < PER; ++q) {
                    s_start[lane * PER + q] = run;
                    run += (s_cnt[lane * PER + q] + 15) & ~15;
                    s_cnt[lane * PER + q] = 0;
                }
                if (lane == 31) s_npad = inc;
            }
            __syncthreads();
            const int npad = s_npad;
            for (int i = tid; i < npad; i += FT) s_sorted[i] = NOKEY;
            __syncthreads();
            for (int i = tid; i < ITEMS; i += FT) {
                const uint16_t key = s_key[i];
                if (key != NOKEY) s_sorted[s_start[key] + atomicAdd(&s_cnt[key], 1)] = (uint16_t)i;
            }
            __syncthreads();
            // gather: half-warp groups of 16 items sharing one key
            {
                const int ngroups = npad >> 4, npairs = (ngroups + 1) >> 1, half = lane >> 4;
                int flags = 0;
                for (int k = warp; k < npairs; k += FT / 32) {
                    const int g = 2 * k + half;
                    if (g >= ngroups) continue;
                    const int i0 = s_sorted[g * 16];
                    int idx = s_sorted[g * 16 + (lane & 15)];
                    const bool real = idx != NOKEY;
                    if (!real) idx = i0;  // dummy lanes repeat the group's first item
                    const int key = s_key[i0];
                    const int b = key / (NVAR * MAX_REG), var = (key / MAX_REG) % NVAR, reg = key % MAX_REG;
                    const int p = c0 + idx / NTAP, t = idx % NTAP;
                    double Dx, Dy;
                    int cf;
                    fused_tap<R>(s_ap + 4 * p, b, var - 1, t, Dx, Dy, cf);
                    const double flx = floor(Dx), fly = floor(Dy);
                    const int x = x0 + (p % TILE), y = y0 + p / TILE;
                    const int bx = x + (int)flx - s_dom[b][0], by = y + (int)fly - s_dom[b][1];
                    const double2 *G = scr + s_poff[b * NVAR + var];
                    double Fh, Fl;
                    int fl = 0;
                    if (var == 0)
                        fused_item<4 * R - 2>(G, s_dom[b][2], s_dom[b][3], bx, by, luts[b].var[0], reg, Dx - flx,
                                              Dy - fly, Fh, Fl, fl);
                    else
                        fused_item<3 * R - 2>(G, s_dom[b][2], s_dom[b][3], bx, by, luts[b].var[var], reg, Dx - flx,
                                              Dy - fly, Fh, Fl, fl);
                    if (real) {
                        s_F[idx] = make_double2(Fh, Fl);
                        flags |= fl;
                    }
                }
                if (flags && a.stats) atomicOr(a.stats + 4, (unsigned long long)flags);
            }
            __syncthreads();
            // per-pixel signed accumulation and normalisation (a7)
            if (tid < P) {
                const int p = c0 + tid;
                const int w = s_info[p];
                const int x = x0 + (p % TILE), y = y0 + p / TILE;
                const bool valid = x < a.W && y < a.H;
                const bool mine = a.pts ? (p == want) : valid;
                if (mine) {
                    double res = __longlong_as_double(0x7ff8000000000000LL);
                    const int b = info_basis(w), var = info_var(w);
                    if (info_live(w)) {
                        const int ntap = var ? NTAP / (R + 1) : NTAP;
                        dd S = {0.0, 0.0};
                        for (int t = 0; t < ntap; ++t) {
                            double Dx, Dy;
                            int cf;
                            fused_tap<R>(s_ap + 4 * p, b, var - 1, t, Dx, Dy, cf);
                            const double2 F = s_F[tid * NTAP + t];
                            S = dd_add(S, dd_mul_d({F.x, F.y}, (double)cf));
                        }
                        double norm = 1.0;
                        for (int k = 0; k < 4; ++k) {
                            if (k == var - 1) continue;
                            const double ia = 1.0 / s_ap[4 * p + k];
                            for (int i = 0; i < R; ++i) norm *= ia;
                        }
                        res = ldexp(dd_to_d(S), s_pe[b * NVAR + var]) * norm / luts[b].var[var].L;
                    }
                    const long long oidx = a.pts ? item : (long long)img * ipl + (size_t)y * a.W + x;
                    if (a.aux) {
                        double *ax = a.aux + BSF_AUX * oidx;
                        ax[0] = b;
                        ax[1] = var - 1;
                        ax[2] = (w >> 5) & 1;
                        ax[3] = w >> 8;
                        for (int k = 0; k < 4; ++k) ax[4 + k] = s_ap[4 * p + k];
                        ax[8] = 0.0;
                        ax[9] = ax[10] = ax[11] = 0.0;
                    }
                    if (a.out_f32 && !a.pts)
                        ((float *)a.out)[oidx] = (float)res;
                    else
                        ((double *)a.out)[oidx] = res;
                    if (a.stats) {
                        atomicAdd(a.stats + 0, 1ull);
                        if ((w >> 5) & 1) atomicAdd(a.stats + 1, 1ull);
                        if (var) atomicAdd(a.stats + 2, 1ull);
                        if (b == BASIS_THETA_PRIME) atomicAdd(a.stats + 3, 1ull);
                        if (w >> 8) atomicOr(a.stats + 4, (unsigned long long)(w >> 8));
                    }
                }
            }
            __syncthreads();
        }
    }
}

template <int R>
static cudaError_t launch_fused_r(const TileArgs &a, int slots, cudaStream_t st, const LutBasis *luts) {
    constexpr size_t sm = fused_smem_bytes<R>();
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(fused_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    fused_kernel<R><<<slots, FT, sm, st>>>(a, luts);
    return cudaGetLastError();
}

int fused_slots() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

cudaError_t launch_fused_impl(const TileArgs &a, int order, int slots, cudaStream_t st, const LutBasis *luts,
                              long long *nl) {
    cudaMemsetAsync(a.counter, 0, sizeof(int), st);
    cudaError_t e;
    switch (order) {
        case 1: e = launch_fused_r<1>(a, slots, st, luts); break;
        case 2: e = launch_fused_r<2>(a, slots, st, luts); break;
        case 3: e = launch_fused_r<3>(a, slots, st, luts); break;
        case 4: e = launch_fused_r<4>(a, slots, st, luts); break;
        default: return cudaErrorInvalidValue;
    }
    ++*nl;
    return e;
}
