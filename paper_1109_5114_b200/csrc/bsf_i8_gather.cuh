// Order-3 gather on the 5th-generation tensor cores (plan option "i8_tc";
// included inside fused_kernel<3, ..., I8 = true> phase 4).
//
// The exact part of Eq. (11)'s window contraction (the
// split of §7), E12_mu = sum_s (G1 2^k + G2)_s n_{s,mu}, is formed as byte-slice
// products on tcgen05.mma kind::i8 with s32 accumulators in TMEM:
//   G12 = sum_{b<8} 2^{8b} B_b,  n = sum_{a<na} 2^{8a} A_a  (top slices signed)
//   E12 = sum_c 2^{8c} D_c,      D_c = sum_{a+b=c} A_a^T B_b  (exact in int32)
// per TILE of up to four consecutive sorted groups (8 items each) sharing a
// key and a pre-split plane: A = the region's numerator slices (pre-sliced on
// the host in the UMMA canonical layout, bulk-copied per 32-slot chunk and
// moved to TMEM by tcgen05.cp), B = the 32 items' window values, byte-
// transposed by all threads into shared memory, M = 128 table columns, N = 32
// items, K = 32 slots.  The tile's E12 (times 2^-k, double-double) goes to
// shared memory; each group's warp then contracts only the rounded G0 limb on
// DMMA and runs the unchanged compensated Horner (fused_group_g3<..., I8>).
// Groups on planes too large to pre-split, or tables without a slice form,
// take the DMMA path one warp per group, as in the default kernel.
{
    const int ngroups = npad / GS;
    int flags = 0;
    uint8_t *sA = smem + i8_smem_off<R>();
    uint8_t *sB = sA + 7 * 4096;
    double2 *sE = reinterpret_cast<double2 *>(sB + 8 * 1024);
    const uint32_t a_addr = (uint32_t)__cvta_generic_to_shared(sA), b_addr = (uint32_t)__cvta_generic_to_shared(sB);
    const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&s_i8bar[0]);
    const uint32_t bar_m = (uint32_t)__cvta_generic_to_shared(&s_i8bar[1]);
    const uint32_t tm = s_tmem;
    // one group (8 items) on one warp; e12: its rows of the tile's E12, or null
    // for the DMMA path
    auto run_group = [&](int g, const double2 *e12) {
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
        double Fh[MT], Fl[MT];
        if (a.stats) {  // algorithmic work: window x monomials per real item
            const unsigned nreal = __popc(__ballot_sync(0xffffffffu, real));
            if (lane == 0)
                atomicAdd(&s_stats[6], (unsigned long long)nreal * __ldg(V.counts + reg) *
                                           (var == 0 ? DegCfg<4 * R - 2>::NMON : DegCfg<3 * R - 2>::NMON));
        }
        const size_t ro = (size_t)reg * V.nslot4 * V.nmonp;
        const double *G0 = scr0 + s_poff[b * NVAR + var];
        const double sce = ldexp(1.0, -s_pe[b * NVAR + var]);
        const bool pre = NX * NY <= G3_PRESPLIT_MAX;
        if (e12) {  // exact limbs from the tile (pre-split planes only)
            if (V.nsplit == 2) {
                const float *nc = V.num32 + 2 * ro;
                if (var == 0)
                    fused_group_g3<4 * R - 2, 2, BSF_G3_NP2, MT, true, true>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                           V.nmonp, n4, V.shift, G0, sce, V.kbits,
                                                                           Fh, Fl, flags, e12);
                else
                    fused_group_g3<3 * R - 2, 2, BSF_G3_NP2, MT, true, true>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                           V.nmonp, n4, V.shift, G0, sce, V.kbits,
                                                                           Fh, Fl, flags, e12);
            } else {
                const float *nc = V.num32 + ro;
                if (var == 0)
                    fused_group_g3<4 * R - 2, 1, BSF_G3_NP1, MT, true, true>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                           V.nmonp, n4, 0, G0, sce, V.kbits, Fh,
                                                                           Fl, flags, e12);
                else
                    fused_group_g3<3 * R - 2, 1, BSF_G3_NP1, MT, true, true>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                           V.nmonp, n4, 0, G0, sce, V.kbits, Fh,
                                                                           Fl, flags, e12);
            }
        } else if (V.nsplit == 2) {
            const float *nc = V.num32 + 2 * ro;
            if (var == 0)
                (pre ? (fused_group_g3<4 * R - 2, 2, BSF_G3_NP2, MT, true>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                        V.nmonp, n4, V.shift, G0, sce, V.kbits, Fh,
                                                                        Fl, flags))
                     : (fused_group_g3<4 * R - 2, 2, BSF_G3_NP2, MT, false>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                          V.nmonp, n4, V.shift, G0, sce, V.kbits, Fh,
                                                                          Fl, flags)));
            else
                (pre ? (fused_group_g3<3 * R - 2, 2, BSF_G3_NP2, MT, true>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                        V.nmonp, n4, V.shift, G0, sce, V.kbits, Fh,
                                                                        Fl, flags))
                     : (fused_group_g3<3 * R - 2, 2, BSF_G3_NP2, MT, false>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                          V.nmonp, n4, V.shift, G0, sce, V.kbits, Fh,
                                                                          Fl, flags)));
        } else {
            const float *nc = V.num32 + ro;
            if (var == 0)
                (pre ? (fused_group_g3<4 * R - 2, 1, BSF_G3_NP1, MT, true>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                        V.nmonp, n4, 0, G0, sce, V.kbits, Fh, Fl,
                                                                        flags))
                     : (fused_group_g3<4 * R - 2, 1, BSF_G3_NP1, MT, false>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                          V.nmonp, n4, 0, G0, sce, V.kbits, Fh, Fl,
                                                                          flags)));
            else
                (pre ? (fused_group_g3<3 * R - 2, 1, BSF_G3_NP1, MT, true>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                        V.nmonp, n4, 0, G0, sce, V.kbits, Fh, Fl,
                                                                        flags))
                     : (fused_group_g3<3 * R - 2, 1, BSF_G3_NP1, MT, false>(G, NX, NY, bxt, byt, fx, fy, offs, nc,
                                                                          V.nmonp, n4, 0, G0, sce, V.kbits, Fh, Fl,
                                                                          flags)));
        }
#pragma unroll
        for (int q = 0; q < MT; ++q) {  // item lane/4 + 8q's result, from its quad's lane 0
            const int src = (lane >> 2) + 8 * q;
            const int iq = __shfl_sync(0xffffffffu, idx, src);
            const bool rq = __shfl_sync(0xffffffffu, (int)real, src) != 0;
            if ((lane & 3) == 0 && rq) s_F[iq] = make_double2(Fh[q], Fl[q]);
        }
    };
    // which groups go to the tensor-core tiles: the full kernel (variant 0)
    // with split numerators (Theta': 5 DMMA products per multiply-add, 4 of
    // them exact) on a pre-split plane with a slice table; every other group
    // is contracted on DMMA first, all warps in parallel as in the default
    // kernel
    auto tiled = [&](int key) {
        const int b = key / (NVAR * MAX_REG), var = (key / MAX_REG) % NVAR;
        const LutVar &V = luts[b].var[var];
        return var == 0 && V.nsplit == 2 && V.i8tab != nullptr && s_dom[b][2] * s_dom[b][3] <= G3_PRESPLIT_MAX;
    };
    for (int g = warp; g < ngroups; g += FT / 32)
        if (!tiled(s_key[s_sorted[g * GS]])) run_group(g, nullptr);
    for (int g = 0; g < ngroups;) {
        const int i0 = s_sorted[g * GS];
        const int key = s_key[i0];
        if (!tiled(key)) {
            ++g;
            continue;
        }
        int ng = 1;
        while (ng < 4 && g + ng < ngroups && s_key[s_sorted[(g + ng) * GS]] == key) ++ng;
        const int b = key / (NVAR * MAX_REG), var = (key / MAX_REG) % NVAR, reg = key % MAX_REG;
        const int NX = s_dom[b][2];
        const LutVar &V = luts[b].var[var];
        // ---- the tile's items: thread = (item i, four slots of a chunk)
        const int it = tid >> 3, sq = tid & 7;
        int idx = NOKEY;
        if ((it >> 3) < ng) idx = s_sorted[(g + (it >> 3)) * GS + (it & 7)];
        if (idx == NOKEY) idx = i0;  // padding items repeat the tile's first item (never read back)
        const int p = c0 + idx % P, t = idx / P;
        double Dx, Dy;
        fused_tap_v<R>(s_tv + 5 * p, var - 1, t, Dx, Dy);
        const int bx = x0 + (p % TILE) + (int)floor(Dx) - s_dom[b][0];
        const int by = y0 + p / TILE + (int)floor(Dy) - s_dom[b][1];
        const double2 *Gp = scr + s_poff[b * NVAR + var];
        const int2 *offs = V.offs4 + (size_t)reg * V.nslot4;
        const int k = V.kbits, na = V.i8na, nch = V.i8nchunk;
        const double S = ldexp(1.0, k);
        const uint8_t *tab = V.i8tab + (size_t)reg * nch * na * 4096;
        for (int ch = 0; ch < nch; ++ch) {
            if (tid == 0) {  // A: the chunk's na slices, one bulk copy
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"(na * 4096)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        a_addr),
                    "l"(tab + (size_t)ch * na * 4096), "r"(na * 4096), "r"(bar_a)
                    : "memory");
            }
            {  // B: G12 = G1 2^k + G2 (exact integers) of four slots, byte-transposed
                unsigned long long gv[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int sl = ch * 32 + sq * 4 + q;
                    const int2 o = sl < V.nslot4 ? __ldg(offs + sl) : make_int2(0, 0);
                    const double2 v = __ldcg(Gp + (size_t)(by + o.y) * NX + (bx + o.x));
                    gv[q] = (unsigned long long)((long long)(v.x * S) + (long long)v.y);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const unsigned w0 = (unsigned)(gv[0] >> (32 * h)), w1 = (unsigned)(gv[1] >> (32 * h));
                    const unsigned w2 = (unsigned)(gv[2] >> (32 * h)), w3 = (unsigned)(gv[3] >> (32 * h));
                    const unsigned a01 = __byte_perm(w0, w1, 0x5140), a23 = __byte_perm(w2, w3, 0x5140);
                    const unsigned b01 = __byte_perm(w0, w1, 0x7362), b23 = __byte_perm(w2, w3, 0x7362);
                    const unsigned pl[4] = {__byte_perm(a01, a23, 0x5410), __byte_perm(a01, a23, 0x7632),
                                            __byte_perm(b01, b23, 0x5410), __byte_perm(b01, b23, 0x7632)};
                    const int off = (it >> 3) * 256 + (sq >> 2) * 128 + (it & 7) * 16 + (sq & 3) * 4;
#pragma unroll
                    for (int q = 0; q < 4; ++q) *reinterpret_cast<unsigned *>(sB + (4 * h + q) * 1024 + off) = pl[q];
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (warp == 0) {
                asm volatile(
                    "{\n\t.reg .pred P;\n"
                    "WAIT_%=:\n\t"
                    "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
                    "@!P bra WAIT_%=;\n}" ::"r"(bar_a),
                    "r"(i8_pa)
                    : "memory");
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                uint32_t leader = 0;
                asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                             : "=r"(leader));
                if (leader) {
                    auto sdesc = [](uint32_t addr) -> uint64_t {  // K-major, no swizzle: LBO 128, SBO 256, sm_100
                        return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
                               ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
                    };
                    for (int aa = 0; aa < na; ++aa)
                        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tm + 448u + 8u * aa),
                                     "l"(sdesc(a_addr + aa * 4096))
                                     : "memory");
                    for (int aa = 0; aa < na; ++aa)
                        for (int bb = 0; bb < 8; ++bb) {
                            const int c = aa + bb;
                            const bool first = ch == 0 && aa == (c > 7 ? c - 7 : 0);
                            const uint32_t idesc = (2u << 4) | ((uint32_t)(aa == na - 1) << 7) |
                                                   ((uint32_t)(bb == 7) << 10) | ((uint32_t)(32 >> 3) << 17) |
                                                   ((uint32_t)(128 >> 4) << 24);
                            asm volatile(
                                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(
                                    tm + (uint32_t)(c * 32)),
                                "r"(tm + 448u + 8u * aa), "l"(sdesc(b_addr + bb * 1024)), "r"(idesc),
                                "r"(first ? 0u : 1u)
                                : "memory");
                        }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     bar_m)
                                 : "memory");
                }
                __syncwarp();
            }
            asm volatile(
                "{\n\t.reg .pred P;\n"
                "WAIT_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
                "@!P bra WAIT_%=;\n}" ::"r"(bar_m),
                "r"(i8_pm)
                : "memory");
            i8_pa ^= 1u;
            i8_pm ^= 1u;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        // ---- E12 (times 2^-k, double-double) of the tile into shared memory:
        // warp w < 3 reads TMEM lanes 32w.. (the table columns), all classes
        if (warp < 3) {
            const int m = warp * 32 + lane;
            const int ncls = na + 7;
            for (int i0e = 0; i0e < 32; i0e += 4) {
                uint32_t r[14][4];
#pragma unroll
                for (int c = 0; c < 14; ++c) {
                    if (c < ncls) {
                        const uint32_t taddr = tm + ((uint32_t)(warp * 32) << 16) + (uint32_t)(c * 32 + i0e);
                        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(r[c][0]), "=r"(r[c][1]), "=r"(r[c][2]), "=r"(r[c][3])
                                     : "r"(taddr));
                    } else {
                        r[c][0] = r[c][1] = r[c][2] = r[c][3] = 0u;
                    }
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    long long P4[4] = {0, 0, 0, 0};  // four classes at a time, exact in int64 (< 2^57)
#pragma unroll
                    for (int c = 0; c < 14; ++c) P4[c >> 2] += (long long)(int)r[c][q] * (1ll << (8 * (c & 3)));
                    const __int128 e = (__int128)P4[0] + ((__int128)P4[1] << 32) + ((__int128)P4[2] << 64) +
                                       ((__int128)P4[3] << 96);
                    // exact double-double: three 40-bit pieces, then 2^-k
                    const __int128 m40 = ((__int128)1 << 40) - 1;
                    const double e0 = (double)(long long)(e & m40), e1 = (double)(long long)((e >> 40) & m40);
                    const double e2 = (double)(long long)(e >> 80);
                    const dd x = dd_add_d(two_sum(ldexp(e2, 80 - k), ldexp(e1, 40 - k)), ldexp(e0, -k));
                    if (m < E12S) sE[(i0e + q) * E12S + m] = make_double2(x.hi, x.lo);
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (warp < ng) run_group(g + warp, sE + warp * 8 * E12S);
        __syncthreads();
        g += ng;
    }
    if (flags) atomicOr(&s_stats[4], (unsigned long long)flags);
}
