// Global pre-integration (PAPER.md:106-110, 119-123,
// Alg. 3 step 2 PAPER.md:395-399): the 4r nested running sums
//     G_l(p) = V_l(p) + G_l(p - s_l),   V_1 = f,  V_{l+1} = G_l,
// on the zero-padded domain x in [0, GW), y in [0, GH) (zero state outside,
// DESIGN.md R3), levels in the order of c_scan_order, repeated r times.
//
// One launch per level, single pass (read V once, write G once), no carries
// between thread blocks:
//
//  * s = (1, 0): one warp per row walks the row in chunks of 32*EPL columns
//    (element j of a lane at x = 32 j + lane: coalesced), a warp-shuffle scan
//    per j plus the running total; the next chunk's loads are in flight
//    while the current one is scanned.  GH * nimg warps.
//  * s = (sx, sy), sy >= 1: in skewed coordinates u = x - sx*floor(y/sy)
//    every line is a column (u, y mod sy).  One warp owns a strip of 32
//    u-columns and walks it top to bottom with the running sums in
//    registers: row y of the strip is 32 consecutive x (coalesced), so no
//    transpose is needed.  The rows stream through a shared-memory ring
//    filled by cp.async (ND groups of RG rows in flight per warp, zero-fill
//    outside the domain), which keeps the HBM pipe full with a few warps
//    per SM.
//
// The first level of each basis reads the image f directly (u8 or f32, zero
// outside the image): no separate fill pass.
//
// Included by bsf_kernels.cu inside namespace bsf.

// element of the level input V at domain point (x, y) of image img:
// the running sums of the previous level, or (first level) the image itself
template <class Op, class In>
__device__ __forceinline__ typename Op::T scan_load(const In *__restrict__ in, const Geometry &geo, int img, int x,
                                                    int y) {
    typedef typename Op::T T;
    if constexpr (sizeof(In) == sizeof(T) && !std::is_same<In, float>::value) {
        return in[((size_t)img * geo.GH + y) * geo.GW + x];
    } else {
        const int xi = x - geo.P;
        if (y >= geo.H || xi < 0 || xi >= geo.W) return Op::zero();
        const In v = __ldg(in + ((size_t)img * geo.H + y) * geo.W + xi);
        if constexpr (sizeof(T) == 16)
            return make_double2((double)v, 0.0);
        else
            return (T)v;
    }
}


__device__ __forceinline__ int floordiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }  // b > 0
__device__ __forceinline__ int ceildiv(int a, int b) { return -floordiv(-a, b); }

// async copy of one element of the level input into shared memory (zero
// outside the domain / image); u8 input is fetched as the aligned 32-bit word
// that contains it
template <class Op, class In>
__device__ __forceinline__ void strip_copy(unsigned dst, const In *in, const Geometry &geo, int img, int x, int y,
                                           bool ok) {
    typedef typename Op::T T;
    const void *src = in;
    int bytes = 0;
    if (std::is_same<In, T>::value) {
        if (ok) {
            src = in + ((size_t)img * geo.GH + y) * geo.GW + x;
            bytes = sizeof(T);
        }
    } else {
        const int xi = x - geo.P;
        if (ok && y < geo.H && xi >= 0 && xi < geo.W) {
            const size_t a = (size_t)(in + ((size_t)img * geo.H + y) * geo.W + xi);
            src = (const void *)(a & ~(size_t)3);
            bytes = 4;
        }
    }
    if constexpr (sizeof(In) == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
    else if constexpr (sizeof(In) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}

template <class Op, class In>
__device__ __forceinline__ typename Op::T strip_value(const unsigned char *slot, const Geometry &geo, int img, int x,
                                                      int y) {
    typedef typename Op::T T;
    if constexpr (std::is_same<In, T>::value) {
        return *(const T *)slot;
    } else {
        In v;
        if constexpr (sizeof(In) == 1) {
            // byte offset of f[img][y][x - P] modulo 4 (the allocation is 4-aligned)
            const unsigned off = (unsigned)(img * geo.H + y) * (unsigned)geo.W + (unsigned)(x - geo.P);
            v = slot[off & 3u];
        } else {
            v = *(const In *)slot;
        }
        if constexpr (sizeof(T) == 16)
            return make_double2((double)v, 0.0);
        else
            return (T)v;
    }
}

// One block (NW warps) per strip of 32 u-columns, walking it top to bottom in
// blocks of NW*RPW rows: warp w scans rows RPW*w .. RPW*w + RPW-1 of the
// block in registers (lane = u-column), the NW warp totals are combined
// through shared memory, and the running carry of the strip stays in
// registers.  The rows stream through a cp.async ring of ND row blocks.
template <class Op, class In, int SX, int SY, int NW, int RPW, int ND>
__global__ void __launch_bounds__(32 * NW) scan_strip_kernel(const In *in, typename Op::T *out, Geometry geo, int U0,
                                                              int NS, const typename Op::T *carry_in) {
    typedef typename Op::T T;
    static_assert(RPW % 2 == 0, "phases of SY = 2 lines need an even row count per warp");
    constexpr int SLOT = sizeof(T);  // >= 4: also holds a u8 word or an f32
    constexpr int BR = NW * RPW;     // rows per block
    constexpr int NT = 32 * NW;
    extern __shared__ __align__(16) unsigned char scan_smem[];
    __shared__ T tot[2][NW][SY][32];  // [block parity][warp][phase][column]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int img = blockIdx.x / NS, ua = U0 + 32 * (blockIdx.x % NS), u = ua + lane;
    // rows where the strip meets the domain: SX * floor(y / SY) in [-ua - 31, GW - 1 - ua]
    int qlo = 0, qhi = (geo.GH - 1) / SY;
    if (SX > 0) {
        qlo = max(qlo, ceildiv(-ua - 31, SX));
        qhi = min(qhi, floordiv(geo.GW - 1 - ua, SX));
    } else if (SX < 0) {
        qlo = max(qlo, ceildiv(ua - geo.GW + 1, -SX));
        qhi = min(qhi, floordiv(ua + 31, -SX));
    } else if (ua + 31 < 0 || ua >= geo.GW) {
        return;
    }
    if (qlo > qhi) return;
    const int ylo = qlo * SY, yhi = min(geo.GH - 1, qhi * SY + SY - 1);  // ylo even when SY = 2
    const int nblk = (yhi - ylo + BR) / BR;
    const unsigned ring_s = (unsigned)__cvta_generic_to_shared(scan_smem) + threadIdx.x * SLOT;
    auto issue = [&](int j) {
        if (j < nblk) {
#pragma unroll
            for (int k = 0; k < RPW; ++k) {
                const int y = ylo + j * BR + RPW * warp + k, x = u + SX * (y / SY);
                const bool ok = y <= yhi && x >= 0 && x < geo.GW;
                strip_copy<Op, In>(ring_s + (unsigned)(((j % ND) * RPW + k) * NT * SLOT), in, geo, img, x, y, ok);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int j = 0; j < ND - 1; ++j) issue(j);
    T carry[SY];  // strip carry of the lines y even / odd (odd only for SY = 2)
#pragma unroll
    for (int ph = 0; ph < SY; ++ph) {
        // a row strip of a larger domain (multi-GPU GLOBAL mode): the line through
        // (u, ph) continues the level's running sum at (u - SX, ph - SY), which is
        // row ph of carry_in ([nimg][SY][GW], the SY domain rows above the strip)
        carry[ph] = Op::zero();
        if (carry_in && ph < geo.GH && u >= 0 && u < geo.GW && u - SX >= 0 && u - SX < geo.GW)
            carry[ph] = carry_in[((size_t)img * SY + ph) * geo.GW + (size_t)(u - SX)];
    }
    T *o = out + (size_t)img * geo.GH * geo.GW;
    for (int j = 0; j < nblk; ++j) {
        issue(j + ND - 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(ND - 1) : "memory");
        const unsigned char *grp = scan_smem + (size_t)(j % ND) * RPW * NT * SLOT + threadIdx.x * SLOT;
        const int yb = ylo + j * BR + RPW * warp;
        T v[RPW];
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const int y = yb + k, x = u + SX * (y / SY);
            const bool ok = y <= yhi && x >= 0 && x < geo.GW;
            v[k] = ok ? strip_value<Op, In>(grp + k * NT * SLOT, geo, img, x, y) : Op::zero();
        }
        // local inclusive scan along the lines (row yb + k is on phase k % SY)
#pragma unroll
        for (int k = SY; k < RPW; ++k) v[k] = Op::add(v[k - SY], v[k]);
        T(*tb)[SY][32] = tot[j & 1];
#pragma unroll
        for (int ph = 0; ph < SY; ++ph) tb[warp][ph][lane] = v[RPW - SY + ph];
        __syncthreads();
        T ex[SY];
#pragma unroll
        for (int ph = 0; ph < SY; ++ph) {
            T acc = carry[ph];
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                if (w == warp) ex[ph] = acc;
                acc = Op::add(acc, tb[w][ph][lane]);
            }
            carry[ph] = acc;
        }
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const int y = yb + k, x = u + SX * (y / SY);
            if (y <= yhi && x >= 0 && x < geo.GW) o[(size_t)y * geo.GW + x] = Op::add(ex[k % SY], v[k]);
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// s = (1, 0): one warp per row, chunks of 32 * EPL columns, next chunk prefetched
template <class Op, class In, int EPL, int WPC>
__global__ void __launch_bounds__(32 * WPC) scan_row_kernel(const In *in, typename Op::T *out, Geometry geo) {
    typedef typename Op::T T;
    const int lane = threadIdx.x & 31;
    const long long rid = (long long)blockIdx.x * WPC + (threadIdx.x >> 5);
    if (rid >= (long long)geo.nimg * geo.GH) return;
    const int img = (int)(rid / geo.GH), y = (int)(rid % geo.GH);
    constexpr int CW = 32 * EPL;
    const int nch = (geo.GW + CW - 1) / CW;
    T *o = out + ((size_t)img * geo.GH + y) * geo.GW;
    T cur[EPL], nxt[EPL];
    auto load = [&](int ch, T (&v)[EPL]) {
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
            const int x = ch * CW + 32 * j + lane;
            v[j] = (ch < nch && x < geo.GW) ? scan_load<Op>(in, geo, img, x, y) : Op::zero();
        }
    };
    load(0, cur);
    T run = Op::zero();
    for (int ch = 0; ch < nch; ++ch) {
        load(ch + 1, nxt);
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
            T a = cur[j];
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const T t = Op::shfl_up(a, dd);
                if (lane >= dd) a = Op::add(t, a);
            }
            a = Op::add(run, a);
            run = Op::shfl_idx(a, 31);
            const int x = ch * CW + 32 * j + lane;
            if (x < geo.GW) o[x] = a;
        }
#pragma unroll
        for (int j = 0; j < EPL; ++j) cur[j] = nxt[j];
    }
}

// ---------------------------------------------------------------------------
// The same strip scan with its rows streamed by TMA (cp.async.bulk.tensor):
// each warp owns RPW rows per block of rows and fetches each of them with ONE
// 3-D tensor copy (box {BX, 1, 1}) into a 128-byte aligned shared-memory row,
// completing on the warp's mbarrier of that ring stage (arrive.expect_tx by
// lane 0, then the lanes issue one row each).  A box's first x coordinate
// must sit on a 16-byte boundary of the row (measured: an unaligned start is
// an illegal instruction on sm_100a), so the box starts at the aligned
// coordinate below the warp's 32 elements and is A - 1 elements wider; each
// lane reads its element at the row's offset.  The tensor map's bounds give
// the zero state outside the domain (levels >= 1) or outside the image
// (level 0: the u8 / f32 image itself, zero-extended) for free: no
// per-element predicates in the copy.  Used when the base address and row
// pitch meet TMA's 16-byte rules (scan_strips checks), else the cp.async
// kernel above runs.  The scan arithmetic is identical (bit-exact int64, same
// double-double order).
// ---------------------------------------------------------------------------
template <class In>
struct TmaRow {
    static constexpr int XS = sizeof(In) == 16 ? 2 : 1;     // double-double rows are fp64 pairs in the map
    static constexpr int ES = (int)sizeof(In) / XS;          // map element size
    static constexpr int A = 16 / ES;                        // map elements per 16-byte boundary
    static constexpr int BX = (32 * XS + (A > XS ? A - XS : 0) + A - 1) / A * A;  // box width (map elements)
    static constexpr unsigned BYTES = (unsigned)(BX * ES);   // bytes one row copy delivers
    static constexpr int PITCH = (int)((BYTES + 127) / 128 * 128);
};
template <class In>
constexpr int tma_row_bytes() {
    return TmaRow<In>::PITCH;
}

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_row(unsigned dst, const CUtensorMap *map, int x, int y, int z, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(bar)
        : "memory");
}

template <class Op, class In, int SX, int SY, int NW, int RPW, int ND>
__global__ void __launch_bounds__(32 * NW) scan_strip_tma_kernel(const __grid_constant__ CUtensorMap map,
                                                                  typename Op::T *out, Geometry geo, int U0, int NS,
                                                                  const typename Op::T *carry_in) {
    typedef typename Op::T T;
    static_assert(RPW % 2 == 0 && RPW <= 32, "phases of SY = 2 lines need an even row count per warp");
    constexpr int BR = NW * RPW;
    typedef TmaRow<In> TR;
    constexpr int PITCH = TR::PITCH;
    extern __shared__ __align__(128) unsigned char scan_tma_smem[];
    __shared__ T tot[2][NW][SY][32];
    __shared__ __align__(8) unsigned long long bars[ND][NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int img = blockIdx.x / NS, ua = U0 + 32 * (blockIdx.x % NS), u = ua + lane;
    int qlo = 0, qhi = (geo.GH - 1) / SY;
    if (SX > 0) {
        qlo = max(qlo, ceildiv(-ua - 31, SX));
        qhi = min(qhi, floordiv(geo.GW - 1 - ua, SX));
    } else if (SX < 0) {
        qlo = max(qlo, ceildiv(ua - geo.GW + 1, -SX));
        qhi = min(qhi, floordiv(ua + 31, -SX));
    } else if (ua + 31 < 0 || ua >= geo.GW) {
        return;
    }
    if (qlo > qhi) return;
    const int ylo = qlo * SY, yhi = min(geo.GH - 1, qhi * SY + SY - 1);
    const int nblk = (yhi - ylo + BR) / BR;
    // 128-byte aligned TMA destinations (the launch adds 128 bytes of slack)
    const unsigned ring = ((unsigned)__cvta_generic_to_shared(scan_tma_smem) + 127u) & ~127u;
    const unsigned char *ring_g = scan_tma_smem + (ring - (unsigned)__cvta_generic_to_shared(scan_tma_smem));
    const unsigned bar0 = (unsigned)__cvta_generic_to_shared(&bars[0][0]);
    if (lane == 0)
        for (int s = 0; s < ND; ++s) mbar_init(bar0 + 8u * (s * NW + warp), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    // level 0 reads the image (coordinates x - P, y, img: zero outside it);
    // later levels read the domain (x, y, img: zero outside [0, GW))
    constexpr bool IMG = !std::is_same<In, T>::value;
    auto issue = [&](int j) {
        if (j >= nblk) return;
        const int s = j % ND;
        const unsigned bar = bar0 + 8u * (s * NW + warp);
        const int yb = ylo + j * BR + RPW * warp;
        const int nrow = max(0, min(RPW, yhi - yb + 1));
        if (nrow == 0) return;
        if (lane == 0) mbar_expect_tx(bar, TR::BYTES * (unsigned)nrow);
        __syncwarp();
        if (lane < nrow) {
            const int y = yb + lane, x = ua + SX * (y / SY);
            const unsigned dst = ring + (unsigned)(((s * NW + warp) * RPW + lane) * PITCH);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the row was read through the generic proxy
            const int xc = TR::XS * (IMG ? x - geo.P : x);
            tma_load_row(dst, &map, xc - (int)((unsigned)xc % TR::A), y, img, bar);  // 16-byte aligned box start
        }
    };
#pragma unroll
    for (int j = 0; j < ND - 1; ++j) issue(j);
    T carry[SY];
#pragma unroll
    for (int ph = 0; ph < SY; ++ph) {
        carry[ph] = Op::zero();
        if (carry_in && ph < geo.GH && u >= 0 && u < geo.GW && u - SX >= 0 && u - SX < geo.GW)
            carry[ph] = carry_in[((size_t)img * SY + ph) * geo.GW + (size_t)(u - SX)];
    }
    T *o = out + (size_t)img * geo.GH * geo.GW;
    for (int j = 0; j < nblk; ++j) {
        issue(j + ND - 1);
        const int s = j % ND;
        const int yb = ylo + j * BR + RPW * warp;
        const int nrow = max(0, min(RPW, yhi - yb + 1));
        if (nrow) mbar_wait(bar0 + 8u * (s * NW + warp), (unsigned)((j / ND) & 1));
        const unsigned char *rows = ring_g + (size_t)((s * NW + warp) * RPW) * PITCH;
        T v[RPW];
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const int y = yb + k, x = u + SX * (y / SY);
            const bool ok = k < nrow && x >= 0 && x < geo.GW;
            T t = Op::zero();
            if (ok) {
                const int xc = TR::XS * (IMG ? ua + SX * (y / SY) - geo.P : ua + SX * (y / SY));
                const int off = (int)((unsigned)xc % TR::A) / TR::XS;  // the warp's first element in the box
                const In e = reinterpret_cast<const In *>(rows + k * PITCH)[off + lane];
                if constexpr (sizeof(T) == 16 && !std::is_same<In, T>::value)
                    t = make_double2((double)e, 0.0);
                else if constexpr (std::is_same<In, T>::value)
                    t = e;
                else
                    t = (T)e;
            }
            v[k] = t;
        }
        __syncwarp();  // every lane read the stage before lane < nrow refills it (issue above, next iterations)
#pragma unroll
        for (int k = SY; k < RPW; ++k) v[k] = Op::add(v[k - SY], v[k]);
        T(*tb)[SY][32] = tot[j & 1];
#pragma unroll
        for (int ph = 0; ph < SY; ++ph) tb[warp][ph][lane] = v[RPW - SY + ph];
        __syncthreads();
        T ex[SY];
#pragma unroll
        for (int ph = 0; ph < SY; ++ph) {
            T acc = carry[ph];
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                if (w == warp) ex[ph] = acc;
                acc = Op::add(acc, tb[w][ph][lane]);
            }
            carry[ph] = acc;
        }
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const int y = yb + k, x = u + SX * (y / SY);
            if (y <= yhi && x >= 0 && x < geo.GW) o[(size_t)y * geo.GW + x] = Op::add(ex[k % SY], v[k]);
        }
    }
}
