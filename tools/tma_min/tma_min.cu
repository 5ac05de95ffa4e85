// Minimal TMA row-load check (diagnostics for the TMA-fed scan): one CTA,
// one warp, each lane loads one 32-element row of a 3-D tensor map.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap map, unsigned char *out, int nrow, int x0) {
    __shared__ __align__(128) unsigned char buf[32 * 128];
    __shared__ __align__(8) unsigned long long bar;
    const int lane = threadIdx.x;
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    unsigned d = (unsigned)__cvta_generic_to_shared(buf);
    if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(1) : "memory");
    if (MODE >= 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(32 * nrow) : "memory");
    __syncwarp();
    if (lane < nrow) {
        if (MODE >= 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
            ::"r"(d + 128 * lane), "l"(&map), "r"(x0), "r"(lane), "r"(0), "r"(b) : "memory");
    }
    asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n}" ::"r"(b), "r"(0) : "memory");
    for (int r = 0; r < nrow; ++r) out[r * 32 + lane] = buf[128 * r + lane];
}

int main() {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeTiledFn fn = (EncodeTiledFn)p;
    const int W = 128, H = 96;
    std::vector<unsigned char> h(W * H);
    for (int i = 0; i < W * H; ++i) h[i] = (unsigned char)(i * 7 + 3);
    unsigned char *dimg, *dout;
    cudaMalloc(&dimg, W * H);
    cudaMalloc(&dout, 32 * 32);
    cudaMemcpy(dimg, h.data(), W * H, cudaMemcpyHostToDevice);
    CUtensorMap map;
    cuuint64_t dims[3] = {W, H, 1}, str[2] = {W, (cuuint64_t)W * H};
    cuuint32_t box[3] = {32, 1, 1}, es[3] = {1, 1, 1};
    CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, dimg, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    for (int mode = 0; mode < 3; ++mode) {
        for (int x0 : {0, 16, -48, 112, -40}) {
            if (mode == 0) k<0><<<1, 32>>>(map, dout, 8, x0);
            if (mode == 1) k<1><<<1, 32>>>(map, dout, 8, x0);
            if (mode == 2) k<2><<<1, 32>>>(map, dout, 8, x0);
            cudaError_t e = cudaDeviceSynchronize();
            printf("mode %d x0 %d: %s\n", mode, x0, cudaGetErrorString(e));
            if (e != cudaSuccess) return 1;
            std::vector<unsigned char> o(32 * 8);
            cudaMemcpy(o.data(), dout, o.size(), cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int rr = 0; rr < 8; ++rr)
                for (int c = 0; c < 32; ++c) {
                    int x = x0 + c;
                    unsigned char want = (x >= 0 && x < W) ? h[rr * W + x] : 0;
                    bad += o[rr * 32 + c] != want;
                }
            printf("  mismatches %d\n", bad);
        }
    }
    return 0;
}
