// Issue rate of int32 IMAD vs IDP4A (dp4a.u32.s32) on this GPU: every thread
// runs NACC independent accumulator chains; the result is stored so nothing
// is dead.  Prints warp instructions per SM clock for both.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dp4a_rate tools/dp4a_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NACC = 12, ITERS = 4096;

__global__ void imad_kernel(int *out, int a0, int b0) {
    int acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x + i;
    int a = a0 + threadIdx.x, b = b0;
#pragma unroll 4
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) acc[i] = acc[i] * a + b;  // IMAD
        a ^= it;
    }
    int s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dp4a_kernel(int *out, unsigned a0, int b0) {
    int acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x + i;
    unsigned a = a0 + threadIdx.x;
    int b = b0;
#pragma unroll 4
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) asm volatile("dp4a.u32.s32 %0, %1, %2, %0;" : "+r"(acc[i]) : "r"(a), "r"(b));
        a ^= it;
    }
    int s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, threads = 256;
    int *out;
    cudaMalloc(&out, sizeof(int) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int k = 0; k < 2; ++k) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (k == 0) imad_kernel<<<blocks, threads>>>(out, 3, 5);
            else dp4a_kernel<<<blocks, threads>>>(out, 0x01020304u, 0x05060708);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            const double warp_instr = (double)blocks * threads / 32 * ITERS * NACC;
            const double per_sm_clk = warp_instr / sms / (ms * 1e-3 * clk * 1e3);
            if (rep == 2)
                printf("{\"op\": \"%s\", \"ms\": %.4f, \"warp_instr_per_sm_clk\": %.3f, \"lanes_per_sm_clk\": %.1f, "
                       "\"clock_attr_mhz\": %d}\n",
                       k == 0 ? "IMAD" : "IDP4A", ms, per_sm_clk, 32 * per_sm_clk, clk / 1000);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
