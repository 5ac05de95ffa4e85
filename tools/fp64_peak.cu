// FP64 peak microbenchmarks on the GPU box (the roofline denominator of the
// gather; MEASURED_PEAKS.json has no FP64 figure):
//   dfma  : independent DFMA chains, 8 warps/SM x 148 SMs x many blocks
//   dmma  : mma.sync m8n8k4 f64 (legacy FP64 tensor-core path) in a loop
//   dmma16: mma.sync m16n8k16 f64 (sm_90+ shape)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void dfma_kernel(double *out, double a, double b) {
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == 1.2345) out[threadIdx.x] = s;
}

__global__ void dmma_kernel(double *out, double a) {
    double A = a + threadIdx.x, B = a - threadIdx.x;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(A), "d"(B));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[threadIdx.x] = s;
}

__global__ void dmma16_kernel(double *out, double a) {
    double A[8], B[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) A[i] = a + i + threadIdx.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) B[i] = a - i;
    double c[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
                "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                : "d"(A[0]), "d"(A[1]), "d"(A[2]), "d"(A[3]), "d"(A[4]), "d"(A[5]), "d"(A[6]), "d"(A[7]), "d"(B[0]),
                  "d"(B[1]), "d"(B[2]), "d"(B[3]));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 1.2345) out[threadIdx.x] = s;
}

// half the warps run DFMA chains, half DMMA: do the two FP64 paths overlap?
__global__ void mixed_kernel(double *out, double a, double b) {
    if ((threadIdx.x >> 5) & 1) {
        double acc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
        for (int it = 0; it < ITERS; ++it) {
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
        }
        double s = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) s += acc[i];
        if (s == 1.2345) out[threadIdx.x] = s;
    } else {
        double A = a + threadIdx.x, B = a - threadIdx.x;
        double c[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
        for (int it = 0; it < ITERS; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c[i][0]), "+d"(c[i][1])
                             : "d"(A), "d"(B));
        }
        double s = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
        if (s == 1.2345) out[threadIdx.x] = s;
    }
}

template <class F>
static float timeit(F launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    return best;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 1 << 20);
    for (int warps : {4, 8, 16, 32}) {
        int blocks = sms * 4, threads = warps * 32 / 4;
        float ms = timeit([&] { dfma_kernel<<<blocks, threads>>>(out, 1.0000001, 1e-9); });
        double flops = 2.0 * 16 * ITERS * (double)blocks * threads;
        printf("{\"kernel\": \"dfma\", \"warps_per_sm\": %d, \"tflops\": %.2f}\n", warps, flops / ms / 1e9);
        ms = timeit([&] { dmma_kernel<<<blocks, threads>>>(out, 1.0); });
        flops = 2.0 * 8 * 8 * 4 * 8 * (double)ITERS * blocks * (threads / 32);
        printf("{\"kernel\": \"dmma_m8n8k4\", \"warps_per_sm\": %d, \"tflops\": %.2f}\n", warps, flops / ms / 1e9);
        ms = timeit([&] { dmma16_kernel<<<blocks, threads>>>(out, 1.0); });
        flops = 2.0 * 16 * 8 * 16 * 4 * (double)(ITERS / 4) * blocks * (threads / 32);
        printf("{\"kernel\": \"dmma_m16n8k16\", \"warps_per_sm\": %d, \"tflops\": %.2f}\n", warps, flops / ms / 1e9);
    }
    {
        // mixed: blocks of 8 warps, 4 DFMA + 4 DMMA; each half does the same work as above per warp
        int blocks = sms * 4, threads = 256;
        float ms = timeit([&] { mixed_kernel<<<blocks, threads>>>(out, 1.0000001, 1e-9); });
        double dfma = 2.0 * 16 * ITERS * (double)blocks * threads / 2;
        double dmma = 2.0 * 8 * 8 * 4 * 8 * (double)ITERS * blocks * (threads / 64);
        printf("{\"kernel\": \"mixed dfma+dmma\", \"warps_per_sm\": 32, \"tflops_total\": %.2f, "
               "\"dfma_share\": %.3f}\n", (dfma + dmma) / ms / 1e9, dfma / (dfma + dmma));
    }
    cudaError_t e = cudaGetLastError();
    printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
