// Empirical check of the mma.sync m16n8k8 .f64 fragment layout assumed by
// bsf_fused.cuh:  A[16x8]: a_i (i < 4) at row gid + 8 (i % 2), col tig + 4 (i / 2)
//                 B[8x8]:  b_i (i < 2) at row tig + 4 i, col gid
//                 C[16x8]: c_i (i < 4) at row gid + 8 (i / 2), col 2 tig + i % 2
// (gid = lane / 4, tig = lane % 4).  Prints "ok" or the first mismatch.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(const double *A, const double *B, double *D) {
    const int lane = threadIdx.x, gid = lane >> 2, tig = lane & 3;
    double a[4], b[2], c[4] = {0, 0, 0, 0};
    for (int i = 0; i < 4; ++i) a[i] = A[(gid + 8 * (i % 2)) * 8 + tig + 4 * (i / 2)];
    for (int i = 0; i < 2; ++i) b[i] = B[(tig + 4 * i) * 8 + gid];
    asm("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
    for (int i = 0; i < 4; ++i) D[(gid + 8 * (i / 2)) * 8 + 2 * tig + i % 2] = c[i];
}

// m16n8k16 .f64: a_i (i < 8) at row gid + 8 (i % 2), col tig + 4 (i / 2);
// b_i (i < 4) at row tig + 4 i, col gid; C as m16n8k8
__global__ void k16(const double *A, const double *B, double *D) {
    const int lane = threadIdx.x, gid = lane >> 2, tig = lane & 3;
    double a[8], b[4], c[4] = {0, 0, 0, 0};
    for (int i = 0; i < 8; ++i) a[i] = A[(gid + 8 * (i % 2)) * 16 + tig + 4 * (i / 2)];
    for (int i = 0; i < 4; ++i) b[i] = B[(tig + 4 * i) * 8 + gid];
    asm("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
        "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
          "d"(b[1]), "d"(b[2]), "d"(b[3]));
    for (int i = 0; i < 4; ++i) D[(gid + 8 * (i / 2)) * 8 + 2 * tig + i % 2] = c[i];
}

static int check16() {
    double A[256], B[128], D[128], R[128];
    for (int i = 0; i < 256; ++i) A[i] = (i * 37 % 101) - 50;
    for (int i = 0; i < 128; ++i) B[i] = (i * 53 % 97) - 48;
    for (int r = 0; r < 16; ++r)
        for (int c = 0; c < 8; ++c) {
            double s = 0;
            for (int kk = 0; kk < 16; ++kk) s += A[r * 16 + kk] * B[kk * 8 + c];
            R[r * 8 + c] = s;
        }
    double *dA, *dB, *dD;
    cudaMalloc(&dA, sizeof A);
    cudaMalloc(&dB, sizeof B);
    cudaMalloc(&dD, sizeof D);
    cudaMemcpy(dA, A, sizeof A, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, sizeof B, cudaMemcpyHostToDevice);
    k16<<<1, 32>>>(dA, dB, dD);
    cudaMemcpy(D, dD, sizeof D, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 128; ++i)
        if (D[i] != R[i]) {
            printf("k16 mismatch at row %d col %d: %g vs %g\n", i / 8, i % 8, D[i], R[i]);
            return 1;
        }
    printf("ok m16n8k16 f64 layout\n");
    return 0;
}

int main() {
    if (check16()) return 1;
    double A[128], B[64], D[128], R[128];
    for (int i = 0; i < 128; ++i) A[i] = (i * 37 % 101) - 50;
    for (int i = 0; i < 64; ++i) B[i] = (i * 53 % 97) - 48;
    for (int r = 0; r < 16; ++r)
        for (int c = 0; c < 8; ++c) {
            double s = 0;
            for (int kk = 0; kk < 8; ++kk) s += A[r * 8 + kk] * B[kk * 8 + c];
            R[r * 8 + c] = s;
        }
    double *dA, *dB, *dD;
    cudaMalloc(&dA, sizeof A);
    cudaMalloc(&dB, sizeof B);
    cudaMalloc(&dD, sizeof D);
    cudaMemcpy(dA, A, sizeof A, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, sizeof B, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dA, dB, dD);
    cudaMemcpy(D, dD, sizeof D, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 128; ++i)
        if (D[i] != R[i]) {
            printf("mismatch at row %d col %d: %g vs %g\n", i / 8, i % 8, D[i], R[i]);
            return 1;
        }
    printf("ok m16n8k8 f64 layout\n");
    return 0;
}
