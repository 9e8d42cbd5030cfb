// FFMA vs FFMA2 (fma.rn.f32x2) issue rate on sm_100a, GEMM-like register
// reuse pattern: acc[i][j] = fma(a[i], b[j], acc[i][j]). Prints FMA/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void kern(float *out, int iters, float s) {
    float a[8], b[8], acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = s * (threadIdx.x + i); b[i] = s * (i + 1); }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                    unsigned long long A, B, C, D;
                    asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a[i]));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b[j]), "f"(b[j + 1]));
                    asm("mov.b64 %0, {%1, %2};" : "=l"(C) : "f"(acc[i][j]), "f"(acc[i][j + 1]));
                    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(D) : "l"(A), "l"(B), "l"(C));
                    asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[i][j]), "=f"(acc[i][j + 1]) : "l"(D));
                }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = a[i] * 0.999f;
    }
    long long t1 = clock64();
    float r = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) r += acc[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}

int main() {
    float *d;
    cudaMalloc(&d, 148 * 8 * 1024 * 4);
    int iters = 4096;
    for (int mode = 0; mode < 2; ++mode)
        for (int thr : {128, 256, 512}) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (mode == 0) kern<0><<<148 * 2, thr>>>(d, iters, 1e-3f);
                else kern<1><<<148 * 2, thr>>>(d, iters, 1e-3f);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double fma = 148.0 * 2 * thr * iters * 64.0;
            printf("mode %s threads %d: %.3f ms, %.2f TFMA/s = %.1f TFLOP/s (%s)\n", mode ? "ffma2" : "ffma ", thr, ms,
                   fma / ms / 1e9, 2 * fma / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
