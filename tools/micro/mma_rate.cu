// Microbenchmark: issue rate of tcgen05.mma (SS operands, K-major, no
// swizzle, M=128) per kind and N. One CTA per SM, one thread issues R MMAs
// into one TMEM accumulator; prints cycles per MMA.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
template <int KIND>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    if (KIND == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc));
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc));
}

template <int KIND>
__global__ void bench(int N, int R, int nsplit, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        // A: 128 rows, padded-layout style: LBO = npix*16 (next K core matrix), SBO = 128
        const uint32_t npix = 168;
        const uint32_t abase = smem_u32(smem), bbase = abase + 96 * 1024;
        const uint32_t idesc = (KIND == 0 ? ((1u << 4) | (2u << 7) | (2u << 10)) : ((1u << 4) | (1u << 7) | (1u << 10)))
                               | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        uint64_t da[8], db[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            da[j] = umma_desc(abase + (uint32_t)((j % 3) * 19) * 16u + (uint32_t)((j & 3) * 2) * npix * 16u, npix * 16u, 128u);
            db[j] = umma_desc(bbase + (uint32_t)j * 2048u, (uint32_t)N * 16u, 128u);
        }
        long long t0 = clock64();
        if (nsplit == 1) {
            for (int r = 0; r < R; r += 8) {
#pragma unroll
                for (int j = 0; j < 8; ++j) mma<KIND>(tmem, da[j], db[j], idesc);
            }
        } else {
            for (int r = 0; r < R; r += 8) {
#pragma unroll
                for (int j = 0; j < 8; ++j) mma<KIND>(tmem + (uint32_t)((j & 1) * 256), da[j], db[j], idesc);
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main(int argc, char **argv) {
    const int NSPLIT = argc > 1 ? atoi(argv[1]) : 1;
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    long long h[148];
    const int R = 4096;
    cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    int Ns[] = {16, 32, 64, 96, 128, 192, 256};
    for (int kind = 0; kind < 2; ++kind)
        for (int N : Ns) {
            for (int rep = 0; rep < 2; ++rep) {
                if (kind == 0) bench<0><<<148, 128, 160 * 1024>>>(N, R, NSPLIT, d);
                else bench<1><<<148, 128, 160 * 1024>>>(N, R, NSPLIT, d);
            }
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double s = 0;
            for (int i = 0; i < 148; ++i) s += h[i];
            const double cyc = s / 148 / R;
            const double macs = 128.0 * N * (kind == 0 ? 8 : 16);
            printf("%s N=%3d: %6.1f cyc/mma  %7.0f MAC/cyc/SM  floor %5.1f  %s\n", kind == 0 ? "tf32" : "f16 ", N, cyc,
                   macs / cyc, 128.0 * N / 256, cudaGetErrorString(e));
        }
    return 0;
}
