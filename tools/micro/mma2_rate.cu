// Microbenchmark: tcgen05.mma issue rate, cta_group::1 (M=128, one SM) vs
// cta_group::2 (M=256 over a CTA pair, issued by the leader), kind::f16, SS
// operands, K-major, no swizzle. Patterns: one N per MMA, and the encoder's
// h / l pair (N=64 then N=32 on different A descriptors). Prints cycles per
// MMA instruction as seen by the issuing SM. A cta_group::2 instruction
// covers both SMs' 128-row halves, each SM reading its own A rows; measured,
// it costs the same ~44 cycles as a cta_group::1 M=128 MMA for N <= 64, so
// each SM still advances 128 rows per ~44 cycles: the pair halves the
// instructions to issue, not the time per row.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma2_rate mma2_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
template <int CG>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    if (CG == 1)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc));
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc));
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// mode 0: every MMA N (idesc n); mode 1: pairs N=64 (A_hi) + N=32 (A_lo)
template <int CG>
__global__ void bench(int N, int R, int mode, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (CG == 2) cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (threadIdx.x == 0 && rank == 0) {
        const uint32_t npix = 168;
        const uint32_t abase = smem_u32(smem), bbase = abase + 96 * 1024;
        const int M = 128 * CG;
        uint64_t da[8], db[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            da[j] = umma_desc(abase + (uint32_t)((j % 3) * 19) * 16u + (uint32_t)((j & 3) * 2) * npix * 16u, npix * 16u, 128u);
            db[j] = umma_desc(bbase + (uint32_t)j * 2048u, (uint32_t)(mode ? 64 : N) / CG * 16u, 128u);
        }
        const uint32_t id = idesc_f16(M, N), id64 = idesc_f16(M, 64), id32 = idesc_f16(M, 32);
        long long t0 = clock64();
        if (mode == 0) {
            for (int r = 0; r < R; r += 8) {
#pragma unroll
                for (int j = 0; j < 8; ++j) mma<CG>(tmem, da[j], db[j], id);
            }
        } else {
            for (int r = 0; r < R; r += 8) {
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                    mma<CG>(tmem, da[j], db[j], id64);
                    mma<CG>(tmem + 32, da[j + 1], db[j], id32);
                }
            }
        }
        if (CG == 1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
        asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    if (CG == 2 && threadIdx.x == 0 && rank == 1) {  // the peer's commit arrival
        asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (CG == 2) cluster_sync();
    if (warp == 0) {
        if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
        else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

int main() {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    long long h[148];
    const int R = 4096;
    cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    int Ns[] = {16, 32, 64, 128, 256};
    for (int mode = 0; mode < 2; ++mode)
        for (int cg = 1; cg <= 2; ++cg)
            for (int N : Ns) {
                if (mode == 1 && N != 64) continue;
                cudaMemset(d, 0, sizeof(h));
                for (int rep = 0; rep < 2; ++rep) {
                    if (cg == 1) {
                        bench<1><<<148, 128, 160 * 1024>>>(N, R, mode, d);
                    } else {
                        cudaLaunchConfig_t cfg = {};
                        cfg.gridDim = dim3(148);
                        cfg.blockDim = dim3(128);
                        cfg.dynamicSmemBytes = 160 * 1024;
                        cudaLaunchAttribute at[1];
                        at[0].id = cudaLaunchAttributeClusterDimension;
                        at[0].val.clusterDim.x = 2;
                        at[0].val.clusterDim.y = 1;
                        at[0].val.clusterDim.z = 1;
                        cfg.attrs = at;
                        cfg.numAttrs = 1;
                        cudaLaunchKernelEx(&cfg, bench<2>, N, R, mode, d);
                    }
                }
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                double s = 0;
                int k = 0;
                for (int i = 0; i < 148; ++i)
                    if (h[i]) s += h[i], ++k;
                const double cyc = s / (k ? k : 1) / R;
                printf("cta_group::%d %s N=%3d: %6.1f cycles per MMA instruction (each SM: one 128-row half)  %s\n", cg,
                       mode ? "pair 64+32" : "single    ", N, cyc, cudaGetErrorString(e));
            }
    return 0;
}
