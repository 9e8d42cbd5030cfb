// Microbenchmark: tcgen05.mma issue styles for the encoder's per-tile loop
// (9 taps x 2 K steps x {N=64, N=32} MMAs, A offset per tap, B offset per
// K group): (0) one thread, descriptors precomputed per MMA; (1) the
// warp-uniform loop with one elect per MMA and 32-bit descriptor adds (the
// kernels' style); (2) as (1) with one elect per tap (4 MMAs per asm block).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_issue mma_issue.cu
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
__device__ __forceinline__ void mma1(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_w(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\tmov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %6, 0;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t}\n" ::"r"(d), "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(id), "r"(acc));
}
// one elect for a tap's four MMAs
__device__ __forceinline__ void mma_tap(uint32_t d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t ahi,
                                        uint32_t b0, uint32_t b1, uint32_t bhi, uint32_t id64, uint32_t id32, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 x0, x1, x2, x3, y0, y1;\n\t"
        "mov.b64 x0, {%1, %5};\n\tmov.b64 x1, {%2, %5};\n\tmov.b64 x2, {%3, %5};\n\tmov.b64 x3, {%4, %5};\n\t"
        "mov.b64 y0, {%6, %8};\n\tmov.b64 y1, {%7, %8};\n\t"
        "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %11, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x0, y0, %9, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%12], x1, y0, %10, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x2, y1, %9, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%12], x3, y1, %10, 1;\n\t}\n"
        ::"r"(d), "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(ahi), "r"(b0), "r"(b1), "r"(bhi), "r"(id64), "r"(id32), "r"(acc),
        "r"(d + 32));
}

__global__ void bench(int mode, int tiles, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar, tb[2];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tb[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tb[1])));
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
    const uint32_t tmem = __shfl_sync(0xFFFFFFFFu, slot, 0);
    const uint32_t Wp = 18, rx = 422;
    const uint64_t dA = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(smem), 0), rx * 16u, 128u);
    const uint64_t dB = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(smem + 140 * 1024), 0), 64u * 16u, 128u);
    constexpr uint32_t id64 = idesc_f16(128, 64), id32 = idesc_f16(128, 32);
    long long t0 = clock64();
    if (warp == 1) {
        if (mode == 0) {
            if (threadIdx.x == 32) {
                for (int t = 0; t < tiles; ++t) {
                    const uint32_t d = tmem + (uint32_t)((t & 1) * 64);
                    const uint64_t dAt = dA + (uint64_t)(uint32_t)(19 + 128 * (t % 3) - Wp - 1);
#pragma unroll
                    for (int tap = 0; tap < 9; ++tap) {
                        const uint32_t off = (uint32_t)((tap / 3) * Wp + tap % 3);
#pragma unroll
                        for (int ks = 0; ks < 2; ++ks) {
                            const uint64_t ao = (uint64_t)(2u * ks * rx + off);
                            const uint64_t bo = (uint64_t)((tap * 4 + 2 * ks) * 64);
                            mma1(d, dAt + ao, dB + bo, id64, (tap | ks) ? 1u : 0u);
                            mma1(d + 32, dAt + ao + 4 * rx, dB + bo, id32, 1u);
                        }
                    }
                }
            }
        } else if (mode == 1) {
            const uint32_t ah = (uint32_t)(dA >> 32), bl = (uint32_t)dB, bh = (uint32_t)(dB >> 32);
            for (int t = 0; t < tiles; ++t) {
                const uint32_t d = tmem + (uint32_t)((t & 1) * 64);
                const uint32_t al = (uint32_t)dA + (uint32_t)(19 + 128 * (t % 3) - Wp - 1);
#pragma unroll
                for (int tap = 0; tap < 9; ++tap) {
                    const uint32_t off = (uint32_t)((tap / 3) * Wp + tap % 3);
#pragma unroll
                    for (int ks = 0; ks < 2; ++ks) {
                        const uint32_t ao = 2u * ks * rx + off;
                        const uint32_t bo = (uint32_t)((tap * 4 + 2 * ks) * 64);
                        mma_w(d, al + ao, ah, bl + bo, bh, id64, (tap | ks) ? 1u : 0u);
                        mma_w(d + 32, al + ao + 4 * rx, ah, bl + bo, bh, id32, 1u);
                    }
                }
            }
        } else if (mode == 2) {
            const uint32_t ah = (uint32_t)(dA >> 32), bl = (uint32_t)dB, bh = (uint32_t)(dB >> 32);
            for (int t = 0; t < tiles; ++t) {
                const uint32_t d = tmem + (uint32_t)((t & 1) * 64);
                const uint32_t al = (uint32_t)dA + (uint32_t)(19 + 128 * (t % 3) - Wp - 1);
#pragma unroll
                for (int tap = 0; tap < 9; ++tap) {
                    const uint32_t off = (uint32_t)((tap / 3) * Wp + tap % 3);
                    const uint32_t b0 = bl + (uint32_t)(tap * 4 * 64), b1 = b0 + 128u;
                    mma_tap(d, al + off, al + off + 4 * rx, al + off + 2 * rx, al + off + 6 * rx, ah, b0, b1, bh, id64, id32,
                            tap ? 1u : 0u);
                }
            }
        } else {
            // modes 3 / 4: as mode 1 plus a commit per tile onto the tile's
            // accumulator barrier; mode 4 also waits, before tile t, for tile
            // t - 2's commit (the accumulator it reuses) -- the trunk kernels'
            // loop with an instantaneous epilogue
            const uint32_t ah = (uint32_t)(dA >> 32), bl = (uint32_t)dB, bh = (uint32_t)(dB >> 32);
            for (int t = 0; t < tiles; ++t) {
                const int a = t & 1;
                if (mode == 4 && t >= 2) {
                    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(&tb[a])), "r"((uint32_t)(((t - 2) >> 1) & 1)) : "memory");
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                }
                const uint32_t d = tmem + (uint32_t)(a * 64);
                const uint32_t al = (uint32_t)dA + (uint32_t)(19 + 128 * (t % 3) - Wp - 1);
#pragma unroll
                for (int tap = 0; tap < 9; ++tap) {
                    const uint32_t off = (uint32_t)((tap / 3) * Wp + tap % 3);
#pragma unroll
                    for (int ks = 0; ks < 2; ++ks) {
                        const uint32_t ao = 2u * ks * rx + off;
                        const uint32_t bo = (uint32_t)((tap * 4 + 2 * ks) * 64);
                        mma_w(d, al + ao, ah, bl + bo, bh, id64, (tap | ks) ? 1u : 0u);
                        mma_w(d + 32, al + ao + 4 * rx, ah, bl + bo, bh, id32, 1u);
                    }
                }
                asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&tb[a])) : "memory");
            }
        }
        if (threadIdx.x == 32)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        long long t1 = clock64();
        if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    long long h[148];
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int tiles = 300;
    for (int mode = 0; mode < 5; ++mode) {
        for (int rep = 0; rep < 2; ++rep) bench<<<148, 128, 200 * 1024>>>(mode, tiles, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double s = 0;
        for (int i = 0; i < 148; ++i) s += h[i];
        printf("mode %d: %.1f cycles per MMA (%s)\n", mode, s / 148 / (tiles * 36.0), cudaGetErrorString(e));
    }
    return 0;
}
