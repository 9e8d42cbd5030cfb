// tcgen05 implicit-GEMM convolutions for the VQ-VAE decoder (sm_100a).
//
// Reference: vqvae.decode_to_params (vqvae.py:79-113) over nn.conv2d
// (nn.py:15-34), residual_block, pixel_shuffle and the logistic head.
//
// Activation layout ("padded group-major", bf16): for a batch of n images
// of H x W with a one-pixel edge-replicated border, Hp = H+2, Wp = W+2, the
// global pixel index q = n*Hp*Wp + y*Wp + x runs over every padded pixel of
// every image, and channel group g (8 channels, 16 bytes) lives in its own
// slab: elem(g, q, e) = act[(g*gstride + MARGIN + q)*8 + e]. Borders hold
// copies of the edge pixels, so nn.conv2d's edge padding is already in
// memory.
//
// GEMM view of a 3x3 conv: M = output pixels (virtual rows q: every padded
// position, outputs at border positions are discarded), N = output
// channels, K = 9 taps x C. A 128-row tile starting at q0 needs input
// pixels [q0 - Wp - 1, q0 + 128 + Wp + 1); one bulk copy per channel group
// brings that halo range into shared memory, and tap (i, j) is the same
// K-major no-swizzle UMMA operand shifted by (i*Wp + j) rows (16 bytes per
// row): no im2col, no per-tap copies. 9 taps x (C/16) tcgen05.mma
// (M=128, K=16) accumulate in TMEM.
//
// Warp roles (320 threads): warp 0 = bulk-copy producer (8-stage ring),
// warp 1 = TMEM allocator + MMA issuer (warp-uniform loop, elected lane),
// warps 2..9 = epilogue in two groups of four, one per TMEM accumulator
// (TMEM -> registers -> bias/residual/ReLU/pixel-shuffle/head -> global), so
// the epilogues of tiles i and i+1 overlap each other and the MMAs of i+2. Deterministic: fixed tiles, fixed K order, no
// atomics -- so a blob compressed on one GPU decodes on any other.

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "common.cuh"
#include "tc_conv.cuh"

namespace {

constexpr int kStages = 8;
constexpr int kThreadsTC = 320;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// waiting threads ask to be suspended until the phase completes (the hint
// bounds the suspension): a plain try_wait loop spins, and in these
// issue-bound kernels the spinning warps took ~30% of the issue slots
// (ncu, enc_front_tc_kernel)
constexpr uint32_t kSuspendNs = 0x989680;
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n\t"
        "DONE:\n\t"
        "}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(kSuspendNs)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, no swizzle (canonical interleave:
// core matrix = 8 rows x 16 B contiguous; LBO = next core matrix along K,
// SBO = next 8-row group along M/N).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// issued by one elected lane of a converged warp: the issue loop stays
// warp-uniform, so descriptors live in uniform registers and no per-MMA
// single-lane branch is needed
__device__ __forceinline__ void mma_bf16_elect(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t"
        ".reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit_elect(uint64_t *bar);

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// 32 consecutive f32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float *v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
        "[%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);  // .x = a (low half)
    return *reinterpret_cast<const uint32_t *>(&v);
}

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ float sigmoid_f32(float x) {
    if (x >= 0.f) return __fdiv_rn(1.f, __fadd_rn(1.f, expf(-x)));
    const float e = expf(x);
    return __fdiv_rn(e, __fadd_rn(1.f, e));
}

// q / d for q < 2^32 without the XU pipe: m = floor(2^32 / d) (host), the
// high product underestimates by at most one.
struct FastDiv {
    uint32_t d, m;
};
__host__ inline FastDiv make_fastdiv(uint32_t d) { return FastDiv{d, (uint32_t)(0x100000000ull / d)}; }
__device__ __forceinline__ uint32_t fdiv(uint32_t q, FastDiv f) {
    uint32_t n = __umulhi(q, f.m);
    if (q - n * f.d >= f.d) ++n;
    return n;
}

// store one 16-byte group at padded pixel q, plus its border copies
__device__ __forceinline__ void store_px(uint16_t *slab, int64_t q, uint4 v, int y, int x, int H, int W, int Wp) {
    uint4 *p = reinterpret_cast<uint4 *>(slab);
    p[q] = v;
    const int dy = (y == 1 ? -1 : 0), dy2 = (y == H ? 1 : 0);
    const int dx = (x == 1 ? -1 : 0), dx2 = (x == W ? 1 : 0);
    if (dy) p[q - Wp] = v;
    if (dy2) p[q + Wp] = v;
    if (dx) p[q - 1] = v;
    if (dx2) p[q + 1] = v;
    if (dy && dx) p[q - Wp - 1] = v;
    if (dy && dx2) p[q - Wp + 1] = v;
    if (dy2 && dx) p[q + Wp - 1] = v;
    if (dy2 && dx2) p[q + Wp + 1] = v;
}

// store_px into the pixel-pair layout: pixel q, channel group z lives in
// group z + 4 (q & 1) at row q / 2 (padded widths are even)
__device__ __forceinline__ void store_px_pair(uint16_t *out, int64_t gs, int64_t mg, int z, int64_t q, uint4 v, int y,
                                              int x, int H, int W, int Wp) {
    auto put = [&](int64_t qq) { reinterpret_cast<uint4 *>(out + ((int64_t)(z + 4 * (int)(qq & 1)) * gs + mg) * 8)[qq >> 1] = v; };
    put(q);
    const int dy = (y == 1 ? -1 : 0), dy2 = (y == H ? 1 : 0);
    const int dx = (x == 1 ? -1 : 0), dx2 = (x == W ? 1 : 0);
    if (dy) put(q - Wp);
    if (dy2) put(q + Wp);
    if (dx) put(q - 1);
    if (dx2) put(q + 1);
    if (dy && dx) put(q - Wp - 1);
    if (dy && dx2) put(q - Wp + 1);
    if (dy2 && dx) put(q + Wp - 1);
    if (dy2 && dx2) put(q + Wp + 1);
}

template <int N, int KS, int MODE>
__global__ void __launch_bounds__(kThreadsTC, 1) tc_conv_kernel(TcLayer L) {
    const int kS = L.n_stages;  // copy ring depth (launcher: as many as fit, <= kStages)
    // HEAD2: the head over pixel pairs (pair layout: row = two horizontally
    // adjacent pixels, 8 channel groups: even pixel 0..3, odd pixel 4..7)
    constexpr bool PAIR = MODE == TC_OUT_HEAD2;
    constexpr bool HEADM = MODE == TC_OUT_HEAD || PAIR;
    constexpr int C = PAIR ? 64 : 32;   // input channels per row
    constexpr int NG = C / 8;
    constexpr int KG = PAIR ? 48 : KS * KS * NG;  // K core-matrix groups (HEAD2: 3 row taps x 128)
    constexpr int TMEM_COLS = (2 * N < 32) ? 32 : 2 * N;
    const int Wp = L.Wp;
    const int npix = KS == 3 ? ((128 + 2 * Wp + 2 + 7) & ~7) : 128;
    const uint32_t stage_bytes = (uint32_t)NG * npix * 16;

    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *s_w = smem;                                   // KG x N x 16 B
    uint8_t *s_a = smem + (size_t)KG * N * 16;             // kStages x NG x npix x 16 B
    uint64_t *bars = reinterpret_cast<uint64_t *>(s_a + (size_t)kS * stage_bytes);
    uint64_t *full = bars;                 // [kStages]
    uint64_t *empty = bars + kS;      // [kStages]
    uint64_t *tfull = bars + 2 * kS;  // [2]
    uint64_t *tempty = tfull + 2;          // [2]
    uint64_t *wbar = tempty + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(wbar + 1);
    float *s_bias = reinterpret_cast<float *>(wbar + 2);  // N floats
    float *s_thr = s_bias + N;                            // head: n_thresh floats

    const int warp = __shfl_sync(0xFFFFFFFFu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    for (int c = threadIdx.x; c < N; c += blockDim.x) s_bias[c] = c < (HEADM ? 6 : N) ? L.bias[c] : 0.f;
    if constexpr (HEADM) {
        for (int k = threadIdx.x; k < L.n_thresh; k += blockDim.x) s_thr[k] = __double2float_rd(L.thresh[k]);
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);
        }
        mbar_init(wbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"((uint32_t)TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xFFFFFFFFu, *tmem_slot, 0);

    const int64_t n_tiles = L.n_tiles;
    if (warp == 0) {
        if (lane == 0) {
            const uint32_t wbytes = (uint32_t)KG * N * 16;
            mbar_expect_tx(wbar, wbytes);
            bulk_g2s(s_w, L.wts, wbytes, wbar);
            int i = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
                const int s = i % kS;
                const int r = i / kS;
                if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
                const int64_t q_lo = t * 128 - (KS == 3 ? (Wp + 1) : 0);
                mbar_expect_tx(&full[s], stage_bytes);
                uint8_t *dst = s_a + (size_t)s * stage_bytes;
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    const uint16_t *src = L.in + ((int64_t)g * L.gstride + L.margin + q_lo) * 8;
                    bulk_g2s(dst + (size_t)g * npix * 16, src, (uint32_t)npix * 16, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        // warp-uniform issue loop, one elected lane per MMA (see tc3)
        constexpr uint32_t idesc = idesc_bf16(128, N);
        mbar_wait(wbar, 0);
        tc_fence_after();
        const uint64_t dA0 = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_a), 0), (uint32_t)npix * 16u, 128u);
        const uint64_t dB0 = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_w), 0), (uint32_t)N * 16u, 128u);
        const uint32_t npx = (uint32_t)npix;
        int i = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
            const int s = i % kS;
            const int a = i & 1;
            const int u = i >> 1;
            if (u > 0) mbar_wait(&tempty[a], (u - 1) & 1);
            mbar_wait(&full[s], (i / kS) & 1);
            tc_fence_after();
            const uint64_t dA = dA0 + (uint64_t)((uint32_t)s * (stage_bytes >> 4));
            const uint32_t d = tmem + (uint32_t)(a * N);
            if constexpr (PAIR) {
                // per row tap di, 8 K steps of 16 channels: the left pair's odd
                // pixel (groups 4-7, one row back), this pair (0-7), the right
                // pair's even pixel (0-3, one row on)
#pragma unroll
                for (int di = 0; di < 3; ++di) {
#pragma unroll
                    for (int sg = 0; sg < 8; ++sg) {
                        const uint32_t slab = (sg < 2) ? 4u + 2u * sg : (sg < 6 ? 2u * (sg - 2) : 2u * (sg - 6));
                        const uint32_t dj = sg < 2 ? 0u : (sg < 6 ? 1u : 2u);
                        const uint32_t off = (uint32_t)di * (uint32_t)Wp + dj;
                        mma_bf16_elect(d, dA + (uint64_t)(slab * npx + off), dB0 + (uint64_t)((2 * (di * 8 + sg)) * N),
                                       idesc, (di | sg) ? 1u : 0u);
                    }
                }
            } else {
#pragma unroll
                for (int tap = 0; tap < KS * KS; ++tap) {
                    const uint32_t off = KS == 3 ? (uint32_t)((tap / KS) * Wp + tap % KS) : 0u;
#pragma unroll
                    for (int ks = 0; ks < NG / 2; ++ks)
                        mma_bf16_elect(d, dA + (uint64_t)(2u * ks * npx + off), dB0 + (uint64_t)((tap * NG + 2 * ks) * N),
                                       idesc, (tap | ks) ? 1u : 0u);
                }
            }
            mma_commit_elect(&empty[s]);
            mma_commit_elect(&tfull[a]);
        }
    } else {
        // epilogue: two groups of four warps (2..5, 6..9), group g owns the
        // tiles with i % 2 == g and accumulator buffer g, so one group's
        // epilogue overlaps the other's; warp w reads TMEM lanes 32*(w%4) .. +31
        const int grp = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int H = L.H, W = L.W;
        const FastDiv div_hw{(uint32_t)(L.Hp * Wp), (uint32_t)(0x100000000ull / (uint32_t)(L.Hp * Wp))};
        const FastDiv div_w{(uint32_t)Wp, (uint32_t)(0x100000000ull / (uint32_t)Wp)};
        constexpr int NB = HEADM ? 6 : N;
        float bias[MODE == TC_OUT_ACT ? NB : 1];
        if constexpr (MODE == TC_OUT_ACT) {
#pragma unroll
            for (int c = 0; c < NB; ++c) bias[c] = L.bias[c];
        }
        int i = grp;
        for (int64_t t = blockIdx.x + (int64_t)grp * gridDim.x; t < n_tiles; t += 2 * (int64_t)gridDim.x, i += 2) {
            const int a = grp;
            const int u = i >> 1;
            const uint32_t q = (uint32_t)t * 128u + (uint32_t)row;
            const uint32_t n = fdiv(q, div_hw);
            const uint32_t rem = q - n * div_hw.d;
            const int y = (int)fdiv(rem, div_w);
            // HEAD2 rows are pixel pairs: x is the even pixel of the pair
            const int x = PAIR ? 2 * (int)(rem - (uint32_t)y * div_w.d) : (int)(rem - (uint32_t)y * div_w.d);
            const bool valid = n < (uint64_t)L.n_img && y >= 1 && y <= H && x >= 1 && x <= W;
            // residual prefetch: independent of the accumulator, issue before the wait
            uint4 rv[4];
            if constexpr (MODE == TC_OUT_ACT) {
                if (L.resid && valid) {
#pragma unroll
                    for (int g = 0; g < 4; ++g)
                        rv[g] = reinterpret_cast<const uint4 *>(L.resid + ((int64_t)g * L.gstride + L.margin) * 8)[q];
                }
            }
            mbar_wait(&tfull[a], u & 1);
            tc_fence_after();
            const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(a * N);
            if constexpr (MODE == TC_OUT_ACT) {
                float v[32];
                tmem_ld32(taddr, v);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[a]);
                if (valid) {
                    uint4 w4[4];
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        float o[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) o[e] = __fadd_rn(v[8 * g + e], bias[8 * g + e]);
                        if (L.resid) {
                            const uint32_t rw[4] = {rv[g].x, rv[g].y, rv[g].z, rv[g].w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                o[2 * e] = __fadd_rn(bf16_lo(rw[e]), o[2 * e]);
                                o[2 * e + 1] = __fadd_rn(bf16_hi(rw[e]), o[2 * e + 1]);
                            }
                        }
                        if (L.relu) {
#pragma unroll
                            for (int e = 0; e < 8; ++e) o[e] = fmaxf(o[e], 0.f);
                        }
                        w4[g] = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]),
                                           pack_bf16(o[6], o[7]));
                    }
#pragma unroll
                    for (int g = 0; g < 4; ++g)
                        store_px(L.out + ((int64_t)g * L.out_gstride + L.out_margin) * 8, q, w4[g], y, x, H, W, Wp);
                }
            } else if constexpr (MODE == TC_OUT_SHUFFLE) {
                // N = 128 = 4 chunks of 32 columns: chunk z holds output
                // channels c = 8z..8z+7 at all four (dy, dx) sub-positions
                const int H2 = 2 * H, W2 = 2 * W, Wp2 = W2 + 2;
                const int64_t hw2 = (int64_t)(H2 + 2) * Wp2;
#pragma unroll 1
                for (int z = 0; z < 4; ++z) {
                    float v[32];
                    tmem_ld32(taddr + (uint32_t)(32 * z), v);
                    if (z == 3) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[a]);
                    }
                    if (!valid) continue;
                    float bz[32];  // this chunk's 32 biases: 8 vector loads instead of 32 scalar ones
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float4 b4 = reinterpret_cast<const float4 *>(s_bias + 32 * z)[e];
                        bz[4 * e] = b4.x;
                        bz[4 * e + 1] = b4.y;
                        bz[4 * e + 2] = b4.z;
                        bz[4 * e + 3] = b4.w;
                    }
#pragma unroll
                    for (int sub = 0; sub < 4; ++sub) {
                        const int dy = sub >> 1, dx = sub & 1;
                        float o[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) o[e] = fmaxf(__fadd_rn(v[4 * e + sub], bz[4 * e + sub]), 0.f);
                        const int Y = 2 * (y - 1) + dy + 1, X = 2 * (x - 1) + dx + 1;
                        const int64_t q2 = (int64_t)n * hw2 + (int64_t)Y * Wp2 + X;
                        const uint4 w4 = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]),
                                                    pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
                        if (L.pair_out)
                            store_px_pair(L.out, L.out_gstride, L.out_margin, z, q2, w4, Y, X, H2, W2, Wp2);
                        else
                            store_px(L.out + ((int64_t)z * L.out_gstride + L.out_margin) * 8, q2, w4, Y, X, H2, W2, Wp2);
                    }
                }
            } else {
                // logistic head (vqvae.py:105-112, logistic.py:36-40, 109-114)
                float v[16];
                tmem_ld16(taddr, v);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[a]);
                auto head_px = [&](const float *vv, int xx) {
                    if (!(n < (uint64_t)L.n_img && y >= 1 && y <= H && xx >= 1 && xx <= W)) return;
                    if (!((y - 1) < L.crop_h && (xx - 1) < L.crop_w)) return;
                    const int64_t px = ((int64_t)n * L.crop_h + (y - 1)) * (int64_t)L.crop_w + (xx - 1);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        float av = __fadd_rn(vv[c], s_bias[c]);
                        av = fminf(fmaxf(av, -15.f), 15.f);
                        // fast intrinsics: the decoder is its own reference (compress
                        // and decompress run this same code), so only determinism
                        // matters, and mu / s stay within ~1e-6 of the f32 formulas
                        const float mu = __fmul_rn(255.f, __fdividef(1.f, 1.f + __expf(-av)));
                        float bv = __fadd_rn(vv[3 + c], s_bias[3 + c]);
                        bv = fminf(fmaxf(bv, L.log_s_min), L.log_s_max);
                        float sv = fminf(fmaxf(__expf(bv), 0.5f), 64.f);
                        // round_half_away(mu), mu >= 0, exact in f32: frac is exact
                        const float fl = floorf(mu);
                        const int shift = (int)fl + (__fsub_rn(mu, fl) >= 0.5f ? 1 : 0);
                        // s > t_k (f64)  <=>  s > rd32(t_k): no float lies in (rd32, t_k]
                        int d = 0;
                        for (int k = 0; k < L.n_thresh; ++k) d += sv > s_thr[k];
                        L.shift[px * 3 + c] = (uint8_t)shift;
                        L.dsel[px * 3 + c] = (uint8_t)d;
                        if (L.mu) L.mu[px * 3 + c] = mu;
                        if (L.s) L.s[px * 3 + c] = sv;
                    }
                };
                head_px(v, x);
                if constexpr (PAIR) head_px(v + 6, x + 1);  // columns 6..11: the odd pixel
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)TMEM_COLS));
    }
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// Round to tf32 (10 mantissa bits), nearest with ties away from zero, in
// integer ops (cvt.rna.tf32 issues on the XU pipe). Finite inputs only.
__device__ __forceinline__ float tf32_rna(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// Encoder conv, C = 32 in, N = 32 out, as a 3-product fp16 split on
// tcgen05 kind::f16: fp32-class accuracy at twice the tf32 MMA rate (an
// SS-mode MMA with N <= 64 is bound by reading its operands from shared
// memory, and an fp16 K=16 step reads as many bytes as a tf32 K=8 step).
//
// Operands. Each activation tensor A_j is stored as two fp16 slab sets per
// image scale 2^k (k = kx[j][n] for image n): x 2^k = h + l 2^-11 with
// h = fp16(x 2^k), l = fp16((x 2^k - h) 2^11) (error <= 2^-22 |x 2^k|; tiny
// values stay exact to 2^-36 absolute); weights likewise with 2^kw. Then
//   conv = [sum h hw + 2^-11 sum (h lw + l hw)] 2^-(k + kw),
// the dropped l lw term being <= 2^-22 |x||w|. D[0:32] = sum h hw and
// D[32:64] = sum (h lw + l hw) accumulate in fp32 TMEM: per K=16 step one MMA
// A_hi x [W_hi | W_lo] (N=64) and one A_lo x W_hi (N=32) into D[32:64].
//
// Scales. The epilogue writing A_j must pick k before A_j is complete, so it
// uses a rigorous per-image bound: |out| <= max|in| L1 + max|b| (+ max|res|),
// L1 = max_co sum |w|, from the exact per-image maxima of its inputs (which
// earlier kernels recorded with atomicMax: order-independent, so nothing
// depends on the batch or the tiling); k puts the bound below 2^15 < 65504.
// It also records the exact max of its own output for the next layer.
// Block outputs are kept in fp32 as well: the residual add is exact.
//
// Warps: 0 bulk-copy producer (hi / lo slabs, ring of kStages3), 1 TMEM +
// MMA issuer (warp-uniform loop, elected lane), 2..9 epilogue in two groups
// of four (one per accumulator buffer, so one group's epilogue overlaps the
// other's), 10 residual producer (bulk copies of the fp32 block input).
constexpr int kStages3 = 6;
constexpr int kThreadsTC3 = 352;

// kind::f16 instruction descriptor: D f32, A/B fp16, both K-major.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// issued by one elected lane of a converged warp (keeps the issue loop
// warp-uniform: descriptors stay in uniform registers)
__device__ __forceinline__ void mma_f16_elect(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t"
        ".reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// as mma_f16_elect with the descriptors as (low, high) words: the address
// offsets are added to the low word only (shared-memory addresses < 2^18 never
// carry out of the 14-bit field), one 32-bit add per descriptor
__device__ __forceinline__ void mma_f16_elect_w(uint32_t d_tmem, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi,
                                                uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t"
        ".reg .pred p, e;\n\t"
        ".reg .b64 da, db;\n\t"
        "mov.b64 da, {%1, %2};\n\t"
        "mov.b64 db, {%3, %4};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t"
        "}\n" ::"r"(d_tmem),
        "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc));
}

// bf16 twin of mma_f16_elect_w
__device__ __forceinline__ void mma_bf16_elect_w(uint32_t d_tmem, uint32_t alo, uint32_t ahi, uint32_t blo,
                                                 uint32_t bhi, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t"
        ".reg .pred p, e;\n\t"
        ".reg .b64 da, db;\n\t"
        "mov.b64 da, {%1, %2};\n\t"
        "mov.b64 db, {%3, %4};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t"
        "}\n" ::"r"(d_tmem),
        "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit_elect(uint64_t *bar) {
    asm volatile(
        "{\n\t"
        ".reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t"
        "}\n" ::"r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ float exp2i(int k) { return __int_as_float((127 + k) << 23); }

// scale exponent k for a per-image bound with float bits `mb`: |x 2^k| < 2^15.
// k in [-90, 90] and kw in [-30, 30] keep 2^k and 2^-(k + kw) normal.
__device__ __forceinline__ int act_exp(uint32_t mb) {
    int k = 0;
    if (mb != 0u && mb < 0x7F800000u) k = 14 - ((int)(mb >> 23) - 127);
    return min(max(k, -90), 90);
}

// fp16 pair (h, l) of two scaled values, packed two per 32-bit word
__device__ __forceinline__ void split2(float a, float b, uint32_t &h, uint32_t &l) {
    const __half2 hh = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(hh);
    const __half2 ll = __floats2half2_rn(__fmul_rn(__fsub_rn(a, hf.x), 2048.f), __fmul_rn(__fsub_rn(b, hf.y), 2048.f));
    h = *reinterpret_cast<const uint32_t *>(&hh);
    l = *reinterpret_cast<const uint32_t *>(&ll);
}

template <int KS, int MODE>
__global__ void __launch_bounds__(kThreadsTC3, 1) tc3_conv_kernel(Tc3Layer L) {
    const int kS = L.n_stages;  // copy ring depth (launcher: as many as fit, <= kStages3)
    constexpr int N = 32;
    constexpr int N2 = 64;  // B' = [W_hi | W_lo] along N
    constexpr int NH = 4;   // 8-channel fp16 groups
    constexpr int KG = KS * KS * NH;
    constexpr int TMEM_COLS = 2 * N2;
    const int Wp = L.Wp;
    const int npix = KS == 3 ? ((128 + 2 * Wp + 2 + 7) & ~7) : 128;
    const uint32_t h_bytes = (uint32_t)NH * npix * 16;
    const uint32_t stage_bytes = 2 * h_bytes;
    const uint32_t wbytes = (uint32_t)KG * N2 * 16;

    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *s_w = smem;
    uint8_t *s_a = smem + (size_t)wbytes;
    const bool has_res = MODE == TC3_ACT && L.res != nullptr;
    float4 *s_res = reinterpret_cast<float4 *>(s_a + (size_t)kS * stage_bytes);  // [2][8][128]
    uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(s_res) + (has_res ? 2 * 8 * 128 * 16 : 0));
    uint64_t *full = bars;
    uint64_t *empty = bars + kS;
    uint64_t *tfull = bars + 2 * kS;
    uint64_t *tempty = tfull + 2;
    uint64_t *rfull = tempty + 2;
    uint64_t *rempty = rfull + 2;
    uint64_t *wbar = rempty + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(wbar + 1);

    const int warp = __shfl_sync(0xFFFFFFFFu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);
            mbar_init(&rfull[a], 1);
            mbar_init(&rempty[a], 4);
        }
        mbar_init(wbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"((uint32_t)TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xFFFFFFFFu, *tmem_slot, 0);
    const int64_t n_tiles = L.n_tiles;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(wbar, wbytes);
            bulk_g2s(s_w, L.w, wbytes, wbar);
            int i = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
                const int s = i % kS;
                const int r = i / kS;
                if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
                const int64_t q_lo = t * 128 - (KS == 3 ? (Wp + 1) : 0);
                mbar_expect_tx(&full[s], stage_bytes);
                uint8_t *dst = s_a + (size_t)s * stage_bytes;
#pragma unroll
                for (int g = 0; g < 2 * NH; ++g) {  // hi groups 0..3, lo groups 4..7
                    const int64_t off = ((int64_t)g * L.gstride + L.margin + q_lo) * 8;
                    bulk_g2s(dst + (size_t)g * npix * 16, L.in + off, (uint32_t)npix * 16, &full[s]);
                }
            }
        }
    } else if (warp == 10) {
        // residual producer: the block input rows of tile i (8 fp32 groups x
        // 128 rows) into buffer i % 2 for the epilogue group that owns it
        if (has_res && lane == 0) {
            int i = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
                const int a = i & 1;
                const int u = i >> 1;
                if (u > 0) mbar_wait(&rempty[a], (u - 1) & 1);
                mbar_expect_tx(&rfull[a], 8 * 128 * 16);
#pragma unroll
                for (int g = 0; g < 8; ++g)
                    bulk_g2s(s_res + (a * 8 + g) * 128, L.res + ((int64_t)g * L.gstride + L.margin + t * 128) * 4,
                             128 * 16, &rfull[a]);
            }
        }
    } else if (warp == 1) {
        // the whole warp runs the (warp-uniform) issue loop; one elected lane
        // issues each MMA. Descriptors: base + offsets in 16-byte units (the
        // address field cannot carry: smem addresses are < 2^18).
        constexpr uint32_t idesc64 = idesc_f16(128, N2);
        constexpr uint32_t idesc32 = idesc_f16(128, N);
        mbar_wait(wbar, 0);
        tc_fence_after();
        const uint64_t dA0 = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_a), 0), (uint32_t)npix * 16u, 128u);
        const uint64_t dB0 = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_w), 0), (uint32_t)N2 * 16u, 128u);
        const uint32_t npx = (uint32_t)npix;
        int i = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
            const int s = i % kS;
            const int a = i & 1;
            const int u = i >> 1;
            if (u > 0) mbar_wait(&tempty[a], (u - 1) & 1);
            mbar_wait(&full[s], (i / kS) & 1);
            tc_fence_after();
            const uint64_t dAh = dA0 + (uint64_t)((uint32_t)s * (stage_bytes >> 4));
            const uint64_t dAl = dAh + (uint64_t)(h_bytes >> 4);
            const uint32_t d = tmem + (uint32_t)(a * N2);
#pragma unroll
            for (int tap = 0; tap < KS * KS; ++tap) {
                const uint32_t off = KS == 3 ? (uint32_t)((tap / KS) * Wp + tap % KS) : 0u;
#pragma unroll
                for (int ks = 0; ks < NH / 2; ++ks) {
                    const uint64_t ao = (uint64_t)(2u * ks * npx + off);
                    const uint64_t bo = (uint64_t)((tap * NH + 2 * ks) * N2);
                    mma_f16_elect(d, dAh + ao, dB0 + bo, idesc64, (tap | ks) ? 1u : 0u);  // D[0:32] += h hw, D[32:64] += h lw
                    mma_f16_elect(d + N, dAl + ao, dB0 + bo, idesc32, 1u);                // D[32:64] += l hw
                }
            }
            mma_commit_elect(&empty[s]);
            mma_commit_elect(&tfull[a]);
        }
    } else {
        // two epilogue groups of four warps (one per TMEM lane quarter);
        // group g owns the tiles with i % 2 == g and accumulator buffer g
        const int grp = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int H = L.H, W = L.W;
        const uint32_t img_px = (uint32_t)(L.Hp * Wp);
        const FastDiv div_hw{img_px, (uint32_t)(0x100000000ull / img_px)};
        const FastDiv div_w{(uint32_t)Wp, (uint32_t)(0x100000000ull / (uint32_t)Wp)};
        const int kw = __float_as_int(L.meta[0]);
        const float l1 = L.meta[1], bmax = L.meta[2];
        float bias[N];
#pragma unroll
        for (int c = 0; c < N; ++c) bias[c] = L.bias[c];
        // per-row image scalars are fetched one tile ahead
        int kx_n = 0;
        uint32_t mx_n = 0, mr_n = 0;
        auto fetch = [&](int64_t t) {
            const uint32_t q = (uint32_t)t * 128u + (uint32_t)row;
            const uint32_t n = fdiv(q, div_hw);
            if (t < n_tiles && n < (uint64_t)L.n_img) {
                kx_n = L.kx_in[n];
                if constexpr (MODE == TC3_ACT) {
                    mx_n = L.mx_in[n];
                    if (L.res) mr_n = L.mx_res[n];
                }
            }
        };
        int i = grp;
        int64_t t = blockIdx.x + (int64_t)grp * gridDim.x;
        fetch(t);
        for (; t < n_tiles; t += 2 * (int64_t)gridDim.x, i += 2) {
            const int a = grp;
            const int u = i >> 1;
            const uint32_t q = (uint32_t)t * 128u + (uint32_t)row;
            const uint32_t n = fdiv(q, div_hw);
            const uint32_t rem = q - n * div_hw.d;
            const int y = (int)fdiv(rem, div_w), x = (int)(rem - (uint32_t)y * div_w.d);
            const bool valid = n < (uint64_t)L.n_img && y >= 1 && y <= H && x >= 1 && x <= W;
            const int kxi = kx_n;
            const uint32_t mxi = mx_n, mri = mr_n;
            fetch(t + 2 * (int64_t)gridDim.x);
            float inv = 1.f, osc = 1.f;
            int ko = 0;
            if (valid) {
                inv = exp2i(-kxi - kw);
                if constexpr (MODE == TC3_ACT) {
                    // rigorous bound on |out| for this image -> output scale 2^ko
                    float bound = __fadd_rn(__fmul_rn(__uint_as_float(mxi), l1), bmax);
                    if (L.res) bound = __fadd_rn(bound, __uint_as_float(mri));
                    ko = act_exp(__float_as_uint(bound));
                    osc = exp2i(ko);
                }
            }
            mbar_wait(&tfull[a], u & 1);
            tc_fence_after();
            const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(a * N2);
            float v[32];
            {
                float w[32];
                tmem_ld32(taddr, v);
                tmem_ld32(taddr + 32, w);
#pragma unroll
                for (int c = 0; c < 32; ++c)  // products by powers of two are exact: 2 roundings, as unfused
                    v[c] = __fmaf_rn(__fmaf_rn(w[c], 0.00048828125f, v[c]), inv, bias[c]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[a]);
            if constexpr (MODE == TC3_ACT) {
                float mx = 0.f;
                if (has_res) mbar_wait(&rfull[a], u & 1);
                if (valid) {
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        if (has_res) {
                            const float4 r = s_res[(a * 8 + g) * 128 + row];
                            v[4 * g + 0] = __fadd_rn(r.x, v[4 * g + 0]);
                            v[4 * g + 1] = __fadd_rn(r.y, v[4 * g + 1]);
                            v[4 * g + 2] = __fadd_rn(r.z, v[4 * g + 2]);
                            v[4 * g + 3] = __fadd_rn(r.w, v[4 * g + 3]);
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            if (L.relu) v[4 * g + e] = fmaxf(v[4 * g + e], 0.f);
                            mx = fmaxf(mx, fabsf(v[4 * g + e]));
                        }
                        if (L.out32) {
                            const int64_t so = ((int64_t)g * L.gstride + L.margin) * 4;
                            // fp32 copy: valid pixels only (no reader uses its edge copies)
                            reinterpret_cast<float4 *>(L.out32 + so)[q] =
                                make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < NH; ++j) {
                        uint4 h, l;
                        split2(__fmul_rn(v[8 * j + 0], osc), __fmul_rn(v[8 * j + 1], osc), h.x, l.x);
                        split2(__fmul_rn(v[8 * j + 2], osc), __fmul_rn(v[8 * j + 3], osc), h.y, l.y);
                        split2(__fmul_rn(v[8 * j + 4], osc), __fmul_rn(v[8 * j + 5], osc), h.z, l.z);
                        split2(__fmul_rn(v[8 * j + 6], osc), __fmul_rn(v[8 * j + 7], osc), h.w, l.w);
                        store_px(L.out + ((int64_t)j * L.gstride + L.margin) * 8, q, h, y, x, H, W, Wp);
                        store_px(L.out + ((int64_t)(NH + j) * L.gstride + L.margin) * 8, q, l, y, x, H, W, Wp);
                    }
                }
                if (has_res) {  // loads consumed above; the next fill is an async-proxy write
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&rempty[a]);
                }
                // per-image exact max |out| and the output scale: one write
                // per warp when the warp's rows share an image
                const uint32_t n_ref = __shfl_sync(0xFFFFFFFFu, n, 0);
                const bool same = __all_sync(0xFFFFFFFFu, n == n_ref && valid);
                if (same) {
                    const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(mx));
                    if (lane == 0) {
                        if (m != 0u) atomicMax(L.mx_out + n_ref, m);
                        L.kx_out[n_ref] = ko;
                    }
                } else if (valid) {
                    if (mx != 0.f) atomicMax(L.mx_out + n, __float_as_uint(mx));
                    L.kx_out[n] = ko;
                }
            } else {
                if (!valid) continue;
                // z = acc + bias, written as tf32 hi / fp32 lo into 128-latent
                // tiles in the UMMA K-major layout the argmin GEMM reads
                const int64_t vix = ((int64_t)n * H + (y - 1)) * (int64_t)W + (x - 1);
                float4 *zo = L.z ? reinterpret_cast<float4 *>(L.z + vix * 32) : nullptr;
                float4 *zt = reinterpret_cast<float4 *>(L.zt) + (vix >> 7) * (2 * 8 * 128) + (vix & 127);
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    float hi[4], lo[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        hi[e] = tf32_rna(v[4 * g + e]);
                        lo[e] = __fsub_rn(v[4 * g + e], hi[e]);
                    }
                    if (zo) zo[g] = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
                    zt[g * 128] = make_float4(hi[0], hi[1], hi[2], hi[3]);
                    zt[(8 + g) * 128] = make_float4(lo[0], lo[1], lo[2], lo[3]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)TMEM_COLS));
    }
}

template <int KS, int MODE>
int launch_tc3(const Tc3Layer &L, cudaStream_t s) {
    constexpr int KG = KS * KS * 4;
    const int npix = KS == 3 ? ((128 + 2 * L.Wp + 2 + 7) & ~7) : 128;
    // ring depth: kStages3, or as many stages as fit for wide images (>= 2)
    auto smem_of = [&](int k) {
        return (size_t)KG * 64 * 16 + (size_t)k * 8 * npix * 16 + (L.res ? 2 * 8 * 128 * 16 : 0) + 8 * (2 * k + 9) + 16;
    };
    int st = kStages3;
    while (st > 2 && smem_of(st) > 227 * 1024) --st;
    const size_t smem = smem_of(st);
    if ((uint64_t)L.n_img * L.Hp * L.Wp >= (1ull << 31)) return PILC_E_UNSUPPORTED;  // 32-bit pixel index
    if (smem > 227 * 1024) return PILC_E_UNSUPPORTED;
    Tc3Layer Ls = L;
    Ls.n_stages = st;
    auto kern = tc3_conv_kernel<KS, MODE>;
    allow_dyn_smem(reinterpret_cast<const void *>(kern));
    int per_sm = (int)((227 * 1024) / (smem + 1024));
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)sm_count() * per_sm;
    if (grid > L.n_tiles) grid = L.n_tiles;
    if (grid < 1) return PILC_OK;
    const double flops = 2.0 * L.n_img * L.H * L.W * 32.0 * 32 * KS * KS;
    ProfScope _ps(PROF_TC3_CONV, s, flops);
    kern<<<(unsigned)grid, kThreadsTC3, smem, s>>>(Ls);
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

// ---- one encoder residual block per launch (vqvae.py:60-62) -----------------
// conv1 and conv2 of a block with the intermediate T = relu(conv1(X)) kept in
// shared memory: per CTA iteration one image's padded X hi / lo rows (tile
// halo included) come in by bulk copy, conv1's epilogue writes T hi / lo
// (edge copies included) into shared memory, and conv2 reads it from there.
// The arithmetic is exactly that of two tc3 ACT launches (same MMAs in the
// same K order, same epilogue roundings, same per-image scales), so results
// are bit-identical to the unfused path; what goes away is T's HBM round
// trip and one launch.
//
// Schedule (one image i per iteration, T = ceil(Hp Wp / 128) tiles per
// conv): MMA issues conv1 tiles of i, commits `xfree` (X(i+1) may load),
// then conv2 tile j as soon as conv1 tiles j - 1 .. j + 1 are in T
// (`hrdy[j]`, per tile). Accumulators alternate over a global tile counter
// as in tc3; conv2 residual rows are loaded by the epilogue threads while
// the MMAs run. The per-image max of T (the conv2 output bound) is reduced
// through per-(tile, quarter) slots, double-buffered by image parity, and
// read after `hready` (all conv1 epilogues of the image done).
//
// Measured (B200, 8192 CIFAR images): ~460 us per block vs 525 us for the
// two tc3 launches. The epilogue (global fp32 + hi / lo stores, residual
// loads) and the MMA issue loop (~115 cycles per h/l MMA pair against a
// ~96-cycle operand floor) bound it, not the conv1 -> conv2 dependency.
constexpr int kThreadsBK = 320;
constexpr int kBkMaxTiles = 8;

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__global__ void __launch_bounds__(kThreadsBK, 1) tc3_block_kernel(Tc3Block L) {
    constexpr int N = 32, N2 = 64, NH = 4, KG = 36;
    constexpr uint32_t WB = KG * N2 * 16;
    const int Wp = L.Wp, HW = L.Hp * Wp;
    const int T = (HW + 127) >> 7;
    const int M0 = (Wp + 1 + 7) & ~7;
    const int RX = M0 + T * 128 + M0;
    const uint32_t slab = (uint32_t)RX * 16u;
    const int nrows = HW + 2 * (Wp + 1);

    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *s_w1 = smem;
    uint8_t *s_w2 = smem + WB;
    uint8_t *s_x = smem + 2 * WB;
    uint8_t *s_h = s_x + 8 * (size_t)slab;
    uint64_t *bars = reinterpret_cast<uint64_t *>(s_h + 8 * (size_t)slab);
    uint64_t *xfull = bars, *xfree = bars + 1, *hready = bars + 2, *wbar = bars + 3;
    uint64_t *tfull = bars + 4, *tempty = bars + 6;
    uint64_t *hrdy = bars + 12;  // [kBkMaxTiles]: conv1 tile j of the image is in T
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 12 + kBkMaxTiles);
    uint32_t *part = tmem_slot + 4;            // [2][kBkMaxTiles][4] max |T| per tile quarter
    float *s_b = reinterpret_cast<float *>(part + 2 * kBkMaxTiles * 4);  // bias1 | bias2

    // warp index broadcast from lane 0: ptxas then knows role branches are
    // warp-uniform and keeps the MMA issue loop on the uniform datapath
    const int warp = __shfl_sync(0xFFFFFFFFu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    if (threadIdx.x < 2 * N) s_b[threadIdx.x] = threadIdx.x < N ? L.bias1[threadIdx.x] : L.bias2[threadIdx.x - N];
    if (threadIdx.x == 0) {
        mbar_init(xfull, 1);
        mbar_init(xfree, 1);
        mbar_init(hready, 8);
        mbar_init(wbar, 1);
        for (int j = 0; j < kBkMaxTiles; ++j) mbar_init(&hrdy[j], 4);
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(2u * N2));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xFFFFFFFFu, *tmem_slot, 0);
    const int64_t n_img = L.n_img;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(wbar, 2 * WB);
            bulk_g2s(s_w1, L.w1, WB, wbar);
            bulk_g2s(s_w2, L.w2, WB, wbar);
            int it = 0;
            for (int64_t n = blockIdx.x; n < n_img; n += gridDim.x, ++it) {
                if (it > 0) mbar_wait(xfree, (it - 1) & 1);
                mbar_expect_tx(xfull, 8u * (uint32_t)nrows * 16u);
                const int64_t q_lo = n * HW - (Wp + 1);
#pragma unroll 1
                for (int g = 0; g < 2 * NH; ++g)
                    bulk_g2s(s_x + (size_t)g * slab + (size_t)(M0 - Wp - 1) * 16,
                             L.in + ((int64_t)g * L.gstride + L.margin + q_lo) * 8, (uint32_t)nrows * 16u, xfull);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc64 = idesc_f16(128, N2);
        constexpr uint32_t idesc32 = idesc_f16(128, N);
        mbar_wait(wbar, 0);
        tc_fence_after();
        const uint64_t dX = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_x), 0), slab, 128u);
        const uint64_t dH = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_h), 0), slab, 128u);
        const uint64_t dW1 = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_w1), 0), (uint32_t)N2 * 16u, 128u);
        const uint64_t dW2 = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_w2), 0), (uint32_t)N2 * 16u, 128u);
        const uint32_t rx = (uint32_t)RX;
        int64_t ti = 0;
        int it = 0;
        for (int64_t n = blockIdx.x; n < n_img; n += gridDim.x, ++it) {
            // two passes per image: conv1 over X, then conv2 over T; inline
            // (no lambda) so the descriptors stay in uniform registers
#pragma unroll 1
            for (int pass = 0; pass < 2; ++pass) {
                if (pass == 0) {
                    mbar_wait(xfull, it & 1);
                    tc_fence_after();
                }
                const uint64_t dA = pass ? dH : dX;
                const uint64_t dB = pass ? dW2 : dW1;
#pragma unroll 1
                for (int j = 0; j < T; ++j, ++ti) {
                    if (pass) {  // conv2 tile j reads T rows of conv1 tiles j - 1 .. j + 1
                        if (j == 0) mbar_wait(&hrdy[0], it & 1);
                        if (j + 1 < T) mbar_wait(&hrdy[j + 1], it & 1);
                        tc_fence_after();
                    }
                    const int a = (int)(ti & 1);
                    const int64_t u = ti >> 1;
                    if (u > 0) mbar_wait(&tempty[a], (uint32_t)((u - 1) & 1));
                    tc_fence_after();
                    const uint32_t d = tmem + (uint32_t)(a * N2);
                    const uint64_t dAt = dA + (uint64_t)(uint32_t)(M0 + 128 * j - Wp - 1);
#pragma unroll
                    for (int tap = 0; tap < 9; ++tap) {
                        const uint32_t off = (uint32_t)((tap / 3) * Wp + tap % 3);
#pragma unroll
                        for (int ks = 0; ks < NH / 2; ++ks) {
                            const uint64_t ao = (uint64_t)(2u * ks * rx + off);
                            const uint64_t bo = (uint64_t)((tap * NH + 2 * ks) * N2);
                            mma_f16_elect(d, dAt + ao, dB + bo, idesc64, (tap | ks) ? 1u : 0u);
                            mma_f16_elect(d + N, dAt + ao + (uint64_t)(NH * rx), dB + bo, idesc32, 1u);
                        }
                    }
                    mma_commit_elect(&tfull[a]);
                }
                if (pass == 0) mma_commit_elect(xfree);
            }
        }
    } else {
        const int grp = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int H = L.H, W = L.W;
        const int kw1 = __float_as_int(L.meta1[0]), kw2 = __float_as_int(L.meta2[0]);
        const float l1a = L.meta1[1], bm1 = L.meta1[2], l1b = L.meta2[1], bm2 = L.meta2[2];
        int64_t ti = 0;
        int it = 0;
        // per-image scalars are fetched one image ahead (a global load per
        // image would otherwise stall every iteration)
        int kx_nx = 0;
        uint32_t mx_nx = 0;
        if (blockIdx.x < n_img) {
            kx_nx = L.kx_in[blockIdx.x];
            mx_nx = L.mx_in[blockIdx.x];
        }
        for (int64_t n = blockIdx.x; n < n_img; n += gridDim.x, ++it) {
            const int kxi = kx_nx;
            const float mxi = __uint_as_float(mx_nx);
            if (n + gridDim.x < n_img) {
                kx_nx = L.kx_in[n + gridDim.x];
                mx_nx = L.mx_in[n + gridDim.x];
            }
            // conv1: T = relu(conv1(X)), scale 2^k1 from the bound on |T|
            const int k1 = act_exp(__float_as_uint(__fadd_rn(__fmul_rn(mxi, l1a), bm1)));
            uint32_t *pt = part + (it & 1) * kBkMaxTiles * 4;
            for (int j = 0; j < T; ++j, ++ti) {
                if ((int)(ti & 1) != grp) continue;
                const uint32_t u = (uint32_t)(ti >> 1);
                const int r = 128 * j + row;
                const int y = r / Wp, x = r - (r / Wp) * Wp;
                const bool valid = r < HW && y >= 1 && y <= H && x >= 1 && x <= W;
                const float inv = exp2i(-kxi - kw1), osc = exp2i(k1);
                mbar_wait(&tfull[grp], u & 1);
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(grp * N2);
                float v[32];
                {
                    float w[32];
                    tmem_ld32(taddr, v);
                    tmem_ld32(taddr + 32, w);
#pragma unroll
                    for (int c = 0; c < 32; ++c) v[c] = __fmaf_rn(__fmaf_rn(w[c], 0.00048828125f, v[c]), inv, s_b[c]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[grp]);
                float mx = 0.f;
                if (valid) {
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        v[c] = fmaxf(v[c], 0.f);
                        mx = fmaxf(mx, fabsf(v[c]));
                    }
#pragma unroll
                    for (int g = 0; g < NH; ++g) {
                        uint4 h, l;
                        split2(__fmul_rn(v[8 * g + 0], osc), __fmul_rn(v[8 * g + 1], osc), h.x, l.x);
                        split2(__fmul_rn(v[8 * g + 2], osc), __fmul_rn(v[8 * g + 3], osc), h.y, l.y);
                        split2(__fmul_rn(v[8 * g + 4], osc), __fmul_rn(v[8 * g + 5], osc), h.z, l.z);
                        split2(__fmul_rn(v[8 * g + 6], osc), __fmul_rn(v[8 * g + 7], osc), h.w, l.w);
                        store_px(reinterpret_cast<uint16_t *>(s_h + (size_t)g * slab + (size_t)M0 * 16), r, h, y, x,
                                 H, W, Wp);
                        store_px(reinterpret_cast<uint16_t *>(s_h + (size_t)(NH + g) * slab + (size_t)M0 * 16), r, l,
                                 y, x, H, W, Wp);
                    }
                }
                const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(mx));
                fence_async_smem();  // T rows -> conv2's MMA operand
                __syncwarp();
                if (lane == 0) {
                    pt[j * 4 + quarter] = m;
                    mbar_arrive(&hrdy[j]);
                }
            }
            if (lane == 0) mbar_arrive(hready);
            mbar_wait(hready, it & 1);
            uint32_t mt = 0;
            for (int k = 0; k < 4 * T; ++k) mt = max(mt, pt[k]);
            // conv2: X' = relu(X + conv2(T)), scale from |T| L1 + max|b| + max|X|
            const float bound = __fadd_rn(__fadd_rn(__fmul_rn(__uint_as_float(mt), l1b), bm2), mxi);
            const int k2 = act_exp(__float_as_uint(bound));
            for (int j = 0; j < T; ++j, ++ti) {
                if ((int)(ti & 1) != grp) continue;
                const uint32_t u = (uint32_t)(ti >> 1);
                const int r = 128 * j + row;
                const int y = r / Wp, x = r - (r / Wp) * Wp;
                const bool valid = r < HW && y >= 1 && y <= H && x >= 1 && x <= W;
                const float inv = exp2i(-k1 - kw2), osc = exp2i(k2);
                const int64_t q = n * HW + r;
                float4 rr[8] = {};  // residual rows, in flight while the MMAs finish
                if (valid) {
#pragma unroll
                    for (int g = 0; g < 8; ++g)
                        rr[g] = __ldg(reinterpret_cast<const float4 *>(L.res) + (int64_t)g * L.gstride + L.margin + q);
                }
                mbar_wait(&tfull[grp], u & 1);
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(grp * N2);
                float v[32];
                {
                    float w[32];
                    tmem_ld32(taddr, v);
                    tmem_ld32(taddr + 32, w);
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        v[c] = __fmaf_rn(__fmaf_rn(w[c], 0.00048828125f, v[c]), inv, s_b[N + c]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[grp]);
                float mx = 0.f;
                if (valid) {
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        v[4 * g + 0] = fmaxf(__fadd_rn(rr[g].x, v[4 * g + 0]), 0.f);
                        v[4 * g + 1] = fmaxf(__fadd_rn(rr[g].y, v[4 * g + 1]), 0.f);
                        v[4 * g + 2] = fmaxf(__fadd_rn(rr[g].z, v[4 * g + 2]), 0.f);
                        v[4 * g + 3] = fmaxf(__fadd_rn(rr[g].w, v[4 * g + 3]), 0.f);
#pragma unroll
                        for (int e = 0; e < 4; ++e) mx = fmaxf(mx, fabsf(v[4 * g + e]));
                        if (L.out32)
                            // fp32 copy: valid pixels only (no reader uses its edge copies)
                            reinterpret_cast<float4 *>(L.out32 + ((int64_t)g * L.gstride + L.margin) * 4)[q] =
                                make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
                    }
#pragma unroll
                    for (int g = 0; g < NH; ++g) {
                        uint4 h, l;
                        split2(__fmul_rn(v[8 * g + 0], osc), __fmul_rn(v[8 * g + 1], osc), h.x, l.x);
                        split2(__fmul_rn(v[8 * g + 2], osc), __fmul_rn(v[8 * g + 3], osc), h.y, l.y);
                        split2(__fmul_rn(v[8 * g + 4], osc), __fmul_rn(v[8 * g + 5], osc), h.z, l.z);
                        split2(__fmul_rn(v[8 * g + 6], osc), __fmul_rn(v[8 * g + 7], osc), h.w, l.w);
                        store_px(L.out + ((int64_t)g * L.gstride + L.margin) * 8, q, h, y, x, H, W, Wp);
                        store_px(L.out + ((int64_t)(NH + g) * L.gstride + L.margin) * 8, q, l, y, x, H, W, Wp);
                    }
                }
                const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(mx));
                if (lane == 0) {
                    if (m != 0u) atomicMax(L.mx_out + n, m);
                    L.kx_out[n] = k2;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2u * N2));
    }
}

size_t tc3_block_smem(int Hp, int Wp) {
    const int T = (Hp * Wp + 127) / 128;
    const int M0 = (Wp + 1 + 7) & ~7;
    const size_t RX = (size_t)M0 + (size_t)T * 128 + M0;
    return 2 * 36 * 64 * 16 + 2 * 8 * RX * 16 + (12 + kBkMaxTiles) * 8 + 16 +
           2 * kBkMaxTiles * 4 * 4 + 64 * 4;
}

// ---- encoder trunk in shared memory (vqvae.py:58-64) ------------------------
// All B residual blocks and the 1x1 projection of one image per CTA
// iteration: X (hi / lo operands, updated in place by each conv2 epilogue)
// and T (conv1 output) stay in shared memory, the fp32 block input (the
// exact residual) and the biases in tensor memory; only z leaves, as the
// argmin's 128-latent tiles.
//
// Per layer the T = ceil(Hp Wp / 128) tiles are issued in order and tile j of
// layer l + 1 waits for tiles j - 1 .. j + 1 of layer l (`hrdy`, one phase
// per layer); MMAs complete in issue order, so no epilogue overwrites a
// buffer an earlier MMA still reads. Weights stream through a two-slot ring.
// Two operand buffers alternate by image: image i's X lives in buffer i & 1
// and its T in the other, which is free once i's last conv2 MMAs are done --
// so image i + 1's X loads into it while i's last epilogues and projection
// run.
//
// The MMAs (M=128, N=64 + N=32 per K=16 step) cost ~44 cycles each whatever
// their N, so the kernel is bound by MMA count (36 per tile) plus the
// bubbles at layer boundaries, where tile 0 of layer l + 1 waits for the
// epilogues of tiles 0 and 1 of layer l: both epilogue groups therefore work
// on every tile (group g: channels 16g .. 16g + 15), halving the epilogue
// latency per tile. The epilogue keeps its non-operand traffic out of shared
// memory (the MMAs' operand reads use most of its bandwidth): residual and
// biases in TMEM columns, one merged predicated store per edge direction,
// partial maxima reduced across lanes. TMEM (512 columns): [0, 128) two
// accumulators (hi x hi | cross terms), [128, 128 + 32 T) the fp32 block
// input per tile, [224, 224 + 32 NL) every layer's bias (the same in all
// 128 lanes).
//
// Measured and rejected: CTA pairs (cta_group::2, M=256 MMAs issued by the
// leader over both CTAs' tiles). An M=256 pair MMA costs the same ~44 cycles
// as an M=128 one (tools/micro/mma2_rate.cu), i.e. no more rows per SM per
// cycle, and the cross-CTA tile / accumulator barriers added latency: 1.89
// ms per CIFAR-8192 launch against 1.63 for single CTAs.
//
// Scales (the per-image bounds of tc3_block_kernel): each epilogue layer
// needs the exact max of its input over the whole image, so the epilogue
// warps meet at a named barrier after every conv layer and reduce per-tile
// partial maxima. Arithmetic (MMA K order, epilogue roundings, scales) is
// that of tc3_block_kernel + tc3_conv_kernel<1, TC3_Z>: z is bit-identical
// to the per-block path.
constexpr int kThreadsET = 320;
constexpr int kEtMaxTiles = 3;
constexpr int kEtMaxLayers = 9;  // 2B + 1 with B <= 4: the biases fill TMEM columns 224 .. 511
constexpr uint32_t kEtX32Col = 128, kEtBiasCol = 224;

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float *v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
        "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
        "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
        "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float *v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
        "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
        : "memory");
}
// 16 consecutive f32 columns of this thread's lane, no wait (tmem_wait_ld before use)
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, float *v) {
    uint32_t *r = reinterpret_cast<uint32_t *>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// store_px with the edge copies merged per direction: ex = -1 / +1 (left /
// right column), ey = -Wp / +Wp (top / bottom row); `rows` / `corner` are
// warp-uniform (some lane of the warp has an edge row / a corner), so most
// warps issue the main store and one column-edge store only
__device__ __forceinline__ void store_px_m(uint8_t *slab_base, int r, uint4 v, bool valid, int ex, int ey,
                                           bool rows, bool corner) {
    uint4 *p = reinterpret_cast<uint4 *>(slab_base);
    if (valid) p[r] = v;
    if (valid && ex) p[r + ex] = v;
    if (rows) {
        if (valid && ey) p[r + ey] = v;
        if (corner && valid && ex && ey) p[r + ey + ex] = v;
    }
}

__global__ void __launch_bounds__(kThreadsET, 1) enc_trunk_kernel(EncTrunk P) {
    constexpr int N = 32, N2 = 64, NH = 4;
    constexpr uint32_t WB = 36 * N2 * 16;
    const int Wp = P.Wp, HW = P.Hp * Wp;
    const int T = (HW + 127) >> 7;
    const int M0 = Wp + 1;
    const int RX = M0 + 128 * T + M0;
    const uint32_t slab = (uint32_t)RX * 16u;
    const int nrows = HW + 2 * M0;
    const int B = P.n_blocks, NL = 2 * B + 1;

    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *s_w = smem;                   // [2][WB] weight ring
    uint8_t *s_buf = s_w + 2 * WB;         // [2][8 slabs] operand buffers
    uint64_t *bars = reinterpret_cast<uint64_t *>(s_buf + 16 * (size_t)slab);
    uint64_t *wfull = bars, *wempty = bars + 2, *xfull = bars + 4, *xfree = bars + 6;
    uint64_t *tfull = bars + 8, *tempty = bars + 10;
    uint64_t *hrdy = bars + 12;  // [kEtMaxTiles]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(hrdy + kEtMaxTiles);
    uint32_t *part = tmem_slot + 4;                                   // [2][kEtMaxTiles][4][2]
    float *s_m = reinterpret_cast<float *>(part + 2 * kEtMaxTiles * 8);  // [NL][4] {kw, L1, max|b|, -}

    const int warp = __shfl_sync(0xFFFFFFFFu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < NL * 4; i += blockDim.x) s_m[i] = (i & 3) < 3 ? P.meta[i >> 2][i & 3] : 0.f;
    if (threadIdx.x == 0) {
        for (int a = 0; a < 2; ++a) {
            mbar_init(&wfull[a], 1);
            mbar_init(&wempty[a], 1);
            mbar_init(&xfull[a], 1);
            mbar_init(&xfree[a], 1);
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8);  // both epilogue groups read every accumulator
        }
        for (int j = 0; j < kEtMaxTiles; ++j) mbar_init(&hrdy[j], 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xFFFFFFFFu, *tmem_slot, 0);
    const int64_t n_img = P.n_img;

    if (warp == 0) {
        if (lane == 0) {
            int lc = 0, it = 0;
            for (int64_t n = blockIdx.x; n < n_img; n += gridDim.x, ++it) {
                const int b = it & 1;
                // X hi / lo (tile halos included) into buffer b, once the image
                // that used b for its T has issued its last conv2 MMAs
                if (it > 0) mbar_wait(&xfree[b], ((it - 1) >> 1) & 1);
                mbar_expect_tx(&xfull[b], 8u * (uint32_t)nrows * 16u);
                const int64_t q_lo = n * HW - M0;
#pragma unroll 1
                for (int g = 0; g < 8; ++g)
                    bulk_g2s(s_buf + (size_t)(b * 8 + g) * slab, P.in + ((int64_t)g * P.gstride + P.margin + q_lo) * 8,
                             (uint32_t)nrows * 16u, &xfull[b]);
#pragma unroll 1
                for (int l = 0; l < NL; ++l, ++lc) {
                    const int s = lc & 1;
                    if (lc >= 2) mbar_wait(&wempty[s], ((lc >> 1) - 1) & 1);
                    const uint32_t bytes = l < 2 * B ? WB : 4u * N2 * 16u;
                    mbar_expect_tx(&wfull[s], bytes);
                    bulk_g2s(s_w + (size_t)s * WB, P.w[l], bytes, &wfull[s]);
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc64 = idesc_f16(128, N2);
        constexpr uint32_t idesc32 = idesc_f16(128, N);
        const uint64_t dBuf = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_buf), 0), slab, 128u);
        const uint64_t dW = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_w), 0), (uint32_t)N2 * 16u, 128u);
        const uint32_t rx = (uint32_t)RX;
        const uint32_t bstep = (8u * slab) >> 4;
        const uint32_t d0 = tmem, d1 = tmem + (uint32_t)N2;
        int64_t ti = 0;
        int lc = 0, it = 0;
        for (int64_t n = blockIdx.x; n < n_img; n += gridDim.x, ++it) {
            const int bx = it & 1;
            mbar_wait(&xfull[bx], (it >> 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int l = 0; l < NL; ++l, ++lc) {
                const int s = lc & 1;
                mbar_wait(&wfull[s], (lc >> 1) & 1);
                tc_fence_after();
                const bool conv = l < 2 * B;
                const int ab = (conv && (l & 1)) ? (bx ^ 1) : bx;  // conv2 reads T, conv1 / proj read X
                const uint64_t dA = dBuf + (uint64_t)((uint32_t)ab * bstep);
                const uint64_t dB = dW + (uint64_t)((uint32_t)s * (WB >> 4));
#pragma unroll 1
                for (int j = 0; j < T; ++j, ++ti) {
                    if (l > 0) {  // the previous layer's tiles j - 1 .. j + 1 (proj: j) are in place
                        if (conv) {
                            if (j == 0) mbar_wait(&hrdy[0], (lc - 1) & 1);
                            if (j + 1 < T) mbar_wait(&hrdy[j + 1], (lc - 1) & 1);
                        } else {
                            mbar_wait(&hrdy[j], (lc - 1) & 1);
                        }
                    }
                    const int a = (int)(ti & 1);
                    const int64_t u = ti >> 1;
                    if (u > 0) mbar_wait(&tempty[a], (uint32_t)((u - 1) & 1));
                    tc_fence_after();
                    const uint32_t d = a ? d1 : d0;
                    const uint32_t bl = (uint32_t)dB, bh = (uint32_t)(dB >> 32), ah = (uint32_t)(dA >> 32);
                    if (conv) {
                        const uint32_t al = (uint32_t)dA + (uint32_t)(M0 + 128 * j - Wp - 1);
#pragma unroll
                        for (int tap = 0; tap < 9; ++tap) {
                            const uint32_t off = (uint32_t)((tap / 3) * Wp + tap % 3);
#pragma unroll
                            for (int ks = 0; ks < NH / 2; ++ks) {
                                const uint32_t ao = 2u * ks * rx + off;
                                const uint32_t bo = (uint32_t)((tap * NH + 2 * ks) * N2);
                                mma_f16_elect_w(d, al + ao, ah, bl + bo, bh, idesc64, (tap | ks) ? 1u : 0u);
                                mma_f16_elect_w(d + N, al + ao + NH * rx, ah, bl + bo, bh, idesc32, 1u);
                            }
                        }
                    } else {
                        const uint32_t al = (uint32_t)dA + (uint32_t)(M0 + 128 * j);
#pragma unroll
                        for (int ks = 0; ks < NH / 2; ++ks) {
                            const uint32_t ao = 2u * ks * rx;
                            const uint32_t bo = (uint32_t)(2 * ks * N2);
                            mma_f16_elect_w(d, al + ao, ah, bl + bo, bh, idesc64, ks ? 1u : 0u);
                            mma_f16_elect_w(d + N, al + ao + NH * rx, ah, bl + bo, bh, idesc32, 1u);
                        }
                    }
                    mma_commit_elect(&tfull[a]);
                }
                mma_commit_elect(&wempty[s]);
                if (l == 2 * B - 1) mma_commit_elect(&xfree[bx ^ 1]);  // T buffer: the next image's X
            }
        }
    } else if (warp >= 2) {
        // two epilogue groups of four warps (one per TMEM lane quarter); both
        // take every tile, group g its channels 16g .. 16g + 15
        const int grp = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int H = P.H, W = P.W;
        const bool thin = H == 1 || W == 1;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        const uint32_t ch = 16u * (uint32_t)grp;  // this group's first channel
        // biases into TMEM, every lane: group g writes layers l = g mod 2
        for (int l = grp; l < NL; l += 2) {
            float bv[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) bv[c] = __ldg(P.bias[l] + c);
            tmem_st32(lane_base + kEtBiasCol + 32u * l, bv);
        }
        tmem_wait_st();
        tc_fence_before();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        tc_fence_after();
        int64_t ti = 0;
        int it = 0;
        int kx_nx = 0;
        uint32_t mx_nx = 0;
        if (blockIdx.x < n_img) {
            kx_nx = P.kx_in[blockIdx.x];
            mx_nx = P.mx_in[blockIdx.x];
        }
        for (int64_t n = blockIdx.x; n < n_img; n += gridDim.x, ++it) {
            const int bx = it & 1;
            uint8_t *bufX = s_buf + (size_t)bx * 8 * slab + (size_t)M0 * 16;
            uint8_t *bufT = s_buf + (size_t)(bx ^ 1) * 8 * slab + (size_t)M0 * 16;
            int kX = kx_nx;
            float mxX = __uint_as_float(mx_nx);
            if (n + gridDim.x < n_img) {
                kx_nx = P.kx_in[n + gridDim.x];
                mx_nx = P.mx_in[n + gridDim.x];
            }
            int kT = 0;
            float mxT = 0.f;
#pragma unroll 1
            for (int l = 0; l < NL; ++l) {
                const int kw = __float_as_int(s_m[4 * l]);
                const float l1 = s_m[4 * l + 1], bm = s_m[4 * l + 2];
                const bool conv = l < 2 * B, conv2 = conv && (l & 1);
                // this layer's input scale and its output scale
                int ko = 0;
                float inv;
                if (!conv) {
                    inv = exp2i(-kX - kw);
                } else if (!conv2) {  // T = relu(conv1(X)), |T| <= max|X| L1 + max|b|
                    ko = act_exp(__float_as_uint(__fadd_rn(__fmul_rn(mxX, l1), bm)));
                    inv = exp2i(-kX - kw);
                } else {              // X' = relu(X + conv2(T)), |X'| <= max|T| L1 + max|b| + max|X|
                    ko = act_exp(__float_as_uint(__fadd_rn(__fadd_rn(__fmul_rn(mxT, l1), bm), mxX)));
                    inv = exp2i(-kT - kw);
                }
                const float osc = exp2i(ko);
                uint32_t *pt = part + (l & 1) * kEtMaxTiles * 8;
                uint8_t *dst = conv2 ? bufX : bufT;
#pragma unroll 1
                for (int j = 0; j < T; ++j, ++ti) {
                    const int a = (int)(ti & 1);
                    const uint32_t u = (uint32_t)(ti >> 1);
                    const int r = 128 * j + row;
                    const int y = r / Wp, x = r - (r / Wp) * Wp;
                    const bool valid = r < HW && y >= 1 && y <= H && x >= 1 && x <= W;
                    const uint32_t x32col = lane_base + kEtX32Col + 32u * j + ch;
                    float rr[16];  // conv2: the fp32 block input of this row (this group's channels)
                    if (l == 1) {  // block 0's input from the front's fp32 slabs, in flight during the MMAs
#pragma unroll
                        for (int g = 0; g < 4; ++g) {
                            float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
                            if (valid)
                                f = __ldg(reinterpret_cast<const float4 *>(P.in32) + (int64_t)(4 * grp + g) * P.gstride +
                                          P.margin + n * HW + r);
                            rr[4 * g] = f.x;
                            rr[4 * g + 1] = f.y;
                            rr[4 * g + 2] = f.z;
                            rr[4 * g + 3] = f.w;
                        }
                    }
                    mbar_wait(&tfull[a], u & 1);
                    tc_fence_after();
                    const uint32_t taddr = lane_base + (uint32_t)(a * N2) + ch;
                    float v[16];
                    {
                        float w[16], bias[16];
                        tmem_ld16_nw(taddr, v);
                        tmem_ld16_nw(taddr + 32, w);
                        tmem_ld16_nw(lane_base + kEtBiasCol + 32u * l + ch, bias);
                        if (conv2 && l > 1) tmem_ld16_nw(x32col, rr);
                        tmem_wait_ld();
#pragma unroll
                        for (int c = 0; c < 16; ++c) v[c] = __fmaf_rn(__fmaf_rn(w[c], 0.00048828125f, v[c]), inv, bias[c]);
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[a]);
                    if (!conv) {
                        // z = acc + bias as tf32 hi / fp32 lo 128-latent tiles (tc3_conv_kernel<1, TC3_Z>)
                        if (valid) {
                            const int64_t vix = ((int64_t)n * H + (y - 1)) * (int64_t)W + (x - 1);
                            float4 *zo = P.z ? reinterpret_cast<float4 *>(P.z + vix * 32) + 4 * grp : nullptr;
                            float4 *zt = reinterpret_cast<float4 *>(P.zt) + (vix >> 7) * (2 * 8 * 128) + (vix & 127) +
                                         4 * grp * 128;
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                float hi[4], lo[4];
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    hi[e] = tf32_rna(v[4 * g + e]);
                                    lo[e] = __fsub_rn(v[4 * g + e], hi[e]);
                                }
                                if (zo) zo[g] = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
                                zt[g * 128] = make_float4(hi[0], hi[1], hi[2], hi[3]);
                                zt[(8 + g) * 128] = make_float4(lo[0], lo[1], lo[2], lo[3]);
                            }
                        }
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&hrdy[j]);
                        continue;
                    }
                    float mx = 0.f;
                    if (conv2) {
#pragma unroll
                        for (int c = 0; c < 16; ++c) v[c] = fmaxf(__fadd_rn(rr[c], v[c]), 0.f);
                        if (l < 2 * B - 1) tmem_st16(x32col, v);  // the next block's residual
                    } else {
#pragma unroll
                        for (int c = 0; c < 16; ++c) v[c] = fmaxf(v[c], 0.f);
                    }
                    if (valid) {
#pragma unroll
                        for (int c = 0; c < 16; ++c) mx = fmaxf(mx, fabsf(v[c]));
                    }
                    const int ex = x == 1 ? -1 : (x == W ? 1 : 0);
                    const int ey = y == 1 ? -Wp : (y == H ? Wp : 0);
                    const bool rows = __any_sync(0xFFFFFFFFu, valid && ey != 0);
                    const bool corner = __any_sync(0xFFFFFFFFu, valid && ey != 0 && ex != 0);
#pragma unroll
                    for (int gg = 0; gg < 2; ++gg) {
                        const int g = 2 * grp + gg;  // channel group (8 channels)
                        uint4 h, lo;
                        split2(__fmul_rn(v[8 * gg + 0], osc), __fmul_rn(v[8 * gg + 1], osc), h.x, lo.x);
                        split2(__fmul_rn(v[8 * gg + 2], osc), __fmul_rn(v[8 * gg + 3], osc), h.y, lo.y);
                        split2(__fmul_rn(v[8 * gg + 4], osc), __fmul_rn(v[8 * gg + 5], osc), h.z, lo.z);
                        split2(__fmul_rn(v[8 * gg + 6], osc), __fmul_rn(v[8 * gg + 7], osc), h.w, lo.w);
                        if (thin) {  // one-pixel-wide grids: a pixel is both edges
                            if (valid) {
                                store_px(reinterpret_cast<uint16_t *>(dst + (size_t)g * slab), r, h, y, x, H, W, Wp);
                                store_px(reinterpret_cast<uint16_t *>(dst + (size_t)(NH + g) * slab), r, lo, y, x, H, W, Wp);
                            }
                        } else {
                            store_px_m(dst + (size_t)g * slab, r, h, valid, ex, ey, rows, corner);
                            store_px_m(dst + (size_t)(NH + g) * slab, r, lo, valid, ex, ey, rows, corner);
                        }
                    }
                    const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(mx));
                    fence_async_smem();  // operand rows -> the next layer's MMAs
                    __syncwarp();
                    if (lane == 0) {
                        pt[(j * 4 + quarter) * 2 + grp] = m;
                        mbar_arrive(&hrdy[j]);
                    }
                }
                if (!conv) break;
                // every tile of the layer is through: the image's exact max |out|
                // (and the residual columns written above are visible to all)
                if (conv2) tmem_wait_st();
                tc_fence_before();
                asm volatile("bar.sync 1, 256;" ::: "memory");
                tc_fence_after();
                const uint32_t mt = __reduce_max_sync(0xFFFFFFFFu, lane < 8 * T ? pt[lane] : 0u);
                if (conv2) {
                    mxX = __uint_as_float(mt);
                    kX = ko;
                } else {
                    mxT = __uint_as_float(mt);
                    kT = ko;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
    }
}

size_t enc_trunk_smem(int Hp, int Wp, int B) {
    const int HW = Hp * Wp, T = (HW + 127) / 128, M0 = Wp + 1;
    const size_t RX = (size_t)2 * M0 + (size_t)T * 128;
    const int NL = 2 * B + 1;
    (void)HW;
    return 2 * 36 * 64 * 16 + 2 * 8 * RX * 16 + (12 + kEtMaxTiles) * 8 + 16 + 2 * kEtMaxTiles * 8 * 4 +
           (size_t)NL * 4 * 4;
}

// ---- decoder trunk in shared memory (vqvae.py:80-100) -----------------------
// dec.proj (as the gathered table T[idx], see dec_table_kernel) and all 2B
// residual-block convs of a group of G images in one persistent kernel: the
// latent activations never leave shared memory. X (block input / output,
// updated in place by conv2's epilogue) and H (conv1 output) are padded
// group-major slab sets as in tc_conv_kernel, with the G images' padded
// grids back to back; taps are shifted descriptors into them. Only the
// trunk output goes to HBM (for the up conv).
//
// Per layer the T = ceil(G Hp Wp / 128) tiles are issued in order; tile j of
// layer l + 1 waits for tiles j - 1 .. j + 1 of layer l (`hrdy`, one
// mbarrier per tile position, one phase per layer). MMAs complete in issue
// order, so an epilogue writing a buffer can never overtake an earlier
// layer's MMA still reading it. Weights stream through a two-slot ring.
// Arithmetic (MMA K order, fadd order, bf16 rounding) is that of
// tc_conv_kernel, so the output is bit-identical to the per-layer path.
constexpr int kDtGroups = 3;  // epilogue groups of four warps, one TMEM accumulator each
constexpr int kThreadsDT = 64 + 128 * kDtGroups;
constexpr int kDtMaxTiles = 16;
constexpr int kDtMaxConvs = 16;

__global__ void __launch_bounds__(kThreadsDT, 1) dec_trunk_kernel(DecTrunk P) {
    constexpr int N = 32, NG = 4;
    constexpr uint32_t WB = 36 * N * 16;
    const int Wp = P.Wp, HW = P.Hp * Wp, G = P.G;
    const int rows = G * HW;
    const int T = (rows + 127) >> 7;
    const int M0 = Wp + 1;
    const int RS = M0 + rows + M0;
    const uint32_t slab = (uint32_t)RS * 16u;
    const int L = P.n_conv;

    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *s_w = smem;                                         // [2][36][32][8] bf16
    uint8_t *s_tab = s_w + 2 * WB;                               // K x 64 B
    uint8_t *s_x = s_tab + (size_t)P.K * 64;
    uint8_t *s_h = s_x + NG * (size_t)slab;
    uint64_t *bars = reinterpret_cast<uint64_t *>(s_h + NG * (size_t)slab + P.pad_bytes);
    uint64_t *wfull = bars, *wempty = bars + 2, *tfull = bars + 4, *tempty = bars + 4 + kDtGroups;
    uint64_t *xready = bars + 4 + 2 * kDtGroups, *tbar = xready + 1, *hrdy = xready + 2;  // hrdy[kDtMaxTiles]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(hrdy + kDtMaxTiles);
    float *s_b = reinterpret_cast<float *>(tmem_slot + 4);      // [L][32]

    const int warp = __shfl_sync(0xFFFFFFFFu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < L * N; i += blockDim.x) s_b[i] = P.bias[i / N][i % N];
    if (threadIdx.x == 0) {
        for (int a = 0; a < 2; ++a) {
            mbar_init(&wfull[a], 1);
            mbar_init(&wempty[a], 1);
        }
        for (int a = 0; a < kDtGroups; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);
        }
        mbar_init(xready, 4 * kDtGroups);
        mbar_init(tbar, 1);
        for (int j = 0; j < kDtMaxTiles; ++j) mbar_init(&hrdy[j], 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(128u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xFFFFFFFFu, *tmem_slot, 0);
    const int64_t n_groups = (P.n_img + G - 1) / G;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(tbar, (uint32_t)P.K * 64u);
            bulk_g2s(s_tab, P.table, (uint32_t)P.K * 64u, tbar);
            int lc = 0;
            for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
                for (int l = 0; l < L; ++l, ++lc) {
                    const int s = lc & 1;
                    if (lc >= 2) mbar_wait(&wempty[s], ((lc >> 1) - 1) & 1);
                    mbar_expect_tx(&wfull[s], WB);
                    bulk_g2s(s_w + (size_t)s * WB, P.w + (size_t)l * (WB / 2), WB, &wfull[s]);
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_bf16(128, N);
        const uint64_t dX = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_x), 0), slab, 128u);
        const uint64_t dH = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_h), 0), slab, 128u);
        const uint64_t dW = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_w), 0), N * 16u, 128u);
        const uint32_t rs = (uint32_t)RS;
        int64_t ti = 0;
        int lc = 0, gc = 0;
        for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x, ++gc) {
            mbar_wait(xready, gc & 1);
            tc_fence_after();
            for (int l = 0; l < L; ++l, ++lc) {
                const int s = lc & 1;
                mbar_wait(&wfull[s], (lc >> 1) & 1);
                tc_fence_after();
                const uint64_t dA = (l & 1) ? dH : dX;
                const uint64_t dB = dW + (uint64_t)((uint32_t)s * (WB >> 4));
                for (int j = 0; j < T; ++j, ++ti) {
                    if (l > 0) {  // tiles j - 1 .. j + 1 of the previous layer are in place
                        if (j == 0) mbar_wait(&hrdy[0], (lc - 1) & 1);
                        if (j + 1 < T) mbar_wait(&hrdy[j + 1], (lc - 1) & 1);
                        tc_fence_after();
                    }
                    const int a = (int)(ti % kDtGroups);
                    const int64_t u = ti / kDtGroups;
                    if (u > 0) mbar_wait(&tempty[a], (uint32_t)((u - 1) & 1));
                    tc_fence_after();
                    const uint32_t d = tmem + (uint32_t)(a * N);
                    const uint32_t al = (uint32_t)dA + (uint32_t)(M0 + 128 * j - Wp - 1), ah = (uint32_t)(dA >> 32);
                    const uint32_t bl = (uint32_t)dB, bh = (uint32_t)(dB >> 32);
#pragma unroll
                    for (int tap = 0; tap < 9; ++tap) {
                        const uint32_t off = (uint32_t)((tap / 3) * Wp + tap % 3);
#pragma unroll
                        for (int ks = 0; ks < NG / 2; ++ks)
                            mma_bf16_elect_w(d, al + 2u * ks * rs + off, ah, bl + (uint32_t)((tap * NG + 2 * ks) * N), bh,
                                             idesc, (tap | ks) ? 1u : 0u);
                    }
                    mma_commit_elect(&tfull[a]);
                }
                mma_commit_elect(&wempty[s]);
            }
        }
    } else {
        const int grp = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int et = threadIdx.x - 64;  // 0 .. 128 kDtGroups - 1
        const int gh = P.Hp - 2, gw = Wp - 2;
        const FastDiv div_hw{(uint32_t)HW, (uint32_t)(0x100000000ull / (uint32_t)HW)};
        const FastDiv div_w{(uint32_t)Wp, (uint32_t)(0x100000000ull / (uint32_t)Wp)};
        mbar_wait(tbar, 0);
        int64_t ti = 0;
        int lc = 0;
        for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
            const int64_t n0 = gi * G;
            const int g_act = (int)min((int64_t)G, P.n_img - n0);
            // gather: X = T[idx] at every padded position of the group (edges by clamping)
            for (int p = et; p < g_act * HW; p += 128 * kDtGroups) {
                const int n = (int)fdiv((uint32_t)p, div_hw), rem = p - n * HW;
                const int yy = (int)fdiv((uint32_t)rem, div_w);
                int y = yy - 1, x = rem - yy * Wp - 1;
                y = y < 0 ? 0 : (y >= gh ? gh - 1 : y);
                x = x < 0 ? 0 : (x >= gw ? gw - 1 : x);
                const int k = P.idx[((n0 + n) * gh + y) * gw + x];
                const uint4 *src = reinterpret_cast<const uint4 *>(s_tab + (size_t)k * 64);
#pragma unroll
                for (int g = 0; g < NG; ++g)
                    reinterpret_cast<uint4 *>(s_x + (size_t)g * slab + (size_t)(M0 + p) * 16)[0] = src[g];
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(xready);
            for (int l = 0; l < L; ++l, ++lc) {
                const bool conv2 = (l & 1) != 0, last = l == L - 1;
                const float *bias = s_b + l * N;
                uint8_t *dst = conv2 ? s_x : s_h;
                for (int j = 0; j < T; ++j, ++ti) {
                    if ((int)(ti % kDtGroups) != grp) continue;
                    const uint32_t u = (uint32_t)(ti / kDtGroups);
                    const int r = 128 * j + row;
                    const int n = (int)fdiv((uint32_t)r, div_hw), rem = r - n * HW;
                    const int y = (int)fdiv((uint32_t)rem, div_w), x = rem - y * Wp;
                    const bool valid = n < g_act && y >= 1 && y <= gh && x >= 1 && x <= gw;
                    mbar_wait(&tfull[grp], u & 1);
                    tc_fence_after();
                    float v[32];
                    tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(grp * N), v);
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[grp]);
                    if (valid) {
                        uint4 w4[NG];
#pragma unroll
                        for (int g = 0; g < NG; ++g) {
                            float o[8];
#pragma unroll
                            for (int e = 0; e < 8; ++e) o[e] = __fadd_rn(v[8 * g + e], bias[8 * g + e]);
                            if (conv2) {
                                const uint4 rv = reinterpret_cast<const uint4 *>(s_x + (size_t)g * slab +
                                                                                (size_t)(M0 + r) * 16)[0];
                                const uint32_t rw[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    o[2 * e] = __fadd_rn(bf16_lo(rw[e]), o[2 * e]);
                                    o[2 * e + 1] = __fadd_rn(bf16_hi(rw[e]), o[2 * e + 1]);
                                }
                            }
#pragma unroll
                            for (int e = 0; e < 8; ++e) o[e] = fmaxf(o[e], 0.f);
                            w4[g] = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]),
                                               pack_bf16(o[6], o[7]));
                        }
                        if (last) {
                            const int64_t q = (n0 + n) * HW + rem;
#pragma unroll
                            for (int g = 0; g < NG; ++g)
                                store_px(P.out + ((int64_t)g * P.out_gstride + P.out_margin) * 8, q, w4[g], y, x, gh,
                                         gw, Wp);
                        } else {
#pragma unroll
                            for (int g = 0; g < NG; ++g)
                                store_px(reinterpret_cast<uint16_t *>(dst + (size_t)g * slab + (size_t)M0 * 16), r,
                                         w4[g], y, x, gh, gw, Wp);
                        }
                    }
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&hrdy[j]);
                }
            }
            // the next group's gather overwrites X: every epilogue warp is past its residual reads
            asm volatile("bar.sync 1, %0;" ::"n"(128 * kDtGroups) : "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u));
    }
}

size_t dec_trunk_smem(int Hp, int Wp, int G, int K, int n_conv, int *pad) {
    const int rows = G * Hp * Wp, T = (rows + 127) / 128, M0 = Wp + 1;
    const size_t RS = (size_t)M0 + rows + M0;
    // the last slab's MMA reads run past its end by up to (128 T + M0) - (rows + M0) rows
    const int p = ((128 * T - rows + 16) * 16 + 127) / 128 * 128;
    if (pad) *pad = p;
    return 2 * 36 * 32 * 16 + (size_t)K * 64 + 2 * 4 * RS * 16 + p + (6 + 2 * kDtGroups + kDtMaxTiles) * 8 + 16 +
           (size_t)n_conv * 32 * 4;
}

// ---- decoder trunk over pixel pairs (vqvae.py:80-100) ------------------------
// dec_trunk_kernel with the activations in the pair layout of the head (row
// = two horizontally adjacent pixels of the padded grid, 8 channel groups:
// even pixel 0..3, odd pixel 4..7; padded width rounded up to even), so one
// MMA row produces both pixels' 32 outputs (N = 64): per row tap 8 K steps
// (the left pair's odd pixel, this pair, the right pair's even pixel, 16
// channels each), 24 MMAs per 256 pixels instead of 36, and each 4 KB A tile
// feeds 64 outputs instead of 32 -- the N=32 convs are bound by the MMAs'
// shared-memory operand reads. Per output pixel the non-zero K chunks come
// in the per-pixel kernel's order (taps row-major, 16 channels per chunk)
// with zero-weight chunks in between, which add exact zeros: the output is
// bit-identical to dec_trunk_kernel / the per-layer path.
//
// The pair weights (48 K groups x 64 rows, 48 KB per conv) stream through a
// ring of four 16 KB slots, one per row tap: a layer's three taps stay
// resident for all its tiles, the fourth slot prefetches the next layer's
// first tap, and each tap's slot is released as soon as the layer's last
// tile has issued that tap's MMAs.
constexpr int kD2Slots = 4;
constexpr uint32_t kD2Chunk = 16 * 64 * 16;  // one row tap: 16 K groups x 64 rows x 16 B
constexpr int kD2MaxTiles = 16;
constexpr int kD2Groups = 3;  // epilogue groups of four warps, one 64-column accumulator each (4: within 1%)
constexpr int kThreadsD2 = 64 + 128 * kD2Groups;


__global__ void __launch_bounds__(kThreadsD2, 1) dec_trunk2_kernel(DecTrunk P) {
    constexpr int NG = 4;
    const int Wp = P.Wp, Wpp = (Wp + 1) & ~1, Wq = Wpp >> 1, gh = P.Hp - 2, gw = Wp - 2;
    const int HWq = P.Hp * Wq;  // pair rows per image
    const int G = P.G;
    const int rows = G * HWq;
    const int T = (rows + 127) >> 7;
    const int M0 = Wq + 1;
    const int RS = M0 + rows + M0;
    const uint32_t slab = (uint32_t)RS * 16u;
    const int L = P.n_conv;

    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *s_w = smem;                                         // [4][16][64][8] bf16
    uint8_t *s_tab = s_w + kD2Slots * kD2Chunk;                  // K x 64 B
    uint8_t *s_x = s_tab + (size_t)P.K * 64;                     // 8 slabs
    uint8_t *s_h = s_x + 8 * (size_t)slab;                       // 8 slabs
    uint64_t *bars = reinterpret_cast<uint64_t *>(s_h + 8 * (size_t)slab + P.pad_bytes);
    uint64_t *wfull = bars, *wempty = bars + kD2Slots, *tfull = bars + 2 * kD2Slots, *tempty = tfull + kD2Groups;
    uint64_t *xready = tempty + kD2Groups, *tbar = xready + 1, *hrdy = xready + 2;  // hrdy[kD2MaxTiles]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(hrdy + kD2MaxTiles);
    float *s_b = reinterpret_cast<float *>(tmem_slot + 4);      // [L][32]

    const int warp = __shfl_sync(0xFFFFFFFFu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < L * 32; i += blockDim.x) s_b[i] = P.bias[i / 32][i % 32];
    if (threadIdx.x == 0) {
        for (int a = 0; a < kD2Slots; ++a) {
            mbar_init(&wfull[a], 1);
            mbar_init(&wempty[a], 1);
        }
        for (int a = 0; a < kD2Groups; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8);
        }
        mbar_init(xready, 4 * kD2Groups);
        mbar_init(tbar, 1);
        for (int j = 0; j < kD2MaxTiles; ++j) mbar_init(&hrdy[j], 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // finite operands in the rows no image writes (margins, tile tails): the
    // zero-weight K chunks read them (0 x NaN = NaN)
    {
        uint4 *z = reinterpret_cast<uint4 *>(s_x);
        const int n16 = 2 * 8 * RS + P.pad_bytes / 16;
        for (int e = threadIdx.x; e < n16; e += blockDim.x) z[e] = make_uint4(0u, 0u, 0u, 0u);
        fence_async_smem();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(256u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xFFFFFFFFu, *tmem_slot, 0);
    const int64_t n_groups = (P.n_img + G - 1) / G;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(tbar, (uint32_t)P.K * 64u);
            bulk_g2s(s_tab, P.table, (uint32_t)P.K * 64u, tbar);
            int cs = 0;  // chunk sequence: (group, layer, row tap)
            for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
                for (int l = 0; l < L; ++l) {
                    for (int c = 0; c < 3; ++c, ++cs) {
                        const int s = cs & (kD2Slots - 1);
                        if (cs >= kD2Slots) mbar_wait(&wempty[s], ((cs / kD2Slots) - 1) & 1);
                        mbar_expect_tx(&wfull[s], kD2Chunk);
                        bulk_g2s(s_w + (size_t)s * kD2Chunk, P.w + ((size_t)l * 3 + c) * (kD2Chunk / 2), kD2Chunk,
                                 &wfull[s]);
                    }
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_bf16(128, 64);
        const uint64_t dX = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_x), 0), slab, 128u);
        const uint64_t dH = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_h), 0), slab, 128u);
        const uint64_t dW = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_w), 0), 64u * 16u, 128u);
        const uint32_t rs = (uint32_t)RS;
        int64_t ti = 0;
        int cs = 0, gc = 0;
        for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x, ++gc) {
            mbar_wait(xready, gc & 1);
            tc_fence_after();
            for (int l = 0; l < L; ++l, cs += 3) {
                const uint64_t dA = (l & 1) ? dH : dX;
                for (int j = 0; j < T; ++j, ++ti) {
                    if (l > 0) {  // tiles j - 1 .. j + 1 of the previous layer are in place
                        if (j == 0) mbar_wait(&hrdy[0], (cs / 3 - 1) & 1);
                        if (j + 1 < T) mbar_wait(&hrdy[j + 1], (cs / 3 - 1) & 1);
                        tc_fence_after();
                    }
                    const int a = (int)(ti % kD2Groups);
                    const int64_t u = ti / kD2Groups;
                    if (u > 0) mbar_wait(&tempty[a], (uint32_t)((u - 1) & 1));
                    tc_fence_after();
                    const uint32_t d = tmem + (uint32_t)(a * 64);
                    const uint32_t al = (uint32_t)dA + (uint32_t)(128 * j), ah = (uint32_t)(dA >> 32);
                    const uint32_t bh = (uint32_t)(dW >> 32);
#pragma unroll
                    for (int di = 0; di < 3; ++di) {
                        if (j == 0) {  // each row tap's weights just before its first use (the ring refills late)
                            mbar_wait(&wfull[(cs + di) & (kD2Slots - 1)], ((cs + di) / kD2Slots) & 1);
                            tc_fence_after();
                        }
                        const uint32_t bl = (uint32_t)dW + (uint32_t)(((cs + di) & (kD2Slots - 1)) * (kD2Chunk >> 4));
#pragma unroll
                        for (int sg = 0; sg < 8; ++sg) {
                            const uint32_t sl = (sg < 2) ? 4u + 2u * sg : (sg < 6 ? 2u * (sg - 2) : 2u * (sg - 6));
                            const uint32_t dj = sg < 2 ? 0u : (sg < 6 ? 1u : 2u);
                            mma_bf16_elect_w(d, al + sl * rs + (uint32_t)di * (uint32_t)Wq + dj, ah,
                                             bl + (uint32_t)(2 * sg * 64), bh, idesc, (di | sg) ? 1u : 0u);
                        }
                        if (j == T - 1) mma_commit_elect(&wempty[(cs + di) & (kD2Slots - 1)]);
                    }
                    mma_commit_elect(&tfull[a]);
                }
            }
        }
    } else {
        const int grp = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int et = threadIdx.x - 64;  // 0 .. 128 kD2Groups - 1
        const int HWpp = P.Hp * Wpp, HW = P.Hp * Wp;
        const FastDiv div_hw{(uint32_t)HWq, (uint32_t)(0x100000000ull / (uint32_t)HWq)};
        const FastDiv div_w{(uint32_t)Wq, (uint32_t)(0x100000000ull / (uint32_t)Wq)};
        const FastDiv div_hwp{(uint32_t)HWpp, (uint32_t)(0x100000000ull / (uint32_t)HWpp)};
        const FastDiv div_wp{(uint32_t)Wpp, (uint32_t)(0x100000000ull / (uint32_t)Wpp)};
        mbar_wait(tbar, 0);
        int64_t ti = 0;
        int lc = 0;
        for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
            const int64_t n0 = gi * G;
            const int g_act = (int)min((int64_t)G, P.n_img - n0);
            // gather: X = T[idx] at every padded position of the group (edges by
            // clamping; the extra even-width column too)
            constexpr int kStep = 128 * kD2Groups;
            for (int p0 = et; p0 < g_act * HWpp; p0 += 4 * kStep) {
                int kk[4];  // four index loads in flight before any use
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int p = p0 + u * kStep;
                    kk[u] = 0;
                    if (p < g_act * HWpp) {
                        const int n = (int)fdiv((uint32_t)p, div_hwp), rem = p - n * HWpp;
                        const int yy = (int)fdiv((uint32_t)rem, div_wp), xx = rem - yy * Wpp;
                        int y = yy - 1, x = xx - 1;
                        y = y < 0 ? 0 : (y >= gh ? gh - 1 : y);
                        x = x < 0 ? 0 : (x >= gw ? gw - 1 : x);
                        kk[u] = P.idx[((n0 + n) * gh + y) * gw + x];
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int p = p0 + u * kStep;
                    if (p >= g_act * HWpp) break;
                    const uint4 *src = reinterpret_cast<const uint4 *>(s_tab + (size_t)kk[u] * 64);
                    uint8_t *dst = s_x + ((size_t)(4 * (p & 1)) * slab + (size_t)(M0 + (p >> 1)) * 16);
#pragma unroll
                    for (int g = 0; g < NG; ++g) reinterpret_cast<uint4 *>(dst + (size_t)g * slab)[0] = src[g];
                }
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(xready);
            for (int l = 0; l < L; ++l, ++lc) {
                const bool conv2 = (l & 1) != 0, last = l == L - 1;
                const float *bias = s_b + l * 32;
                uint8_t *dst = conv2 ? s_x : s_h;
                for (int j = 0; j < T; ++j, ++ti) {
                    // tile ti: accumulator a = ti % 3; its even pixels go to group
                    // a, its odd pixels to group a + 1 (mod 3), halving the
                    // epilogue latency per tile (a layer has few tiles, and tile
                    // j of the next layer waits for tiles j - 1 .. j + 1)
                    const int a = (int)(ti % kD2Groups);
                    const int h = a == grp ? 0 : (a == (grp + kD2Groups - 1) % kD2Groups ? 1 : -1);
                    if (h < 0) continue;
                    const uint32_t u = (uint32_t)(ti / kD2Groups);
                    const int r = 128 * j + row;
                    const int n = (int)fdiv((uint32_t)r, div_hw), rem = r - n * HWq;
                    const int y = (int)fdiv((uint32_t)rem, div_w), x = 2 * (rem - y * Wq) + h;
                    mbar_wait(&tfull[a], u & 1);
                    tc_fence_after();
                    {
                        float v[32];
                        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(a * 64 + 32 * h), v);
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[a]);
                        if (!(n < g_act && y >= 1 && y <= gh && x >= 1 && x <= gw)) goto tile_done;
                        uint4 w4[NG];
#pragma unroll
                        for (int g = 0; g < NG; ++g) {
                            float o[8];
#pragma unroll
                            for (int e = 0; e < 8; ++e) o[e] = __fadd_rn(v[8 * g + e], bias[8 * g + e]);
                            if (conv2) {
                                const uint4 rv = reinterpret_cast<const uint4 *>(
                                    s_x + (size_t)(g + 4 * h) * slab + (size_t)(M0 + r) * 16)[0];
                                const uint32_t rw[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    o[2 * e] = __fadd_rn(bf16_lo(rw[e]), o[2 * e]);
                                    o[2 * e + 1] = __fadd_rn(bf16_hi(rw[e]), o[2 * e + 1]);
                                }
                            }
#pragma unroll
                            for (int e = 0; e < 8; ++e) o[e] = fmaxf(o[e], 0.f);
                            w4[g] = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]),
                                               pack_bf16(o[6], o[7]));
                        }
                        if (last) {
                            const int64_t q = (n0 + n) * HW + (int64_t)y * Wp + x;
#pragma unroll
                            for (int g = 0; g < NG; ++g)
                                store_px(P.out + ((int64_t)g * P.out_gstride + P.out_margin) * 8, q, w4[g], y, x, gh,
                                         gw, Wp);
                        } else {
                            // pixel q of the group at slab g + 4 (q & 1), row q / 2, plus its edge copies
                            const int q = n * HWpp + y * Wpp + x;
                            const int ey = (y == 1 ? -Wpp : (y == gh ? Wpp : 0)), ey2 = (y == 1 && y == gh) ? Wpp : 0;
                            const int ex = (x == 1 ? -1 : (x == gw ? 1 : 0)), ex2 = (x == 1 && x == gw) ? 1 : 0;
#pragma unroll
                            for (int g = 0; g < NG; ++g) {
                                auto put = [&](int qq) {
                                    reinterpret_cast<uint4 *>(dst + (size_t)(g + 4 * (qq & 1)) * slab +
                                                              (size_t)(M0 + (qq >> 1)) * 16)[0] = w4[g];
                                };
                                put(q);
                                if (ex) put(q + ex);
                                if (ex2) put(q + ex2);
                                if (ey) {
                                    put(q + ey);
                                    if (ex) put(q + ey + ex);
                                    if (ex2) put(q + ey + ex2);
                                }
                                if (ey2) {
                                    put(q + ey2);
                                    if (ex) put(q + ey2 + ex);
                                    if (ex2) put(q + ey2 + ex2);
                                }
                            }
                        }
                    }
                tile_done:
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&hrdy[j]);
                }
            }
            // the next group's gather overwrites X: every epilogue warp is past its residual reads
            asm volatile("bar.sync 1, %0;" ::"n"(128 * kD2Groups) : "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u));
    }
}

size_t dec_trunk2_smem(int Hp, int Wp, int G, int K, int n_conv, int *pad) {
    const int Wq = ((Wp + 1) & ~1) / 2;
    const int rows = G * Hp * Wq, T = (rows + 127) / 128, M0 = Wq + 1;
    const size_t RS = (size_t)M0 + rows + M0;
    const int p = ((128 * T - rows + 16) * 16 + 127) / 128 * 128;
    if (pad) *pad = p;
    return kD2Slots * kD2Chunk + (size_t)K * 64 + 2 * 8 * RS * 16 + p +
           (2 * kD2Slots + 2 * kD2Groups + 2 + kD2MaxTiles) * 8 + 16 + (size_t)n_conv * 32 * 4;
}

// ---- decoder output stage in shared memory (vqvae.py:101-112) ---------------
// The up conv (3x3, 32 -> 128), pixel shuffle + ReLU and the logistic head of
// one image per CTA iteration; the 2x hi-res activations (the largest tensor
// of the decoder) never leave shared memory. The image's padded latent grid
// arrives by one bulk copy per channel group; the up conv runs as
// tc_conv_kernel<128, 3, SHUFFLE> (18 MMAs of N = 128 per 128-row tile), its
// epilogue writes the shuffled bf16 activations in the pair head's layout
// (row = two horizontally adjacent pixels, 8 channel groups; edges
// replicated) into a shared buffer, and the head runs as tc_conv_kernel<16,
// 3, HEAD2> (24 MMAs of N = 16 per tile) from there. Same MMAs, same K order,
// same epilogue roundings: shift / d / mu / s are bit-identical to the two
// launches.
//
// Overlap: every tile of an image has its own TMEM accumulator (up tiles at
// columns 128 t, head tiles at 384 + 16 k), so the tensor core runs image i's
// up tiles, then its head tiles (each waiting only for the up tile that
// writes its last input row, `hrdy`), then image i + 1's up tiles while
// image i's head epilogue drains. The hi-res buffer is single: image i + 1's
// up epilogue waits for image i's head MMAs (`hfree`), which the tensor core
// has finished before image i + 1's up MMAs anyway. The latent buffer is
// reloaded as soon as an image's up MMAs complete.
//
// Warps: 0 bulk-copy producer, 1 TMEM allocator + MMA issuer, 2..5 up
// epilogue, 6..13 head epilogue (two groups of four, alternate tiles).
constexpr int kUhMaxUp = 3, kUhMaxHead = 8;  // tiles per image: TMEM 128 x 3 + 16 x 8 = 512 columns
constexpr int kThreadsUH = 448;
constexpr uint32_t kUhWUp = 36 * 128 * 16, kUhWHead = 48 * 16 * 16;
constexpr int kUhBars = 32;  // >= 4 + 3 kUhMaxUp + 2 kUhMaxHead, even
static_assert(kUhBars >= 4 + 3 * kUhMaxUp + 2 * kUhMaxHead && kUhBars % 2 == 0, "barrier block");

struct UhGeom {
    int Wp, HW, Tu, M0, RSu;  // latent grid, up tiles, slab rows
    int Wq, HWq, Th, M0q, RSh;  // hi-res pair grid, head tiles, slab rows
};
__host__ __device__ inline UhGeom uh_geom(int gh, int gw) {
    UhGeom g;
    g.Wp = gw + 2;
    g.HW = (gh + 2) * g.Wp;
    g.Tu = (g.HW + 127) / 128;
    g.M0 = g.Wp + 1;
    g.RSu = g.M0 + 128 * g.Tu + g.M0;
    g.Wq = gw + 1;
    g.HWq = (2 * gh + 2) * g.Wq;
    g.Th = (g.HWq + 127) / 128;
    g.M0q = g.Wq + 1;
    g.RSh = g.M0q + 128 * g.Th + g.M0q;
    return g;
}
size_t dec_uphead_smem(const UhGeom &g) {
    return kUhWUp + kUhWHead + 4 * (size_t)g.RSu * 16 + 8 * (size_t)g.RSh * 16 +
           8 * kUhBars + 16 + (128 + 16 + 256) * 4;
}

__global__ void __launch_bounds__(kThreadsUH, 1) dec_uphead_kernel(DecUpHead P) {
    const UhGeom G = uh_geom(P.gh, P.gw);
    const int gh = P.gh, gw = P.gw, Wp = G.Wp, Wq = G.Wq, Tu = G.Tu, Th = G.Th;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *s_wu = smem;                                   // [36][128][8] bf16
    uint8_t *s_wh = s_wu + kUhWUp;                          // [48][16][8] bf16
    uint8_t *s_x = s_wh + kUhWHead;                         // 4 slabs x RSu rows: latent
    uint8_t *s_q = s_x + 4 * (size_t)G.RSu * 16;            // 8 slabs x RSh rows: hi-res pairs
    uint64_t *bars = reinterpret_cast<uint64_t *>(s_q + 8 * (size_t)G.RSh * 16);
    uint64_t *wbar = bars, *lfull = bars + 1, *lempty = bars + 2, *hfree = bars + 3;
    uint64_t *ufull = bars + 4, *uempty = ufull + kUhMaxUp, *hrdy = uempty + kUhMaxUp;
    uint64_t *qfull = hrdy + kUhMaxUp, *qempty = qfull + kUhMaxHead;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + kUhBars);
    float *s_bu = reinterpret_cast<float *>(tmem_slot + 4);  // 128 up biases (16-byte aligned: float4 reads)
    float *s_bh = s_bu + 128;                                // 6 head biases
    float *s_thr = s_bh + 16;                                // rd32 thresholds

    const int warp = __shfl_sync(0xFFFFFFFFu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    for (int c = threadIdx.x; c < 128; c += blockDim.x) s_bu[c] = P.b_up[c];
    for (int c = threadIdx.x; c < 16; c += blockDim.x) s_bh[c] = c < 6 ? P.b_head[c] : 0.f;
    for (int k = threadIdx.x; k < P.n_thresh; k += blockDim.x) s_thr[k] = __double2float_rd(P.thresh[k]);
    // finite operands everywhere: rows no image writes (tile tails, margins)
    // are read by the pair head's zero-weight K segments (0 x NaN = NaN)
    {
        uint4 *z = reinterpret_cast<uint4 *>(s_x);
        const int n16 = 4 * G.RSu + 8 * G.RSh;
        for (int e = threadIdx.x; e < n16; e += blockDim.x) z[e] = make_uint4(0u, 0u, 0u, 0u);
        fence_async_smem();
    }
    if (threadIdx.x == 0) {
        mbar_init(wbar, 1);
        mbar_init(lfull, 1);
        mbar_init(lempty, 1);
        mbar_init(hfree, 1);
        for (int t = 0; t < kUhMaxUp; ++t) {
            mbar_init(&ufull[t], 1);
            mbar_init(&uempty[t], 4);
            mbar_init(&hrdy[t], 4);
        }
        for (int k = 0; k < kUhMaxHead; ++k) {
            mbar_init(&qfull[k], 1);
            mbar_init(&qempty[k], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xFFFFFFFFu, *tmem_slot, 0);

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(wbar, kUhWUp + kUhWHead);
            bulk_g2s(s_wu, P.w_up, kUhWUp, wbar);
            bulk_g2s(s_wh, P.w_head, kUhWHead, wbar);
            const uint32_t bytes = (uint32_t)G.HW * 16u;
            int i = 0;
            for (int64_t n = blockIdx.x; n < P.n_img; n += gridDim.x, ++i) {
                if (i > 0) mbar_wait(lempty, (i - 1) & 1);
                mbar_expect_tx(lfull, 4 * bytes);
#pragma unroll
                for (int g = 0; g < 4; ++g)
                    bulk_g2s(s_x + ((size_t)g * G.RSu + G.M0) * 16,
                             P.in + ((int64_t)g * P.gstride + P.margin + n * G.HW) * 8, bytes, lfull);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idu = idesc_bf16(128, 128), idh = idesc_bf16(128, 16);
        mbar_wait(wbar, 0);
        tc_fence_after();
        const uint64_t dX = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_x), 0), (uint32_t)G.RSu * 16u, 128u);
        const uint64_t dQ = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_q), 0), (uint32_t)G.RSh * 16u, 128u);
        const uint64_t dWu = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_wu), 0), 128u * 16u, 128u);
        const uint64_t dWh = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_wh), 0), 16u * 16u, 128u);
        const uint32_t rsu = (uint32_t)G.RSu, rsh = (uint32_t)G.RSh;
        int i = 0;
        for (int64_t n = blockIdx.x; n < P.n_img; n += gridDim.x, ++i) {
            mbar_wait(lfull, i & 1);
            tc_fence_after();
            for (int t = 0; t < Tu; ++t) {
                if (i > 0) mbar_wait(&uempty[t], (i - 1) & 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(128 * t);
                // tile rows q0 = 128 t; tap (di, dj) reads from q0 - Wp - 1 + di Wp + dj (slab row + M0)
                const uint32_t al = (uint32_t)dX + (uint32_t)(128 * t), ah = (uint32_t)(dX >> 32);
                const uint32_t bl = (uint32_t)dWu, bh = (uint32_t)(dWu >> 32);
#pragma unroll
                for (int tap = 0; tap < 9; ++tap) {
                    const uint32_t off = (uint32_t)((tap / 3) * Wp + tap % 3);
#pragma unroll
                    for (int ks = 0; ks < 2; ++ks)
                        mma_bf16_elect_w(d, al + 2u * ks * rsu + off, ah, bl + (uint32_t)((tap * 4 + 2 * ks) * 128), bh,
                                         idu, (tap | ks) ? 1u : 0u);
                }
                mma_commit_elect(&ufull[t]);
            }
            mma_commit_elect(lempty);
            int waited = -1;
            for (int k = 0; k < Th; ++k) {
                // the up tile writing this head tile's last input row (pair row
                // 128 k + 128 + Wq): hi-res row Y comes from latent row (Y + 1) / 2
                int Y = (128 * k + 128 + Wq) / Wq;
                Y = Y > 2 * gh + 1 ? 2 * gh + 1 : Y;
                int y = (Y + 1) >> 1;
                y = y < 1 ? 1 : (y > gh ? gh : y);
                int tn = (y * Wp + gw) >> 7;
                tn = tn > Tu - 1 ? Tu - 1 : tn;
                if (tn > waited) {
                    mbar_wait(&hrdy[tn], i & 1);
                    waited = tn;
                }
                if (i > 0) mbar_wait(&qempty[k], (i - 1) & 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(384 + 16 * k);
                const uint32_t al = (uint32_t)dQ + (uint32_t)(128 * k), ah = (uint32_t)(dQ >> 32);
                const uint32_t bl = (uint32_t)dWh, bh = (uint32_t)(dWh >> 32);
                // per row tap di, 8 K steps: the left pair's odd pixel (groups
                // 4-7), this pair (0-7), the right pair's even pixel (0-3)
#pragma unroll
                for (int di = 0; di < 3; ++di) {
#pragma unroll
                    for (int sg = 0; sg < 8; ++sg) {
                        const uint32_t slab = (sg < 2) ? 4u + 2u * sg : (sg < 6 ? 2u * (sg - 2) : 2u * (sg - 6));
                        const uint32_t dj = sg < 2 ? 0u : (sg < 6 ? 1u : 2u);
                        const uint32_t off = (uint32_t)di * (uint32_t)Wq + dj;
                        mma_bf16_elect_w(d, al + slab * rsh + off, ah, bl + (uint32_t)((2 * (di * 8 + sg)) * 16), bh,
                                         idh, (di | sg) ? 1u : 0u);
                    }
                }
                mma_commit_elect(&qfull[k]);
            }
            mma_commit_elect(hfree);
        }
    } else if (warp < 6) {
        // up epilogue: bias, ReLU, bf16, pixel shuffle into the pair buffer
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int H2 = 2 * gh, W2 = 2 * gw, Wp2 = 2 * Wq;
        int i = 0;
        for (int64_t n = blockIdx.x; n < P.n_img; n += gridDim.x, ++i) {
            for (int t = 0; t < Tu; ++t) {
                const int q = 128 * t + row;
                const int y = q / Wp, x = q - y * Wp;
                const bool valid = q < G.HW && y >= 1 && y <= gh && x >= 1 && x <= gw;
                mbar_wait(&ufull[t], i & 1);
                if (t == 0 && i > 0) mbar_wait(hfree, (i - 1) & 1);  // image i - 1's head MMAs are done reading
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(128 * t);
#pragma unroll 1
                for (int z = 0; z < 4; ++z) {
                    float v[32];
                    tmem_ld32(taddr + (uint32_t)(32 * z), v);
                    if (z == 3) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&uempty[t]);
                    }
                    if (!valid) continue;
                    float bz[32];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float4 b4 = reinterpret_cast<const float4 *>(s_bu + 32 * z)[e];
                        bz[4 * e] = b4.x;
                        bz[4 * e + 1] = b4.y;
                        bz[4 * e + 2] = b4.z;
                        bz[4 * e + 3] = b4.w;
                    }
#pragma unroll
                    for (int sub = 0; sub < 4; ++sub) {
                        const int dy = sub >> 1, dx = sub & 1;
                        float o[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) o[e] = fmaxf(__fadd_rn(v[4 * e + sub], bz[4 * e + sub]), 0.f);
                        const int Y = 2 * (y - 1) + dy + 1, X = 2 * (x - 1) + dx + 1;
                        const uint4 w4 = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]),
                                                    pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
                        auto put = [&](int qq) {
                            reinterpret_cast<uint4 *>(s_q + ((size_t)(z + 4 * (qq & 1)) * G.RSh + G.M0q) * 16)[qq >> 1] =
                                w4;
                        };
                        const int q2 = Y * Wp2 + X;
                        put(q2);
                        const int ey = (Y == 1 ? -Wp2 : (Y == H2 ? Wp2 : 0));
                        const int ex = (X == 1 ? -1 : (X == W2 ? 1 : 0));
                        if (ex) put(q2 + ex);
                        if (ey) put(q2 + ey);
                        if (ex && ey) put(q2 + ey + ex);
                    }
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&hrdy[t]);
            }
        }
    } else {
        // head epilogue (vqvae.py:105-112, logistic.py:36-40, 109-114): as
        // tc_conv_kernel's TC_OUT_HEAD2, two groups of four warps taking
        // alternate tiles (the epilogue is math-heavy: one group cannot keep up
        // with the tensor core)
        const int hg = (warp - 6) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int H2 = 2 * gh, W2 = 2 * gw;
        const int nt = P.n_thresh;
        float thr[8];  // the usual grids (D <= 9) compare against registers
#pragma unroll
        for (int e = 0; e < 8; ++e) thr[e] = e < nt ? s_thr[e] : __int_as_float(0x7f800000);
        int i = 0;
        for (int64_t n = blockIdx.x; n < P.n_img; n += gridDim.x, ++i) {
            for (int k = hg; k < Th; k += 2) {
                const int p = 128 * k + row;
                const int Y = p / Wq, X = 2 * (p - Y * Wq);
                mbar_wait(&qfull[k], i & 1);
                tc_fence_after();
                float v[16];
                tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(384 + 16 * k), v);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&qempty[k]);
                auto head_px = [&](const float *vv, int xx) {
                    if (!(Y >= 1 && Y <= H2 && xx >= 1 && xx <= W2)) return;
                    if (!((Y - 1) < P.crop_h && (xx - 1) < P.crop_w)) return;
                    const int64_t px = ((int64_t)n * P.crop_h + (Y - 1)) * (int64_t)P.crop_w + (xx - 1);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        float av = __fadd_rn(vv[c], s_bh[c]);
                        av = fminf(fmaxf(av, -15.f), 15.f);
                        const float mu = __fmul_rn(255.f, __fdividef(1.f, 1.f + __expf(-av)));
                        float bv = __fadd_rn(vv[3 + c], s_bh[3 + c]);
                        bv = fminf(fmaxf(bv, P.log_s_min), P.log_s_max);
                        float sv = fminf(fmaxf(__expf(bv), 0.5f), 64.f);
                        const float fl = floorf(mu);
                        const int shift = (int)fl + (__fsub_rn(mu, fl) >= 0.5f ? 1 : 0);
                        int d = 0;
                        if (nt <= 8) {
#pragma unroll
                            for (int e = 0; e < 8; ++e) d += sv > thr[e];
                        } else {
                            for (int e = 0; e < nt; ++e) d += sv > s_thr[e];
                        }
                        P.shift[px * 3 + c] = (uint8_t)shift;
                        P.dsel[px * 3 + c] = (uint8_t)d;
                        if (P.mu) P.mu[px * 3 + c] = mu;
                        if (P.s) P.s[px * 3 + c] = sv;
                    }
                };
                head_px(v, X);
                head_px(v + 6, X + 1);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
    }
}

// ---- encoder front on tcgen05 (vqvae.py:55-57) -----------------------------
// stem (3x3, 3 -> 32, ReLU) and down (3x3 stride 2, 32 -> 32, ReLU), both as
// 3-product fp16 MMAs, in one kernel: the stem never leaves the SM.
//
// Down. The stride-2 conv is a stride-1 implicit GEMM over the space-to-depth
// view of the stem output: s2d cell (a, b) of the latent grid holds stem
// pixels (2a + pi, 2b + pj), four phases x 32 channels. Down output (u, v)
// tap (i, j) reads stem (2u + i - 1, 2v + j - 1) = s2d cell (u + di, v + dj)
// phase (pi, pj) with (di, pi) = (-1, 1), (0, 0), (0, 1) for i = 0, 1, 2
// (likewise j). With s2d cells on the padded latent indexing (borders
// included) each tap is the stage's K-major operand shifted by
// (di + 1) Wp + (dj + 1) rows and offset to the phase's channel groups --
// the tap-shift trick of the block convs. Clamping (nn.conv2d edge padding,
// _even_pad) is exact: every s2d cell, border cells included, is the stem at
// clamp(2a + pi) x clamp(2b + pj), which is what the reference's padded down
// conv reads. Cells no valid output reads stay zero.
//
// Stem. Per down tile the needed stem pixels m = phase * npix + s2d row are
// cut into 128-pixel chunks: an im2col row per pixel (27 normalised inputs
// in the reference's channel-tap order, padded to K = 32, scaled by 2^14 and
// split into fp16 hi / lo), one 128 x 32 x 32 3-product MMA per chunk, and an
// epilogue (bias, ReLU, 2^k_stem scale, split) that writes the chunk into
// the down stage.
//
// Warps: 0 weight copies, 1 MMA issuer (stem chunks of tile i + 1 are issued
// before the down GEMM of tile i), 2..5 down epilogue, 6..9 and 14..17 stem
// epilogue, 10..13 and 18..21 im2col producers (pairs of groups take
// alternate chunks).
constexpr int kEfThreads = 704;
constexpr int kEfRing = 4;     // im2col chunk buffers
constexpr int kEfSlots = 6;    // stem accumulators in TMEM (>= chunks per tile)
constexpr int kEfMaxQ = 8;     // down-stage phase quarters, at most
constexpr int kEfChunkBytes = 2 * 4 * 128 * 16;  // hi + lo, 4 K groups, 128 rows

__global__ void __launch_bounds__(kEfThreads, 1) enc_front_tc_kernel(EncFrontTc a) {
    constexpr int N = 32, N2 = 64;
    const int Wp = a.gw + 2, Hp = a.gh + 2;
    const int npix = (128 + Wp + 1 + 7) & ~7;
    const int nch = (4 * npix + 127) >> 7;  // stem chunks per down tile
    // the down stage is a ring of nq phase quarters (one phase's 4 hi + 4 lo
    // channel groups, npix rows each): tile i phase ph lives in quarter
    // (4 i + ph) % nq, so the stem epilogue of the next tile writes a phase
    // as soon as the down GEMM's last tap reading that quarter is done
    const int nq = a.n_quarters;
    const uint32_t q_bytes = 8u * npix * 16u;
    constexpr uint32_t wd_bytes = 36 * N2 * 16, ws_bytes = 4 * N2 * 16;

    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *s_wd = smem;
    uint8_t *s_wsb = smem + wd_bytes;
    uint8_t *s_a = s_wsb + ws_bytes;                             // down stage quarters [nq]
    uint8_t *s_c = s_a + (size_t)nq * q_bytes;                   // im2col ring
    float *s_bs = reinterpret_cast<float *>(s_c + kEfRing * kEfChunkBytes);
    float *s_bd = s_bs + N;
    // per byte value: the fp16 hi | lo << 16 split of (x / 127.5 - 1) 2^14
    // (vqvae.py:41-43): the stem operand is a function of the byte alone
    uint32_t *s_hl = reinterpret_cast<uint32_t *>(s_bd + N);
    uint64_t *bars = reinterpret_cast<uint64_t *>(s_hl + 256);
    uint64_t *afull = bars, *aempty = afull + kEfRing;
    uint64_t *sfull = aempty + kEfRing, *sempty = sfull + kEfSlots;
    uint64_t *dfull = sempty + kEfSlots, *qempty = dfull + 1;  // qempty[kEfMaxQ]
    uint64_t *tfull = qempty + kEfMaxQ, *tempty = tfull + 2;
    uint64_t *wbar = tempty + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(wbar + 1);

    const int warp = __shfl_sync(0xFFFFFFFFu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    if (threadIdx.x < N) {
        s_bs[threadIdx.x] = a.b_stem[threadIdx.x];
        s_bd[threadIdx.x] = a.b_down[threadIdx.x];
    }
    for (int e = threadIdx.x; e < 256; e += blockDim.x) {
        const float xn = __fmul_rn(__fsub_rn(__fdiv_rn((float)e, 127.5f), 1.f), 16384.f);
        uint32_t h, l;
        split2(xn, 0.f, h, l);
        s_hl[e] = (h & 0xFFFFu) | (l << 16);
    }
    if (threadIdx.x == 0) {
        for (int r = 0; r < kEfRing; ++r) {
            mbar_init(&afull[r], 4);
            mbar_init(&aempty[r], 1);
        }
        for (int r = 0; r < kEfSlots; ++r) {
            mbar_init(&sfull[r], 1);
            mbar_init(&sempty[r], 4);
        }
        mbar_init(dfull, 8);
        for (int q = 0; q < kEfMaxQ; ++q) mbar_init(&qempty[q], 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        mbar_init(wbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xFFFFFFFFu, *tmem_slot, 0);
    const uint32_t tmem_down = tmem + 64u * kEfSlots;
    const int64_t n_tiles = a.n_tiles;
    const uint32_t img_px = (uint32_t)(Hp * Wp);
    const FastDiv div_hw{img_px, (uint32_t)(0x100000000ull / img_px)};
    const FastDiv div_w{(uint32_t)Wp, (uint32_t)(0x100000000ull / (uint32_t)Wp)};
    const FastDiv div_np{(uint32_t)npix, (uint32_t)(0x100000000ull / (uint32_t)npix)};
    const int He = 2 * a.gh, We = 2 * a.gw;
    // stem pixel m of tile t: s2d row p = m % npix, phase ph = m / npix;
    // live when some valid down output reads it
    auto stem_px = [&](int64_t t, int m, int &ph, int &p, uint32_t &n, int &sy, int &sx) -> bool {
        ph = (int)fdiv((uint32_t)m, div_np);
        p = m - ph * npix;
        if (ph > 3) return false;
        const int64_t q = t * 128 - (Wp + 1) + p;
        if (q < 0) return false;
        n = fdiv((uint32_t)q, div_hw);
        const uint32_t rem = (uint32_t)q - n * img_px;
        const int yy = (int)fdiv(rem, div_w), xx = (int)(rem - (uint32_t)yy * div_w.d);
        // latent rows -1 .. gh-1 (row -1 only in phase pi = 1), likewise columns
        if (n >= (uint64_t)a.n_img || yy > a.gh || xx > a.gw || (yy < 1 && !(ph >> 1)) || (xx < 1 && !(ph & 1)))
            return false;
        sy = min(max(2 * (yy - 1) + (ph >> 1), 0), He - 1);
        sx = min(max(2 * (xx - 1) + (ph & 1), 0), We - 1);
        return true;
    };

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(wbar, wd_bytes + ws_bytes);
            bulk_g2s(s_wd, a.w_down, wd_bytes, wbar);
            bulk_g2s(s_wsb, a.w_stem16, ws_bytes, wbar);
        }
    } else if ((warp >= 10 && warp < 14) || warp >= 18) {
        // im2col producers, two groups of four warps (10..13, 18..21) taking
        // alternate chunks; one stem pixel (row of the chunk) per thread
        const int pg = warp >= 18 ? 1 : 0;
        const int row = threadIdx.x - (pg ? 18 : 10) * 32;
        int64_t g = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
            for (int c = 0; c < nch; ++c, ++g) {
                if ((int)(g & 1) != pg) continue;
                const int slot = (int)(g % kEfRing);
                if (g >= kEfRing) mbar_wait(&aempty[slot], (uint32_t)((g / kEfRing) - 1) & 1);
                uint4 *hs = reinterpret_cast<uint4 *>(s_c + (size_t)slot * kEfChunkBytes);
                uint4 *ls = hs + 4 * 128;
                int ph, p, sy = 0, sx = 0;
                uint32_t n = 0;
                const bool live = stem_px(t, c * 128 + row, ph, p, n, sy, sx);
                uint32_t hw[16], lw[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) hw[e] = lw[e] = 0u;
                if (live) {
                    const uint8_t *img = a.img + (int64_t)n * a.H * a.W * 3;
                    uint32_t xv[28];  // per tap the byte's hi | lo << 16 (K = c*9 + tap, 27 -> 28)
#pragma unroll
                    for (int ki = 0; ki < 3; ++ki) {
                        const uint8_t *rp = img + (int64_t)min(max(sy + ki - 1, 0), a.H - 1) * a.W * 3;
#pragma unroll
                        for (int kj = 0; kj < 3; ++kj) {
                            const uint8_t *px = rp + min(max(sx + kj - 1, 0), a.W - 1) * 3;
#pragma unroll
                            for (int ch = 0; ch < 3; ++ch) xv[ch * 9 + ki * 3 + kj] = s_hl[__ldg(px + ch)];
                        }
                    }
                    xv[27] = 0u;
#pragma unroll
                    for (int e = 0; e < 14; ++e) {  // k = 2e, 2e + 1 (the same split2 of x 2^14, by table)
                        hw[e] = __byte_perm(xv[2 * e], xv[2 * e + 1], 0x5410);
                        lw[e] = __byte_perm(xv[2 * e], xv[2 * e + 1], 0x7632);
                    }
                }
#pragma unroll
                for (int kg = 0; kg < 4; ++kg) {
                    hs[kg * 128 + row] = make_uint4(hw[4 * kg], hw[4 * kg + 1], hw[4 * kg + 2], hw[4 * kg + 3]);
                    ls[kg * 128 + row] = make_uint4(lw[4 * kg], lw[4 * kg + 1], lw[4 * kg + 2], lw[4 * kg + 3]);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&afull[slot]);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc64 = idesc_f16(128, N2);
        constexpr uint32_t idesc32 = idesc_f16(128, N);
        mbar_wait(wbar, 0);
        tc_fence_after();
        const uint64_t dA0 = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_a), 0), (uint32_t)npix * 16u, 128u);
        const uint64_t dB0 = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_wd), 0), (uint32_t)N2 * 16u, 128u);
        const uint64_t dC0 = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_c), 0), 128u * 16u, 128u);
        const uint64_t dS0 = umma_desc(__shfl_sync(0xFFFFFFFFu, smem_u32(s_wsb), 0), (uint32_t)N2 * 16u, 128u);
        const uint32_t npx = (uint32_t)npix;
        int64_t gi = 0;  // next stem chunk to issue (global index)
        // stem chunks of one tile: A (im2col) x [Ws_hi | Ws_lo] and A_lo x Ws_hi
        auto issue_stem = [&]() {
            for (int c = 0; c < nch; ++c, ++gi) {
                const int r = (int)(gi % kEfRing), sl = (int)(gi % kEfSlots);
                mbar_wait(&afull[r], (uint32_t)(gi / kEfRing) & 1);
                if (gi >= kEfSlots) mbar_wait(&sempty[sl], (uint32_t)((gi / kEfSlots) - 1) & 1);
                tc_fence_after();
                const uint64_t dh = dC0 + (uint64_t)((uint32_t)r * (kEfChunkBytes >> 4));
                const uint64_t dl = dh + (uint64_t)(4 * 128);
                const uint32_t d = tmem + 64u * sl;
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const uint64_t ao = (uint64_t)(2 * ks * 128);
                    const uint64_t bo = (uint64_t)(2 * ks * N2);
                    mma_f16_elect(d, dh + ao, dS0 + bo, idesc64, ks ? 1u : 0u);
                    mma_f16_elect(d + N, dl + ao, dS0 + bo, idesc32, 1u);
                }
                mma_commit_elect(&aempty[r]);
                mma_commit_elect(&sfull[sl]);
            }
        };
        if (blockIdx.x < n_tiles) issue_stem();
        int i = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
            if (t + gridDim.x < n_tiles) issue_stem();  // next tile's stem overlaps this tile's down GEMM
            const int b = i & 1;
            const int u = i >> 1;
            if (u > 0) mbar_wait(&tempty[b], (u - 1) & 1);
            mbar_wait(dfull, (uint32_t)i & 1);
            tc_fence_after();
            const uint32_t d = tmem_down + (uint32_t)(b * N2);
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) {
                const int ti = tap / 3, tj = tap % 3;
                const uint32_t rows = (uint32_t)((ti == 0 ? 0 : Wp) + (tj == 0 ? 0 : 1));  // (di + 1) Wp + (dj + 1)
                const uint32_t ph = (uint32_t)((ti == 1 ? 0 : 2) + (tj == 1 ? 0 : 1));     // pi * 2 + pj
                const uint32_t qs = (uint32_t)((4 * i + (int)ph) % nq);
                const uint64_t dq = dA0 + (uint64_t)(qs * (q_bytes >> 4));
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const uint64_t ao = (uint64_t)(2u * ks * npx + rows);
                    const uint64_t bo = (uint64_t)((tap * 4 + 2 * ks) * N2);
                    mma_f16_elect(d, dq + ao, dB0 + bo, idesc64, (tap | ks) ? 1u : 0u);
                    mma_f16_elect(d + N, dq + ao + (uint64_t)(4u * npx), dB0 + bo, idesc32, 1u);
                }
                // taps 4, 5, 7, 8 are the last readers of phases 0, 1, 2, 3
                if (tap == 4 || tap == 5 || tap == 7 || tap == 8) mma_commit_elect(&qempty[qs]);
            }
            mma_commit_elect(&tfull[b]);
        }
    } else if (warp >= 6) {
        // stem epilogue, two groups of four warps (6..9, 14..17) taking
        // alternate chunks: chunk row -> stem pixel; bias, ReLU, 2^k_stem,
        // split into the down stage (phase ph's 4 hi / 4 lo groups, row p)
        const int grp = warp >= 14 ? 1 : 0;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int kws = __float_as_int(a.meta_stem[0]);
        const float inv = exp2i(-14 - kws);
        const float sc = exp2i(__float_as_int(a.meta_down[3]));
        uint4 *hs0 = reinterpret_cast<uint4 *>(s_a);
        int64_t g = 0;
        int i = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
            for (int c = 0; c < nch; ++c, ++g) {
                if ((int)(g & 1) != grp) continue;
                // the quarters this chunk writes must be free: their previous
                // tile's last reading tap has completed
                const int ph_lo = min(3, (128 * c) / npix), ph_hi = min(3, (128 * c + 127) / npix);
                for (int q = ph_lo; q <= ph_hi; ++q) {
                    const int qg = 4 * i + q;
                    if (qg >= nq) mbar_wait(&qempty[qg % nq], (uint32_t)((qg / nq) - 1) & 1);
                }
                const int sl = (int)(g % kEfSlots);
                int ph, p, sy, sx;
                uint32_t n;
                const bool live = stem_px(t, c * 128 + row, ph, p, n, sy, sx);
                mbar_wait(&sfull[sl], (uint32_t)(g / kEfSlots) & 1);
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + 64u * sl;
                float v[32];
                {
                    float w[32];
                    tmem_ld32(taddr, v);
                    tmem_ld32(taddr + 32, w);
#pragma unroll
                    for (int k = 0; k < 32; ++k)
                        v[k] = __fmul_rn(fmaxf(__fmaf_rn(__fmaf_rn(w[k], 0.00048828125f, v[k]), inv, s_bs[k]), 0.f),
                                         live ? sc : 0.f);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&sempty[sl]);
                if (ph < 4) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        uint4 h, l;
                        split2(v[8 * j + 0], v[8 * j + 1], h.x, l.x);
                        split2(v[8 * j + 2], v[8 * j + 3], h.y, l.y);
                        split2(v[8 * j + 4], v[8 * j + 5], h.z, l.z);
                        split2(v[8 * j + 6], v[8 * j + 7], h.w, l.w);
                        uint4 *hq = hs0 + (size_t)((4 * i + ph) % nq) * (q_bytes / 16);
                        hq[j * npix + p] = h;
                        hq[(4 + j) * npix + p] = l;
                    }
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(dfull);
        }
    } else {
        // down epilogue
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int H = a.gh, W = a.gw;
        const float inv = exp2i(-__float_as_int(a.meta_down[3]) - __float_as_int(a.meta_down[0]));
        const int ko = *a.k0;
        const float osc = exp2i(ko);
        int i = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
            const int b = i & 1;
            const int u = i >> 1;
            const uint32_t q = (uint32_t)t * 128u + (uint32_t)row;
            const uint32_t n = fdiv(q, div_hw);
            const uint32_t rem = q - n * div_hw.d;
            const int y = (int)fdiv(rem, div_w), x = (int)(rem - (uint32_t)y * div_w.d);
            const bool valid = n < (uint64_t)a.n_img && y >= 1 && y <= H && x >= 1 && x <= W;
            mbar_wait(&tfull[b], u & 1);
            tc_fence_after();
            const uint32_t taddr = tmem_down + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * N2);
            float v[32];
            {
                float w[32];
                tmem_ld32(taddr, v);
                tmem_ld32(taddr + 32, w);
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    v[c] = fmaxf(__fmaf_rn(__fmaf_rn(w[c], 0.00048828125f, v[c]), inv, s_bd[c]), 0.f);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[b]);
            float mx = 0.f;
            if (valid) {
#pragma unroll
                for (int g = 0; g < 8; ++g) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) mx = fmaxf(mx, v[4 * g + e]);
                    const int64_t so = ((int64_t)g * a.gstride + a.margin) * 4;
                    // fp32 copy: valid pixels only (no reader uses its edge copies)
                    reinterpret_cast<float4 *>(a.out32 + so)[q] =
                        make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint4 h, l;
                    split2(__fmul_rn(v[8 * j + 0], osc), __fmul_rn(v[8 * j + 1], osc), h.x, l.x);
                    split2(__fmul_rn(v[8 * j + 2], osc), __fmul_rn(v[8 * j + 3], osc), h.y, l.y);
                    split2(__fmul_rn(v[8 * j + 4], osc), __fmul_rn(v[8 * j + 5], osc), h.z, l.z);
                    split2(__fmul_rn(v[8 * j + 6], osc), __fmul_rn(v[8 * j + 7], osc), h.w, l.w);
                    store_px(a.out + ((int64_t)j * a.gstride + a.margin) * 8, q, h, y, x, H, W, Wp);
                    store_px(a.out + ((int64_t)(4 + j) * a.gstride + a.margin) * 8, q, l, y, x, H, W, Wp);
                }
            }
            const uint32_t n_ref = __shfl_sync(0xFFFFFFFFu, n, 0);
            const bool same = __all_sync(0xFFFFFFFFu, n == n_ref && valid);
            if (same) {
                const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(mx));
                if (lane == 0) {
                    if (m != 0u) atomicMax(a.out_max + n_ref, m);
                    a.kx_out[n_ref] = ko;
                }
            } else if (valid) {
                if (mx != 0.f) atomicMax(a.out_max + n, __float_as_uint(mx));
                a.kx_out[n] = ko;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
    }
}

// ---- codebook argmin on tcgen05 (vqvae.py:66-76) ---------------------------
// Per 128-latent tile: dot[r][k] = z_r . c_k for all 256 codes as a 3xTF32
// GEMM (z_hi c_hi + z_hi c_lo + z_lo c_hi, fp32 TMEM accumulators, M=128,
// N=256, K=32). The epilogue ranks codes by f_k = |c_k|^2 - 2 dot_k (|z|^2 is
// common to the row and cannot change the order). f_k is within
// e_k = a1 |z| |c_k| + a2 |c_k|^2 of the exact value: the dot product of the
// split operands is off by at most eps |z||c_k| (Cauchy-Schwarz) with
// eps = 2^-21 + 2^-21 + 2^-22 (tf32-truncated lo parts, dropped lo x lo) +
// 96 x 2^-23 (fp32 accumulation of 96 products, even with truncating adds)
// ~ 1.3e-5, |c_k|^2 in fp32 is within 32 x 2^-24, plus one rounding of f_k;
// a1 = 5.3e-5 and a2 = 4e-6 are twice those worst cases (the reference's own
// float64 rounding, ~1e-13 relative, is far inside the margin). With
// E = max_k e_k (a row constant), d1 < d2 the two smallest f and k1 the
// code of d1: if d2 - d1 > 2E every other code is strictly farther than k1
// under the reference's arithmetic, so k1 is its answer. Otherwise (~0.3% of
// rows) every code with f_k <= d1 + 2E -- a superset of the reference's
// possible winners -- is re-scored exactly as the reference does (float64,
// component order, no FMA) and the first minimum wins.
// Warps: 0 producer (bulk copies of z tiles), 1 TMEM + MMA, 2..9 epilogue
// in two groups of four (one per TMEM lane quarter); group g owns the tiles
// with i % 2 == g and TMEM buffer g, so a group re-scoring a rare ambiguous
// row never stalls the other, and no barrier spans the groups.
constexpr int kAmThreads = 320;
constexpr int kAmStages = 3;

__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float *v) {
    uint32_t r[64];
#pragma unroll
    for (int h = 0; h < 2; ++h)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[32 * h + 0]), "=r"(r[32 * h + 1]), "=r"(r[32 * h + 2]), "=r"(r[32 * h + 3]),
              "=r"(r[32 * h + 4]), "=r"(r[32 * h + 5]), "=r"(r[32 * h + 6]), "=r"(r[32 * h + 7]),
              "=r"(r[32 * h + 8]), "=r"(r[32 * h + 9]), "=r"(r[32 * h + 10]), "=r"(r[32 * h + 11]),
              "=r"(r[32 * h + 12]), "=r"(r[32 * h + 13]), "=r"(r[32 * h + 14]), "=r"(r[32 * h + 15]),
              "=r"(r[32 * h + 16]), "=r"(r[32 * h + 17]), "=r"(r[32 * h + 18]), "=r"(r[32 * h + 19]),
              "=r"(r[32 * h + 20]), "=r"(r[32 * h + 21]), "=r"(r[32 * h + 22]), "=r"(r[32 * h + 23]),
              "=r"(r[32 * h + 24]), "=r"(r[32 * h + 25]), "=r"(r[32 * h + 26]), "=r"(r[32 * h + 27]),
              "=r"(r[32 * h + 28]), "=r"(r[32 * h + 29]), "=r"(r[32 * h + 30]), "=r"(r[32 * h + 31])
            : "r"(taddr + 32u * h));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}

__global__ void __launch_bounds__(kAmThreads, 1) argmin_tc_kernel(ArgminTc a) {
    constexpr int NC = 256;                    // codes (N)
    constexpr uint32_t ZB = 2 * 8 * 128 * 16;  // z tile bytes (hi + lo)
    constexpr uint32_t CB = 2 * 8 * NC * 16;   // codebook operand bytes
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *s_cb = smem;                                            // [hi|lo][8][256][16 B]
    uint8_t *s_z = smem + CB;                                        // kAmStages x ZB
    float *s_cn = reinterpret_cast<float *>(s_z + kAmStages * ZB);   // |c_k|^2, +inf for k >= K
    uint32_t *s_max = reinterpret_cast<uint32_t *>(s_cn + NC);       // max |c_k|, max |c_k|^2 (f32 bits)
    uint64_t *bars = reinterpret_cast<uint64_t *>(s_max + 4);
    uint64_t *full = bars, *empty = bars + kAmStages, *tfull = bars + 2 * kAmStages, *tempty = tfull + 2;
    uint64_t *wbar = tempty + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(wbar + 1);
    const float a1 = 5.3e-5f, a2 = 4e-6f;

    const int warp = __shfl_sync(0xFFFFFFFFu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kAmStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1 + 4);  // MMA commit + the epilogue warps reading |z|^2
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        mbar_init(wbar, 1);
        s_max[0] = s_max[1] = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(wbar, CB);
        bulk_g2s(s_cb, a.cbt, CB, wbar);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xFFFFFFFFu, *tmem_slot, 0);
    mbar_wait(wbar, 0);
    const float *cb_hi = reinterpret_cast<const float *>(s_cb);
    const float *cb_lo = cb_hi + 8 * NC * 4;
    for (int k = threadIdx.x; k < NC; k += blockDim.x) {
        float acc = 0.f;
        for (int c = 0; c < 32; ++c) {
            const int e = ((c >> 2) * NC + k) * 4 + (c & 3);
            const float v = __fadd_rn(cb_hi[e], cb_lo[e]);
            acc = fmaf(v, v, acc);
        }
        s_cn[k] = k < a.K ? acc : INFINITY;  // codes >= K can never win
        if (k < a.K) {  // non-negative floats order as their bit patterns
            atomicMax(&s_max[0], __float_as_uint(sqrtf(acc) * 1.000001f));
            atomicMax(&s_max[1], __float_as_uint(acc));
        }
    }
    __syncthreads();

    const int64_t n_tiles = a.n_tiles;
    if (warp == 0) {
        if (lane == 0) {
            int i = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
                const int s = i % kAmStages, r = i / kAmStages;
                if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
                mbar_expect_tx(&full[s], ZB);
                bulk_g2s(s_z + (size_t)s * ZB, a.zt + t * (ZB / 4), ZB, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(128, NC);
            tc_fence_after();
            const uint32_t bhi = smem_u32(s_cb), blo = bhi + CB / 2;
            int i = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
                const int s = i % kAmStages, b = i & 1, u = i >> 1;
                if (u > 0) mbar_wait(&tempty[b], (u - 1) & 1);
                mbar_wait(&full[s], (i / kAmStages) & 1);
                tc_fence_after();
                const uint32_t ahi = smem_u32(s_z + (size_t)s * ZB), alo = ahi + ZB / 2;
                const uint32_t d = tmem + (uint32_t)(b * NC);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint32_t ao = (uint32_t)(2 * ks) * 128 * 16, bo = (uint32_t)(2 * ks) * NC * 16;
                    const uint64_t dah = umma_desc(ahi + ao, 128 * 16, 128), dal = umma_desc(alo + ao, 128 * 16, 128);
                    const uint64_t dbh = umma_desc(bhi + bo, NC * 16, 128), dbl = umma_desc(blo + bo, NC * 16, 128);
                    mma_tf32(d, dah, dbh, idesc, ks ? 1u : 0u);
                    mma_tf32(d, dah, dbl, idesc, 1u);
                    mma_tf32(d, dal, dbh, idesc, 1u);
                }
                mma_commit(&empty[s]);
                mma_commit(&tfull[b]);
            }
        }
    } else {
        const int grp = (warp - 2) >> 2;  // tiles i with i % 2 == grp, TMEM buffer grp
        const int quarter = warp & 3;     // TMEM lane quarter (warp % 4)
        const int row = quarter * 32 + lane;
        const float cmax = __uint_as_float(s_max[0]), cnmax = __uint_as_float(s_max[1]);
        const float4 *cn4 = reinterpret_cast<const float4 *>(s_cn);
        const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(grp * NC);
        int i = grp;
        for (int64_t t = blockIdx.x + (int64_t)grp * gridDim.x; t < n_tiles; t += 2 * (int64_t)gridDim.x, i += 2) {
            const int s = i % kAmStages, u = i >> 1;
            const int64_t v = t * 128 + row;
            const bool live = v < a.n_vec;
            // |z|^2 from the staged tile (z = hi + lo exactly)
            mbar_wait(&full[s], (i / kAmStages) & 1);
            const float4 *zs = reinterpret_cast<const float4 *>(s_z + (size_t)s * ZB) + row;
            float zn = 0.f;
#pragma unroll
            for (int gq = 0; gq < 8; ++gq) {
                const float4 h = zs[gq * 128], l = zs[(8 + gq) * 128];
                zn = fmaf(__fadd_rn(h.x, l.x), __fadd_rn(h.x, l.x), zn);
                zn = fmaf(__fadd_rn(h.y, l.y), __fadd_rn(h.y, l.y), zn);
                zn = fmaf(__fadd_rn(h.z, l.z), __fadd_rn(h.z, l.z), zn);
                zn = fmaf(__fadd_rn(h.w, l.w), __fadd_rn(h.w, l.w), zn);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            // 2E, E = max_k e_k; the 1.000001 covers the roundings of |z|^2, sqrt and the products
            const float e2 = 2.f * fmaf(a1 * sqrtf(zn) * 1.000001f, cmax, a2 * cnmax) * 1.000001f;

            mbar_wait(&tfull[grp], u & 1);
            tc_fence_after();
            // two interleaved chains of (smallest, its code, second smallest)
            float d1a = INFINITY, d2a = INFINITY, d1b = INFINITY, d2b = INFINITY;
            int k1a = 0, k1b = 0;
#pragma unroll 1
            for (int c = 0; c < NC / 64; ++c) {
                float dv[64];
                tmem_ld64(tbase + 64 * c, dv);
#pragma unroll
                for (int j = 0; j < 64; j += 4) {
                    const float4 cn = cn4[(64 * c + j) >> 2];
                    const int k = 64 * c + j;
                    float f = fmaf(-2.f, dv[j], cn.x);
                    d2a = fminf(d2a, fmaxf(d1a, f));
                    k1a = f < d1a ? k : k1a;
                    d1a = fminf(d1a, f);
                    f = fmaf(-2.f, dv[j + 1], cn.y);
                    d2b = fminf(d2b, fmaxf(d1b, f));
                    k1b = f < d1b ? k + 1 : k1b;
                    d1b = fminf(d1b, f);
                    f = fmaf(-2.f, dv[j + 2], cn.z);
                    d2a = fminf(d2a, fmaxf(d1a, f));
                    k1a = f < d1a ? k + 2 : k1a;
                    d1a = fminf(d1a, f);
                    f = fmaf(-2.f, dv[j + 3], cn.w);
                    d2b = fminf(d2b, fmaxf(d1b, f));
                    k1b = f < d1b ? k + 3 : k1b;
                    d1b = fminf(d1b, f);
                }
            }
            float d1, d2;
            int k1;
            if (d1b < d1a) {
                d1 = d1b, k1 = k1b, d2 = fminf(d1a, d2b);
            } else {
                d1 = d1a, k1 = k1a, d2 = fminf(d2a, d1b);
            }
            const bool amb = live && !(d2 - d1 > e2);
            if (__any_sync(0xffffffffu, amb)) {
                // rare: re-score every code with f_k <= d1 + 2E exactly as vqvae.py:71-75
                float zv[32];
                if (amb) {
                    const float4 *zt = reinterpret_cast<const float4 *>(a.zt) + t * (2 * 8 * 128) + row;
#pragma unroll
                    for (int gq = 0; gq < 8; ++gq) {
                        const float4 h = zt[gq * 128], l = zt[(8 + gq) * 128];
                        zv[4 * gq + 0] = __fadd_rn(h.x, l.x);
                        zv[4 * gq + 1] = __fadd_rn(h.y, l.y);
                        zv[4 * gq + 2] = __fadd_rn(h.z, l.z);
                        zv[4 * gq + 3] = __fadd_rn(h.w, l.w);
                    }
                }
                const float thr = d1 + e2;
                double best = INFINITY;
#pragma unroll 1
                for (int c = 0; c < NC / 64; ++c) {
                    float dv[64];
                    tmem_ld64(tbase + 64 * c, dv);
                    if (!amb) continue;
                    uint64_t cand = 0;
#pragma unroll
                    for (int j = 0; j < 64; ++j)
                        cand |= (uint64_t)(fmaf(-2.f, dv[j], s_cn[64 * c + j]) <= thr) << j;
#pragma unroll 1
                    for (; cand; cand &= cand - 1) {  // codes in increasing order
                        const int k = 64 * c + __ffsll((long long)cand) - 1;
                        double dist = 0.0;
#pragma unroll
                        for (int cc = 0; cc < 32; ++cc) {
                            const int e = ((cc >> 2) * NC + k) * 4 + (cc & 3);
                            const double diff = __dsub_rn((double)zv[cc], (double)__fadd_rn(cb_hi[e], cb_lo[e]));
                            dist = __dadd_rn(dist, __dmul_rn(diff, diff));
                        }
                        if (dist < best) {  // equal distances keep the lower code
                            best = dist;
                            k1 = k;
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[grp]);
            if (live) a.idx[v] = (uint8_t)k1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
    }
}

// shared-memory plan of one tc_conv_kernel launch: ring depth kStages, or as
// many stages as fit for wide images (>= 2); 0 when even that does not fit
template <int N, int KS, int MODE>
size_t tc_smem_plan(int Wp, int *stages) {
    constexpr int NG = MODE == TC_OUT_HEAD2 ? 8 : 4;
    constexpr int KG = MODE == TC_OUT_HEAD2 ? 48 : KS * KS * NG;
    const int npix = KS == 3 ? ((128 + 2 * Wp + 2 + 7) & ~7) : 128;
    auto smem_of = [&](int k) {
        return (size_t)KG * N * 16 + (size_t)k * NG * npix * 16 + 8 * (2 * k + 6) + 4 * N +
               4 * ((MODE == TC_OUT_HEAD || MODE == TC_OUT_HEAD2) ? 256 : 0) + 16;
    };
    int st = kStages;
    // the heads run two CTAs per SM: half the shared memory each
    const size_t cap = (MODE == TC_OUT_HEAD || MODE == TC_OUT_HEAD2) ? 113 * 1024 : 227 * 1024;
    while (st > 2 && smem_of(st) > cap) --st;
    *stages = st;
    return smem_of(st) > 227 * 1024 ? 0 : smem_of(st);
}

template <int N, int KS, int MODE>
int launch_tc(const TcLayer &L, cudaStream_t s) {
    int st = 0;
    const size_t smem = tc_smem_plan<N, KS, MODE>(L.Wp, &st);
    TcLayer Ls = L;
    Ls.n_stages = st;
    if ((uint64_t)L.n_img * L.Hp * L.Wp >= (1ull << 31)) return PILC_E_UNSUPPORTED;  // 32-bit pixel index
    if (smem == 0) return PILC_E_UNSUPPORTED;
    auto kern = tc_conv_kernel<N, KS, MODE>;
    allow_dyn_smem(reinterpret_cast<const void *>(kern));
    // one persistent CTA per SM (two epilogue groups, an 8-deep copy ring);
    // the head's math-heavy epilogue (few registers) runs two CTAs per SM
    int64_t grid = (int64_t)sm_count() * ((MODE == TC_OUT_HEAD || MODE == TC_OUT_HEAD2) ? 2 : 1);
    if (grid > L.n_tiles) grid = L.n_tiles;
    if (grid < 1) return PILC_OK;
    const double flops = 2.0 * L.n_img * L.H * L.W * (double)((MODE == TC_OUT_HEAD || MODE == TC_OUT_HEAD2) ? 6 : N) *
                         32 * KS * KS;
    ProfScope _ps(PROF_TC_CONV, s, flops);
    kern<<<(unsigned)grid, kThreadsTC, smem, s>>>(Ls);
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

// dec.proj folded into a table: T[k] = relu(W cb[k] + b), bf16 (K x 32)
__global__ void dec_table_kernel(const float *__restrict__ cb, const float *__restrict__ w,
                                 const float *__restrict__ b, int K, int Dc, int ci_pad, int co_pad,
                                 uint16_t *__restrict__ table) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K * 32) return;
    const int k = i / 32, c = i % 32;
    float acc = 0.f;
    for (int j = 0; j < Dc; ++j) acc = fmaf(cb[k * Dc + j], w[(int64_t)j * co_pad + c], acc);
    acc = fmaxf(__fadd_rn(acc, b[c]), 0.f);
    table[i] = __bfloat16_as_ushort(__float2bfloat16_rn(acc));
}

// X = T[idx] at every padded position (borders replicate by clamping)
__global__ void gather_kernel(const uint8_t *__restrict__ idx, const uint16_t *__restrict__ table,
                              int64_t n_img, int gh, int gw, uint16_t *__restrict__ x, int64_t gstride,
                              int64_t margin) {
    const int Hp = gh + 2, Wp = gw + 2;
    const int64_t total = n_img * Hp * Wp;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = q / ((int64_t)Hp * Wp);
        const int rem = (int)(q - n * Hp * Wp);
        int y = rem / Wp - 1, xx = rem % Wp - 1;
        y = y < 0 ? 0 : (y >= gh ? gh - 1 : y);
        xx = xx < 0 ? 0 : (xx >= gw ? gw - 1 : xx);
        const int k = idx[(n * gh + y) * gw + xx];
        const uint4 *row = reinterpret_cast<const uint4 *>(table + k * 32);
#pragma unroll
        for (int g = 0; g < 4; ++g) reinterpret_cast<uint4 *>(x + ((int64_t)g * gstride + margin) * 8)[q] = row[g];
    }
}

}  // namespace

__global__ void pack_z_tiles_kernel(const float *__restrict__ z, int64_t n, float *__restrict__ zt) {
    const int64_t nt = (n + 127) / 128;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nt * 128 * 8;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i >> 3;  // latent
        const int g = (int)(i & 7);  // 4-component group
        float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
        if (v < n) f = reinterpret_cast<const float4 *>(z)[v * 8 + g];
        const float in[4] = {f.x, f.y, f.z, f.w};
        float hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            hi[e] = tf32_rna(in[e]);
            lo[e] = __fsub_rn(in[e], hi[e]);
        }
        float4 *t = reinterpret_cast<float4 *>(zt) + (v >> 7) * (2 * 8 * 128) + (v & 127);
        t[g * 128] = make_float4(hi[0], hi[1], hi[2], hi[3]);
        t[(8 + g) * 128] = make_float4(lo[0], lo[1], lo[2], lo[3]);
    }
}

int tc_launch_act(const TcLayer &L, cudaStream_t s) { return launch_tc<32, 3, TC_OUT_ACT>(L, s); }
int pack_z_tiles(const float *z, int64_t n, float *zt, cudaStream_t s) {
    if (n <= 0) return PILC_OK;
    const int64_t work = ((n + 127) / 128) * 128 * 8;
    int64_t blocks = ceil_div64(work, 256);
    const int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    ProfScope _ps(PROF_GATHER, s, (double)n);
    pack_z_tiles_kernel<<<(unsigned)blocks, 256, 0, s>>>(z, n, zt);
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}
int argmin_tc_launch(const ArgminTc &a, cudaStream_t s) {
    if (a.n_tiles <= 0) return PILC_OK;
    if (a.K < 1 || a.K > 256) return PILC_E_ARG;
    const size_t smem = 2 * 8 * 256 * 16 + (size_t)kAmStages * 2 * 8 * 128 * 16 + 4 * 256 + 16 +
                        8 * (2 * kAmStages + 5) + 16;
    allow_dyn_smem(reinterpret_cast<const void *>(argmin_tc_kernel));
    int64_t grid = sm_count();
    if (grid > a.n_tiles) grid = a.n_tiles;
    ProfScope _ps(PROF_ARGMIN, s, 3.0 * a.n_vec * a.K * 32);
    argmin_tc_kernel<<<(unsigned)grid, kAmThreads, smem, s>>>(a);
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

int enc_front_tc_launch(const EncFrontTc &a, cudaStream_t s) {
    const int Wp = a.gw + 2;
    const int npix = (128 + Wp + 1 + 7) & ~7;
    if ((4 * npix + 127) / 128 > kEfSlots) return PILC_E_UNSUPPORTED;
    // as many down-stage phase quarters (>= 4, one full stage) as fit
    auto smem_of = [&](int nq) {
        return 36 * 64 * 16 + 4 * 64 * 16 + (size_t)nq * 8 * npix * 16 + (size_t)kEfRing * kEfChunkBytes +
               (32 + 32 + 256) * 4 + 8 * (2 * kEfRing + 2 * kEfSlots + kEfMaxQ + 6) + 16;
    };
    EncFrontTc b = a;
    b.n_quarters = kEfMaxQ;
    while (b.n_quarters > 4 && smem_of(b.n_quarters) > 227 * 1024) --b.n_quarters;
    const size_t smem = smem_of(b.n_quarters);
    if ((uint64_t)a.n_img * (a.gh + 2) * Wp >= (1ull << 31)) return PILC_E_UNSUPPORTED;
    if (smem > 227 * 1024) return PILC_E_UNSUPPORTED;
    allow_dyn_smem(reinterpret_cast<const void *>(enc_front_tc_kernel));
    int64_t grid = sm_count();
    if (grid > a.n_tiles) grid = a.n_tiles;
    if (grid < 1) return PILC_OK;
    const double flops = 2.0 * a.n_img * (4.0 * a.gh * a.gw * 32 * 27 + (double)a.gh * a.gw * 32 * 32 * 9);
    ProfScope _ps(PROF_ENC_FRONT, s, flops);
    enc_front_tc_kernel<<<(unsigned)grid, kEfThreads, smem, s>>>(b);
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

int tc3_launch(const Tc3Layer &L, int ks, int mode, cudaStream_t s) {
    if (ks == 3 && mode == TC3_ACT) return launch_tc3<3, TC3_ACT>(L, s);
    if (ks == 1 && mode == TC3_Z) return launch_tc3<1, TC3_Z>(L, s);
    return PILC_E_UNSUPPORTED;
}
int tc3_block_launch(const Tc3Block &b, cudaStream_t s) {
    const size_t smem = tc3_block_smem(b.Hp, b.Wp);
    if ((b.Hp * b.Wp + 127) / 128 > kBkMaxTiles || smem > 227 * 1024) return PILC_E_UNSUPPORTED;
    if ((uint64_t)b.n_img * b.Hp * b.Wp >= (1ull << 31)) return PILC_E_UNSUPPORTED;
    allow_dyn_smem(reinterpret_cast<const void *>(tc3_block_kernel));
    int64_t grid = sm_count();
    if (grid > b.n_img) grid = b.n_img;
    if (grid < 1) return PILC_OK;
    const double flops = 2.0 * 2.0 * b.n_img * b.H * b.W * 32.0 * 32 * 9;
    ProfScope _ps(PROF_TC3_BLOCK, s, flops);
    tc3_block_kernel<<<(unsigned)grid, kThreadsBK, smem, s>>>(b);
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}
int enc_trunk_launch(const EncTrunk &p, cudaStream_t s) {
    if (p.n_blocks < 1 || 2 * p.n_blocks + 1 > kEtMaxLayers) return PILC_E_UNSUPPORTED;
    const int HW = p.Hp * p.Wp;
    if ((HW + 127) / 128 > kEtMaxTiles) return PILC_E_UNSUPPORTED;
    const size_t smem = enc_trunk_smem(p.Hp, p.Wp, p.n_blocks);
    if (smem > 227 * 1024) return PILC_E_UNSUPPORTED;
    if ((uint64_t)p.n_img * HW >= (1ull << 31)) return PILC_E_UNSUPPORTED;
    allow_dyn_smem(reinterpret_cast<const void *>(enc_trunk_kernel));
    int64_t grid = sm_count();
    if (grid > p.n_img) grid = p.n_img;
    if (grid < 1) return PILC_OK;
    const double flops = 2.0 * p.n_img * p.H * p.W * 32.0 * 32 * (18.0 * p.n_blocks + 1);
    ProfScope _ps(PROF_ENC_TRUNK, s, flops);
    enc_trunk_kernel<<<(unsigned)grid, kThreadsET, smem, s>>>(p);
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}
int dec_trunk_launch(const DecTrunk &p0, cudaStream_t s) {
    DecTrunk p = p0;
    if (p.n_conv < 1 || p.n_conv > kDtMaxConvs || p.K < 1 || p.K > 256) return PILC_E_UNSUPPORTED;
    if ((uint64_t)p.n_img * p.Hp * p.Wp >= (1ull << 31)) return PILC_E_UNSUPPORTED;
    int G = 0, pad = 0;
    size_t smem = 0;
    for (int g = 1; g <= 64; ++g) {  // images per group: the most that fit
        int pd;
        const size_t sm = dec_trunk_smem(p.Hp, p.Wp, g, p.K, p.n_conv, &pd);
        if (sm > 227 * 1024 || (g * p.Hp * p.Wp + 127) / 128 > kDtMaxTiles) break;
        G = g;
        pad = pd;
        smem = sm;
    }
    if (G == 0) return PILC_E_UNSUPPORTED;
    p.G = G;
    p.pad_bytes = pad;
    allow_dyn_smem(reinterpret_cast<const void *>(dec_trunk_kernel));
    const int64_t groups = (p.n_img + G - 1) / G;
    int64_t grid = sm_count();
    if (grid > groups) grid = groups;
    if (grid < 1) return PILC_OK;
    const double flops = 2.0 * p.n_img * (p.Hp - 2) * (p.Wp - 2) * 32.0 * 32 * 9 * p.n_conv;
    ProfScope _ps(PROF_DEC_TRUNK, s, flops);
    dec_trunk_kernel<<<(unsigned)grid, kThreadsDT, smem, s>>>(p);
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}
int dec_uphead_launch(const DecUpHead &p, cudaStream_t s) {
    if (p.gh < 1 || p.gw < 1 || p.n_thresh < 0 || p.n_thresh > 255) return PILC_E_UNSUPPORTED;
    const UhGeom g = uh_geom(p.gh, p.gw);
    if (g.Tu > kUhMaxUp || g.Th > kUhMaxHead) return PILC_E_UNSUPPORTED;
    const size_t smem = dec_uphead_smem(g);
    if (smem > 227 * 1024) return PILC_E_UNSUPPORTED;
    if ((uint64_t)p.n_img * g.HW >= (1ull << 31)) return PILC_E_UNSUPPORTED;
    allow_dyn_smem(reinterpret_cast<const void *>(dec_uphead_kernel));
    int64_t grid = sm_count();
    if (grid > p.n_img) grid = p.n_img;
    if (grid < 1) return PILC_OK;
    const double flops = 2.0 * p.n_img * p.gh * p.gw * 32.0 * 9 * (128 + 4 * 6);
    ProfScope _ps(PROF_DEC_UPHEAD, s, flops);
    dec_uphead_kernel<<<(unsigned)grid, kThreadsUH, smem, s>>>(p);
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}
int dec_trunk2_launch(const DecTrunk &p0, cudaStream_t s) {
    DecTrunk p = p0;
    if (p.n_conv < 1 || p.n_conv > kDtMaxConvs || p.K < 1 || p.K > 256) return PILC_E_UNSUPPORTED;
    const int Wq = ((p.Wp + 1) & ~1) / 2;
    if (Wq + 1 > 128) return PILC_E_UNSUPPORTED;  // a tile's halo reaches one tile either way
    if ((uint64_t)p.n_img * p.Hp * 2 * Wq >= (1ull << 31)) return PILC_E_UNSUPPORTED;
    // images per group: the most images per MMA tile (fewest padded rows), then the most images
    int G = 0, pad = 0, bestT = 1;
    size_t smem = 0;
    for (int g = 1; g <= 64; ++g) {
        int pd;
        const size_t sm = dec_trunk2_smem(p.Hp, p.Wp, g, p.K, p.n_conv, &pd);
        const int T = (g * p.Hp * Wq + 127) / 128;
        if (sm > 227 * 1024 || T > kD2MaxTiles) break;
        if (G == 0 || (int64_t)g * bestT >= (int64_t)G * T) {
            G = g;
            bestT = T;
            pad = pd;
            smem = sm;
        }
    }
    if (G == 0) return PILC_E_UNSUPPORTED;
    p.G = G;
    p.pad_bytes = pad;
    allow_dyn_smem(reinterpret_cast<const void *>(dec_trunk2_kernel));
    const int64_t groups = (p.n_img + G - 1) / G;
    int64_t grid = sm_count();
    if (grid > groups) grid = groups;
    if (grid < 1) return PILC_OK;
    const double flops = 2.0 * p.n_img * (p.Hp - 2) * (p.Wp - 2) * 32.0 * 32 * 9 * p.n_conv;
    ProfScope _ps(PROF_DEC_TRUNK2, s, flops);
    dec_trunk2_kernel<<<(unsigned)grid, kThreadsD2, smem, s>>>(p);
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}
int tc_launch_shuffle(const TcLayer &L, cudaStream_t s) { return launch_tc<128, 3, TC_OUT_SHUFFLE>(L, s); }
// Whether the tcgen05 decoder runs for a latent grid gh x gw (a function of
// the shape only, never of the batch size: vq_decode splits batches below the
// 32-bit pixel-index limit). The per-layer block convs, the up conv and the
// head must fit shared memory; the fused trunk falls back to the per-layer
// convs with bit-identical results.
bool tc_decoder_supported(int gh, int gw, bool pairs) {
    int st;
    if (!tc_smem_plan<32, 3, TC_OUT_ACT>(gw + 2, &st)) return false;
    if (!tc_smem_plan<128, 3, TC_OUT_SHUFFLE>(gw + 2, &st)) return false;
    (void)pairs;
    return tc_smem_plan<16, 3, TC_OUT_HEAD2>(gw + 1, &st) != 0;
}
int tc_launch_head2(const TcLayer &L, cudaStream_t s) { return launch_tc<16, 3, TC_OUT_HEAD2>(L, s); }

int tc_dec_table(const float *cb, const float *w, const float *b, int K, int Dc, int ci_pad, int co_pad,
                 uint16_t *table, cudaStream_t s) {
    ProfScope _ps(PROF_GATHER, s, (double)K * 32);
    dec_table_kernel<<<(K * 32 + 255) / 256, 256, 0, s>>>(cb, w, b, K, Dc, ci_pad, co_pad, table);
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

int tc_gather(const uint8_t *idx, const uint16_t *table, int64_t n_img, int gh, int gw, uint16_t *x,
              int64_t gstride, int64_t margin, cudaStream_t s) {
    const int64_t total = n_img * (gh + 2) * (int64_t)(gw + 2);
    int64_t blocks = ceil_div64(total, 256);
    const int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    ProfScope _ps(PROF_GATHER, s, (double)total);
    gather_kernel<<<(unsigned)blocks, 256, 0, s>>>(idx, table, n_img, gh, gw, x, gstride, margin);
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}
