// Fused encoder front for the 3xTF32 encoder: stem (3x3, 3 -> 32, ReLU) and
// down (3x3 stride 2, 32 -> 32, ReLU) in one kernel, stem tile kept in
// shared memory, output written straight into the fp32 slab the tcgen05
// block convs read (tc_conv.cu).
//
// Reference: vqvae.encode_to_indices (vqvae.py:55-57) with _even_pad,
// _normalize (vqvae.py:33-43) and nn.conv2d's edge-replicate padding
// (nn.py:15-34). Both pads are clamps: the stem at (even-padded) position
// (sy, sx) reads image pixels clamp(sy-1..sy+1, 0, H-1); the down conv at
// (y, x) reads stem positions clamp(2y-1..2y+1, 0, He-1).
//
// CTA = one image x (16 x 16) down outputs, 256 threads (~199 KB smem):
//   1. image patch (35 x 35 x 3) -> normalized f32 in smem
//   2. stem at the 33 x 33 clamped positions the tile needs, one position
//      x 32 channels per thread per round -> smem (channel-planar)
//   3. down conv: 4 outputs x 8 channels per thread
//   4. bias + ReLU -> the fp32 slab set and the scaled fp16 hi / lo operand
//      slabs of the first block conv (+ border copies)
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "enc_front.cuh"
#include <cuda_fp16.h>

namespace {

constexpr int TH = 16, TW = 16;          // down-output tile
constexpr int SR = 2 * TH + 1, SC = 2 * TW + 1;   // stem patch 17 x 33
constexpr int SCP = SC + 1;              // pitch
constexpr int IR = SR + 2, IC = SC + 2;  // image patch 19 x 35
constexpr int kThreads = 256;
constexpr int C = 32;
constexpr int kImgF = (3 * IR * IC + 3) & ~3;  // image patch floats, rounded for float4 alignment

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ void store4(float *slab, int64_t q, float4 v, int y, int x, int H, int W, int Wp) {
    float4 *p = reinterpret_cast<float4 *>(slab);
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

__device__ __forceinline__ void store16(uint16_t *slab, int64_t q, uint4 v, int y, int x, int H, int W, int Wp) {
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

__global__ void __launch_bounds__(kThreads) enc_front_kernel(EncFront a) {
    extern __shared__ __align__(16) float sm[];
    float *s_img = sm;                      // [3][IR][IC]
    float *s_ws = s_img + kImgF;            // stem weights [27][32] (k = c*9 + i*3 + j), 16-B aligned
    float *s_bs = s_ws + 27 * C;            // [32]
    float *s_wd = s_bs + C;                 // down weights [9][32 ci][32 co]
    float *s_bd = s_wd + 9 * C * C;         // [32]
    float *s_st = s_bd + C;                 // stem out [32][SR][SCP]

    const int t = threadIdx.x;
    const int tiles_x = (a.gw + TW - 1) / TW;
    const int tiles = tiles_x * ((a.gh + TH - 1) / TH);
    const int64_t n = blockIdx.x / tiles;
    const int tile = blockIdx.x - (int)n * tiles;
    const int oy0 = (tile / tiles_x) * TH, ox0 = (tile % tiles_x) * TW;
    const int He = 2 * a.gh, We = 2 * a.gw;

    // weights (model layout [tap][ci_pad][co_pad], co fastest)
    for (int e = t; e < 27 * C; e += kThreads) {
        const int k = e / C, co = e % C;  // k = c*9 + tap
        const int c = k / 9, tap = k % 9;
        s_ws[e] = a.w_stem[((int64_t)tap * a.stem_ci_pad + c) * a.stem_co_pad + co];
    }
    for (int e = t; e < 9 * C * C; e += kThreads) {
        const int tap = e / (C * C), rem = e % (C * C);
        const int ci = rem / C, co = rem % C;
        s_wd[e] = a.w_down[((int64_t)tap * a.down_ci_pad + ci) * a.down_co_pad + co];
    }
    if (t < C) {
        s_bs[t] = a.b_stem[t];
        s_bd[t] = a.b_down[t];
    }
    // 1. image patch: staged row r holds image row clamp(2*oy0 - 2 + r)
    const uint8_t *img = a.img + n * (int64_t)a.H * a.W * 3;
    for (int e = t; e < IR * IC; e += kThreads) {
        const int r = e / IC, cc = e % IC;
        const int y = clampi(2 * oy0 - 2 + r, 0, a.H - 1), x = clampi(2 * ox0 - 2 + cc, 0, a.W - 1);
        const uint8_t *px = img + ((int64_t)y * a.W + x) * 3;
#pragma unroll
        for (int c = 0; c < 3; ++c) s_img[(c * IR + r) * IC + cc] = __fsub_rn(__fdiv_rn((float)px[c], 127.5f), 1.f);
    }
    __syncthreads();
    // 2. stem at patch position (r, cc) = stem (clamp(2*oy0-1+r, 0, He-1), clamp(2*ox0-1+cc, 0, We-1))
    for (int p = t; p < SR * SC; p += kThreads) {
        asm volatile("" ::: "memory");  // keep the weight loads inside the loop (no 864-value hoist)
        const int pr = p / SC, pc = p - (p / SC) * SC;
        const int sy = clampi(2 * oy0 - 1 + pr, 0, He - 1), sx = clampi(2 * ox0 - 1 + pc, 0, We - 1);
        // image rows sy-1..sy+1 live at staged rows (sy - 1 + i) - (2*oy0 - 2)
        const int rb = sy - 1 - (2 * oy0 - 2), cb = sx - 1 - (2 * ox0 - 2);
        float acc[C];
#pragma unroll
        for (int co = 0; co < C; ++co) acc[co] = s_bs[co];
#pragma unroll
        for (int k = 0; k < 27; ++k) {
            const int c = k / 9, i = (k % 9) / 3, j = k % 3;
            const float xv = s_img[(c * IR + rb + i) * IC + cb + j];
            const float4 *w4 = reinterpret_cast<const float4 *>(s_ws + k * C);
#pragma unroll
            for (int q = 0; q < C / 4; ++q) {
                const float4 w = w4[q];
                acc[4 * q + 0] = fmaf(xv, w.x, acc[4 * q + 0]);
                acc[4 * q + 1] = fmaf(xv, w.y, acc[4 * q + 1]);
                acc[4 * q + 2] = fmaf(xv, w.z, acc[4 * q + 2]);
                acc[4 * q + 3] = fmaf(xv, w.w, acc[4 * q + 3]);
            }
        }
#pragma unroll
        for (int co = 0; co < C; ++co) s_st[(co * SR + pr) * SCP + pc] = fmaxf(acc[co], 0.f);
    }
    __syncthreads();
    // 3. down conv: thread = 4 outputs (rows ry, ry+4, ry+8, ry+12 of column cx) x 8 channels
    const int cgrp = t >> 6;            // channels 8*cgrp .. +7
    const int cx = t & 15, ry = (t >> 4) & 3;
    float acc[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[u][e] = 0.f;
    for (int ci = 0; ci < C; ++ci) {
        asm volatile("" ::: "memory");
        const float *sp = s_st + ci * SR * SCP;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const float4 *w4 = reinterpret_cast<const float4 *>(s_wd + ((i * 3 + j) * C + ci) * C + 8 * cgrp);
                const float4 wa = w4[0], wb = w4[1];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float xv = sp[(2 * (ry + 4 * u) + i) * SCP + 2 * cx + j];
                    acc[u][0] = fmaf(xv, wa.x, acc[u][0]);
                    acc[u][1] = fmaf(xv, wa.y, acc[u][1]);
                    acc[u][2] = fmaf(xv, wa.z, acc[u][2]);
                    acc[u][3] = fmaf(xv, wa.w, acc[u][3]);
                    acc[u][4] = fmaf(xv, wb.x, acc[u][4]);
                    acc[u][5] = fmaf(xv, wb.y, acc[u][5]);
                    acc[u][6] = fmaf(xv, wb.z, acc[u][6]);
                    acc[u][7] = fmaf(xv, wb.w, acc[u][7]);
                }
            }
    }
    // 4. bias + ReLU -> the fp32 slab set and the scaled fp16 hi / lo operands
    const int Wp = a.gw + 2;
    const int k0 = *a.k0;
    const float sc = __int_as_float((127 + k0) << 23);
    float mx = 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int oy = oy0 + ry + 4 * u, ox = ox0 + cx;
        if (oy >= a.gh || ox >= a.gw) continue;
        const int64_t q = (n * (a.gh + 2) + oy + 1) * (int64_t)Wp + ox + 1;
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            v[e] = fmaxf(__fadd_rn(acc[u][e], s_bd[8 * cgrp + e]), 0.f);
            mx = fmaxf(mx, v[e]);
        }
#pragma unroll
        for (int g2 = 0; g2 < 2; ++g2) {
            const int64_t so = ((int64_t)(2 * cgrp + g2) * a.gstride + a.margin) * 4;
            store4(a.out32 + so, q, make_float4(v[4 * g2], v[4 * g2 + 1], v[4 * g2 + 2], v[4 * g2 + 3]), oy + 1,
                   ox + 1, a.gh, a.gw, Wp);
        }
        uint32_t h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float x0 = __fmul_rn(v[2 * e], sc), x1 = __fmul_rn(v[2 * e + 1], sc);
            const __half2 hh = __floats2half2_rn(x0, x1);
            const float2 hf = __half22float2(hh);
            const __half2 ll = __floats2half2_rn(__fmul_rn(__fsub_rn(x0, hf.x), 2048.f),
                                                 __fmul_rn(__fsub_rn(x1, hf.y), 2048.f));
            h[e] = *reinterpret_cast<const uint32_t *>(&hh);
            l[e] = *reinterpret_cast<const uint32_t *>(&ll);
        }
        store16(a.out + ((int64_t)cgrp * a.gstride + a.margin) * 8, q, make_uint4(h[0], h[1], h[2], h[3]), oy + 1,
                ox + 1, a.gh, a.gw, Wp);
        store16(a.out + ((int64_t)(4 + cgrp) * a.gstride + a.margin) * 8, q, make_uint4(l[0], l[1], l[2], l[3]),
                oy + 1, ox + 1, a.gh, a.gw, Wp);
    }
    // per-image max (bound input of the first block conv) and the scale
    const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(mx));
    if ((t & 31) == 0 && m != 0u) atomicMax(a.out_max + n, m);
    if (t == 0) a.kx_out[n] = k0;
}

}  // namespace

size_t enc_front_smem() {
    return sizeof(float) * (kImgF + 27 * C + C + 9 * C * C + C + C * SR * SCP);
}

int enc_front_launch(const EncFront &a, cudaStream_t s) {
    const int tiles = ((a.gw + TW - 1) / TW) * ((a.gh + TH - 1) / TH);
    const int64_t blocks = a.n_img * tiles;
    if (blocks > 0x7FFFFFFF) return PILC_E_UNSUPPORTED;
    const size_t smem = enc_front_smem();
    cudaFuncSetAttribute(enc_front_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const double flops = 2.0 * a.n_img * (4.0 * a.gh * a.gw * C * 27 + (double)a.gh * a.gw * C * C * 9);
    ProfScope _ps(PROF_ENC_FRONT, s, flops);
    enc_front_kernel<<<(unsigned)blocks, kThreads, smem, s>>>(a);
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}
