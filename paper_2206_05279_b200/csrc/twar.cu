// TWAR three-neighbour predictor: forward residual and wavefront inverse.
//
// Numeric contract (_kernels.py:69-88, predictor.py:106-111, 183-190):
// acc = w0*c0; acc += w1*c1; acc += w2*c2; acc += bias, all float32 with no
// FMA contraction (explicit __fmul_rn/__fadd_rn), then round half away from
// zero in float64 and reduce mod 256. Out-of-image context reads as 0.
//   R: (up-left, up, left)       G: (left, R-left, R-here)
//   B: (left, G-left, G-here)    (predictor.py:36-40)

#include "common.cuh"

namespace {

struct Params {
    float w[9];
    float b[3];
    // every weight an integer with |w| <= 2^13 and every bias an integer
    // with |b| <= 2^22 (the default predictor): with byte contexts each
    // float32 product and partial sum is an exact integer below 2^24, so the
    // round-half-away step is the identity and only the mod 256 remains
    int integral;
};

__device__ __forceinline__ uint32_t round_mod256(float acc) {
    // |acc| < 2^22: acc +- 0.5 is exact in float32, so floor / ceil there
    // equal the float64 ones (the common case: unit weights, byte contexts)
    if (fabsf(acc) < 4194304.f) {
        const float r = acc >= 0.f ? floorf(__fadd_rn(acc, 0.5f)) : ceilf(__fsub_rn(acc, 0.5f));
        return (uint32_t)((int)r & 255);
    }
    const double p = (double)acc;
    const double r = p >= 0.0 ? floor(p + 0.5) : ceil(p - 0.5);
    if (fabs(r) < 4.0e18) return (uint32_t)((long long)r & 255LL);
    double m = fmod(r, 256.0);
    if (m < 0.0) m += 256.0;
    return (uint32_t)m;
}

__device__ __forceinline__ uint32_t predict(float c0, float c1, float c2, const float *w, float b,
                                            int integral = 0) {
    float acc = __fmul_rn(w[0], c0);
    acc = __fadd_rn(acc, __fmul_rn(w[1], c1));
    acc = __fadd_rn(acc, __fmul_rn(w[2], c2));
    acc = __fadd_rn(acc, b);
    if (integral) return (uint32_t)__float2int_rz(acc) & 255u;  // acc is an exact integer (see Params)
    return round_mod256(acc);
}

// One thread per pixel, all three channels (predictor.py:173-195).
__global__ void twar_forward_kernel(const uint8_t *__restrict__ img, uint8_t *__restrict__ res,
                                    int64_t n_px, int H, int W, Params p) {
    const int64_t hw = (int64_t)H * W;
    const bool small = n_px < (1ll << 32) && hw < (1ll << 32);
    const uint32_t hw32 = (uint32_t)hw, w32 = (uint32_t)W;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_px;
         g += (int64_t)gridDim.x * blockDim.x) {
        int64_t n;
        int rem;
        if (small) {  // 32-bit divisions (the 64-bit ones are a long software sequence)
            const uint32_t n32 = (uint32_t)g / hw32;
            n = n32;
            rem = (int)((uint32_t)g - n32 * hw32);
        } else {
            n = g / hw;
            rem = (int)(g - n * hw);
        }
        const int u = (int)((uint32_t)rem / w32), v = rem - u * W;
        const uint8_t *x = img + n * hw * 3;
        const int64_t o = (int64_t)rem * 3;
        const float r = x[o], gg = x[o + 1], bb = x[o + 2];
        float rl = 0.f, gl = 0.f, bl = 0.f, ru = 0.f, rul = 0.f;
        if (v > 0) {
            rl = x[o - 3];
            gl = x[o - 2];
            bl = x[o - 1];
        }
        if (u > 0) {
            ru = x[o - 3 * W];
            if (v > 0) rul = x[o - 3 * W - 3];
        }
        const uint32_t pr = predict(rul, ru, rl, p.w, p.b[0], p.integral);
        const uint32_t pg = predict(gl, rl, r, p.w + 3, p.b[1], p.integral);
        const uint32_t pb = predict(bl, gl, gg, p.w + 6, p.b[2], p.integral);
        uint8_t *t = res + n * hw * 3 + o;
        t[0] = (uint8_t)(((uint32_t)r - pr + 128u) & 0xFFu);
        t[1] = (uint8_t)(((uint32_t)gg - pg + 128u) & 0xFFu);
        t[2] = (uint8_t)(((uint32_t)bb - pb + 128u) & 0xFFu);
    }
}

// Rows of W = 8 m pixels: a thread per 8-pixel run (24 bytes) of a row,
// loaded as three 8-byte vectors (plus the same run of the row above and
// the 4 bytes before each, for the left / up-left neighbours), 24 residual
// bytes stored as three vectors. Same arithmetic per pixel as
// twar_forward_kernel (INTEGRAL: the integer-weight predictor in integer
// arithmetic, exact as in predict()); the scalar kernel is issue bound at
// ~85 instructions per pixel, this one at ~10 per subpixel and HBM.
__device__ __forceinline__ uint32_t byte_at(const uint32_t *w, int i) { return (w[i >> 2] >> (8 * (i & 3))) & 0xFFu; }

template <int INTEGRAL>
__device__ __forceinline__ uint32_t predict8(uint32_t c0, uint32_t c1, uint32_t c2, const Params &p, const int *wi, int k) {
    if (INTEGRAL) return (uint32_t)(wi[3 * k] * (int)c0 + wi[3 * k + 1] * (int)c1 + wi[3 * k + 2] * (int)c2 + wi[9 + k]) & 255u;
    return predict((float)c0, (float)c1, (float)c2, p.w + 3 * k, p.b[k], 0);
}

// the residual bytes of an npx-pixel run (npx = 8 or 16) from its bytes c,
// the same run of the row above a, and the 4 bytes before each (cl, al).
// INTEGRAL == 2: the default predictor (W_r = (-1, 1, 1), W_g = W_b =
// (1, -1, 1), no bias) four bytes at a time: t = x + X - Y - Z + 128 (mod
// 256) with (X, Y, Z) = (up-left, up, left) on red bytes and (the left
// pixel's red / green, the left subpixel, the previous subpixel) on green /
// blue ones; even and odd bytes go through 16-bit lanes.
template <int INTEGRAL>
__device__ __forceinline__ void run_residual(const uint32_t *c, const uint32_t *a, uint32_t cl, uint32_t al, int npx,
                                             const Params &p, const int *wi, uint32_t *o) {
    if (INTEGRAL == 2) {
#pragma unroll
        for (int j = 0; j < 3 * npx / 4; ++j) {
            const uint32_t M = (j % 3 == 0) ? 0xFF0000FFu : (j % 3 == 1 ? 0x00FF0000u : 0x0000FF00u);
            const uint32_t Cm = j ? c[j - 1] : cl, Um = j ? a[j - 1] : al;
            const uint32_t c3 = __funnelshift_l(Cm, c[j], 24), c1 = __funnelshift_l(Cm, c[j], 8);
            const uint32_t u3 = __funnelshift_l(Um, a[j], 24);
            const uint32_t X = (Cm & ~M) | (u3 & M), Y = (c3 & ~M) | (a[j] & M), Z = (c1 & ~M) | (c3 & M);
            constexpr uint32_t LO = 0x00FF00FFu, K = 0x02800280u;
            const uint32_t e = (c[j] & LO) + (X & LO) + K - (Y & LO) - (Z & LO);
            const uint32_t d = ((c[j] >> 8) & LO) + ((X >> 8) & LO) + K - ((Y >> 8) & LO) - ((Z >> 8) & LO);
            o[j] = (e & LO) | ((d & LO) << 8);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 3 * npx / 4; ++j) o[j] = 0u;
#pragma unroll
        for (int i = 0; i < npx; ++i) {
            const uint32_t r = byte_at(c, 3 * i), gg = byte_at(c, 3 * i + 1), bb = byte_at(c, 3 * i + 2);
            const uint32_t rl = i ? byte_at(c, 3 * i - 3) : (cl >> 8) & 0xFFu;
            const uint32_t gl = i ? byte_at(c, 3 * i - 2) : (cl >> 16) & 0xFFu;
            const uint32_t bl = i ? byte_at(c, 3 * i - 1) : cl >> 24;
            const uint32_t ru = byte_at(a, 3 * i);
            const uint32_t rul = i ? byte_at(a, 3 * i - 3) : (al >> 8) & 0xFFu;
            const uint32_t pr = predict8<INTEGRAL>(rul, ru, rl, p, wi, 0);
            const uint32_t pg = predict8<INTEGRAL>(gl, rl, r, p, wi, 1);
            const uint32_t pb = predict8<INTEGRAL>(bl, gl, gg, p, wi, 2);
            o[(3 * i) >> 2] |= ((r - pr + 128u) & 0xFFu) << (8 * ((3 * i) & 3));
            o[(3 * i + 1) >> 2] |= ((gg - pg + 128u) & 0xFFu) << (8 * ((3 * i + 1) & 3));
            o[(3 * i + 2) >> 2] |= ((bb - pb + 128u) & 0xFFu) << (8 * ((3 * i + 2) & 3));
        }
    }
}

// one 8-pixel run's inputs: the run, the same run of the row above, and
// the 4 bytes before each (left / up-left neighbours in bytes 1..3)
struct Run8 {
    uint32_t c[6], a[6], cl, al;
};

__device__ __forceinline__ void load_run8(Run8 &r, const uint8_t *img, int64_t g, int upr, int rb, int H) {
    int64_t R;  // global row (image n, row u)
    int k, u;   // run within the row, row within the image
    if (g < (1ll << 32) / 2) {  // 32-bit divisions (the 64-bit ones are a long software sequence)
        const uint32_t R32 = (uint32_t)g / (uint32_t)upr;
        R = R32;
        k = (int)((uint32_t)g - R32 * (uint32_t)upr);
        u = (int)(R32 % (uint32_t)H);
    } else {
        R = g / upr;
        k = (int)(g - R * upr);
        u = (int)(R % H);
    }
    const uint8_t *rp = img + R * rb + 24 * k;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(rp) + q);
        r.c[2 * q] = v.x, r.c[2 * q + 1] = v.y;
    }
    r.cl = k > 0 ? __ldg(reinterpret_cast<const uint32_t *>(rp) - 1) : 0u;
    r.al = 0u;
#pragma unroll
    for (int q = 0; q < 6; ++q) r.a[q] = 0u;
    if (u > 0) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const uint2 v = __ldg(reinterpret_cast<const uint2 *>(rp - rb) + q);
            r.a[2 * q] = v.x, r.a[2 * q + 1] = v.y;
        }
        if (k > 0) r.al = __ldg(reinterpret_cast<const uint32_t *>(rp - rb) - 1);
    }
}

template <int INTEGRAL>
__global__ void __launch_bounds__(256) twar_forward8_kernel(const uint8_t *__restrict__ img, uint8_t *__restrict__ res,
                                                            int64_t n_units, int H, int W, Params p) {
    const int upr = W >> 3;  // 8-pixel runs per row
    const int rb = 3 * W;    // row bytes
    int wi[12];
#pragma unroll
    for (int k = 0; k < 9; ++k) wi[k] = (int)p.w[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) wi[9 + k] = (int)p.b[k];
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_units; g += (int64_t)gridDim.x * blockDim.x) {
        Run8 cur;
        load_run8(cur, img, g, upr, rb, H);
        const uint32_t *c = cur.c, *a = cur.a;
        const uint32_t cl = cur.cl, al = cur.al;
        uint32_t o[6];
        run_residual<INTEGRAL>(c, a, cl, al, 8, p, wi, o);
        uint2 *op = reinterpret_cast<uint2 *>(res + g * 24);
#pragma unroll
        for (int q = 0; q < 3; ++q) op[q] = make_uint2(o[2 * q], o[2 * q + 1]);
    }
}

// Whole images through shared memory (W = 16 m, at most 12 KB per image):
// each block takes G images at a time, brought in by one bulk copy (TMA
// engine, double-buffered one group ahead) and written back by one bulk
// store from a staged output buffer, so HBM sees only long contiguous
// transfers; a thread computes 16-pixel runs from shared memory (the row
// above included: no second global read of it). Per pixel the arithmetic of
// twar_forward8_kernel.
__device__ __forceinline__ uint32_t s_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kTwTileBytes = 12288;  // input (and output) bytes per group buffer

template <int INTEGRAL>
__global__ void __launch_bounds__(256) twar_forward_tile_kernel(const uint8_t *__restrict__ img, uint8_t *__restrict__ res,
                                                                int64_t n_img, int H, int W, int G, Params p) {
    extern __shared__ __align__(128) uint8_t s_tw[];  // in[2][kTwTileBytes], out[2][kTwTileBytes]
    uint8_t(*s_in)[kTwTileBytes] = reinterpret_cast<uint8_t(*)[kTwTileBytes]>(s_tw);
    uint8_t(*s_out)[kTwTileBytes] = reinterpret_cast<uint8_t(*)[kTwTileBytes]>(s_tw + 2 * kTwTileBytes);
    __shared__ uint64_t bar[2];
    const int rb = 3 * W, ib = H * rb;  // row / image bytes
    const int upr = W >> 4;             // 16-pixel runs per row
    int wi[12];
#pragma unroll
    for (int k = 0; k < 9; ++k) wi[k] = (int)p.w[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) wi[9 + k] = (int)p.b[k];
    const int64_t n_groups = (n_img + G - 1) / G;
    auto load = [&](int64_t gi, int b) {  // thread 0: group gi into buffer b
        const int64_t n0 = gi * G;
        const uint32_t bytes = (uint32_t)(min((int64_t)G, n_img - n0) * ib);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&bar[b])), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         s_u32(s_in[b])),
                     "l"(img + n0 * ib), "r"(bytes), "r"(s_u32(&bar[b]))
                     : "memory");
    };
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (blockIdx.x < n_groups) load(blockIdx.x, 0);
    }
    __syncthreads();
    int it = 0;
    for (int64_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x, ++it) {
        const int b = it & 1;
        if (threadIdx.x == 0) {
            if (gi + gridDim.x < n_groups) load(gi + gridDim.x, b ^ 1);  // its buffer was released by the last __syncthreads
            // s_out[b] is reused: its bulk store of two groups ago must have read it
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        asm volatile(
            "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(
                s_u32(&bar[b])),
            "r"((uint32_t)((it >> 1) & 1))
            : "memory");
        __syncthreads();  // s_out[b] free (thread 0 waited above)
        const int64_t n0 = gi * G;
        const int g_act = (int)min((int64_t)G, n_img - n0);
        const int units = g_act * H * upr;
        for (int t = threadIdx.x; t < units; t += blockDim.x) {
            const int R = t / upr, k = t - R * upr;  // row within the group, run within the row
            const int u = R % H;
            const uint8_t *rp = s_in[b] + R * rb + 48 * k;
            uint32_t c[12], a[12], cl = 0u, al = 0u;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const uint4 v = reinterpret_cast<const uint4 *>(rp)[q];
                c[4 * q] = v.x, c[4 * q + 1] = v.y, c[4 * q + 2] = v.z, c[4 * q + 3] = v.w;
            }
            if (k > 0) cl = reinterpret_cast<const uint32_t *>(rp)[-1];
            if (u > 0) {
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const uint4 v = reinterpret_cast<const uint4 *>(rp - rb)[q];
                    a[4 * q] = v.x, a[4 * q + 1] = v.y, a[4 * q + 2] = v.z, a[4 * q + 3] = v.w;
                }
                if (k > 0) al = reinterpret_cast<const uint32_t *>(rp - rb)[-1];
            } else {
#pragma unroll
                for (int q = 0; q < 12; ++q) a[q] = 0u;
            }
            uint32_t o[12];
            run_residual<INTEGRAL>(c, a, cl, al, 16, p, wi, o);
            uint4 *op = reinterpret_cast<uint4 *>(s_out[b] + R * rb + 48 * k);
#pragma unroll
            for (int q = 0; q < 3; ++q) op[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the staged bytes -> the bulk store
        __syncthreads();  // s_in[b] consumed, s_out[b] complete
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(res + n0 * ib),
                         "r"(s_u32(s_out[b])), "r"((uint32_t)(g_act * ib))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Inverse (_kernels.py:146-170 wavefront schedule). One warp per image;
// the image is staged in shared memory when it fits, else decoded in place
// in the output buffer. Red: lanes take rows of two 32-row strips at a time
// and march a skewed wavefront (lane u handles columns step - u and
// step - u - 32), receiving the up / up-left values from lane u-1 by
// shuffle. Green, blue: rows are independent; one sweep per row decodes
// both channels, each lane walking two rows. Every pixel's arithmetic is the
// reference's; only the order across independent pixels changes.
constexpr int kDecWarps = 4;

__device__ __forceinline__ uint32_t unrec(const uint8_t *coded, const uint8_t *shift, int64_t i) {
    uint32_t t = coded[i];
    if (shift) t = (t + shift[i] + 128u) & 0xFFu;
    return t;
}

__global__ void __launch_bounds__(32 * kDecWarps) twar_decode_kernel(
    const uint8_t *__restrict__ coded, const uint8_t *__restrict__ shift, uint8_t *__restrict__ out,
    int64_t n_img, int H, int W, Params p, int stage_in_smem, int rp) {
    // rp: row pitch in bytes of the working image (3 W in global memory; in
    // shared memory padded so the lanes' rows -- and the red wavefront's
    // skewed diagonals -- fall in different banks: unpadded 64-pixel rows
    // put all 32 lanes in two banks)
    extern __shared__ uint8_t s_img[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t hw3 = (int64_t)H * W * 3;
    for (int64_t n = (int64_t)blockIdx.x * kDecWarps + warp; n < n_img;
         n += (int64_t)gridDim.x * kDecWarps) {
        const uint8_t *cd = coded + n * hw3;
        const uint8_t *sh = shift ? shift + n * hw3 : nullptr;
        uint8_t *o_g = out + n * hw3;
        const int64_t img_b = (int64_t)H * rp;  // bytes of one working image
        // staged: one buffer per warp, decoded in place (every residual byte is
        // read once, just before its pixel's output overwrites it)
        uint8_t *o = stage_in_smem ? s_img + (int64_t)warp * img_b : o_g;
        const int w3 = 3 * W;
        const bool vec = stage_in_smem && (w3 & 15) == 0 && (rp & 3) == 0 &&
                         ((reinterpret_cast<uintptr_t>(cd) | reinterpret_cast<uintptr_t>(o_g) |
                           (sh ? reinterpret_cast<uintptr_t>(sh) : 0)) & 15) == 0;
        if (stage_in_smem) {
            // stage the un-recentred residual t in shared memory (coalesced
            // 16-byte loads, rows re-pitched): the wavefront below reads it at
            // smem latency
            uint8_t *tb = o;
            if (vec) {
                const int cpr = w3 >> 4;  // 16-byte chunks per row
                for (int c = lane; c < H * cpr; c += 32) {
                    const int u = c / cpr, j = (c - u * cpr) * 16;
                    const int64_t i = (int64_t)u * w3 + j;
                    uint4 c4 = *reinterpret_cast<const uint4 *>(cd + i);
                    if (sh) {
                        const uint4 s4 = *reinterpret_cast<const uint4 *>(sh + i);
                        uint32_t *cw = reinterpret_cast<uint32_t *>(&c4);
                        const uint32_t *sw = reinterpret_cast<const uint32_t *>(&s4);
#pragma unroll
                        for (int e = 0; e < 4; ++e) cw[e] = __vadd4(__vadd4(cw[e], sw[e]), 0x80808080u);  // bytewise mod 256
                    }
                    uint32_t *d = reinterpret_cast<uint32_t *>(tb + (int64_t)u * rp + j);
                    d[0] = c4.x;
                    d[1] = c4.y;
                    d[2] = c4.z;
                    d[3] = c4.w;
                }
            } else {
                for (int64_t i = lane; i < hw3; i += 32) {
                    const int u = (int)(i / w3), j = (int)(i - (int64_t)u * w3);
                    tb[(int64_t)u * rp + j] = (uint8_t)unrec(cd, sh, i);
                }
            }
            __syncwarp();
            cd = tb;
            sh = nullptr;
        }
        // ---- red: skewed wavefront over pairs of 32-row strips. At step s
        // lane u decodes (u0 + u, s - u) in strip a and (u0 + 32 + u, s - u - 32)
        // in strip b; up / up-left come from lane u - 1's outputs one / two
        // steps earlier (strip b's lane 0 takes strip a's lane 31), so the two
        // strips' chains overlap and a pair costs W + 63 steps, not 2 (W + 31).
        for (int u0 = 0; u0 < H; u0 += 64) {
            const bool two = u0 + 32 < H;  // warp-uniform
            const int ua = u0 + lane, ub = u0 + 32 + lane;
            const bool ok_a = ua < H, ok_b = two && ub < H;
            float left_a = 0.f, left_b = 0.f;
            float ma1 = 0.f, ma2 = 0.f, mb1 = 0.f, mb2 = 0.f;  // this lane's outputs 1 / 2 steps ago
            const int steps = W + (two ? 63 : 31);
            for (int s = 0; s < steps; ++s) {
                const float na1 = __shfl_up_sync(0xffffffffu, ma1, 1);
                const float na2 = __shfl_up_sync(0xffffffffu, ma2, 1);
                float nb1 = 0.f, nb2 = 0.f;
                if (two) {
                    const int src = (lane + 31) & 31;
                    const float x1 = __shfl_sync(0xffffffffu, mb1, src);
                    const float x2 = __shfl_sync(0xffffffffu, mb2, src);
                    const float y1 = __shfl_sync(0xffffffffu, ma1, 31);
                    const float y2 = __shfl_sync(0xffffffffu, ma2, 31);
                    nb1 = lane == 0 ? y1 : x1;
                    nb2 = lane == 0 ? y2 : x2;
                }
                const int v = s - lane;
                float va = 0.f, vb = 0.f;
                if (ok_a && v >= 0 && v < W) {
                    float up, ul;
                    if (lane == 0) {  // row above the pair: decoded by the previous pair
                        up = ua > 0 ? (float)o[(int64_t)(ua - 1) * rp + v * 3] : 0.f;
                        ul = (ua > 0 && v > 0) ? (float)o[(int64_t)(ua - 1) * rp + (v - 1) * 3] : 0.f;
                    } else {
                        up = na1;
                        ul = v > 0 ? na2 : 0.f;
                    }
                    const float lf = v > 0 ? left_a : 0.f;
                    const uint32_t pr = predict(ul, up, lf, p.w, p.b[0], p.integral);
                    const int64_t i = (int64_t)ua * rp + v * 3;
                    const uint32_t x = (unrec(cd, sh, i) + pr + 128u) & 0xFFu;  // t - 128 + pred
                    o[i] = (uint8_t)x;
                    va = (float)x;
                    left_a = va;
                }
                const int w2 = v - 32;
                if (ok_b && w2 >= 0 && w2 < W) {
                    const float ul = w2 > 0 ? nb2 : 0.f;
                    const float lf = w2 > 0 ? left_b : 0.f;
                    const uint32_t pr = predict(ul, nb1, lf, p.w, p.b[0], p.integral);
                    const int64_t i = (int64_t)ub * rp + w2 * 3;
                    const uint32_t x = (unrec(cd, sh, i) + pr + 128u) & 0xFFu;
                    o[i] = (uint8_t)x;
                    vb = (float)x;
                    left_b = vb;
                }
                ma2 = ma1;
                ma1 = va;
                mb2 = mb1;
                mb1 = vb;
            }
            __syncwarp();
        }
        // ---- green and blue in one column sweep (blue at (u, v) needs green
        // at (u, v) and (u, v - 1) only); rows are independent, each lane
        // walks two of them (lane + 64k and lane + 32 + 64k) side by side
        auto gb = [&](int u, int v, float &rL, float &gL, float &bL) {
            const int64_t i0 = (int64_t)u * rp + v * 3;
            const float r = o[i0];
            const uint32_t pg = predict(gL, rL, r, p.w + 3, p.b[1], p.integral);
            const uint32_t g = (unrec(cd, sh, i0 + 1) + pg + 128u) & 0xFFu;
            o[i0 + 1] = (uint8_t)g;
            const float gf = (float)g;
            const uint32_t pb = predict(bL, gL, gf, p.w + 6, p.b[2], p.integral);
            const uint32_t bb = (unrec(cd, sh, i0 + 2) + pb + 128u) & 0xFFu;
            o[i0 + 2] = (uint8_t)bb;
            rL = r;
            gL = gf;
            bL = (float)bb;
        };
        for (int u = lane; u < H; u += 64) {
            const int u2 = u + 32;
            float rL = 0.f, gL = 0.f, bL = 0.f, rL2 = 0.f, gL2 = 0.f, bL2 = 0.f;
            if (u2 < H) {
                for (int v = 0; v < W; ++v) {
                    gb(u, v, rL, gL, bL);
                    gb(u2, v, rL2, gL2, bL2);
                }
            } else {
                for (int v = 0; v < W; ++v) gb(u, v, rL, gL, bL);
            }
        }
        __syncwarp();
        if (stage_in_smem) {
            // coalesced copy-out, 16 bytes per lane when aligned
            if (vec) {
                const int cpr = w3 >> 4;
                for (int c = lane; c < H * cpr; c += 32) {
                    const int u = c / cpr, j = (c - u * cpr) * 16;
                    const uint32_t *d = reinterpret_cast<const uint32_t *>(o + (int64_t)u * rp + j);
                    *reinterpret_cast<uint4 *>(o_g + (int64_t)u * w3 + j) = make_uint4(d[0], d[1], d[2], d[3]);
                }
            } else {
                for (int64_t i = lane; i < hw3; i += 32) {
                    const int u = (int)(i / w3), j = (int)(i - (int64_t)u * w3);
                    o_g[i] = o[(int64_t)u * rp + j];
                }
            }
            __syncwarp();
        }
    }
}

// Shared-memory row pitch for twar_decode_kernel: a multiple of 4 bytes
// >= 3 W with the fewest bank conflicts for the red wavefront's skewed
// accesses (lane u at byte 3 s + u (rp - 3)) and the green / blue sweep's
// (lane u at byte u rp + 3 v), over the four byte phases.
int decode_pitch(int W) {
    int best_rp = 3 * W, best = 1 << 30;
    for (int rp = (3 * W + 3) & ~3; rp < 3 * W + 260; rp += 4) {
        int worst = 0;
        for (int pat = 0; pat < 2; ++pat)
            for (int ph = 0; ph < 4; ++ph) {
                int words[32][32], cnt[32] = {0};
                for (int u = 0; u < 32; ++u) {
                    const long long a = pat == 0 ? 3LL * (ph + 64) + (long long)u * (rp - 3) : (long long)u * rp + ph;
                    const int wd = (int)(a >> 2), bk = wd & 31;
                    bool dup = false;
                    for (int k = 0; k < cnt[bk]; ++k) dup |= words[bk][k] == wd;
                    if (!dup) words[bk][cnt[bk]++] = wd;
                }
                for (int b = 0; b < 32; ++b) worst = worst > cnt[b] ? worst : cnt[b];
            }
        if (worst < best) {
            best = worst;
            best_rp = rp;
        }
    }
    return best_rp;
}

Params load_params(const float *p12) {
    Params p;
    p.integral = 1;
    for (int c = 0; c < 3; ++c) {
        for (int j = 0; j < 3; ++j) {
            const float w = p12[4 * c + j];
            p.w[3 * c + j] = w;
            p.integral &= (w == floorf(w) && fabsf(w) <= 8192.f) ? 1 : 0;
        }
        const float b = p12[4 * c + 3];
        p.b[c] = b;
        p.integral &= (b == floorf(b) && fabsf(b) <= 4194304.f) ? 1 : 0;
    }
    return p;
}

}  // namespace

extern "C" int pilc_twar_forward(const uint8_t *img, uint8_t *res, int64_t n_img, int32_t H,
                                 int32_t W, const float *params12_host, void *stream) {
    if (n_img < 0 || H < 1 || W < 1 || !params12_host) return PILC_E_ARG;
    const int64_t n_px = n_img * (int64_t)H * W;
    if (n_px == 0) return PILC_OK;
    const int threads = 256;
    const Params prm = load_params(params12_host);
    ProfScope _ps(PROF_TWAR_FWD, as_stream(stream), 3.0 * n_px);
    static const float kDefault[9] = {-1.f, 1.f, 1.f, 1.f, -1.f, 1.f, 1.f, -1.f, 1.f};
    bool unit = prm.b[0] == 0.f && prm.b[1] == 0.f && prm.b[2] == 0.f;
    for (int k = 0; k < 9; ++k) unit = unit && prm.w[k] == kDefault[k];
    const int64_t ib = (int64_t)H * W * 3;
    if ((W & 15) == 0 && ib <= kTwTileBytes && ((reinterpret_cast<uintptr_t>(img) | reinterpret_cast<uintptr_t>(res)) & 15) == 0) {
        const int G = (int)(kTwTileBytes / ib);
        const int64_t groups = (n_img + G - 1) / G;
        int64_t blocks = groups;
        const int64_t cap = (int64_t)sm_count() * 4;
        if (blocks > cap) blocks = cap;
        const int sm = 4 * kTwTileBytes;
        auto kern = unit ? twar_forward_tile_kernel<2> : (prm.integral ? twar_forward_tile_kernel<1> : twar_forward_tile_kernel<0>);
        allow_dyn_smem(reinterpret_cast<const void *>(kern));
        kern<<<(unsigned)blocks, threads, sm, as_stream(stream)>>>(img, res, n_img, H, W, G, prm);
    } else if ((W & 7) == 0 && ((reinterpret_cast<uintptr_t>(img) | reinterpret_cast<uintptr_t>(res)) & 7) == 0) {
        const int64_t n_units = n_px >> 3;
        int64_t blocks = ceil_div64(n_units, threads);
        const int64_t cap = (int64_t)sm_count() * 32;
        if (blocks > cap) blocks = cap;
        if (unit)
            twar_forward8_kernel<2><<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(img, res, n_units, H, W, prm);
        else if (prm.integral)
            twar_forward8_kernel<1><<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(img, res, n_units, H, W, prm);
        else
            twar_forward8_kernel<0><<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(img, res, n_units, H, W, prm);
    } else {
        int64_t blocks = ceil_div64(n_px, threads);
        const int64_t cap = (int64_t)sm_count() * 32;
        if (blocks > cap) blocks = cap;
        twar_forward_kernel<<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(img, res, n_px, H, W, prm);
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

extern "C" int pilc_twar_decode(const uint8_t *coded, const uint8_t *shift, uint8_t *img,
                                int64_t n_img, int32_t H, int32_t W, const float *params12_host,
                                void *stream) {
    if (n_img < 0 || H < 1 || W < 1 || !params12_host) return PILC_E_ARG;
    if (n_img == 0) return PILC_OK;
    const int64_t hw3 = (int64_t)H * W * 3;
    const int rp_s = decode_pitch(W);
    const int stage = (int64_t)H * rp_s * kDecWarps <= 200 * 1024;  // one image per warp, decoded in place
    const int rp = stage ? rp_s : 3 * W;
    const size_t smem = stage ? (size_t)((int64_t)H * rp * kDecWarps) : 0;
    if (smem > 48 * 1024)
        allow_dyn_smem(reinterpret_cast<const void *>(twar_decode_kernel));
    int64_t blocks = ceil_div64(n_img, kDecWarps);
    const int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
{
        ProfScope _ps(PROF_TWAR_DEC, as_stream(stream), (double)n_img * hw3);
        twar_decode_kernel<<<(unsigned)blocks, 32 * kDecWarps, smem, as_stream(stream)>>>(
        coded, shift, img, n_img, H, W, load_params(params12_host), stage, rp);
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}
