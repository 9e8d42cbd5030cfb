/*
 * PILC CPU oracle -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's compiled hot loops
 * (/root/reference/pkg/src/pixelcodec/_kernels.py), used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * as the checker. The product (paper_2206_05279_b200) never links this.
 *
 * Deliberately written like the reference: one bit per inner iteration for
 * the coder, raster order for the inverse predictor. Pinned against the
 * reference's own outputs by tests/test_oracle.py (tests/golden/ fixtures).
 *
 * Build: oracle/Makefile  (gcc -O2 -ffp-contract=off -fopenmp -shared)
 * -ffp-contract=off is part of the contract: the reference accumulates the
 * predictor in float32 without FMA (_kernels.py:82-88).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* _kernels.py:20-40 (encode_lane). Symbols are read at syms[i*stride],
 * i = n-1 .. 0 (reverse order); bits are pushed LSB-first into buf, which
 * the caller zero-fills and sizes for n*(M+1) bits. Returns the final state. */
int64_t oracle_encode_lane(const uint8_t *syms, const uint16_t *ds, int64_t n,
                           int64_t stride, const uint16_t *delta,
                           const uint16_t *phi, int64_t X, int M, uint8_t *buf,
                           int64_t *nbits_out) {
    int64_t state = (int64_t)1 << M;
    int64_t pos = 0;
    for (int64_t i = n - 1; i >= 0; --i) {
        int64_t d = ds[i * stride];
        int64_t x = syms[i * stride];
        int64_t b = ((int64_t)delta[d * X + x] + state) >> M;
        for (int64_t j = 0; j < b; ++j) {
            int64_t bit = (state >> j) & 1;
            buf[pos >> 3] |= (uint8_t)(bit << (pos & 7));
            ++pos;
        }
        state = (state >> b) + (int64_t)phi[d * X + x];
    }
    *nbits_out = pos;
    return state;
}

/* _kernels.py:43-63 (decode_lane). Returns the end state (-1 on underflow)
 * and the number of unread bits in *rem. Output at out[i*stride]. */
int64_t oracle_decode_lane(int64_t state, const uint8_t *buf, int64_t nbits,
                           const uint16_t *ds, int64_t n, int64_t stride,
                           const uint8_t *theta, const uint8_t *bcnt,
                           const uint16_t *nxt, int M, uint8_t *out,
                           int64_t *rem) {
    const int64_t base = (int64_t)1 << M;
    const int64_t T = base;
    int64_t pos = nbits;
    for (int64_t i = 0; i < n; ++i) {
        int64_t idx = state - base;
        int64_t d = ds[i * stride];
        out[i * stride] = theta[d * T + idx];
        int64_t b = bcnt[d * T + idx];
        if (pos < b) {
            *rem = pos;
            return -1;
        }
        int64_t v = 0;
        for (int64_t k = 0; k < b; ++k) {
            --pos;
            v = (v << 1) | ((buf[pos >> 3] >> (pos & 7)) & 1);
        }
        state = (int64_t)nxt[d * T + idx] + v;
    }
    *rem = pos;
    return state;
}

/* _kernels.py:68-79 (_round_mod256): f64 round-half-away, fmod 256. */
static int64_t round_mod256(float p32) {
    double p = (double)p32;
    double r = p >= 0.0 ? floor(p + 0.5) : ceil(p - 0.5);
    double m = fmod(r, 256.0);
    if (m < 0.0) m += 256.0;
    return (int64_t)m;
}

/* _kernels.py:82-88 (_predict3): f32, left to right, bias last, no FMA. */
static int64_t predict3(float c0, float c1, float c2, const float *w, float b) {
    float acc = w[0] * c0;
    acc = acc + w[1] * c1;
    acc = acc + w[2] * c2;
    acc = acc + b;
    return round_mod256(acc);
}

#define PX(img, u, v, c) (img)[((int64_t)(u) * W + (v)) * 3 + (c)]

/* predictor.py:173-195 (predictions + forward_residual), stock k=3 layout
 * (predictor.py:36-40): R <- (ul, up, left); G,B <- (left, prev-left,
 * prev-here); zero outside the image. One image per OpenMP iteration. */
void oracle_twar_forward(const uint8_t *img, int64_t N, int H, int W,
                         const float *w9, const float *b3, uint8_t *res) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t n = 0; n < N; ++n) {
        const uint8_t *x = img + n * (int64_t)H * W * 3;
        uint8_t *t = res + n * (int64_t)H * W * 3;
        for (int u = 0; u < H; ++u)
            for (int v = 0; v < W; ++v)
                for (int c = 0; c < 3; ++c) {
                    float c0, c1, c2;
                    if (c == 0) {
                        c0 = (u > 0 && v > 0) ? (float)PX(x, u - 1, v - 1, 0) : 0.f;
                        c1 = u > 0 ? (float)PX(x, u - 1, v, 0) : 0.f;
                        c2 = v > 0 ? (float)PX(x, u, v - 1, 0) : 0.f;
                    } else {
                        c0 = v > 0 ? (float)PX(x, u, v - 1, c) : 0.f;
                        c1 = v > 0 ? (float)PX(x, u, v - 1, c - 1) : 0.f;
                        c2 = (float)PX(x, u, v, c - 1);
                    }
                    int64_t pred = predict3(c0, c1, c2, w9 + 3 * c, b3[c]);
                    PX(t, u, v, c) = (uint8_t)(((int64_t)PX(x, u, v, c) - pred + 128) & 0xFF);
                }
    }
}

/* _kernels.py:91-112 (seq_decode3), batched like seq_decode3_batch
 * (_kernels.py:173-176). Optional shift plane undoes recentring first
 * (logistic.py:166-168): t = (coded + shift - 128) & 255. */
void oracle_twar_decode(const uint8_t *coded, const uint8_t *shift, int64_t N,
                        int H, int W, const float *w9, const float *b3,
                        uint8_t *out) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t n = 0; n < N; ++n) {
        const int64_t off = n * (int64_t)H * W * 3;
        const uint8_t *r = coded + off;
        const uint8_t *sh = shift ? shift + off : 0;
        uint8_t *o = out + off;
#define RES(u, v, c) ((int64_t)(sh ? (uint8_t)((PX(r, u, v, c) + PX(sh, u, v, c) - 128) & 0xFF) : PX(r, u, v, c)))
        for (int u = 0; u < H; ++u)
            for (int v = 0; v < W; ++v) {
                float c0 = (u > 0 && v > 0) ? (float)PX(o, u - 1, v - 1, 0) : 0.f;
                float c1 = u > 0 ? (float)PX(o, u - 1, v, 0) : 0.f;
                float c2 = v > 0 ? (float)PX(o, u, v - 1, 0) : 0.f;
                int64_t pred = predict3(c0, c1, c2, w9, b3[0]);
                PX(o, u, v, 0) = (uint8_t)((RES(u, v, 0) - 128 + pred) & 0xFF);
            }
        for (int c = 1; c < 3; ++c)
            for (int u = 0; u < H; ++u)
                for (int v = 0; v < W; ++v) {
                    float c0 = v > 0 ? (float)PX(o, u, v - 1, c) : 0.f;
                    float c1 = v > 0 ? (float)PX(o, u, v - 1, c - 1) : 0.f;
                    float c2 = (float)PX(o, u, v, c - 1);
                    int64_t pred = predict3(c0, c1, c2, w9 + 3 * c, b3[c]);
                    PX(o, u, v, c) = (uint8_t)((RES(u, v, c) - 128 + pred) & 0xFF);
                }
#undef RES
    }
}

/* Batched lanes for the CPU baseline: image i owns syms[i*n .. i*n+n),
 * lane l takes symbols l, l+L, ... (tables.py:202-223). Per-lane scratch
 * of cap bytes; outputs nbits/state per (image, lane). */
void oracle_encode_batch(const uint8_t *syms, const uint16_t *ds, int64_t N,
                         int64_t n, int64_t L, const uint16_t *delta,
                         const uint16_t *phi, int64_t X, int M, uint8_t *scratch,
                         int64_t cap, int64_t *nbits, int64_t *states) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t k = 0; k < N * L; ++k) {
        int64_t img = k / L, lane = k % L;
        int64_t cnt = lane < n ? (n - lane + L - 1) / L : 0;
        uint8_t *buf = scratch + k * cap;
        memset(buf, 0, (size_t)cap);
        states[k] = oracle_encode_lane(syms + img * n + lane, ds + img * n + lane,
                                       cnt, L, delta, phi, X, M, buf, &nbits[k]);
    }
}

/* ---------------------------------------------------------------------------
 * The reference network's float arithmetic, stated as explicit operations.
 *
 * nn.py:15-34 computes each conv as `out += np.tensordot(w[:, :, i, j], tap)`
 * tap by tap (i outer, j inner), then `out + b`. The tensordot is an f32
 * GEMM through numpy's OpenBLAS (scipy-openblas 0.3.30 here), whose sgemm
 * microkernels keep one accumulator per output element and walk the
 * contraction index in order with fused multiply-adds, starting from zero
 * (K <= 32 here, so there is a single K block). So, for most pixels:
 *   t_ij[co,p] = fmaf(w[co,ci=K-1], x[K-1,p], ... fmaf(w[co,0], x[0,p], 0))
 *   out = ((0 + t_00) + t_01) + ... + t_22 ;  out = out + b[co]
 * with edge-replicate padding and stride 1 or 2; tap_dot() states the two
 * places where OpenBLAS walks k differently (single-pixel outputs go to
 * sgemv; with K >= 32 the last 1..8 pixels of an image go to a k-vectorised
 * tail kernel). Returns -1 where no order is modelled. tests/test_oracle.py checks
 * this statement bit for bit against the reference's own z, mu and s
 * (tests/golden/vqvae_*.npz), which is what pins the GPU "exact" network.
 * x: [cin][H][W] f32, w: [cout][cin][k][k], out: [cout][Ho][Wo]. */
/* One tap's contraction over the input channels, in the order OpenBLAS
 * evaluates it for an output pixel at position p of an n_px-pixel conv
 * output (n_px = Ho*Wo of one image). -1 = order not modelled. */
static int tap_dot(const float *w, int wstride, const float *x, int xstride, int K, int64_t p, int64_t n_px,
                   int cout, float *res) {
    if (n_px == 1) {
        /* numpy hands a single-column product to sgemv (sgemv_t); its
         * order depends on K: short rows are one fused multiply-add chain,
         * K = 4 and 8 reduce adjacent products pairwise, longer rows keep
         * 8 lanes (k = l mod 8) reduced as ((l0+l4)+(l1+l5))+((l2+l6)+(l3+l7))
         * with K = 9 / 10 leftovers folded in after. Modelled for whole
         * groups of 4 output channels (sgemv_t's column blocks) only. */
        if (cout % 4) return -1;
        if (K == 1) {
            *res = w[0] * x[0];
            return 0;
        }
        float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (K == 4 || K == 8) {
            for (int l = 0; l < K; ++l) a[l] = w[l * wstride] * x[l * xstride];
            float g = (a[0] + a[1]) + (a[2] + a[3]);
            *res = K == 4 ? g : g + ((a[4] + a[5]) + (a[6] + a[7]));
            return 0;
        }
        if (!(K == 9 || K == 10 || (K >= 16 && K % 8 == 0))) return -1;
        const int m = K & ~7;
        for (int k = 0; k < m; ++k) a[k & 7] = fmaf(w[k * wstride], x[k * xstride], a[k & 7]);
        float y = ((a[0] + a[4]) + (a[1] + a[5])) + ((a[2] + a[6]) + (a[3] + a[7]));
        if (K == 9) y = fmaf(w[8 * wstride], x[8 * xstride], y);
        if (K == 10) y = y + fmaf(w[8 * wstride], x[8 * xstride], w[9 * wstride] * x[9 * xstride]);
        *res = y;
        return 0;
    }
    const int64_t r = n_px % 16;
    if (K >= 32 && r >= 1 && r <= 8 && p >= n_px - r) {
        if (cout % 4 && !(cout == 3 && (r == 4 || r == 8))) return -1;  /* modelled: whole column groups, the heads */
        /* sgemm's narrow m-tail (1..8 leftover pixels) vectorises over k:
         * 16 lanes k = l (mod 16), then an adjacent-pair tree */
        float a[16];
        for (int l = 0; l < 16; ++l) a[l] = 0.0f;
        for (int k = 0; k < K; ++k) a[k & 15] = fmaf(w[k * wstride], x[k * xstride], a[k & 15]);
        for (int n = 16; n > 1; n >>= 1)
            for (int l = 0; l < n / 2; ++l) a[l] = a[2 * l] + a[2 * l + 1];
        *res = a[0];
        return 0;
    }
    float t = 0.0f;
    for (int k = 0; k < K; ++k) t = fmaf(w[k * wstride], x[k * xstride], t);
    *res = t;
    return 0;
}

int oracle_conv_fma(const float *x, int cin, int H, int W, const float *w,
                    const float *b, int cout, int k, int stride, float *out) {
    int p = k / 2;
    int Ho = (H + 2 * p - k) / stride + 1, Wo = (W + 2 * p - k) / stride + 1;
    const int64_t n_px = (int64_t)Ho * Wo;
    float col[4096];
    if (cin > 4096) return -1;
    for (int co = 0; co < cout; ++co)
        for (int y = 0; y < Ho; ++y)
            for (int xo = 0; xo < Wo; ++xo) {
                float o = 0.0f;
                for (int i = 0; i < k; ++i)
                    for (int j = 0; j < k; ++j) {
                        int yy = y * stride + i - p, xx = xo * stride + j - p;
                        yy = yy < 0 ? 0 : (yy >= H ? H - 1 : yy);
                        xx = xx < 0 ? 0 : (xx >= W ? W - 1 : xx);
                        for (int ci = 0; ci < cin; ++ci) col[ci] = x[(ci * H + yy) * W + xx];
                        float t;
                        if (tap_dot(w + (co * cin * k + i) * k + j, k * k, col, 1, cin, (int64_t)y * Wo + xo, n_px, cout, &t))
                            return -1;
                        o = o + t;
                    }
                out[(co * Ho + y) * Wo + xo] = o + b[co];
            }
    return 0;
}

/* numpy's float32 exp (the SIMD loop numpy 2.x dispatches to on AVX2/AVX512F
 * hosts, numpy/_core/src/umath/loops_exponent_log.dispatch.c.src
 * simd_exp_f32): Cody-Waite reduction by ln 2 in two parts, a [5/2] rational
 * approximation evaluated with fused multiply-adds, an IEEE division and a
 * scale by 2^q. The reference's sigmoid and s = exp(.) (nn.py:41-48,
 * vqvae.py:108) go through it; tests/test_oracle.py compares this statement
 * with np.exp over every float32 in the head's input ranges. */
float oracle_expf_np(float x) {
    const float log2e = 1.44269504088896341f, magic = 0x1.800000p+23f;
    const float c1 = -6.93145752e-1f, c2 = -1.42860677e-6f;
    const float p0 = 9.999999999980870924916e-01f, p1 = 7.257664613233124478488e-01f,
                p2 = 2.473615434895520810817e-01f, p3 = 5.114512081637298353406e-02f,
                p4 = 6.757896990527504603057e-03f, p5 = 5.082762527590693718096e-04f;
    const float q1 = -2.742335390411667452936e-01f, q2 = 2.159509375685829852307e-02f;
    float q = x * log2e;
    q = q + magic;
    q = q - magic;
    float r = fmaf(q, c1, x);
    r = fmaf(q, c2, r);
    float n = fmaf(p5, r, p4);
    n = fmaf(n, r, p3);
    n = fmaf(n, r, p2);
    n = fmaf(n, r, p1);
    n = fmaf(n, r, p0);
    float d = fmaf(q2, r, q1);
    d = fmaf(d, r, 1.0f);
    return ldexpf(n / d, (int)q);
}

void oracle_expf_np_array(const float *x, float *y, int64_t n) {
    for (int64_t i = 0; i < n; ++i) y[i] = oracle_expf_np(x[i]);
}
