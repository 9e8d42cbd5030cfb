// Shared helpers for the PILC sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pilc.h"

#define PILC_CHECK_LAUNCH()                              \
    do {                                                 \
        if (cudaPeekAtLastError() != cudaSuccess) {      \
            cudaGetLastError();                          \
            return PILC_E_CUDA;                          \
        }                                                \
    } while (0)

// ---- launch accounting / live per-kernel timing (pilc_prof_* in pilc.h) ----
// Every kernel launch goes through a ProfScope: it bumps the launch counter
// and, when timing is enabled, brackets the launch with CUDA events on the
// launching stream together with the launch's algorithmic work units.
enum ProfCat {
    PROF_CONV = 0,
    PROF_ARGMIN,
    PROF_RANS_ENC,
    PROF_RANS_DEC,
    PROF_TWAR_FWD,
    PROF_TWAR_DEC,
    PROF_STATIC_SCALE,
    PROF_SIZES,
    PROF_PACK,
    PROF_PARSE,
    PROF_LANES,
    PROF_CRC,
    PROF_SCHED_CRC,
    PROF_TC_CONV,
    PROF_GATHER,
    PROF_TC3_CONV,
    PROF_ENC_FRONT,
    PROF_TC3_BLOCK,
    PROF_DEC_TRUNK,
    PROF_ENC_TRUNK,
    PROF_DEC_UPHEAD,
    PROF_DEC_TRUNK2,
    PROF_NCAT
};
void *prof_begin(int cat, cudaStream_t s, double units);
void prof_end(void *tok, cudaStream_t s);
struct ProfScope {
    void *tok;
    cudaStream_t s;
    ProfScope(int cat, cudaStream_t st, double units) : s(st) { tok = prof_begin(cat, st, units); }
    ~ProfScope() { prof_end(tok, s); }
};

// Library tuning switches (pilc_set_tuning); defaults are the production path.
enum { PILC_TUNE_BLOCK_FUSION = 0, PILC_TUNE_DEC_TRUNK = 1, PILC_TUNE_ENC_TRUNK = 2, PILC_TUNE_DEC_UPHEAD = 3, PILC_TUNE_N };
extern int g_tuning[PILC_TUNE_N];

static inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Dynamic shared memory: every kernel's limit is raised once to the device
// maximum (less its static shared memory) and launches pick their own,
// smaller, sizes. Setting the attribute to each launch's own size raced
// between host threads launching one kernel with different sizes (one
// thread's setting undercut another's launch, cudaErrorInvalidValue).
int dyn_smem_limit(const void *func);  // api.cu: cached per (device, kernel)
static inline void allow_dyn_smem(const void *func) {
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem_limit(func));
}

static inline int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Grid sizing: the B200 has 148 SMs; cap grids at a multiple of the SM
// count and let kernels grid-stride.
static inline int sm_count() {
    static int cached = 0;
    if (!cached) {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cached = n > 0 ? n : 148;
    }
    return cached;
}

// ---------------------------------------------------------------------------
// CRC-32 (zlib polynomial 0xEDB88320, reflected), warp-cooperative.
//
// The warp walks the blob in rounds of 32 x 64 bytes. Lane i takes the i-th
// 64-byte chunk of the round, computes a standard crc32 of it with a
// byte table, and the chunks are merged with the affine combine rule
//   crc(A||B) = crc(A) * x^(8|B|)  xor  crc(B)     (mod P, reflected)
// (the rule zlib's crc32_combine implements). Powers x^(8*64*j) come from a
// small table; the ragged final round costs two x2nmodp evaluations.

struct CrcConsts {
    uint32_t tab[256];
    uint32_t qpow[33];  // (x^(8*64))^j mod P, j = 0..32
    uint32_t x2n[32];   // x^(2^k) mod P
};

__host__ __device__ inline uint32_t crc_multmodp(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
    }
    return p;
}

// x^(n * 2^k) mod P
__host__ __device__ inline uint32_t crc_x2nmodp(const uint32_t *x2n, uint64_t n, unsigned k) {
    uint32_t p = 1u << 31;
    while (n) {
        if (n & 1) p = crc_multmodp(x2n[k & 31], p);
        n >>= 1;
        k++;
    }
    return p;
}

const CrcConsts &crc_consts();  // host, built once (container.cu)

// Standard crc32 over n bytes (n may be 0) starting at p, table in smem.
__device__ inline uint32_t crc_bytes(const uint32_t *tab, const uint8_t *p, int n) {
    uint32_t c = 0xFFFFFFFFu;
    for (int i = 0; i < n; ++i) c = tab[(c ^ p[i]) & 0xFF] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

__device__ inline uint32_t warp_xor(uint32_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v ^= __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Slice-by-4 tables T1..T3 (T0 = CrcConsts::tab), built in shared memory.
struct CrcSlices {
    uint32_t t[3][256];
};

__device__ inline void build_crc_slices(CrcSlices *sl, const uint32_t *t0) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = t0[i];
        c = (c >> 8) ^ t0[c & 0xFF];
        sl->t[0][i] = c;
        c = (c >> 8) ^ t0[c & 0xFF];
        sl->t[1][i] = c;
        c = (c >> 8) ^ t0[c & 0xFF];
        sl->t[2][i] = c;
    }
}

// crc32 of n <= 64 bytes at a 4-byte aligned smem address, slice-by-4
__device__ inline uint32_t crc_chunk4(const uint32_t *t0, const CrcSlices *sl, const uint8_t *p, int n) {
    uint32_t c = 0xFFFFFFFFu;
    const uint32_t *w = reinterpret_cast<const uint32_t *>(p);
    int j = 0;
    for (; j + 4 <= n; j += 4) {
        c ^= w[j >> 2];
        c = sl->t[2][c & 0xFF] ^ sl->t[1][(c >> 8) & 0xFF] ^ sl->t[0][(c >> 16) & 0xFF] ^ t0[c >> 24];
    }
    for (; j < n; ++j) c = t0[(c ^ p[j]) & 0xFF] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

// Whole-warp crc32 of [p, p+n). stage: 32*68 + 64 bytes of this warp's smem.
// VEC: the bytes are fetched with 16-byte loads from the enclosing aligned
// vectors, so the source must be readable up to 15 bytes past p+n (the
// container buffers carry a 16-byte pad); chunks then use slice-by-4 (sl).
template <bool VEC = false>
__device__ inline uint32_t warp_crc32(const CrcConsts *cc, const uint8_t *p, uint64_t n, uint8_t *stage,
                                      const CrcSlices *sl = nullptr) {
    const int lane = threadIdx.x & 31;
    uint32_t crc = 0;  // crc32 of the empty string
    uint64_t done = 0;
    while (done < n) {
        const uint64_t rem = n - done;
        const int rb = rem >= 2048 ? 2048 : (int)rem;
        // chunk i of the round at stage + i*68 (padded: conflict-free per-lane reads)
        if constexpr (VEC) {
            const uintptr_t a = reinterpret_cast<uintptr_t>(p + done);
            const uint4 *a0 = reinterpret_cast<const uint4 *>(a & ~(uintptr_t)15);
            const int lead = (int)(a & 15);
            const int nv = (lead + rb + 15) >> 4;
            uint4 v[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const int vi = lane + 32 * k;
                v[k] = vi < nv ? a0[vi] : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const int vi = lane + 32 * k;
                const uint32_t w4[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int idx = 16 * vi + e - lead;
                    if (idx >= 0 && idx < rb) stage[(idx >> 6) * 68 + (idx & 63)] = (uint8_t)(w4[e >> 2] >> (8 * (e & 3)));
                }
            }
        } else {
            for (int j = lane; j < rb; j += 32) stage[(j >> 6) * 68 + (j & 63)] = p[done + j];
        }
        __syncwarp();
        const int beg = lane * 64;
        int len = rb - beg;
        len = len < 0 ? 0 : (len > 64 ? 64 : len);
        uint32_t c;
        if constexpr (VEC) c = crc_chunk4(cc->tab, sl, stage + lane * 68, len);
        else c = crc_bytes(cc->tab, stage + lane * 68, len);
        uint32_t term;
        if (rb == 2048) {
            term = crc_multmodp(cc->qpow[31 - lane], c);
        } else {
            // chunks k_last = (rb-1)/64 is ragged with r = rb - 64*k_last bytes
            const int kl = (rb - 1) >> 6;
            const int r = rb - 64 * kl;
            if (lane > kl) {
                term = 0;
            } else if (lane == kl) {
                term = c;
            } else {
                uint32_t xr = crc_x2nmodp(cc->x2n, (uint64_t)r, 3);
                term = crc_multmodp(crc_multmodp(cc->qpow[kl - lane - 1], xr), c);
            }
        }
        const uint32_t round_crc = warp_xor(term);
        if (rb == 2048)
            crc = crc_multmodp(cc->qpow[32], crc) ^ round_crc;
        else
            crc = crc_multmodp(crc_x2nmodp(cc->x2n, (uint64_t)rb, 3), crc) ^ round_crc;
        done += rb;
        __syncwarp();
    }
    return crc;
}

// Raw crc32 register (init 0, no final xor) of 64 bytes held as 16
// little-endian words, slice-by-4.
__device__ inline uint32_t crc_raw64(const uint32_t *t0, const CrcSlices *sl, const uint32_t *w) {
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        c ^= w[i];
        c = sl->t[2][c & 0xFF] ^ sl->t[1][(c >> 8) & 0xFF] ^ sl->t[0][(c >> 16) & 0xFF] ^ t0[c >> 24];
    }
    return c;
}

// Whole-warp crc32 of [p, p+n), no staging and no ragged rounds. The message
// is virtually left-padded with zero bytes to a multiple of 2048 (zero bytes
// leave a raw register at 0), so every round is 32 full 64-byte chunks, one
// per lane, read straight from global memory (16-byte loads re-aligned with
// funnel shifts) and merged pairwise with table multiplications by the
// constants x^(8*64*2^k); the standard init enters as 0xFF XORed into the
// first four bytes and the xorout at the end. The source must be readable up to
// the 16-byte boundary after p + n (the container buffers' pad).
// Multiplication by the constants x^(8*64*s), s = 1, 2, 4, 8, 16, 32, as
// byte-sliced tables (the map c -> c x^k mod P is linear): [6][4][256]
// words, built once on the host (crc_mul_tables, container.cu), read
// through the read-only cache.
constexpr int kCrcMulTables = 6 * 4 * 256;
__device__ inline uint32_t crc_mulk(const uint32_t *__restrict__ mt, int k, uint32_t c) {
    const uint32_t *t = mt + k * 1024;
    return __ldg(t + (c & 0xFF)) ^ __ldg(t + 256 + ((c >> 8) & 0xFF)) ^ __ldg(t + 512 + ((c >> 16) & 0xFF)) ^
           __ldg(t + 768 + (c >> 24));
}

__device__ inline uint32_t warp_crc32_fast(const CrcConsts *cc, const CrcSlices *sl, const uint32_t *__restrict__ mt,
                                           const uint8_t *p, uint64_t n) {
    const int lane = threadIdx.x & 31;
    if (n < 4) return __shfl_sync(0xffffffffu, crc_bytes(cc->tab, p, (int)n), 0);  // tiny messages
    const int64_t pad = (int64_t)((2048 - n % 2048) % 2048);
    uint32_t crc = 0;
    for (int64_t r0 = -pad; r0 < (int64_t)n; r0 += 2048) {
        const int64_t s = r0 + 64 * lane;
        uint32_t c = 0;
        uint32_t w[16];
        if (s >= 0) {
            const uintptr_t a = reinterpret_cast<uintptr_t>(p + s);
            const uint4 *a0 = reinterpret_cast<const uint4 *>(a & ~(uintptr_t)15);
            const int off = (int)(a & 15), q = off >> 2, sh = 8 * (off & 3);
            uint32_t W[20];
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const uint4 v = a0[k];
                W[4 * k] = v.x;
                W[4 * k + 1] = v.y;
                W[4 * k + 2] = v.z;
                W[4 * k + 3] = v.w;
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint32_t lo = q == 0 ? W[i] : q == 1 ? W[i + 1] : q == 2 ? W[i + 2] : W[i + 3];
                const uint32_t hi = q == 0 ? W[i + 1] : q == 1 ? W[i + 2] : q == 2 ? W[i + 3] : W[i + 4];
                w[i] = __funnelshift_r(lo, hi, sh);
            }
            if (s < 4) w[0] ^= 0xFFFFFFFFu >> (8 * s);  // the init register, folded into bytes 0..3
            c = crc_raw64(cc->tab, sl, w);
        } else if (s + 64 > 0) {
            // the chunk holding the first byte: what precedes p is zero. The
            // bytes come from the 16-byte vectors from align_down(p) on (never
            // below the buffer, which is 16-byte aligned), re-aligned to the
            // chunk's start s < 0 relative to p and masked below p
            const uintptr_t a = reinterpret_cast<uintptr_t>(p);
            const uint4 *a0 = reinterpret_cast<const uint4 *>(a & ~(uintptr_t)15);
            const int d = (int)(a & 15);
            uint32_t W[20];
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                const uint4 v = (16 * k < d + (int)(s + 64)) ? a0[k] : make_uint4(0u, 0u, 0u, 0u);
                W[4 * k] = v.x;
                W[4 * k + 1] = v.y;
                W[4 * k + 2] = v.z;
                W[4 * k + 3] = v.w;
            }
            const int s32 = (int)s;  // -63 .. -1
            // words from align_down(p) with 16 zero words in front: word i of
            // the chunk starts at byte s + 4 i + d of that window (one lane per
            // message takes this path; the dynamic index goes to local memory)
            uint32_t Z[37];
#pragma unroll
            for (int k = 0; k < 16; ++k) Z[k] = 0u;
#pragma unroll
            for (int k = 0; k < 20; ++k) Z[16 + k] = W[k];
            Z[36] = 0u;
            const int o0 = s32 + d + 64;  // >= 1
            const int q0 = o0 >> 2, sh = 8 * (o0 & 3);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                uint32_t v = __funnelshift_r(Z[q0 + i], Z[q0 + i + 1], sh);
                const int j0 = s32 + 4 * i;  // offset of the word's byte 0 from p
                if (j0 < 0) v = j0 > -4 ? v & (0xFFFFFFFFu << (8 * -j0)) : 0u;
                if (j0 > -4 && j0 < 4) v ^= j0 >= 0 ? 0xFFFFFFFFu >> (8 * j0) : 0xFFFFFFFFu << (8 * -j0);
                w[i] = v;
            }
            c = crc_raw64(cc->tab, sl, w);
        }
        // merge the 32 chunk registers pairwise: level k joins 64*2^k-byte
        // neighbours, the left one times x^(8*64*2^k); lane 0 ends with the round
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const uint32_t w = __shfl_down_sync(0xffffffffu, c, 1 << k);
            if ((lane & ((2 << k) - 1)) == 0) c = crc_mulk(mt, k, c) ^ w;
        }
        crc = crc_mulk(mt, 5, crc) ^ __shfl_sync(0xffffffffu, c, 0);
    }
    // the standard crc's init register entered as 0xFF XORed into bytes 0..3
    // (crc_I(M) = crc_0(M ^ I) for |M| >= 4); its final xor:
    return crc ^ 0xFFFFFFFFu;
}

__device__ inline void load_crc_consts(CrcConsts *dst, const CrcConsts &src) {
    const uint32_t *s = reinterpret_cast<const uint32_t *>(&src);
    uint32_t *d = reinterpret_cast<uint32_t *>(dst);
    for (int i = threadIdx.x; i < (int)(sizeof(CrcConsts) / 4); i += blockDim.x) d[i] = s[i];
}
