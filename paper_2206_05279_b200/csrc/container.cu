// PILC container on the device: static scale, blob sizing, packing, crc32,
// header parsing and lane extraction.
//
// Layout (container.py:3-25, little-endian):
//   "PILC" | ver u8 | backend u8 | M u8 | pad u8 | flags u8
//   | W u32 | H u32 | L u16 | static_d u16        (static_d at byte 19)
//   | grid: D u16, D x f64 | params hash 8 | [vqvae: model hash 8]
//   | [vqvae: idx table: total u32, L x u32 wire sizes, L x u16 states]
//   | residual table (same) | [flags&1: schedule crc u32]
//   | idx lane blobs | residual lane blobs | crc32 u32 over all of the above
// A lane blob is the BitStack wire form (bits.py:66-87): u64 LE bit count,
// then ceil(nbits/8) payload bytes, tail bits zero.

#include <math.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "common.cuh"

// ---------------------------------------------------------------------------
const CrcConsts &crc_consts() {
    static CrcConsts cc;
    static bool init = false;
    if (!init) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ 0xEDB88320u : c >> 1;
            cc.tab[i] = c;
        }
        uint32_t p = 1u << 30;  // x^1
        for (int k = 0; k < 32; ++k) {
            cc.x2n[k] = p;
            p = crc_multmodp(p, p);
        }
        const uint32_t q = cc.x2n[9];  // x^512 = x^(8*64)
        cc.qpow[0] = 1u << 31;
        for (int j = 1; j <= 32; ++j) cc.qpow[j] = crc_multmodp(cc.qpow[j - 1], q);
        init = true;
    }
    return cc;
}

// Device copy of the constant-multiplication tables (common.cuh), per device.
const uint32_t *crc_mul_tables() {
    static const uint32_t *dev_tab[64] = {};
    static std::mutex mu;
    int d = 0;
    cudaGetDevice(&d);
    std::lock_guard<std::mutex> g(mu);
    if (d < 0 || d >= 64) return nullptr;
    if (!dev_tab[d]) {
        const CrcConsts &cc = crc_consts();
        std::vector<uint32_t> h(kCrcMulTables);
        const int pw[6] = {1, 2, 4, 8, 16, 32};
        for (int k = 0; k < 6; ++k)
            for (int j = 0; j < 4; ++j)
                for (uint32_t v = 0; v < 256; ++v) h[k * 1024 + j * 256 + v] = crc_multmodp(cc.qpow[pw[k]], v << (8 * j));
        void *p = nullptr;
        if (cudaMalloc(&p, h.size() * 4) != cudaSuccess) return nullptr;
        cudaMemcpy(p, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
        dev_tab[d] = static_cast<const uint32_t *>(p);
    }
    return dev_tab[d];
}

namespace {

constexpr int kWarps = 4;  // warps per block for warp-per-blob kernels
constexpr int kStage = 32 * 68 + 64;

__device__ __forceinline__ uint32_t rd_u16(const uint8_t *p) { return p[0] | (p[1] << 8); }
__device__ __forceinline__ uint32_t rd_u32(const uint8_t *p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
__device__ __forceinline__ uint64_t rd_u64(const uint8_t *p) {
    return (uint64_t)rd_u32(p) | ((uint64_t)rd_u32(p + 4) << 32);
}
__device__ __forceinline__ void wr_u16(uint8_t *p, uint32_t v) {
    p[0] = v & 0xFF;
    p[1] = (v >> 8) & 0xFF;
}
__device__ __forceinline__ void wr_u32(uint8_t *p, uint32_t v) {
    p[0] = v & 0xFF;
    p[1] = (v >> 8) & 0xFF;
    p[2] = (v >> 16) & 0xFF;
    p[3] = v >> 24;
}

// ---- static scale (container.py:163-170) ---------------------------------
// Block per image: exact integer sum of |t - 128|; then the reference's f64
// formula  argmin_j |log2(mad / ln 4) - log2 g_j|  (ties to smaller j).
__global__ void static_scale_kernel(const uint8_t *__restrict__ res, int64_t n_sym,
                                    const double *__restrict__ log2g, int D,
                                    uint16_t *__restrict__ d_img) {
    const int64_t img = blockIdx.x;
    const uint8_t *t = res + img * n_sym;
    unsigned long long s = 0;
    for (int64_t i = threadIdx.x; i < n_sym; i += blockDim.x) {
        const int v = (int)t[i] - 128;
        s += (unsigned long long)(v < 0 ? -v : v);
    }
    __shared__ unsigned long long red[32];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tot = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
        // np.mean over float64 values: pairwise summation of exact small
        // integers is exact, so mean = tot / n correctly rounded.
        const double mad = (double)tot / (double)n_sym;
        const double s_est = mad / 1.3862943611198906;  // np.log(4.0), correctly rounded
        int best = 0;
        if (s_est > 0) {
            const double l2 = log2(s_est);
            double bd = fabs(l2 - log2g[0]);
            for (int j = 1; j < D; ++j) {
                const double dj = fabs(l2 - log2g[j]);
                if (dj < bd) {
                    bd = dj;
                    best = j;
                }
            }
        }
        d_img[img] = (uint16_t)best;
    }
}

// ---- sizes -----------------------------------------------------------------
__global__ void blob_sizes_kernel(const uint32_t *__restrict__ idx_nbits,
                                  const uint32_t *__restrict__ res_nbits, int64_t n_img,
                                  int lanes, int64_t fixed_bytes, uint64_t *__restrict__ sizes) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t img = (int64_t)blockIdx.x * kWarps + warp; img < n_img;
         img += (int64_t)gridDim.x * kWarps) {
        uint64_t s = 0;
        for (int l = lane; l < lanes; l += 32) {
            s += 8 + (((uint64_t)res_nbits[img * lanes + l] + 7) >> 3);
            if (idx_nbits) s += 8 + (((uint64_t)idx_nbits[img * lanes + l] + 7) >> 3);
        }
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) sizes[img] = s + (uint64_t)fixed_bytes;
    }
}

// single-block exclusive scan of n sizes into off[0..n]
__global__ void scan_kernel(const uint64_t *__restrict__ sizes, int64_t n, uint64_t *__restrict__ off) {
    __shared__ uint64_t part[1024];
    const int t = threadIdx.x, T = blockDim.x;
    const int64_t per = (n + T - 1) / T;
    const int64_t b = t * per, e = b + per < n ? b + per : n;
    uint64_t s = 0;
    for (int64_t i = b; i < e; ++i) s += sizes[i];
    part[t] = s;
    __syncthreads();
    for (int o = 1; o < T; o <<= 1) {
        uint64_t v = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    uint64_t run = t ? part[t - 1] : 0;
    for (int64_t i = b; i < e; ++i) {
        off[i] = run;
        run += sizes[i];
    }
    if (t == T - 1) off[n] = part[T - 1];
}

// ---- pack -----------------------------------------------------------------
struct PackArgs {
    const uint16_t *d_img;
    const uint8_t *dsched;
    int sched_check;
    int64_t n_img, n_sym;
    int lanes;
    const uint32_t *idx_scratch;
    int64_t idx_cap;
    const uint32_t *idx_nbits;
    const uint16_t *idx_states;
    const uint32_t *res_scratch;
    int64_t res_cap;
    const uint32_t *res_nbits;
    const uint16_t *res_states;
    const uint64_t *blob_off;
    uint8_t *out;
    const uint8_t *tmpl;  // device copy of the header prefix
    int tmpl_len;
};

// Copy one lane blob (u64 nbits + payload bytes from 32-bit scratch words).
// The payload lands at an arbitrary byte offset: whole destination-aligned
// words are assembled from two source words with a funnel shift and stored
// as 32-bit words; the partial words at either end go byte by byte (the
// bytes around belong to the header and to the next blob). Tail bits zero.
__device__ void put_lane(uint8_t *dst, const uint32_t *words, uint32_t nbits, int lane) {
    const uint32_t nbytes = (nbits + 7) >> 3;
    if (lane < 8) dst[lane] = lane < 4 ? (nbits >> (8 * lane)) & 0xFF : 0;
    if (nbytes == 0) return;
    uint8_t *pay = dst + 8;
    const uint32_t tmask = (nbits & 7) ? (1u << (nbits & 7)) - 1u : 0xFFu;
    auto src_byte = [&](uint32_t j) -> uint32_t {
        uint32_t v = (words[j >> 2] >> (8 * (j & 3))) & 0xFF;
        return j == nbytes - 1 ? v & tmask : v;
    };
    const uint32_t a = (uint32_t)(reinterpret_cast<uintptr_t>(pay) & 3);
    const uint32_t head = a ? 4 - a : 0;                       // bytes before the first aligned word
    if (head >= nbytes || nbytes - head < 8) {                 // short: bytes only
        for (uint32_t j = lane; j < nbytes; j += 32) pay[j] = (uint8_t)src_byte(j);
        return;
    }
    const uint32_t nw = (nbytes - head) >> 2;                  // whole aligned words
    const uint32_t tail0 = head + 4 * nw;                      // first byte after them
    if (lane < (int)head) pay[lane] = (uint8_t)src_byte(lane);
    if (lane < (int)(nbytes - tail0)) pay[tail0 + lane] = (uint8_t)src_byte(tail0 + lane);
    uint32_t *pw = reinterpret_cast<uint32_t *>(pay + head);
    // aligned word m holds payload bytes head + 4m .. +3 = source bytes
    // starting at byte (head & 3) of source word (head >> 2) + m
    const uint32_t s0 = head >> 2, sh = 8 * (head & 3);
    for (uint32_t m = lane; m < nw; m += 32) {
        const uint32_t lo = words[s0 + m];
        uint32_t v = sh ? __funnelshift_r(lo, words[s0 + m + 1], sh) : lo;
        if (head + 4 * m + 3 == nbytes - 1) v = (v & 0x00FFFFFFu) | ((v >> 24 & tmask) << 24);
        pw[m] = v;
    }
}

// Writes one stream table and returns its length.
__device__ int put_table(uint8_t *dst, const uint32_t *nbits, const uint16_t *states, int lanes,
                         int lane) {
    uint64_t tot = 0;
    for (int l = lane; l < lanes; l += 32) {
        const uint32_t w = 8 + ((nbits[l] + 7) >> 3);
        tot += w;
        wr_u32(dst + 4 + 4 * l, w);
        wr_u16(dst + 4 + 4 * lanes + 2 * l, states[l]);
    }
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0) wr_u32(dst, (uint32_t)tot);
    return 4 + 6 * lanes;
}

__device__ uint32_t sched_crc_warp(const CrcConsts *cc, const uint8_t *dsched, uint32_t dconst,
                                   int64_t n_sym, uint8_t *stage) {
    // crc32 over n_sym u16 LE values; stage them two bytes at a time
    const int lane = threadIdx.x & 31;
    uint32_t crc = 0;
    const int64_t nbytes = 2 * n_sym;
    int64_t done = 0;
    while (done < nbytes) {
        const int64_t rem = nbytes - done;
        const int rb = rem >= 2048 ? 2048 : (int)rem;
        for (int j = lane; j < rb; j += 32) {
            const int64_t bi = done + j;
            const uint32_t d = dsched ? dsched[bi >> 1] : dconst;
            stage[(j >> 6) * 68 + (j & 63)] = (bi & 1) ? (uint8_t)(d >> 8) : (uint8_t)(d & 0xFF);
        }
        __syncwarp();
        const int beg = lane * 64;
        int len = rb - beg;
        len = len < 0 ? 0 : (len > 64 ? 64 : len);
        const uint32_t c = crc_bytes(cc->tab, stage + lane * 68, len);
        uint32_t term;
        if (rb == 2048) {
            term = crc_multmodp(cc->qpow[31 - lane], c);
        } else {
            const int kl = (rb - 1) >> 6;
            const int r = rb - 64 * kl;
            if (lane > kl) term = 0;
            else if (lane == kl) term = c;
            else term = crc_multmodp(crc_multmodp(cc->qpow[kl - lane - 1], crc_x2nmodp(cc->x2n, r, 3)), c);
        }
        const uint32_t rc = warp_xor(term);
        crc = (rb == 2048) ? (crc_multmodp(cc->qpow[32], crc) ^ rc)
                           : (crc_multmodp(crc_x2nmodp(cc->x2n, rb, 3), crc) ^ rc);
        done += rb;
        __syncwarp();
    }
    return crc;
}

__global__ void __launch_bounds__(32 * kWarps) pack_kernel(PackArgs a, CrcConsts ccv, const uint32_t *__restrict__ mt) {
    __shared__ CrcConsts cc;
    __shared__ CrcSlices sl;
    __shared__ __align__(16) uint8_t stage[kWarps][kStage];
    load_crc_consts(&cc, ccv);
    __syncthreads();
    build_crc_slices(&sl, cc.tab);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = a.lanes;
    for (int64_t img = (int64_t)blockIdx.x * kWarps + warp; img < a.n_img;
         img += (int64_t)gridDim.x * kWarps) {
        uint8_t *blob = a.out + a.blob_off[img];
        const uint64_t size = a.blob_off[img + 1] - a.blob_off[img];
        for (int i = lane; i < a.tmpl_len; i += 32) blob[i] = a.tmpl[i];
        __syncwarp();
        const uint32_t sd = a.d_img ? a.d_img[img] : 0u;
        if (lane == 0) wr_u16(blob + 19, sd);
        int64_t off = a.tmpl_len;
        if (a.idx_nbits)
            off += put_table(blob + off, a.idx_nbits + img * L, a.idx_states + img * L, L, lane);
        off += put_table(blob + off, a.res_nbits + img * L, a.res_states + img * L, L, lane);
        if (a.sched_check) {
            const uint32_t c = sched_crc_warp(&cc, a.dsched ? a.dsched + img * a.n_sym : nullptr, sd,
                                              a.n_sym, stage[warp]);
            if (lane == 0) wr_u32(blob + off, c);
            off += 4;
        }
        // lane blobs: each warp walks lanes in order, sizes are known
        for (int s = 0; s < 2; ++s) {
            const uint32_t *nb = s == 0 ? a.idx_nbits : a.res_nbits;
            if (!nb) continue;
            const uint32_t *scr = s == 0 ? a.idx_scratch : a.res_scratch;
            const int64_t cap = s == 0 ? a.idx_cap : a.res_cap;
            for (int l = 0; l < L; ++l) {
                const uint32_t bits = nb[img * L + l];
                put_lane(blob + off, scr + (img * L + l) * cap, bits, lane);
                off += 8 + ((bits + 7) >> 3);
            }
        }
        __syncwarp();
        __threadfence_block();
        // the output buffer carries 16 bytes of slack (pilc.h): vector reads
        const uint32_t crc = warp_crc32_fast(&cc, &sl, mt, blob, size - 4);
        if (lane == 0) wr_u32(blob + size - 4, crc);
    }
}

// ---- parse (container.py:195-258) ----------------------------------------
__global__ void __launch_bounds__(32 * kWarps) parse_kernel(const uint8_t *__restrict__ buf,
                                                            const uint64_t *__restrict__ blob_off,
                                                            int64_t n_blob, uint64_t params_hash,
                                                            uint64_t model_hash, int has_model,
                                                            pilc_header *hdr, CrcConsts ccv,
                                                            const uint32_t *__restrict__ mt) {
    __shared__ CrcConsts cc;
    __shared__ CrcSlices sl;
    __shared__ __align__(16) uint8_t stage[kWarps][kStage];
    load_crc_consts(&cc, ccv);
    __syncthreads();
    build_crc_slices(&sl, cc.tab);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t i = (int64_t)blockIdx.x * kWarps + warp; i < n_blob;
         i += (int64_t)gridDim.x * kWarps) {
        const uint8_t *b = buf + blob_off[i];
        const uint64_t n = blob_off[i + 1] - blob_off[i];
        pilc_header h;
        memset(&h, 0, sizeof(h));
        int st = 0;
        if (n < 8) st = PILC_ST_TRUNCATED;
        else if (b[0] != 'P' || b[1] != 'I' || b[2] != 'L' || b[3] != 'C') st = PILC_ST_BAD_MAGIC;
        else if (b[4] != 1) {
            st = PILC_ST_BAD_VERSION;
            h.aux = b[4];
        }
        if (!st) {
            // blob buffers are padded by 16 bytes (pilc.h): vector reads
            const uint32_t crc = warp_crc32_fast(&cc, &sl, mt, b, n - 4);
            if (crc != rd_u32(b + n - 4)) st = PILC_ST_CRC;
        }
        // sequential structure walk (lane 0), mirroring _Reader.take
        uint64_t off = 5;
        auto need = [&](uint64_t k) { return off + k <= n; };
        if (!st && lane == 0) {
            if (!need(4)) st = PILC_ST_TRUNCATED;
            if (!st) {
                h.backend = b[5];
                h.M = b[6];
                h.pad_rule = b[7];
                h.flags = b[8];
                off = 9;
                if (h.backend > 1) {
                    st = PILC_ST_BAD_BACKEND;
                    h.aux = h.backend;
                } else if (h.M < 10 || h.M > 12) st = PILC_ST_BAD_M;
                else if (h.pad_rule != 0) st = PILC_ST_BAD_PAD;
                else if ((h.flags & ~0x81u) || ((h.flags & 0x80u) && h.backend != 1)) st = PILC_ST_BAD_FLAGS;  // 0x80: fast decoder (vqvae only)
            }
            if (!st) {
                if (!need(12)) st = PILC_ST_TRUNCATED;
                else {
                    h.width = rd_u32(b + 9);
                    h.height = rd_u32(b + 13);
                    h.lanes = rd_u16(b + 17);
                    h.static_d = rd_u16(b + 19);
                    off = 21;
                    if (h.width < 1 || h.height < 1 || h.lanes < 1) st = PILC_ST_BAD_DIMS;
                }
            }
            if (!st) {
                if (n - off < 2) st = PILC_ST_GRID_TRUNC;
                else {
                    h.D = rd_u16(b + off);
                    if (off + 2 + 8ull * h.D > n) st = PILC_ST_GRID_TRUNC;
                    else off += 2 + 8ull * h.D;
                }
            }
            // ScaleGrid validation (logistic.py:52-64), same IEEE f64 ops
            if (!st) {
                const uint8_t *g = b + 23;
                const int D = h.D;
                if (D < 1) st = PILC_ST_GRID_EMPTY;
                for (int k = 0; !st && k < D; ++k) {
                    const double v = __longlong_as_double((long long)rd_u64(g + 8 * k));
                    if (!isfinite(v) || v <= 0.0) st = PILC_ST_GRID_VALUE;
                }
                for (int k = 1; !st && k < D; ++k) {
                    const double a0 = __longlong_as_double((long long)rd_u64(g + 8 * (k - 1)));
                    const double a1 = __longlong_as_double((long long)rd_u64(g + 8 * k));
                    if (!(a1 - a0 > 0.0)) st = PILC_ST_GRID_ORDER;
                }
                if (!st && D > 2) {
                    const double r0 = __longlong_as_double((long long)rd_u64(g + 8)) /
                                      __longlong_as_double((long long)rd_u64(g));
                    double mx = 0.0;
                    for (int k = 1; k + 1 < D; ++k) {
                        const double r = __longlong_as_double((long long)rd_u64(g + 8 * (k + 1))) /
                                         __longlong_as_double((long long)rd_u64(g + 8 * k));
                        mx = fmax(mx, fabs(r - r0));
                    }
                    if (mx > 1e-9 * r0) st = PILC_ST_GRID_GEOM;
                }
                uint32_t c = 0xFFFFFFFFu;
                for (int k = 0; k < 2 + 8 * D; ++k) c = cc.tab[(c ^ b[21 + k]) & 0xFF] ^ (c >> 8);
                h.grid_crc = c ^ 0xFFFFFFFFu;
            }
            if (!st && h.static_d >= h.D) st = PILC_ST_STATIC_D;
            if (!st) {
                if (!need(8)) st = PILC_ST_TRUNCATED;
                else {
                    h.params_hash_off = (uint32_t)off;
                    off += 8;
                }
            }
            const uint32_t L = h.lanes;
            if (!st && h.backend == 1) {
                if (!need(8)) st = PILC_ST_TRUNCATED;
                else {
                    h.model_hash_off = (uint32_t)off;
                    off += 8;
                }
                if (!st) {
                    if (!need(4 + 4ull * L + 2ull * L)) st = PILC_ST_TRUNCATED;
                    else {
                        h.idx_table_off = (uint32_t)off;
                        const uint32_t tot = rd_u32(b + off);
                        uint64_t s = 0;
                        for (uint32_t l = 0; l < L; ++l) s += rd_u32(b + off + 4 + 4 * l);
                        h.idx_bytes = s;
                        off += 4 + 6ull * L;
                        if (s != tot) st = PILC_ST_IDX_LENS;
                    }
                }
            }
            if (!st) {
                if (!need(4 + 6ull * L)) st = PILC_ST_TRUNCATED;
                else {
                    h.res_table_off = (uint32_t)off;
                    const uint32_t tot = rd_u32(b + off);
                    uint64_t s = 0;
                    for (uint32_t l = 0; l < L; ++l) s += rd_u32(b + off + 4 + 4 * l);
                    h.res_bytes = s;
                    off += 4 + 6ull * L;
                    if (s != tot) st = PILC_ST_RES_LENS;
                }
            }
            if (!st && (h.flags & 1)) {
                if (!need(4)) st = PILC_ST_TRUNCATED;
                else {
                    h.sched_crc = rd_u32(b + off);
                    off += 4;
                }
            }
            if (!st) {
                h.payload_off = (uint32_t)off;
                if (off + h.idx_bytes + h.res_bytes + 4 != n) st = PILC_ST_PAYLOAD_LEN;
            }
            // container.py:288-304: predictor hash, then model hash
            if (!st && rd_u64(b + h.params_hash_off) != params_hash) st = PILC_ST_PARAMS_HASH;
            if (!st && h.backend == 1 && has_model && rd_u64(b + h.model_hash_off) != model_hash)
                st = PILC_ST_MODEL_HASH;
        }
        st = __shfl_sync(0xffffffffu, st, 0);
        if (lane == 0) {
            h.status = st;
            hdr[i] = h;
        }
    }
}

// ---- lanes (container.py:261-271, bits.py:75-85) -------------------------
__global__ void lanes_kernel(const uint8_t *__restrict__ buf, const uint64_t *__restrict__ blob_off,
                             const pilc_header *__restrict__ hdr, const int64_t *__restrict__ blob_idx,
                             int64_t n_group, int lanes, int stream_id, int expect_M, int expect_D,
                             uint64_t *__restrict__ lane_off, uint32_t *__restrict__ nbits,
                             uint16_t *__restrict__ states, uint8_t *__restrict__ lane_status) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t g = (int64_t)blockIdx.x * kWarps + warp; g < n_group;
         g += (int64_t)gridDim.x * kWarps) {
        const int64_t bi = blob_idx[g];
        const pilc_header h = hdr[bi];
        const uint8_t *b = buf + blob_off[bi];
        const uint32_t M = h.M;
        const uint32_t tab = stream_id == 0 ? h.idx_table_off : h.res_table_off;
        uint64_t start = h.payload_off + (stream_id == 0 ? 0 : h.idx_bytes);
        // blobs whose lane count / precision / grid size differ from the
        // group's (a speculated group, container.py) are rejected here, so the
        // coder never indexes its tables with another blob's parameters
        const bool ok = h.status == 0 && tab != 0 && h.lanes == (uint32_t)lanes &&
                        (expect_M == 0 || h.M == (uint32_t)expect_M) && (expect_D == 0 || h.D == (uint32_t)expect_D);
        // lane wire sizes -> running offsets, 32 lanes at a time
        for (int l0 = 0; l0 < lanes; l0 += 32) {
            const int l = l0 + lane;
            uint32_t wsz = 0;
            if (ok && l < lanes) wsz = rd_u32(b + tab + 4 + 4 * l);
            // inclusive scan of wsz over the warp
            uint64_t inc = wsz;
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t v = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += v;
            }
            const uint64_t my = start + inc - wsz;
            if (l < lanes) {
                const int64_t k = g * lanes + l;
                uint8_t st = 0;
                uint64_t nb = 0;
                uint32_t s = 0;
                if (!ok) st = PILC_ST_TRUNCATED;
                else if (wsz < 8) st = PILC_ST_LANE_HDR;
                else {
                    nb = rd_u64(b + my);
                    const uint64_t need = 8 + ((nb + 7) >> 3);
                    if (nb >= (1ull << 32) || need > wsz) st = need > wsz ? PILC_ST_LANE_TRUNC : PILC_ST_LANE_LEN;
                    else if (need != wsz) st = PILC_ST_LANE_LEN;
                }
                if (ok) s = rd_u16(b + tab + 4 + 4 * lanes + 2 * l);
                if (!st && !(s >= (1u << M) && s < (2u << M))) st = PILC_ST_STATE_RANGE;
                lane_off[k] = blob_off[bi] + my + 8;
                nbits[k] = (uint32_t)nb;
                states[k] = (uint16_t)s;
                lane_status[k] = st;
            }
            start += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
}

__global__ void __launch_bounds__(32 * kWarps) crc_kernel(const uint8_t *__restrict__ buf,
                                                          const uint64_t *__restrict__ off,
                                                          const uint64_t *__restrict__ len, int64_t n,
                                                          uint32_t *__restrict__ out, CrcConsts ccv) {
    __shared__ CrcConsts cc;
    __shared__ uint8_t stage[kWarps][kStage];
    load_crc_consts(&cc, ccv);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t i = (int64_t)blockIdx.x * kWarps + warp; i < n; i += (int64_t)gridDim.x * kWarps) {
        const uint32_t c = warp_crc32(&cc, buf + off[i], len[i], stage[warp]);
        if (lane == 0) out[i] = c;
    }
}

__global__ void __launch_bounds__(32 * kWarps) sched_crc_kernel(const uint8_t *__restrict__ dsched,
                                                                const uint16_t *__restrict__ d_img,
                                                                int64_t n_img, int64_t n_sym,
                                                                uint32_t *__restrict__ out, CrcConsts ccv) {
    __shared__ CrcConsts cc;
    __shared__ uint8_t stage[kWarps][kStage];
    load_crc_consts(&cc, ccv);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t i = (int64_t)blockIdx.x * kWarps + warp; i < n_img; i += (int64_t)gridDim.x * kWarps) {
        const uint32_t c = sched_crc_warp(&cc, dsched ? dsched + i * n_sym : nullptr,
                                          d_img ? d_img[i] : 0u, n_sym, stage[warp]);
        if (lane == 0) out[i] = c;
    }
}

unsigned warp_grid(int64_t n) {
    int64_t blocks = ceil_div64(n, kWarps);
    const int64_t cap = (int64_t)sm_count() * 16;
    return (unsigned)(blocks > cap ? cap : (blocks < 1 ? 1 : blocks));
}

// ---- batch summary --------------------------------------------------------
// One block: counts headers with a nonzero status, checks that every header
// shares blob 0's grouping key (dims, backend, M, lanes, flags, D, grid crc)
// and copies blob 0's header and grid bytes, so the host decides the common
// one-group case from one small read instead of every header.
__global__ void summary_kernel(const uint8_t *__restrict__ buf, const uint64_t *__restrict__ blob_off,
                               const pilc_header *__restrict__ hdr, int64_t n, pilc_summary *__restrict__ out) {
    __shared__ int s_bad[32], s_diff[32];
    const pilc_header h0 = hdr[0];
    int bad = 0, diff = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const pilc_header h = hdr[i];
        bad += h.status != 0;
        diff |= h.width != h0.width || h.height != h0.height || h.backend != h0.backend || h.M != h0.M ||
                h.lanes != h0.lanes || h.flags != h0.flags || h.D != h0.D || h.grid_crc != h0.grid_crc;
    }
    for (int o = 16; o; o >>= 1) {
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
        diff |= __shfl_xor_sync(0xffffffffu, diff, o);
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        s_bad[w] = bad;
        s_diff[w] = diff;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int b = 0, d = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            b += s_bad[k];
            d |= s_diff[k];
        }
        out->n_bad = b;
        out->uniform = !d;
        out->h0 = h0;
    }
    // grid bytes of blob 0: u16 D + D f64 at offset 21 (valid when its status is OK)
    const int nb = h0.status == 0 ? 2 + 8 * (int)h0.D : 0;
    for (int k = threadIdx.x; k < nb && k < (int)sizeof(out->grid); k += blockDim.x) out->grid[k] = buf[blob_off[0] + 21 + k];
}

}  // namespace

extern "C" int pilc_static_scale(const uint8_t *res, int64_t n_img, int64_t n_sym, const double *log2_grid,
                                 int32_t D, uint16_t *d_img, void *stream) {
    if (n_img < 0 || n_sym < 1 || D < 1 || D > 65535 || !log2_grid) return PILC_E_ARG;
    if (n_img == 0) return PILC_OK;
    if (n_img > 0x7FFFFFFF) return PILC_E_ARG;
    cudaStream_t s = as_stream(stream);
    {
        ProfScope _ps(PROF_STATIC_SCALE, s, (double)n_img * n_sym);
        static_scale_kernel<<<(unsigned)n_img, 256, 0, s>>>(res, n_sym, log2_grid, D, d_img);
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

extern "C" int pilc_container_sizes(const uint32_t *idx_nbits, const uint32_t *res_nbits, int64_t n_img,
                                    int32_t lanes, int64_t fixed_bytes, uint64_t *sizes, uint64_t *blob_off,
                                    void *stream) {
    if (n_img < 0 || lanes < 1 || !res_nbits || !blob_off || (n_img && !sizes)) return PILC_E_ARG;
    cudaStream_t s = as_stream(stream);
    if (n_img == 0) {
        cudaMemsetAsync(blob_off, 0, sizeof(uint64_t), s);
        PILC_CHECK_LAUNCH();
        return PILC_OK;
    }
    {
        ProfScope _ps(PROF_SIZES, s, (double)n_img);
        blob_sizes_kernel<<<warp_grid(n_img), 32 * kWarps, 0, s>>>(idx_nbits, res_nbits, n_img, lanes,
                                                                   fixed_bytes, sizes);
        scan_kernel<<<1, 1024, 0, s>>>(sizes, n_img, blob_off);
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

extern "C" int pilc_container_pack(const uint8_t *tmpl, int32_t template_len, const uint16_t *d_img,
                                   const uint8_t *dsched, int32_t sched_check, int64_t n_img, int64_t n_sym,
                                   int32_t lanes, const uint32_t *idx_scratch, int64_t idx_cap,
                                   const uint32_t *idx_nbits, const uint16_t *idx_states,
                                   const uint32_t *res_scratch, int64_t res_cap, const uint32_t *res_nbits,
                                   const uint16_t *res_states, const uint64_t *blob_off, uint8_t *out,
                                   void *stream) {
    if (n_img < 0 || lanes < 1 || template_len < 21 || !tmpl || !res_nbits) return PILC_E_ARG;
    if (n_img == 0) return PILC_OK;
    cudaStream_t s = as_stream(stream);
    PackArgs a{d_img,     dsched,      sched_check, n_img,      n_sym,      lanes,
               idx_scratch, idx_cap,   idx_nbits,   idx_states, res_scratch, res_cap,
               res_nbits, res_states,  blob_off,    out,        tmpl,       template_len};
    {
        ProfScope _ps(PROF_PACK, s, (double)n_img);
        const uint32_t *mt = crc_mul_tables();
        if (!mt) return PILC_E_CUDA;
        pack_kernel<<<warp_grid(n_img), 32 * kWarps, 0, s>>>(a, crc_consts(), mt);
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

extern "C" int pilc_container_parse(const uint8_t *buf, const uint64_t *blob_off, int64_t n_blob,
                                    uint64_t params_hash, uint64_t model_hash, int32_t has_model,
                                    pilc_header *hdr, void *stream) {
    if (n_blob < 0 || !blob_off || !hdr) return PILC_E_ARG;
    if (n_blob == 0) return PILC_OK;
    const uint32_t *mt = crc_mul_tables();
    if (!mt) return PILC_E_CUDA;
    {
        ProfScope _ps(PROF_PARSE, as_stream(stream), (double)n_blob);
        parse_kernel<<<warp_grid(n_blob), 32 * kWarps, 0, as_stream(stream)>>>(
            buf, blob_off, n_blob, params_hash, model_hash, has_model, hdr, crc_consts(), mt);
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

extern "C" int pilc_container_summary(const uint8_t *buf, const uint64_t *blob_off, const pilc_header *hdr,
                                      int64_t n_blob, pilc_summary *out, void *stream) {
    if (n_blob < 1 || !buf || !blob_off || !hdr || !out) return PILC_E_ARG;
    {
        ProfScope _ps(PROF_PARSE, as_stream(stream), (double)n_blob);
        summary_kernel<<<1, 1024, 0, as_stream(stream)>>>(buf, blob_off, hdr, n_blob, out);
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

extern "C" int pilc_container_lanes(const uint8_t *buf, const uint64_t *blob_off,
                                    const pilc_header *hdr, const int64_t *blob_idx, int64_t n_group,
                                    int32_t lanes, int32_t stream_id, int32_t expect_M, int32_t expect_D,
                                    uint64_t *lane_off, uint32_t *nbits, uint16_t *states, uint8_t *lane_status,
                                    void *stream) {
    if (n_group < 0 || lanes < 1 || (stream_id != 0 && stream_id != 1)) return PILC_E_ARG;
    if (n_group == 0) return PILC_OK;
{
        ProfScope _ps(PROF_LANES, as_stream(stream), (double)n_group * lanes);
        lanes_kernel<<<warp_grid(n_group), 32 * kWarps, 0, as_stream(stream)>>>(
        buf, blob_off, hdr, blob_idx, n_group, lanes, stream_id, expect_M, expect_D, lane_off, nbits, states,
        lane_status);
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

extern "C" int pilc_crc32(const uint8_t *buf, const uint64_t *off, const uint64_t *len, int64_t n,
                          uint32_t *crc, void *stream) {
    if (n < 0) return PILC_E_ARG;
    if (n == 0) return PILC_OK;
{
        ProfScope _ps(PROF_CRC, as_stream(stream), (double)n);
        crc_kernel<<<warp_grid(n), 32 * kWarps, 0, as_stream(stream)>>>(buf, off, len, n, crc, crc_consts());
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

extern "C" int pilc_sched_crc(const uint8_t *dsched, const uint16_t *d_img, int64_t n_img,
                              int64_t n_sym, uint32_t *crc, void *stream) {
    if (n_img < 0 || n_sym < 0) return PILC_E_ARG;
    if (n_img == 0) return PILC_OK;
{
        ProfScope _ps(PROF_SCHED_CRC, as_stream(stream), (double)n_img * n_sym);
        sched_crc_kernel<<<warp_grid(n_img), 32 * kWarps, 0, as_stream(stream)>>>(dsched, d_img, n_img, n_sym,
                                                                             crc, crc_consts());
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}
