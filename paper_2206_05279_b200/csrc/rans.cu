// Interleaved table-driven rANS lanes on sm_100a.
//
// Reference: tables.interleaved_encode / interleaved_decode
// (tables.py:202-274) over _kernels.encode_lane / decode_lane
// (_kernels.py:20-63). The reference pushes and pops one bit per inner loop
// iteration; here a lane keeps a 64-bit reservoir: encode ORs the low b bits
// of the state in at the current bit position and flushes 32-bit words,
// decode extracts the top b bits below the read position from a 64-bit
// window of aligned words. Both are byte-identical to the bit loops (the
// lane payload is the little-endian integer sum (S_i & (2^b_i - 1)) << pos_i).
//
// One thread per (image, lane). Coder tables live in shared memory when
// they fit (D*X*4 B encode, D*2^M*4 B decode: 8 KB / 128 KB at D=8, M=12),
// else they are read through L1 from global memory.

#include "common.cuh"

namespace {

constexpr int kThreads = 128;
constexpr int kSmemTableMax = 160 * 1024;  // + 32 KB cp.async ring at 512 threads

__device__ __forceinline__ int lane_count(int64_t n_sym, int lanes, int l) {
    return l < n_sym ? (int)((n_sym - l + lanes - 1) / lanes) : 0;
}

// Byte j of a 16-byte vector.
__device__ __forceinline__ uint32_t vbyte(const uint4 &v, int j) {
    const uint32_t w = j < 4 ? v.x : (j < 8 ? v.y : (j < 12 ? v.z : v.w));
    return (w >> (8 * (j & 3))) & 0xFFu;
}

struct EncState {
    uint32_t state;
    uint64_t acc;
    int nacc;
    uint32_t words;
};

__device__ __forceinline__ void enc_step(EncState &e, const uint32_t *tab, int X, int M, uint32_t d,
                                         uint32_t x, uint32_t *out) {
    const uint32_t t = tab[d * X + x];
    const uint32_t b = ((t & 0xFFFFu) + e.state) >> M;
    e.acc |= (uint64_t)(e.state & ((1u << b) - 1u)) << e.nacc;
    e.nacc += b;
    if (e.nacc >= 32) {
        out[e.words++] = (uint32_t)e.acc;
        e.acc >>= 32;
        e.nacc -= 32;
    }
    e.state = (e.state >> b) + (t >> 16);
}

__global__ void __launch_bounds__(kThreads) rans_encode_kernel(
    const uint8_t *__restrict__ syms, const uint8_t *__restrict__ shift,
    const uint8_t *__restrict__ dsched, const uint16_t *__restrict__ d_img,
    int64_t n_img, int64_t n_sym, int lanes, const uint32_t *__restrict__ enc_tab_g,
    int D, int X, int M, int tab_in_smem, uint32_t *__restrict__ scratch,
    int64_t lane_cap, uint32_t *__restrict__ nbits, uint16_t *__restrict__ states) {
    extern __shared__ uint32_t s_tab[];
    const uint32_t *tab = enc_tab_g;
    if (tab_in_smem) {
        const int n = D * X;
        for (int i = threadIdx.x; i < n; i += blockDim.x) s_tab[i] = enc_tab_g[i];
        __syncthreads();
        tab = s_tab;
    }
    const int64_t total = n_img * lanes;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t img = k / lanes;
        const int l = (int)(k - img * lanes);
        const int cnt = lane_count(n_sym, lanes, l);
        const int64_t base = img * n_sym + l;
        const uint32_t dconst = d_img ? d_img[img] : 0u;
        uint32_t *out = scratch + k * lane_cap;
        EncState e{1u << M, 0, 0, 0};
        auto scalar = [&](int i) {
            const int64_t pos = base + (int64_t)i * lanes;
            uint32_t x = syms[pos];
            if (shift) x = (x - shift[pos] + 128u) & 0xFFu;
            enc_step(e, tab, X, M, dsched ? dsched[pos] : dconst, x, out);
        };
        int i = cnt - 1;
        if (lanes == 1) {
            // reverse order; 16-byte vector loads over aligned chunks
            for (; i >= 0 && ((base + i + 1) & 15); --i) scalar(i);
            const uint4 z4 = make_uint4(0, 0, 0, 0);
            uint4 sv = z4, hv = z4, dv = z4;
            if (i >= 15) {
                const int64_t p0 = base + i - 15;
                sv = *reinterpret_cast<const uint4 *>(syms + p0);
                if (shift) hv = *reinterpret_cast<const uint4 *>(shift + p0);
                if (dsched) dv = *reinterpret_cast<const uint4 *>(dsched + p0);
            }
            for (; i >= 15; i -= 16) {
                uint4 sn = z4, hn = z4, dn = z4;  // prefetch the previous chunk
                if (i >= 31) {
                    const int64_t pn = base + i - 31;
                    sn = *reinterpret_cast<const uint4 *>(syms + pn);
                    if (shift) hn = *reinterpret_cast<const uint4 *>(shift + pn);
                    if (dsched) dn = *reinterpret_cast<const uint4 *>(dsched + pn);
                }
#pragma unroll
                for (int j = 15; j >= 0; --j) {
                    uint32_t x = vbyte(sv, j);
                    if (shift) x = (x - vbyte(hv, j) + 128u) & 0xFFu;
                    enc_step(e, tab, X, M, dsched ? vbyte(dv, j) : dconst, x, out);
                }
                sv = sn;
                hv = hn;
                dv = dn;
            }
        }
        // strided lanes: the next (lower) symbol's inputs are fetched one ahead
        if (i >= 0) {
            int64_t pos = base + (int64_t)i * lanes;
            uint32_t xn = syms[pos], hn = shift ? shift[pos] : 0u, dn = dsched ? dsched[pos] : dconst;
            for (; i >= 0; --i, pos -= lanes) {
                const uint32_t xc = xn, hc = hn, dc = dn;
                if (i > 0) {
                    xn = syms[pos - lanes];
                    if (shift) hn = shift[pos - lanes];
                    if (dsched) dn = dsched[pos - lanes];
                }
                enc_step(e, tab, X, M, dc, shift ? ((xc - hc + 128u) & 0xFFu) : xc, out);
            }
        }
        if (e.nacc) out[e.words] = (uint32_t)e.acc;
        nbits[k] = e.words * 32u + (uint32_t)e.nacc;
        states[k] = (uint16_t)e.state;
    }
}

// Backward bit reader, 32-bit arithmetic relative to the lane's first
// 16-byte chunk. A 64-bit window over aligned words is refilled one word at a
// time from the current 16-byte chunk `cur` (registers). Chunks arrive
// through a per-thread ring of kRing slots in shared memory filled with
// cp.async three chunks (~30 symbols) ahead: unlike a register prefetch, a
// pending cp.async never stalls an instruction until cp.async.wait_group
// asks for that very chunk, so the state chain does not wait on memory.
// Chunks stay inside [first chunk, last chunk] of the lane; buffers are padded
// by 16 bytes (pilc.h) so the last chunk is always readable.
constexpr int kRing = 4;

struct BitReader {
    const uint4 *base4;  // chunk 0 = the lane's first chunk
    uint4 *ring;         // this thread's kRing slots (stride = blockDim.x)
    int stride;
    int A, start, wl, cq, hi_c;
    uint64_t win;
    uint4 cur;

    __device__ __forceinline__ void issue(int c) {
        if (c >= 0 && c <= hi_c) {
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + (c & (kRing - 1)) * stride);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(base4 + c) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    __device__ __forceinline__ static uint32_t pick(const uint4 &v, int k) {
        return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
    }
    __device__ __forceinline__ uint4 direct(int c) const {
        return (c >= 0 && c <= hi_c) ? __ldg(base4 + c) : make_uint4(0, 0, 0, 0);
    }
    __device__ __forceinline__ void init(const uint4 *lane_base4, uint4 *my_ring, int ring_stride, int start_bit,
                                         uint32_t nb) {
        base4 = lane_base4;
        ring = my_ring;
        stride = ring_stride;
        start = start_bit;                               // 0..127
        hi_c = nb ? (int)((start_bit + nb - 1) >> 7) : -1;
        A = start_bit + (int)nb;
        wl = ((A - 1) >> 5) - 1;                         // window = bits [32 wl, 32 wl + 64)
        const int c_top = (wl + 1) >> 2, c_lo = wl >> 2;
        const uint4 a = direct(c_top);
        const uint4 b = c_lo == c_top ? a : direct(c_lo);
        win = ((uint64_t)pick(a, (wl + 1) & 3) << 32) | pick(b, wl & 3);
        cq = (wl - 1) >> 2;                              // chunk of the next word to bring in
        cur = direct(cq);
        issue(cq - 1);
        issue(cq - 2);
        issue(cq - 3);
    }
    // false on underflow
    __device__ __forceinline__ bool take(uint32_t b, uint32_t &v) {
        const int lo = A - (int)b;
        if (lo < start) return false;
        if (lo < (wl << 5)) {
            --wl;
            if ((wl >> 2) != cq) {
                --cq;
                asm volatile("cp.async.wait_group 2;" ::: "memory");
                cur = (cq >= 0 && cq <= hi_c) ? ring[(cq & (kRing - 1)) * stride] : make_uint4(0, 0, 0, 0);
                issue(cq - 3);
            }
            win = (win << 32) | pick(cur, wl & 3);
        }
        v = (uint32_t)(win >> (lo - (wl << 5))) & ((1u << b) - 1u);
        A = lo;
        return true;
    }
};

template <bool SMEM>
__global__ void __launch_bounds__(512) rans_decode_kernel(
    const uint8_t *__restrict__ buf, const uint64_t *__restrict__ lane_off,
    const uint32_t *__restrict__ nbits_a, const uint16_t *__restrict__ states,
    const uint8_t *__restrict__ dsched, const uint16_t *__restrict__ d_img, int64_t n_img,
    int64_t n_sym, int lanes, const uint32_t *__restrict__ dec_tab_g, int D, int M,
    const uint8_t *__restrict__ unshift, uint8_t *__restrict__ out,
    uint8_t *__restrict__ lane_status) {
    extern __shared__ __align__(16) uint32_t s_tab[];
    __shared__ __align__(8) uint64_t tbar;
    if constexpr (SMEM) {
        // one bulk copy of the whole table (up to 160 KB)
        const uint32_t bytes = (uint32_t)(D << M) * 4u;
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&tbar);
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    (uint32_t)__cvta_generic_to_shared(s_tab)),
                "l"(dec_tab_g), "r"(bytes), "r"(bar)
                : "memory");
        }
        __syncthreads();
        asm volatile(
            "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
            "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(bar)
            : "memory");
    }
    uint4 *ring_base = reinterpret_cast<uint4 *>(s_tab + (SMEM ? (D << M) : 0));
    uint4 *my_ring = ring_base + threadIdx.x;
    const uint32_t T = 1u << M;
    auto lookup = [&](uint32_t d, uint32_t st) -> uint32_t {
        const uint32_t i = d * T + (st - T);
        if constexpr (SMEM) return s_tab[i];
        else return __ldg(dec_tab_g + i);
    };
    const int64_t total = n_img * lanes;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (lane_status[k]) continue;
        const int64_t img = lanes == 1 ? k : k / lanes;
        const int l = (int)(k - img * lanes);
        const int cnt = lane_count(n_sym, lanes, l);
        const int64_t sbase = img * n_sym + l;
        const uint32_t dconst = d_img ? d_img[img] : 0u;
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(buf) + lane_off[k];
        BitReader br;
        br.init(reinterpret_cast<const uint4 *>(a0 & ~(uintptr_t)15), my_ring, (int)blockDim.x, (int)(a0 & 15) * 8,
                nbits_a[k]);
        uint32_t state = states[k];
        uint8_t st = 0;
        // one symbol: the decoded (optionally un-recentred) byte
        auto step = [&](uint32_t d, uint32_t sh) -> uint32_t {
            const uint32_t e = lookup(d, state);
            uint32_t v = 0;
            if (!br.take((e >> 8) & 0xFFu, v)) st = PILC_ST_UNDERFLOW;
            state = (e >> 16) + v;
            return unshift ? ((e + sh + 128u) & 0xFFu) : (e & 0xFFu);  // (x + shift - 128) mod 256
        };
        int i = 0;
        if (lanes == 1) {
            for (; i < cnt && ((sbase + i) & 15) && !st; ++i) {
                const int64_t pos = sbase + i;
                out[pos] = (uint8_t)step(dsched ? dsched[pos] : dconst, unshift ? unshift[pos] : 0u);
            }
            // 16-symbol chunks; the next chunk's d / shift vectors are loaded
            // one chunk ahead
            const uint4 z4 = make_uint4(0, 0, 0, 0);
            uint4 dv = z4, hv = z4;
            if (i + 16 <= cnt) {
                if (dsched) dv = *reinterpret_cast<const uint4 *>(dsched + sbase + i);
                if (unshift) hv = *reinterpret_cast<const uint4 *>(unshift + sbase + i);
            }
            for (; i + 16 <= cnt && !st; i += 16) {
                const int64_t p0 = sbase + i;  // 16-aligned
                uint4 dn = z4, hn = z4;
                if (i + 32 <= cnt) {
                    if (dsched) dn = *reinterpret_cast<const uint4 *>(dsched + p0 + 16);
                    if (unshift) hn = *reinterpret_cast<const uint4 *>(unshift + p0 + 16);
                }
                uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    o[j >> 2] |= step(dsched ? vbyte(dv, j) : dconst, vbyte(hv, j)) << (8 * (j & 3));
                *reinterpret_cast<uint4 *>(out + p0) = make_uint4(o[0], o[1], o[2], o[3]);
                dv = dn;
                hv = hn;
            }
        }
        // strided lanes: the next symbol's d / shift are fetched one ahead
        uint32_t dn = 0, hn = 0;
        if (i < cnt) {
            const int64_t pos = sbase + (int64_t)i * lanes;
            dn = dsched ? dsched[pos] : dconst;
            hn = unshift ? unshift[pos] : 0u;
        }
        for (; i < cnt && !st; ++i) {
            const int64_t pos = sbase + (int64_t)i * lanes;
            const uint32_t dc = dn, hc = hn;
            if (i + 1 < cnt) {
                dn = dsched ? dsched[pos + lanes] : dconst;
                hn = unshift ? unshift[pos + lanes] : 0u;
            }
            out[pos] = (uint8_t)step(dc, hc);
        }
        if (!st && (state != T || br.A != br.start)) st = PILC_ST_END_STATE;
        lane_status[k] = st;
        asm volatile("cp.async.wait_all;" ::: "memory");  // ring slots are reused by the next lane
    }
}

}  // namespace

extern "C" int pilc_rans_encode(const uint8_t *syms, const uint8_t *shift, const uint8_t *dsched,
                                const uint16_t *d_img, int64_t n_img, int64_t n_sym,
                                int32_t lanes, const uint32_t *enc_tab, int32_t D, int32_t X,
                                int32_t M, uint32_t *scratch, int64_t lane_cap, uint32_t *nbits,
                                uint16_t *states, void *stream) {
    if (n_img < 0 || n_sym < 0 || lanes < 1 || M < 2 || M > 12 || D < 1 || X < 1 || X > 256)
        return PILC_E_ARG;
    const int64_t per_lane = ceil_div64(n_sym, lanes);
    if (lane_cap < (per_lane * M + 31) / 32 + 1) return PILC_E_ARG;
    if (n_img == 0) return PILC_OK;
    const int64_t tab_bytes = (int64_t)D * X * 4;
    const int in_smem = tab_bytes <= kSmemTableMax;
    const size_t smem = in_smem ? (size_t)tab_bytes : 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(rans_encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t total = n_img * lanes;
    int64_t blocks = ceil_div64(total, kThreads);
    const int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
{
        ProfScope _ps(PROF_RANS_ENC, as_stream(stream), (double)n_img * n_sym);
        rans_encode_kernel<<<(unsigned)blocks, kThreads, smem, as_stream(stream)>>>(
        syms, shift, dsched, d_img, n_img, n_sym, lanes, enc_tab, D, X, M, in_smem, scratch,
        lane_cap, nbits, states);
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}

extern "C" int pilc_rans_decode(const uint8_t *buf, const uint64_t *lane_off, const uint32_t *nbits,
                                const uint16_t *states, const uint8_t *dsched, const uint16_t *d_img,
                                int64_t n_img, int64_t n_sym, int32_t lanes, const uint32_t *dec_tab, int32_t D,
                                int32_t M, const uint8_t *unshift, uint8_t *out, uint8_t *lane_status,
                                void *stream) {
    if (n_img < 0 || n_sym < 0 || lanes < 1 || M < 2 || M > 12 || D < 1) return PILC_E_ARG;
    if (n_img == 0) return PILC_OK;
    const int64_t tab_bytes = ((int64_t)D << M) * 4;
    const int in_smem = tab_bytes <= kSmemTableMax;
    const int64_t total = n_img * lanes;
    // one table copy per block; per_sm resident blocks fit in shared memory.
    // Spread the lanes over every SM: threads per block = lanes / (SMs x
    // per_sm), rounded to warps, in [32, 512].
    const int64_t per_sm = in_smem ? (tab_bytes > 96 * 1024 ? 1 : (tab_bytes > 48 * 1024 ? 2 : 8)) : 16;
    const int64_t slots = (int64_t)sm_count() * per_sm;
    int64_t threads = ceil_div64(ceil_div64(total, slots), 32) * 32;
    threads = threads < 32 ? 32 : (threads > 512 ? 512 : threads);
    int64_t blocks = ceil_div64(total, threads);
    if (blocks > slots) blocks = slots;
    const size_t smem = (in_smem ? (size_t)tab_bytes : 0) + (size_t)kRing * 16 * (size_t)threads;
    {
        ProfScope _ps(PROF_RANS_DEC, as_stream(stream), (double)n_img * n_sym);
        if (in_smem) {
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(rans_decode_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            rans_decode_kernel<true><<<(unsigned)blocks, (unsigned)threads, smem, as_stream(stream)>>>(
                buf, lane_off, nbits, states, dsched, d_img, n_img, n_sym, lanes, dec_tab, D, M, unshift, out,
                lane_status);
        } else {
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(rans_decode_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            rans_decode_kernel<false><<<(unsigned)blocks, (unsigned)threads, smem, as_stream(stream)>>>(
                buf, lane_off, nbits, states, dsched, d_img, n_img, n_sym, lanes, dec_tab, D, M, unshift, out,
                lane_status);
        }
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}
