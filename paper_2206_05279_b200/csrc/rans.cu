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

// ---- encoder --------------------------------------------------------------
// The state chain per symbol is four integer ops (b = (delta + S) >> M;
// S = (S >> b) + phi); the table word of every symbol depends only on (d, x)
// and is fetched ahead of the chain. The bit output is branch-free: a 64-bit
// accumulator, one predicated 32-bit store when 32 bits are complete.
struct EncState {
    uint32_t S;
    uint64_t acc;
    uint32_t nacc;
    uint32_t *wp;  // next output word
};

__device__ __forceinline__ void st_if(uint32_t *p, uint32_t v, bool on) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.u32 [%0], %1;\n\t}\n" ::"l"(p), "r"(v),
        "r"(on ? 1u : 0u)
        : "memory");
}

// one symbol's bits into the accumulator, no flush (nacc stays < 64 for two
// symbols after a flush: < 32 + 2 x 12)
__device__ __forceinline__ void enc_bits(EncState &e, uint32_t t, int M) {
    const uint32_t b = ((t & 0xFFFFu) + e.S) >> M;
    e.acc |= (uint64_t)(e.S & ((1u << b) - 1u)) << e.nacc;
    e.nacc += b;
    e.S = (e.S >> b) + (t >> 16);
}

// a complete 32-bit word out, branch-free (leaves nacc < 32)
__device__ __forceinline__ void enc_flush(EncState &e) {
    const bool f = e.nacc >= 32u;
    st_if(e.wp, (uint32_t)e.acc, f);
    e.wp += f ? 1 : 0;
    e.acc = f ? (e.acc >> 32) : e.acc;
    e.nacc -= f ? 32u : 0u;
}

__device__ __forceinline__ void enc_push(EncState &e, uint32_t t, int M) {
    enc_bits(e, t, M);
    enc_flush(e);
}

template <bool SMEM>
__global__ void __launch_bounds__(kThreads) rans_encode_kernel(
    const uint8_t *__restrict__ syms, const uint8_t *__restrict__ shift,
    const uint8_t *__restrict__ dsched, const uint16_t *__restrict__ d_img,
    int64_t n_img, int64_t n_sym, int lanes, const uint32_t *__restrict__ enc_tab_g,
    int D, int X, int M, uint32_t *__restrict__ scratch,
    int64_t lane_cap, uint32_t *__restrict__ nbits, uint16_t *__restrict__ states) {
    extern __shared__ uint32_t s_tab[];
    if constexpr (SMEM) {
        const int n = D * X;
        for (int i = threadIdx.x; i < n; i += blockDim.x) s_tab[i] = enc_tab_g[i];
        __syncthreads();
    }
    auto tab = [&](uint32_t i) -> uint32_t {
        if constexpr (SMEM) return s_tab[i];
        else return __ldg(enc_tab_g + i);
    };
    const int64_t total = n_img * lanes;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t img = k / lanes;
        const int l = (int)(k - img * lanes);
        const int cnt = lane_count(n_sym, lanes, l);
        const int64_t base = img * n_sym + l;
        const uint32_t dconst = d_img ? d_img[img] : 0u;
        uint32_t *out = scratch + k * lane_cap;
        EncState e{1u << M, 0, 0, out};
        auto word = [&](uint32_t x, uint32_t h, uint32_t d) -> uint32_t {
            if (shift) x = (x - h + 128u) & 0xFFu;
            return tab(d * X + x);
        };
        int i = cnt - 1;
        if (lanes == 1) {
            // reverse order; 16-byte vector loads over aligned chunks, the
            // previous chunk prefetched while this one is coded
            for (; i >= 0 && ((base + i + 1) & 15); --i) {
                const int64_t pos = base + i;
                enc_push(e, word(syms[pos], shift ? shift[pos] : 0u, dsched ? dsched[pos] : dconst), M);
            }
            // 16-symbol blocks, a register ring of two blocks: the inputs of
            // block j + 2 are requested as soon as block j is coded (~32
            // symbols ahead, longer than a DRAM round trip at this chain
            // length); two blocks per iteration keep the body in the
            // instruction cache
            const uint4 z4 = make_uint4(0, 0, 0, 0);
            auto ld = [&](int ii, uint4 &sv, uint4 &hv, uint4 &dv) {  // block with top symbol ii
                if (ii >= 15) {
                    const int64_t p0 = base + ii - 15;
                    sv = *reinterpret_cast<const uint4 *>(syms + p0);
                    if (shift) hv = *reinterpret_cast<const uint4 *>(shift + p0);
                    if (dsched) dv = *reinterpret_cast<const uint4 *>(dsched + p0);
                }
            };
            auto blk = [&](const uint4 &sv, const uint4 &hv, const uint4 &dv) {
                uint32_t t[16];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    t[j] = word(vbyte(sv, j), vbyte(hv, j), dsched ? vbyte(dv, j) : dconst);
#pragma unroll
                for (int j = 15; j >= 1; j -= 2) {  // one flush per two symbols
                    enc_bits(e, t[j], M);
                    enc_bits(e, t[j - 1], M);
                    enc_flush(e);
                }
            };
            uint4 s0 = z4, s1 = z4, h0 = z4, h1 = z4, d0 = z4, d1 = z4;
            ld(i, s0, h0, d0);
            ld(i - 16, s1, h1, d1);
            for (; i >= 31; i -= 32) {
                blk(s0, h0, d0);
                ld(i - 32, s0, h0, d0);
                blk(s1, h1, d1);
                ld(i - 48, s1, h1, d1);
            }
            if (i >= 15) {
                blk(s0, h0, d0);
                i -= 16;
            }
        }
        // strided lanes (symbol l + i L): the same two-block register ring as
        // above with 16 scalar loads per block -- consecutive lanes of a warp
        // read consecutive bytes, so every load is one coalesced request, and
        // block j + 2's requests are in flight while block j is coded (~32
        // symbols, several DRAM round trips of chain work ahead)
        if (i >= 0 && lanes > 1) {
            // the loaded bytes stay unpacked in registers until their block is
            // coded: packing them at load time would wait for the loads there
            struct Blk {
                uint32_t s[16], h[16], d[16];
            };
            auto ld = [&](int ii, Blk &b) {  // block with top symbol ii
                if (ii >= 15) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int64_t pos = base + (int64_t)(ii - 15 + j) * lanes;
                        b.s[j] = __ldg(syms + pos);
                        b.h[j] = shift ? __ldg(shift + pos) : 0u;
                        b.d[j] = dsched ? __ldg(dsched + pos) : dconst;
                    }
                }
            };
            auto blk = [&](const Blk &b) {
                uint32_t t[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) t[j] = word(b.s[j], b.h[j], b.d[j]);
#pragma unroll
                for (int j = 15; j >= 1; j -= 2) {  // one flush per two symbols
                    enc_bits(e, t[j], M);
                    enc_bits(e, t[j - 1], M);
                    enc_flush(e);
                }
            };
            Blk b0, b1;
            ld(i, b0);
            ld(i - 16, b1);
            for (; i >= 31; i -= 32) {
                blk(b0);
                ld(i - 32, b0);
                blk(b1);
                ld(i - 48, b1);
            }
            if (i >= 15) {
                blk(b0);
                i -= 16;
            }
        }
        for (; i >= 0; --i) {  // the last < 16 symbols of a lane (lowest indices)
            const int64_t pos = base + (int64_t)i * lanes;
            enc_push(e, word(syms[pos], shift ? shift[pos] : 0u, dsched ? dsched[pos] : dconst), M);
        }
        if (e.nacc) *e.wp = (uint32_t)e.acc;
        nbits[k] = (uint32_t)(e.wp - out) * 32u + e.nacc;
        states[k] = (uint16_t)e.S;
    }
}

// ---- decoder --------------------------------------------------------------
// Backward bit reader, branch-free. Positions are bit indices relative to
// the lane's first 16-byte chunk. The window (hi:lo) holds the cnt >= 32
// unread bits just below position A, left-aligned, so a field of b <= 12
// bits is `hi >> (32 - b)`: the state chain pays one 32-bit shift. A pop
// that leaves fewer than 32 bits ORs in the next lower word (index wn),
// read from a per-thread ring of kRing 16-byte chunks (4 kRing words) in
// shared memory, one predicated 32-bit load. Ring word q of thread t sits at
// (q * blockDim + t) * 4, so the address is one multiply-add of wn and a
// warp's loads never share a bank; chunks land as four 4-byte cp.async.
// cp.async keeps the ring kAhead chunks ahead;
// issuing (predicated, branch-free: at most two chunks, one commit group)
// and waiting happen once per 16-symbol block (sync()): a block pops at
// most 192 bits = 6 words, so it touches at most two chunks, both issued at
// least one block earlier. Lanes of a warp refill at different symbols, so
// the per-symbol path is predicated rather than branched.
constexpr int kRing = 8;
constexpr int kAhead = 4;

struct BitReader {
    const uint4 *base4;  // chunk 0 = the lane's first chunk
    uint32_t ring_s;     // shared address of this thread's ring word 0
    uint32_t ring_stride;  // bytes between ring words q and q + 1 (blockDim.x * 4): word-interleaved
                           // across the block's threads, so same-q reads of a warp hit 32 banks
    int hi_c;            // last chunk holding payload bits
    int cnt, start, wn, ci;  // ci: lowest chunk issued to the ring
    // read position A = 32 (wn + 1) + cnt (the window's bottom is word wn's
    // top); kept implicit so the per-symbol path does not update it
    __device__ __forceinline__ int A() const { return 32 * (wn + 1) + cnt; }
    uint32_t hi, lo;     // window: bits [A - cnt, A), left-aligned (bit A-1 at bit 63 of hi:lo)

    __device__ __forceinline__ uint4 direct(int c) const {
        return (c >= 0 && c <= hi_c) ? __ldg(base4 + c) : make_uint4(0, 0, 0, 0);
    }
    __device__ __forceinline__ static uint32_t pick(const uint4 &v, int j) {
        return j == 0 ? v.x : (j == 1 ? v.y : (j == 2 ? v.z : v.w));
    }
    __device__ __forceinline__ uint32_t word(int wi) const { return wi >= 0 ? pick(direct(wi >> 2), wi & 3) : 0u; }
    // chunk c = ring words 4c .. 4c + 3 (mod 4 kRing), four predicated
    // 4-byte cp.async (no branch: lanes of a warp refill at different blocks)
    __device__ __forceinline__ void issue(int c, bool on) {
        const uint32_t dst = ring_s + (uint32_t)((4 * c) & (4 * kRing - 1)) * ring_stride;
        const uint32_t *src = reinterpret_cast<const uint32_t *>(base4 + c);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p cp.async.ca.shared.global [%0], [%1], 4;\n\t}\n" ::"r"(
                    dst + j * ring_stride),
                "l"(src + j), "r"(on ? 1u : 0u)
                : "memory");
    }
    __device__ __forceinline__ void init(const uint4 *lane_base4, uint32_t my_ring_s, uint32_t stride_bytes,
                                         int start_bit, uint32_t nb) {
        base4 = lane_base4;
        ring_s = my_ring_s;
        ring_stride = stride_bytes;
        start = start_bit;  // 0..127
        hi_c = nb ? (int)((start_bit + nb - 1) >> 7) : -1;
        const int A0 = start_bit + (int)nb;
        const int wt = (A0 - 1) >> 5;  // word holding bit A0-1 (arithmetic: -1 when A0 == 0)
        const int nt = A0 - 32 * wt;   // its valid bits, 1..32
        const uint32_t w2 = word(wt - 1);
        hi = (word(wt) << (32 - nt)) | (nt < 32 ? w2 >> nt : 0u);
        lo = w2 << (32 - nt);
        cnt = nt + 32;
        wn = wt - 2;  // next word to bring in
        ci = (wn >> 2) + 1;
        // prime the ring kAhead chunks deep and wait for it (once per lane)
        const int target = (wn >> 2) - kAhead;
        for (int j = 0; j < kAhead + 1; ++j) {
            const int c = ci - 1;
            const bool on = c >= target;
            issue(c, on && c >= 0 && c <= hi_c);
            ci = on ? c : ci;
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    }
    // once per 16-symbol block: keep the ring kAhead chunks below the
    // current one (a block pops <= 192 bits, so the target moves <= 2 chunks)
    // as one commit group, then wait for every group but this one: the
    // chunks this block reads (the current one and the one below) were
    // issued at least one block earlier
    __device__ __forceinline__ void sync() {
        const int target = (wn >> 2) - kAhead;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int c = ci - 1;
            const bool on = c >= target;
            issue(c, on && c >= 0 && c <= hi_c);
            ci = on ? c : ci;
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 1;" ::: "memory");
    }
    // pop b bits (1 <= b <= 12); underflow shows as A < start at the end.
    // `e8` = table entry >> 8: b in bits 0..7, anything above. The funnel
    // shifts use the shift amount mod 32 (= b), so the state chain pays
    // entry >> 8 and one funnel shift here (no mask, no 32 - b).
    __device__ __forceinline__ uint32_t take(uint32_t e8) {
        const uint32_t b = e8 & 0xFFu;
        const uint32_t v = __funnelshift_l(hi, 0u, e8);  // top b bits of the window
        hi = __funnelshift_l(lo, hi, e8);
        lo <<= b;
        cnt -= (int)b;
        // refill below the valid bits (lo is zero here) with word wn
        const bool p = cnt < 32;
        const uint32_t src = ring_s + (uint32_t)(wn & (4 * kRing - 1)) * ring_stride;
        uint32_t w = 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.u32 %0, [%1];\n\t}\n"
            : "+r"(w)
            : "r"(src), "r"(p ? 1u : 0u)
            : "memory");
        const uint32_t sh = (uint32_t)cnt;  // < 32 when p (the only case whose result is kept)
        hi = p ? (hi | (w >> sh)) : hi;
        lo = p ? (w << (32u - sh)) : lo;
        cnt = p ? cnt + 32 : cnt;
        wn = p ? wn - 1 : wn;
        return v;
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
    const uint32_t my_ring =
        (uint32_t)__cvta_generic_to_shared(s_tab + (SMEM ? (D << M) : 0) + threadIdx.x);
    const uint32_t T = 1u << M;
    // table row of distribution d, pre-offset by -T so the index is the state
    const uint32_t *tabT = (SMEM ? s_tab : dec_tab_g) - T;
    // shared address of row -T: the row base (tabs0 + 4 dT) is formed off
    // the state chain, the state then adds with one multiply-add (the table
    // is read-only once the bulk copy above has landed)
    const uint32_t tabs0 = (uint32_t)__cvta_generic_to_shared(s_tab) - 4u * T;
    auto lookup = [&](uint32_t dT, uint32_t st) -> uint32_t {
        if constexpr (SMEM) {
            const uint32_t rowb = tabs0 + (dT << 2);
            uint32_t a, e;
            asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a) : "r"(st), "r"(rowb));
            asm("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(a));
            return e;
        } else {
            return __ldg(tabT + dT + st);
        }
    };
    const int64_t total = n_img * lanes;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (lane_status[k]) continue;
        const int64_t img = lanes == 1 ? k : k / lanes;
        const int l = (int)(k - img * lanes);
        const int cnt = lane_count(n_sym, lanes, l);
        const int64_t sbase = img * n_sym + l;
        const uint32_t dconstT = (d_img ? (uint32_t)d_img[img] : 0u) << M;
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(buf) + lane_off[k];
        BitReader br;
        br.init(reinterpret_cast<const uint4 *>(a0 & ~(uintptr_t)15), my_ring, blockDim.x * 4u, (int)(a0 & 15) * 8,
                nbits_a[k]);
        uint32_t state = states[k];
        // one symbol: the decoded (optionally un-recentred) byte
        auto step = [&](uint32_t dT, uint32_t sh) -> uint32_t {
            const uint32_t e = lookup(dT, state);
            state = (e >> 16) + br.take(e >> 8);
            return unshift ? ((e + sh + 128u) & 0xFFu) : (e & 0xFFu);  // (x + shift - 128) mod 256
        };
        int i = 0;
        if (lanes == 1) {
            for (; i < cnt && ((sbase + i) & 15); ++i) {
                const int64_t pos = sbase + i;
                br.sync();
                out[pos] = (uint8_t)step(dsched ? ((uint32_t)dsched[pos] << M) : dconstT, unshift ? unshift[pos] : 0u);
            }
            // 16-symbol blocks, a register ring of two blocks for d / shift:
            // block j + 2 is requested as soon as block j is decoded (~32
            // symbols ahead). Two blocks per iteration keep the loop body
            // inside the instruction cache: four were 25% slower (ncu: 14%
            // of stalls on instruction fetch), one (register moves) 15%.
            const uint4 z4 = make_uint4(0, 0, 0, 0);
            auto ld = [&](int ii, uint4 &dv, uint4 &hv) {
                if (ii + 16 <= cnt) {
                    if (dsched) dv = *reinterpret_cast<const uint4 *>(dsched + sbase + ii);
                    if (unshift) hv = *reinterpret_cast<const uint4 *>(unshift + sbase + ii);
                }
            };
            auto blk = [&](const uint4 &dv, const uint4 &hv, int64_t p0) {
                br.sync();
                uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    o[j >> 2] |= step(dsched ? (vbyte(dv, j) << M) : dconstT, vbyte(hv, j)) << (8 * (j & 3));
                *reinterpret_cast<uint4 *>(out + p0) = make_uint4(o[0], o[1], o[2], o[3]);
            };
            uint4 d0 = z4, d1 = z4, h0 = z4, h1 = z4;
            ld(i, d0, h0);
            ld(i + 16, d1, h1);
            for (; i + 32 <= cnt; i += 32) {
                blk(d0, h0, sbase + i);
                ld(i + 32, d0, h0);
                blk(d1, h1, sbase + i + 16);
                ld(i + 48, d1, h1);
            }
            if (i + 16 <= cnt) {
                blk(d0, h0, sbase + i);
                i += 16;
            }
        }
        // strided lanes (symbol l + i L): 16-symbol blocks with a two-block
        // register ring of d / shift (coalesced across the warp's consecutive
        // lanes, requested ~32 symbols ahead), as for one lane above
        if (i < cnt && lanes > 1) {
            struct Blk {
                uint32_t d[16], h[16];  // unpacked: consumed only when the block is decoded
            };
            auto ld = [&](int ii, Blk &b) {
                if (ii + 16 <= cnt) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int64_t pos = sbase + (int64_t)(ii + j) * lanes;
                        b.d[j] = dsched ? (uint32_t)__ldg(dsched + pos) : 0u;  // row shift applied at use
                        b.h[j] = unshift ? (uint32_t)__ldg(unshift + pos) : 0u;
                    }
                }
            };
            auto blk = [&](const Blk &b, int ii) {
                br.sync();
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    out[sbase + (int64_t)(ii + j) * lanes] = (uint8_t)step(dsched ? (b.d[j] << M) : dconstT, b.h[j]);
            };
            Blk b0, b1;
            ld(i, b0);
            ld(i + 16, b1);
            for (; i + 32 <= cnt; i += 32) {
                blk(b0, i);
                ld(i + 32, b0);
                blk(b1, i + 16);
                ld(i + 48, b1);
            }
            if (i + 16 <= cnt) {
                blk(b0, i);
                i += 16;
            }
        }
        for (; i < cnt; ++i) {  // the last < 16 symbols of a lane
            const int64_t pos = sbase + (int64_t)i * lanes;
            br.sync();
            out[pos] = (uint8_t)step(dsched ? ((uint32_t)dsched[pos] << M) : dconstT, unshift ? unshift[pos] : 0u);
        }
        uint8_t st = 0;
        if (br.A() < br.start) st = PILC_ST_UNDERFLOW;
        else if (state != T || br.A() != br.start) st = PILC_ST_END_STATE;
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
    // lane bit positions and counts are 32-bit (< 2^31 bits per lane)
    if (per_lane * M >= ((int64_t)1 << 31)) return PILC_E_ARG;
    if (lane_cap < (per_lane * M + 31) / 32 + 1) return PILC_E_ARG;
    if (n_img == 0) return PILC_OK;
    const int64_t tab_bytes = (int64_t)D * X * 4;
    const int in_smem = tab_bytes <= kSmemTableMax;
    const size_t smem = in_smem ? (size_t)tab_bytes : 0;
    const int64_t total = n_img * lanes;
    // spread the lanes over every SM: threads per block = lanes / SMs,
    // rounded to warps, in [32, kThreads]
    int64_t threads = ceil_div64(ceil_div64(total, sm_count()), 32) * 32;
    threads = threads < 32 ? 32 : (threads > kThreads ? kThreads : threads);
    int64_t blocks = ceil_div64(total, threads);
    const int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    {
        ProfScope _ps(PROF_RANS_ENC, as_stream(stream), (double)n_img * n_sym);
        if (in_smem) {
            if (smem > 48 * 1024)
                allow_dyn_smem(reinterpret_cast<const void *>(rans_encode_kernel<true>));
            rans_encode_kernel<true><<<(unsigned)blocks, (unsigned)threads, smem, as_stream(stream)>>>(
                syms, shift, dsched, d_img, n_img, n_sym, lanes, enc_tab, D, X, M, scratch, lane_cap, nbits, states);
        } else {
            rans_encode_kernel<false><<<(unsigned)blocks, (unsigned)threads, 0, as_stream(stream)>>>(
                syms, shift, dsched, d_img, n_img, n_sym, lanes, enc_tab, D, X, M, scratch, lane_cap, nbits, states);
        }
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
    // lane bit positions are 32-bit: a valid lane holds <= M bits per symbol
    if (ceil_div64(n_sym, lanes) * M >= ((int64_t)1 << 31)) return PILC_E_ARG;
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
                allow_dyn_smem(reinterpret_cast<const void *>(rans_decode_kernel<true>));
            rans_decode_kernel<true><<<(unsigned)blocks, (unsigned)threads, smem, as_stream(stream)>>>(
                buf, lane_off, nbits, states, dsched, d_img, n_img, n_sym, lanes, dec_tab, D, M, unshift, out,
                lane_status);
        } else {
            if (smem > 48 * 1024)
                allow_dyn_smem(reinterpret_cast<const void *>(rans_decode_kernel<false>));
            rans_decode_kernel<false><<<(unsigned)blocks, (unsigned)threads, smem, as_stream(stream)>>>(
                buf, lane_off, nbits, states, dsched, d_img, n_img, n_sym, lanes, dec_tab, D, M, unshift, out,
                lane_status);
        }
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}
