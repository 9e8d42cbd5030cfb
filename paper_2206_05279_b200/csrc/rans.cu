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
constexpr int kSmemTableMax = 160 * 1024;

__device__ __forceinline__ int lane_count(int64_t n_sym, int lanes, int l) {
    return l < n_sym ? (int)((n_sym - l + lanes - 1) / lanes) : 0;
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
        uint32_t state = 1u << M;
        uint64_t acc = 0;
        int nacc = 0;
        uint32_t words = 0;
        for (int i = cnt - 1; i >= 0; --i) {
            const int64_t pos = base + (int64_t)i * lanes;
            uint32_t x = syms[pos];
            if (shift) x = (x - shift[pos] + 128u) & 0xFFu;
            const uint32_t d = dsched ? dsched[pos] : dconst;
            const uint32_t e = tab[d * X + x];
            const uint32_t b = ((e & 0xFFFFu) + state) >> M;
            acc |= (uint64_t)(state & ((1u << b) - 1u)) << nacc;
            nacc += b;
            if (nacc >= 32) {
                out[words++] = (uint32_t)acc;
                acc >>= 32;
                nacc -= 32;
            }
            state = (state >> b) + (e >> 16);
        }
        if (nacc) out[words] = (uint32_t)acc;
        nbits[k] = words * 32u + (uint32_t)nacc;
        states[k] = (uint16_t)state;
    }
}

// Aligned 32-bit word holding absolute byte address 4*w; reads outside
// [lo_w, hi_w] return 0 (never used by a valid stream).
__device__ __forceinline__ uint32_t load_word(const uint32_t *base_w, int64_t w, int64_t lo_w,
                                              int64_t hi_w) {
    return (w >= lo_w && w <= hi_w) ? __ldg(base_w + w) : 0u;
}

__global__ void __launch_bounds__(kThreads) rans_decode_kernel(
    const uint8_t *__restrict__ buf, const uint64_t *__restrict__ lane_off,
    const uint32_t *__restrict__ nbits_a, const uint16_t *__restrict__ states,
    const uint8_t *__restrict__ dsched, const uint16_t *__restrict__ d_img, int64_t n_img,
    int64_t n_sym, int lanes, const uint32_t *__restrict__ dec_tab_g, int D, int M,
    int tab_in_smem, const uint8_t *__restrict__ unshift, uint8_t *__restrict__ out,
    uint8_t *__restrict__ lane_status) {
    extern __shared__ uint32_t s_tab[];
    const uint32_t *tab = dec_tab_g;
    if (tab_in_smem) {
        const int n = D << M;
        for (int i = threadIdx.x; i < n; i += blockDim.x) s_tab[i] = dec_tab_g[i];
        __syncthreads();
        tab = s_tab;
    }
    // word-aligned view of the buffer (buffer base is at least 4-aligned)
    const uintptr_t base_addr = reinterpret_cast<uintptr_t>(buf) & ~(uintptr_t)3;
    const uint32_t *words = reinterpret_cast<const uint32_t *>(base_addr);
    const int64_t head = (int64_t)(reinterpret_cast<uintptr_t>(buf) - base_addr);  // 0..3
    const int64_t total = n_img * lanes;
    const uint32_t T = 1u << M;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (lane_status[k]) continue;
        const int64_t img = k / lanes;
        const int l = (int)(k - img * lanes);
        const int cnt = lane_count(n_sym, lanes, l);
        const int64_t sbase = img * n_sym + l;
        const uint32_t dconst = d_img ? d_img[img] : 0u;
        const uint32_t nb = nbits_a[k];
        // absolute bit addresses relative to `words`
        const int64_t start_bit = (head + (int64_t)lane_off[k]) * 8;
        const int64_t lo_w = start_bit >> 5;
        const int64_t hi_w = (start_bit + (int64_t)nb - 1) >> 5;  // word of the last bit
        int64_t A = start_bit + nb;      // read position (exclusive top)
        int64_t wlo = ((A - 1) >> 5) - 1;  // window = bits [32*wlo, 32*wlo+64)
        uint64_t win = ((uint64_t)load_word(words, wlo + 1, lo_w, hi_w) << 32) |
                       load_word(words, wlo, lo_w, hi_w);
        uint32_t state = states[k];
        uint8_t st = 0;
        for (int i = 0; i < cnt; ++i) {
            const int64_t pos = sbase + (int64_t)i * lanes;
            const uint32_t d = dsched ? dsched[pos] : dconst;
            const uint32_t e = tab[d * T + (state - T)];
            const uint32_t b = (e >> 8) & 0xFFu;
            uint32_t x = e & 0xFFu;
            if (unshift) x = (x + unshift[pos] + 128u) & 0xFFu;  // (x + shift - 128) mod 256
            out[pos] = (uint8_t)x;
            if (A - start_bit < (int64_t)b) {
                st = PILC_ST_UNDERFLOW;
                break;
            }
            const int64_t lo = A - b;
            if (lo < wlo * 32) {  // slide the window down one word
                wlo -= 1;
                win = (win << 32) | load_word(words, wlo, lo_w, hi_w);
            }
            const uint32_t v = (uint32_t)(win >> (lo - wlo * 32)) & ((1u << b) - 1u);
            A = lo;
            state = (e >> 16) + v;
        }
        if (!st && (state != T || A != start_bit)) st = PILC_ST_END_STATE;
        lane_status[k] = st;
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
                                const uint16_t *states, const uint8_t *dsched,
                                const uint16_t *d_img, int64_t n_img, int64_t n_sym,
                                int32_t lanes, const uint32_t *dec_tab, int32_t D, int32_t M,
                                const uint8_t *unshift, uint8_t *out, uint8_t *lane_status,
                                void *stream) {
    if (n_img < 0 || n_sym < 0 || lanes < 1 || M < 2 || M > 12 || D < 1) return PILC_E_ARG;
    if (n_img == 0) return PILC_OK;
    const int64_t tab_bytes = ((int64_t)D << M) * 4;
    const int in_smem = tab_bytes <= kSmemTableMax;
    const size_t smem = in_smem ? (size_t)tab_bytes : 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(rans_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t total = n_img * lanes;
    int64_t blocks = ceil_div64(total, kThreads);
    // one table copy per block: keep the grid at one resident block per SM
    // when the table is large, several when it is small
    const int64_t per_sm = in_smem ? (tab_bytes > 96 * 1024 ? 1 : (tab_bytes > 48 * 1024 ? 2 : 8)) : 16;
    const int64_t cap = (int64_t)sm_count() * per_sm;
    if (blocks > cap) blocks = cap;
{
        ProfScope _ps(PROF_RANS_DEC, as_stream(stream), (double)n_img * n_sym);
        rans_decode_kernel<<<(unsigned)blocks, kThreads, smem, as_stream(stream)>>>(
        buf, lane_off, nbits, states, dsched, d_img, n_img, n_sym, lanes, dec_tab, D, M, in_smem,
        unshift, out, lane_status);
    }
    PILC_CHECK_LAUNCH();
    return PILC_OK;
}
