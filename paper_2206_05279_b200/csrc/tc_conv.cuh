// tcgen05 decoder convolutions (tc_conv.cu), driven from vq.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

enum TcOutMode { TC_OUT_ACT = 0, TC_OUT_SHUFFLE = 1, TC_OUT_HEAD = 2, TC_OUT_HEAD2 = 3 };

struct TcLayer {
    const uint16_t *in;  // padded group-major bf16 activations (32 channels)
    int64_t gstride;     // pixels per channel-group slab (margins included)
    int64_t margin;      // leading margin pixels of each slab
    int Hp, Wp, H, W;    // padded / interior dims of the conv grid
    int64_t n_img, n_tiles;
    const uint16_t *wts;  // B operand, [KG][N][8] bf16
    const float *bias;
    const uint16_t *resid;  // TC_OUT_ACT: same layout as out (nullable)
    uint16_t *out;
    int64_t out_gstride, out_margin;
    int relu;
    // head
    uint8_t *shift, *dsel;
    float *mu, *s;
    int crop_h, crop_w;
    const double *thresh;
    int n_thresh;
    float log_s_min, log_s_max;
    int pair_out;        // TC_OUT_SHUFFLE: write the output in the pixel-pair layout (HEAD2's input)
    int n_stages;        // set by the launcher
};

// Decoder trunk (gather of dec.proj's table + all 2B block convs) with the
// activations resident in shared memory, G images per CTA iteration.
struct DecTrunk {
    const uint8_t *idx;        // (n, gh, gw) codebook indices
    const uint16_t *table;     // K x 32 bf16: relu(proj(codebook)) (dec_table_kernel)
    int K;
    int Hp, Wp;                // padded latent grid
    int64_t n_img;
    int n_conv;                // 2B, <= 16
    const uint16_t *w;         // 2B consecutive [36][32][8] bf16 B operands (pairs: [48][64][8])
    const float *bias[16];
    uint16_t *out;             // padded group-major bf16 slabs (the up conv's input)
    int64_t out_gstride, out_margin;
    int G, pad_bytes;          // set by the launcher
};
int dec_trunk_launch(const DecTrunk &p, cudaStream_t s);
// The same over pixel pairs (N = 64 MMAs, 24 per 256 pixels; w = 2B
// consecutive [48][64][8] bf16 pair operands, vq.cu tc_blk2); bit-identical.
int dec_trunk2_launch(const DecTrunk &p, cudaStream_t s);

// Decoder output stage: up conv + pixel shuffle + logistic head of one image
// per CTA iteration, the hi-res activations kept in shared memory (same
// arithmetic as tc_launch_shuffle + tc_launch_head2). PILC_E_UNSUPPORTED for
// grids whose tiles do not fit; the caller then runs those two kernels.
struct DecUpHead {
    const uint16_t *in;        // trunk output: padded group-major bf16 slabs (32 channels)
    int64_t gstride, margin;
    int gh, gw;                // latent grid (interior)
    int64_t n_img;
    const uint16_t *w_up;      // [36][128][8] bf16
    const float *b_up;         // 128
    const uint16_t *w_head;    // pair head [48][16][8] bf16
    const float *b_head;       // 6
    uint8_t *shift, *dsel;
    float *mu, *s;             // nullable
    int crop_h, crop_w;
    const double *thresh;
    int n_thresh;
    float log_s_min, log_s_max;
};
int dec_uphead_launch(const DecUpHead &p, cudaStream_t s);

// Encoder layers (3-product fp16 split, tc_conv.cu). Operands: the scaled
// fp16 hi / lo slab sets of a tensor (8-channel groups, 16 B per pixel: hi
// groups 0..3 then lo groups 4..7), padded group-major like the bf16 path;
// block outputs also as an fp32 slab set (4-channel groups) for the exact
// residual. kx / mx: per-image scale exponent and exact max |x| (float bits).
enum Tc3Mode { TC3_ACT = 0, TC3_Z = 1 };

struct Tc3Layer {
    const uint16_t *in;  // hi / lo slabs of the input
    int64_t gstride, margin;
    int Hp, Wp, H, W;
    int64_t n_img, n_tiles;
    const uint16_t *w;   // B operand [KG][64][8] fp16: rows 0..31 = hi(w 2^kw), 32..63 = lo
    const float *meta;   // {kw (int bits), L1 = max_co sum|w|, max|b|}
    const int32_t *kx_in;
    const uint32_t *mx_in;
    const float *bias;
    const float *res;         // TC3_ACT residual fp32 slab (nullable)
    const uint32_t *mx_res;   // with res
    uint16_t *out;            // TC3_ACT hi / lo slabs of the output
    float *out32;             // TC3_ACT fp32 copy (nullable)
    int32_t *kx_out;
    uint32_t *mx_out;         // atomicMax; zeroed by the caller
    float *z;                 // TC3_Z: (n, H, W, 32) fp32 (nullable)
    float *zt;                // TC3_Z: 128-latent tiles [tile][hi|lo][8][128][4]
    int relu;
    int n_stages;             // set by the launcher
};

// One encoder residual block, X' = relu(X + conv2(relu(conv1(X)))), both
// convs in one kernel with the intermediate kept in shared memory (one image
// per CTA iteration); same arithmetic as two tc3 ACT launches.
struct Tc3Block {
    const uint16_t *in;   // hi / lo slabs of X
    const float *res;     // fp32 slabs of X
    int64_t gstride, margin;
    int Hp, Wp, H, W;
    int64_t n_img;
    const uint16_t *w1, *w2;      // [36][64][8] fp16 B operands
    const float *meta1, *meta2;   // {kw, L1, max|b|}
    const float *bias1, *bias2;
    const int32_t *kx_in;
    const uint32_t *mx_in;
    uint16_t *out;
    float *out32;                 // nullable
    int32_t *kx_out;
    uint32_t *mx_out;             // atomicMax; zeroed by the caller
};
int tc3_block_launch(const Tc3Block &b, cudaStream_t s);

// Encoder trunk: all B residual blocks and the 1x1 projection of one image
// per CTA iteration with the activations (hi / lo operands and the fp32
// block input) resident in shared memory; z leaves as the argmin's tiles.
// Same arithmetic as the per-block kernels plus the TC3_Z projection.
constexpr int kEtMaxBlocks = 8;
struct EncTrunk {
    const uint16_t *in;   // hi / lo slabs of the front output
    const float *in32;    // its fp32 slabs
    int64_t gstride, margin;
    int Hp, Wp, H, W;
    int64_t n_img;
    int n_blocks;                               // B, 1 .. kEtMaxBlocks
    const uint16_t *w[2 * kEtMaxBlocks + 1];    // [36][64][8] fp16 B operands; [2B] = proj [4][64][8]
    const float *meta[2 * kEtMaxBlocks + 1];    // {kw, L1, max|b|}
    const float *bias[2 * kEtMaxBlocks + 1];
    const int32_t *kx_in;                       // front output scale exponent per image
    const uint32_t *mx_in;                      // front output max |x| per image
    float *z;                                   // (n, H, W, 32) fp32 (nullable)
    float *zt;                                  // 128-latent tiles [tile][hi|lo][8][128][4]
};
int enc_trunk_launch(const EncTrunk &p, cudaStream_t s);

// Encoder front (stem and the stride-2 down conv as 3-product fp16 MMAs, the
// down GEMM over the space-to-depth stem, tc_conv.cu); outputs like the
// block convs.
struct EncFrontTc {
    const uint8_t *img;  // (n, H, W, 3)
    int64_t n_img, n_tiles;
    int H, W, gh, gw;
    const uint16_t *w_stem16;      // [4][64][8] fp16 hi / lo of w_stem 2^kw_stem, K = c*9 + tap (27 -> 32)
    const float *meta_stem;        // {kw_stem (int), ...}
    const float *b_stem;
    const uint16_t *w_down;        // [36][64][8] fp16 hi / lo of w 2^kw_down
    const float *b_down;
    const float *meta_down;        // {kw_down (int), L1, max|b|, k_stem (int)}: weight / stem-output scales
    const int32_t *k0;             // output scale exponent
    float *out32;                  // fp32 slab set
    uint16_t *out;                 // hi / lo slab set (scale 2^k0)
    int64_t gstride, margin;
    uint32_t *out_max;
    int32_t *kx_out;
    int n_quarters;                // set by the launcher
};
int enc_front_tc_launch(const EncFrontTc &a, cudaStream_t s);

// Codebook argmin on tcgen05 (3xTF32 distance GEMM + exact float64 rescore).
struct ArgminTc {
    const float *zt;       // z tiles from the projection epilogue
    int64_t n_vec, n_tiles;
    const float *cbt;      // codebook B operand: [hi|lo][8][256][4]
    int K;
    uint8_t *idx;
};
int argmin_tc_launch(const ArgminTc &a, cudaStream_t s);
// z (n, 32) float32 -> the argmin's 128-latent tiles (tf32 hi / fp32 lo, as
// the projection epilogues write them; tail rows zero)
int pack_z_tiles(const float *z, int64_t n, float *zt, cudaStream_t s);

int tc3_launch(const Tc3Layer &L, int ks, int mode, cudaStream_t s);

int tc_launch_act(const TcLayer &L, cudaStream_t s);
bool tc_decoder_supported(int gh, int gw, bool pairs);
int tc_launch_shuffle(const TcLayer &L, cudaStream_t s);
int tc_launch_head2(const TcLayer &L, cudaStream_t s);  // head over pixel pairs (pair layout input)
int tc_dec_table(const float *cb, const float *w, const float *b, int K, int Dc, int ci_pad, int co_pad,
                 uint16_t *table, cudaStream_t s);
int tc_gather(const uint8_t *idx, const uint16_t *table, int64_t n_img, int gh, int gw, uint16_t *x,
              int64_t gstride, int64_t margin, cudaStream_t s);
