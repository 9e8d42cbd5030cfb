// tcgen05 decoder convolutions (tc_conv.cu), driven from vq.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

enum TcOutMode { TC_OUT_ACT = 0, TC_OUT_SHUFFLE = 1, TC_OUT_HEAD = 2 };

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
};

// 3xTF32 encoder layers: activations are fp32 split into a tf32 "hi" slab
// and an fp32 "lo" residual slab, 4 channels (16 B) per group, same padded
// group-major pixel indexing as the bf16 path.
enum Tc3Mode { TC3_ACT = 0, TC3_Z = 1 };

struct Tc3Layer {
    const float *in_hi, *in_lo;
    int64_t gstride, margin;
    int Hp, Wp, H, W;
    int64_t n_img, n_tiles;
    const float *w_hi, *w_lo;  // B operand hi/lo, [KG][N][4] fp32
    const float *bias;
    const float *res_hi, *res_lo;  // TC3_ACT residual (nullable)
    float *out_hi, *out_lo;        // TC3_ACT
    float *z;                      // TC3_Z: (n, H, W, 32) fp32 (nullable)
    float *zt;                     // TC3_Z: 128-latent tiles [tile][hi|lo][8][128][4]
    int relu;
};

// Codebook argmin on tcgen05 (3xTF32 distance GEMM + exact float64 rescore).
struct ArgminTc {
    const float *zt;       // z tiles from the projection epilogue
    int64_t n_vec, n_tiles;
    const float *cbt;      // codebook B operand: [hi|lo][8][256][4]
    int K;
    uint8_t *idx;
};
int argmin_tc_launch(const ArgminTc &a, cudaStream_t s);

int tc3_launch(const Tc3Layer &L, int ks, int mode, cudaStream_t s);

int tc_launch_act(const TcLayer &L, cudaStream_t s);
int tc_launch_shuffle(const TcLayer &L, cudaStream_t s);
int tc_launch_head(const TcLayer &L, cudaStream_t s);
int tc_dec_table(const float *cb, const float *w, const float *b, int K, int Dc, int ci_pad, int co_pad,
                 uint16_t *table, cudaStream_t s);
int tc_gather(const uint8_t *idx, const uint16_t *table, int64_t n_img, int gh, int gw, uint16_t *x,
              int64_t gstride, int64_t margin, cudaStream_t s);
