// Fused stem + down convolution of the 3xTF32 encoder (enc_front.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

struct EncFront {
    const uint8_t *img;  // (n, H, W, 3)
    int64_t n_img;
    int H, W, gh, gw;    // gh = ceil(H/2)
    const float *w_stem, *b_stem;
    int stem_ci_pad, stem_co_pad;
    const float *w_down, *b_down;
    int down_ci_pad, down_co_pad;
    float *out_hi, *out_lo;  // padded group-major tf32 hi / fp32 lo slabs
    int64_t gstride, margin;
};

size_t enc_front_smem();
int enc_front_launch(const EncFront &a, cudaStream_t s);
