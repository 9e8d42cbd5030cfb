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
    float *out32;       // padded group-major fp32 slab set (tc_conv.cu encoder layout)
    uint16_t *out;      // scaled fp16 hi / lo slab set (scale 2^k0)
    uint32_t *out_max;  // per-image max |out| (float bits, atomicMax)
    int32_t *kx_out;    // per-image scale exponent (= k0)
    const int32_t *k0;  // device: static scale exponent of this output
    int64_t gstride, margin;
};

size_t enc_front_smem();
int enc_front_launch(const EncFront &a, cudaStream_t s);
