/*
 * pilc.h -- C ABI of libpilc_sm100a.so, the B200 (sm_100a) PILC hot path.
 *
 * The reference (`pixelcodec`, /root/reference/pkg/src/pixelcodec) is a
 * Python package whose hot loops are numba @njit functions; these entry
 * points replace them one for one (see INTEGRATION.md for the ctypes
 * binding the reference-side Python would add). Conventions:
 *
 *  - plain pointers and sizes only; no torch types, no structs by value
 *    except the fixed-layout pilc_header record written by the parser;
 *  - every buffer is caller-allocated DEVICE memory unless the argument
 *    name ends in _host; nothing is retained after the call returns;
 *  - `stream` is a cudaStream_t (NULL = legacy default stream); all work is
 *    stream-ordered and asynchronous; the return value is a launch status
 *    (PILC_OK or PILC_E_*), data errors go to per-image/per-lane status
 *    arrays (PILC_ST_*) that the host maps to the reference's exceptions;
 *  - results are bit-identical regardless of batch size, device or GPU
 *    count: no atomics, no split-K, fixed per-image schedules.
 *
 * Layouts: images are (N, H, W, 3) uint8, C-contiguous, exactly as
 * numpy hands them to `pixelcodec.compress`. Symbol planes (residuals,
 * recentring shifts, distribution indices d) share that layout.
 */
#ifndef PILC_H
#define PILC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- launch status ------------------------------------------------------ */
#define PILC_OK 0
#define PILC_E_ARG 1          /* invalid argument (shape, range, null)     */
#define PILC_E_CUDA 2         /* CUDA runtime / launch error               */
#define PILC_E_UNSUPPORTED 3  /* valid but not implemented on this path   */

/* ---- per-image / per-lane data status (reference exception in brackets) -
 * Codes are ordered like the checks in container.parse_header
 * (container.py:195-258), _read_lanes (:261-271) and
 * tables.interleaved_decode (tables.py:226-274). */
#define PILC_ST_OK 0
#define PILC_ST_TRUNCATED 1      /* [FormatError] container truncated        */
#define PILC_ST_BAD_MAGIC 2      /* [FormatError] bad magic                  */
#define PILC_ST_BAD_VERSION 3    /* [FormatError] unsupported version (aux)  */
#define PILC_ST_CRC 4            /* [CorruptStreamError] checksum mismatch   */
#define PILC_ST_BAD_BACKEND 5    /* [FormatError] unknown backend id (aux)   */
#define PILC_ST_BAD_M 6          /* [FormatError] precision M outside [10,12]*/
#define PILC_ST_BAD_PAD 7        /* [FormatError] unknown padding rule       */
#define PILC_ST_BAD_FLAGS 8      /* [FormatError] unknown header flags       */
#define PILC_ST_BAD_DIMS 9       /* [FormatError] bad dimensions/lane count  */
#define PILC_ST_GRID_TRUNC 10    /* [FormatError] scale grid truncated       */
#define PILC_ST_STATIC_D 11      /* [FormatError] static index outside grid  */
#define PILC_ST_IDX_LENS 12      /* [FormatError] index lengths inconsistent */
#define PILC_ST_RES_LENS 13      /* [FormatError] residual lengths inconsist.*/
#define PILC_ST_PAYLOAD_LEN 14   /* [FormatError] payload length mismatch    */
#define PILC_ST_GRID_EMPTY 15    /* [FormatError] bad scale grid: no scale   */
#define PILC_ST_GRID_VALUE 16    /* [FormatError] bad scale grid: finite >0  */
#define PILC_ST_GRID_ORDER 17    /* [FormatError] bad scale grid: increasing */
#define PILC_ST_GRID_GEOM 18     /* [FormatError] bad scale grid: geometric  */
#define PILC_ST_LANE_HDR 20      /* [FormatError] bit stream header truncated*/
#define PILC_ST_LANE_TRUNC 21    /* [FormatError] bit stream payload trunc.  */
#define PILC_ST_LANE_LEN 22      /* [FormatError] lane length field mismatch */
#define PILC_ST_STATE_RANGE 23   /* [CorruptStreamError] state out of range  */
#define PILC_ST_UNDERFLOW 24     /* [CorruptStreamError] bit stream underflow*/
#define PILC_ST_END_STATE 25     /* [CorruptStreamError] not back at 2^M     */
#define PILC_ST_PARAMS_HASH 26   /* [ModelError] predictor params mismatch   */
#define PILC_ST_MODEL_HASH 27    /* [ModelError] model hash mismatch         */

/* Parsed container header, one per blob (written by pilc_container_parse).
 * Offsets are relative to the blob start. 72 bytes, naturally aligned.
 * Checks run in the reference's order and stop at the first failure:
 * structure and crc (container.py:195-258, with ScaleGrid validation,
 * logistic.py:52-64), then the predictor-parameter hash (:288-292) and,
 * when has_model, the model hash (:303-304). */
typedef struct pilc_header {
    int32_t status;        /* PILC_ST_*                                      */
    int32_t aux;           /* offending value for BAD_VERSION / BAD_BACKEND  */
    uint8_t backend, M, pad_rule, flags;
    uint32_t width, height;
    uint16_t lanes, static_d;
    uint16_t D, reserved;
    uint32_t params_hash_off;   /* 8 bytes                                  */
    uint32_t model_hash_off;    /* 8 bytes (vqvae), else 0                  */
    uint32_t idx_table_off;     /* total u32, L x u32, L x u16 (vqvae) or 0 */
    uint32_t res_table_off;     /* same shape                               */
    uint32_t sched_crc;         /* flags bit 0                              */
    uint32_t payload_off;       /* first lane blob                          */
    uint32_t grid_crc;          /* crc32 of the grid bytes (grouping key)   */
    uint64_t idx_bytes;         /* sum of index lane wire sizes             */
    uint64_t res_bytes;         /* sum of residual lane wire sizes          */
} pilc_header;

const char *pilc_version(void);
/* Tuning switches of the fast path (no reference counterpart; for A/B
 * checks). key 0: encoder residual blocks as one fused kernel per block
 * (default 1) instead of two conv launches; key 1: decoder trunk (gather +
 * block convs) as one kernel with activations in shared memory, 2 (default)
 * with the activations in pixel pairs (N = 64 MMAs), 1 one pixel per MMA
 * row, 0 per-layer launches; key 2: encoder trunk (every residual block
 * + the projection in one kernel, default 1); key 3: decoder output stage (up
 * conv + pixel shuffle + head in one kernel with the hi-res activations in
 * shared memory, default 1) instead of two launches through HBM. All
 * bit-identical to the unfused path, so no switch changes any output byte.
 * Returns the previous value, or -PILC_E_ARG for an unknown key. */
int pilc_set_tuning(int32_t key, int32_t value);
/* Device sanity: returns 100 for sm_100 etc., or -1 if no usable device. */
int pilc_device_arch(void);

/* ---- TWAR predictor ------------------------------------------------------
 * Replaces predictor.forward_residual (predictor.py:292 -> :173-195) and
 * predictor.decode_parallel (predictor.py:309 -> _kernels.par_decode3
 * _kernels.py:146-170). params12_host: the 12 float32 of the PILW/wire
 * order (W_r[3], b_r, W_g[3], b_g, W_b[3], b_b), predictor.py:66-74.
 * shift (nullable): recentring shift plane; decode first undoes
 * recentring, t = (coded + shift - 128) & 255 (logistic.py:166-168). */
int pilc_twar_forward(const uint8_t *img, uint8_t *res, int64_t n_img,
                      int32_t H, int32_t W, const float *params12_host,
                      void *stream);
int pilc_twar_decode(const uint8_t *coded, const uint8_t *shift, uint8_t *img,
                     int64_t n_img, int32_t H, int32_t W,
                     const float *params12_host, void *stream);

/* ---- interleaved rANS lanes ----------------------------------------------
 * Replaces tables.interleaved_encode (tables.py:202-223) over
 * _kernels.encode_lane (_kernels.py:20-40), and tables.interleaved_decode
 * (tables.py:226-274) over _kernels.decode_lane (_kernels.py:43-63).
 *
 * Image i owns n_sym symbols at syms + i*n_sym; symbol j goes to lane
 * j mod lanes; each lane is encoded in reverse. The coded symbol is
 *   x = shift ? (syms - shift + 128) & 255 : syms          (recentring)
 * and its distribution index is dsched[i*n_sym + j] if dsched != NULL,
 * else d_img[i] if d_img != NULL, else 0.
 * enc_tab: D*X uint32 = delta | phi << 16 (tables.py:109-134 layout).
 * Encoder output: lane (i, l) writes its bit string (LSB-first, push
 * order, little-endian 32-bit words) to scratch + (i*lanes + l)*lane_cap
 * words; lane_cap >= ceil(ceil(n_sym/lanes) * M / 32) + 1. */
int pilc_rans_encode(const uint8_t *syms, const uint8_t *shift,
                     const uint8_t *dsched, const uint16_t *d_img,
                     int64_t n_img, int64_t n_sym, int32_t lanes,
                     const uint32_t *enc_tab, int32_t D, int32_t X, int32_t M,
                     uint32_t *scratch, int64_t lane_cap, uint32_t *nbits,
                     uint16_t *states, void *stream);

/* dec_tab: D * 2^M uint32 = symbol | pop_count << 8 | next_base << 16
 * (tables.py:115-134). Lane (i, l) payload starts at byte
 * buf + lane_off[i*lanes + l] and holds nbits bits; initial state
 * states[...]. lane_status (in/out, uint8 per lane): lanes whose status is
 * already non-zero (from pilc_container_lanes) are skipped; otherwise set
 * to PILC_ST_UNDERFLOW / PILC_ST_END_STATE / 0. `buf` must stay readable
 * 16 bytes past the last lane payload (16-byte chunked backward reads).
 * Symbols are written to
 * out + i*n_sym + j; if unshift != NULL they are un-recentred on the way
 * out, out = (x + unshift - 128) & 255. */
int pilc_rans_decode(const uint8_t *buf, const uint64_t *lane_off,
                     const uint32_t *nbits, const uint16_t *states,
                     const uint8_t *dsched, const uint16_t *d_img,
                     int64_t n_img, int64_t n_sym, int32_t lanes,
                     const uint32_t *dec_tab, int32_t D, int32_t M,
                     const uint8_t *unshift, uint8_t *out,
                     uint8_t *lane_status, void *stream);

/* ---- VQ-VAE network (vqvae.py:51-119, nn.py:15-67) -----------------------
 * The model lives in one device buffer in the kernel layout produced on
 * the host by pilc_model_pack from the canonical PILW tensor order
 * (weights.py:46-69); pilc_model_floats gives its size. */
int64_t pilc_model_floats(int32_t K, int32_t Dc, int32_t C, int32_t B);
int pilc_model_pack(const float *canonical_host, int32_t K, int32_t Dc,
                    int32_t C, int32_t B, float *packed_host);
/* Scratch bytes for a batch of n_img images of H x W. */
int64_t pilc_vq_workspace_bytes(int64_t n_img, int32_t H, int32_t W,
                                int32_t K, int32_t Dc, int32_t C, int32_t B);
/* encode_to_indices (vqvae.py:51-76): image -> u8 indices (N, gh, gw),
 * gh = ceil(H/2). z_out (nullable) receives the pre-argmin latents
 * (N, gh, gw, Dc) float32. Codebook argmin is float64 in the reference's
 * accumulation order with ties to the lower index. */
int pilc_vq_encode(const uint8_t *img, int64_t n_img, int32_t H, int32_t W,
                   const float *model, int32_t K, int32_t Dc, int32_t C,
                   int32_t B, void *workspace, int64_t ws_bytes,
                   uint8_t *idx_out, float *z_out, void *stream);
/* Same contract, the exact network: the reference's float arithmetic
 * operation for operation (nn.conv2d as OpenBLAS evaluates it, numpy's
 * float32 exp; oracle/pilc_oracle.c states it), so z and the indices are
 * bit-identical to the reference's. pilc_vq_encode (the fast encoder) runs
 * the convs as fp16-split tcgen05 GEMMs when C == Dc == 32 (fp32-class z:
 * hi/lo split of activations and weights, three MMAs per K step) and the
 * exact network otherwise. Returns PILC_E_UNSUPPORTED for the few shapes
 * where OpenBLAS's order is not modelled (single-pixel convs with Ci not a
 * multiple of 8, ...). */
int pilc_vq_encode_exact(const uint8_t *img, int64_t n_img, int32_t H,
                        int32_t W, const float *model, int32_t K, int32_t Dc,
                        int32_t C, int32_t B, void *workspace, int64_t ws_bytes,
                        uint8_t *idx_out, float *z_out, void *stream);
/* 1 when pilc_vq_decode runs the tcgen05 decoder for this model and image
 * shape (C == 32 and the tiles fit shared memory), 0 when it runs the exact
 * network. A function of (config, H, W) only. */
int pilc_vq_fast_decoder(int32_t K, int32_t Dc, int32_t C, int32_t B, int32_t H, int32_t W);
/* Codebook argmin alone: z (n_vec, Dc) float32 -> u8 (vqvae.py:66-76). */
int pilc_vq_argmin(const float *z, int64_t n_vec, const float *model,
                   int32_t K, int32_t Dc, int32_t C, int32_t B, uint8_t *idx_out,
                   void *stream);
/* The same on the tensor cores: the encoders' argmin (3xTF32 distance GEMM,
 * proven error radius, exact float64 rescore), fed from plain z. Dc == 32
 * and C == 32 only (PILC_E_UNSUPPORTED otherwise); workspace >=
 * pilc_vq_argmin_tc_workspace(n_vec) bytes (z as 128-latent tiles). */
int64_t pilc_vq_argmin_tc_workspace(int64_t n_vec);
int pilc_vq_argmin_tc(const float *z, int64_t n_vec, const float *model,
                      int32_t K, int32_t Dc, int32_t C, int32_t B, void *workspace,
                      int64_t ws_bytes, uint8_t *idx_out, void *stream);
/* decode_to_params (vqvae.py:79-113) fused with the logistic head
 * (logistic.round_half_away / scales_to_distributions, logistic.py:36-40,
 * 109-114): indices -> shift = round(mu) and d per subpixel (N, H, W, 3)
 * uint8. d_thresh: D-1 float64 thresholds (device), d = #{k : s > t_k}.
 * mu_out / s_out (nullable) receive the float32 planes. */
int pilc_vq_decode(const uint8_t *idx, int64_t n_img, int32_t H, int32_t W,
                   const float *model, int32_t K, int32_t Dc, int32_t C,
                   int32_t B, const double *d_thresh, int32_t D,
                   void *workspace, int64_t ws_bytes, uint8_t *shift_out,
                   uint8_t *d_out, float *mu_out, float *s_out, void *stream);

/* Same contract, the exact network (see pilc_vq_encode_exact): mu and s are
 * bit-identical to the reference's decode_to_params, so shift and d are
 * too, and containers decode interchangeably with pixelcodec. The fast
 * pilc_vq_decode runs the tcgen05 bf16 decoder when pilc_vq_fast_decoder
 * says so for (model, H, W), else the exact network; containers written
 * with the fast decoder carry header flag 0x80 (container.py). */
int pilc_vq_decode_exact(const uint8_t *idx, int64_t n_img, int32_t H, int32_t W,
                        const float *model, int32_t K, int32_t Dc, int32_t C,
                        int32_t B, const double *d_thresh, int32_t D,
                        void *workspace, int64_t ws_bytes, uint8_t *shift_out,
                        uint8_t *d_out, float *mu_out, float *s_out,
                        void *stream);

/* ---- container (container.py:3-25, 128-335) ------------------------------
 * Static d per image for twar-static (container.py:163-170): exact
 * integer sum of |t - 128|, then argmin |log2(MAD/ln 4) - log2 g|.
 * log2_grid: D float64 log2 of the grid values (device). */
int pilc_static_scale(const uint8_t *res, int64_t n_img, int64_t n_sym,
                      const double *log2_grid, int32_t D,
                      uint16_t *d_img, void *stream);

/* Blob sizes and offsets: blob_off[0..n_img] (exclusive scan, uint64).
 * fixed_bytes = header + stream tables (+ schedule crc) + 4-byte crc.
 * idx_nbits may be NULL (twar-static). sizes: n_img uint64 scratch. */
int pilc_container_sizes(const uint32_t *idx_nbits, const uint32_t *res_nbits,
                         int64_t n_img, int32_t lanes, int64_t fixed_bytes,
                         uint64_t *sizes, uint64_t *blob_off, void *stream);
/* Pack blobs (container.py:174-191): template (device) = header prefix up
 * to and including the params/model hash (static_d at byte 19 is patched
 * per image from d_img); then stream tables, optional schedule crc32 over
 * the u16 LE d schedule (dsched or d_img), lane wire blobs, crc32. */
int pilc_container_pack(const uint8_t *tmpl, int32_t template_len,
                        const uint16_t *d_img, const uint8_t *dsched,
                        int32_t sched_check, int64_t n_img, int64_t n_sym,
                        int32_t lanes, const uint32_t *idx_scratch,
                        int64_t idx_cap, const uint32_t *idx_nbits,
                        const uint16_t *idx_states, const uint32_t *res_scratch,
                        int64_t res_cap, const uint32_t *res_nbits,
                        const uint16_t *res_states, const uint64_t *blob_off,
                        uint8_t *out, void *stream);
/* Parse + validate n_blob blobs laid end to end in buf (blob i spans
 * [blob_off[i], blob_off[i+1])), including the crc32 trailer; buf must be
 * readable 16 bytes past the last blob (vector reads). params_hash
 * and model_hash are the expected 8-byte digests read as little-endian
 * uint64. Writes hdr[i]. */
int pilc_container_parse(const uint8_t *buf, const uint64_t *blob_off,
                         int64_t n_blob, uint64_t params_hash,
                         uint64_t model_hash, int32_t has_model,
                         pilc_header *hdr, void *stream);
/* Batch summary of parsed headers (one small record the host can read in a
 * single transfer): number of headers with a nonzero status, whether all
 * share blob 0's grouping key (width, height, backend, M, lanes, flags, D,
 * grid crc), blob 0's header and its grid bytes (u16 D + D f64, when blob 0
 * parsed OK). Replaces the reference's per-blob parse_header on the hot path
 * (container.py:195-258) for the common one-shape batch. */
typedef struct pilc_summary {
    int32_t n_bad, uniform;
    pilc_header h0;
    uint8_t grid[2 + 8 * 256];
    uint8_t pad[6];
} pilc_summary;
int pilc_container_summary(const uint8_t *buf, const uint64_t *blob_off,
                           const pilc_header *hdr, int64_t n_blob,
                           pilc_summary *out, void *stream);
/* Per-lane extraction for a group of blobs sharing (lanes, backend):
 * blob_idx[g] selects the blob; for stream 0 (index) / 1 (residual) the
 * lane payload offset (absolute, into buf), bit count and state are
 * written at [g*lanes + l], with the _read_lanes checks in lane_status.
 * Blobs whose lane count, or M / D when expect_M / expect_D are nonzero,
 * differ from the group's get a nonzero lane status (the coder skips them). */
int pilc_container_lanes(const uint8_t *buf, const uint64_t *blob_off,
                         const pilc_header *hdr, const int64_t *blob_idx,
                         int64_t n_group, int32_t lanes, int32_t stream_id,
                         int32_t expect_M, int32_t expect_D,
                         uint64_t *lane_off, uint32_t *nbits, uint16_t *states,
                         uint8_t *lane_status, void *stream);
/* crc32 (zlib polynomial) of [off[i], off[i] + len[i]) into crc[i]. */
int pilc_crc32(const uint8_t *buf, const uint64_t *off, const uint64_t *len,
               int64_t n, uint32_t *crc, void *stream);
/* crc32 of each image's u16-LE d schedule (container.py:186, :322-327). */
int pilc_sched_crc(const uint8_t *dsched, const uint16_t *d_img, int64_t n_img,
                   int64_t n_sym, uint32_t *crc, void *stream);

/* ---- launch accounting -----------------------------------------------------
 * Every kernel launch is counted; with timing enabled each launch is also
 * bracketed by CUDA events on its stream, with its algorithmic work units
 * (conv/argmin: FLOPs; coder: symbols; predictor: subpixels; container:
 * blobs). Used by bench.py for the live roofline. */
void pilc_prof_reset(int32_t enable_timing);
int64_t pilc_prof_launches(void);
int32_t pilc_prof_categories(void);
const char *pilc_prof_name(int32_t cat);
int pilc_prof_read(int32_t cat, int64_t *launches, double *total_ms,
                   double *units);
/* Per-launch records in launch order (timing enabled only). */
int64_t pilc_prof_count(void);
int pilc_prof_record(int64_t i, int32_t *cat, double *ms, double *units);

#ifdef __cplusplus
}
#endif
#endif /* PILC_H */
