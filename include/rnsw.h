/*
 * rnsw.h -- C ABI of the B200 (sm_100a) RNS-Winograd exact INT8 convolution.
 *
 * The reference exposes this path only as a Python API (there is no FFI in
 * the reference); each entry point below is what that API's body becomes:
 *
 *   rnsw_plan_create        <- transforms.cached_transforms + reduce_for_system
 *                              + RnsSystem._mrc_inv   (rw/transforms.py:334-342,
 *                              rw/residue.py:70-81)
 *   rnsw_filter_transform   <- layer.precompute_filter_transforms
 *                              (rw/layer.py:161-174, rw/kernel.py:38-41)
 *   rnsw_input_transform    <- _modulus_pass part 1: residue_encode_array +
 *                              input_transform_mod  (rw/layer.py:278-283)
 *   rnsw_input_transform_compact, rnsw_small_channel_product
 *                           <- the same two steps for C <= 4 input channels
 *   rnsw_winograd_gemm      <- _modulus_pass GEMM loop / _modular_gemm
 *                              (rw/layer.py:251-263, 285-291)
 *   rnsw_output_residues    <- _modulus_pass part 2: backward_transform_mod
 *                              (rw/layer.py:293-297)
 *   rnsw_output_transform   <- backward transform + mrc_reconstruct_arrays +
 *                              scatter (rw/layer.py:293-297, 374-388,
 *                              rw/residue.py:180-206)
 *   rnsw_conv_forward       <- winograd_layer_conv body after its pre-flight
 *                              checks (rw/layer.py:343-389)
 *   rnsw_conv_forward_timed <- the same body with the reference's StageTimings
 *                              accounting (rw/layer.py:211-232, 366-376)
 *   rnsw_tile_decompose     <- layer.tile_decompose (rw/layer.py:118-158)
 *   rnsw_mrc_reconstruct    <- residue.mrc_reconstruct_arrays (rw/residue.py:180-206)
 *
 * Conventions
 *   - All tensor pointers are DEVICE pointers owned by the caller; the plan owns
 *     only its constant tables.  Every call is stream-ordered on `stream`
 *     (a cudaStream_t passed as void*, NULL = legacy default stream) and never
 *     synchronises the host.
 *   - Residues are symmetric: [-(m-1)/2, (m-1)/2] for odd m (rw/residue.py:25-33).
 *   - A plan is immutable after creation and may be shared across host threads
 *     and streams.
 *   - Return value 0 is success; the non-zero codes map one-to-one onto the
 *     reference's exception classes (rw/errors.py:4-33).
 */
#ifndef RNSW_H_
#define RNSW_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes. */
#define RNSW_OK 0
#define RNSW_ERR_INVALID 1     /* ValueError                         */
#define RNSW_ERR_SHAPE 2       /* ShapeMismatch                      */
#define RNSW_ERR_STRIDE 3      /* UnsupportedStride                  */
#define RNSW_ERR_RANGE 4       /* DynamicRangeExceeded               */
#define RNSW_ERR_NOT_COPRIME 5 /* NotCoprime                         */
#define RNSW_ERR_OVERFLOW 6    /* OverflowRisk                       */
#define RNSW_ERR_SYSTEM 7      /* SystemMismatch                     */
#define RNSW_ERR_CUDA 8        /* CUDA runtime failure               */
#define RNSW_ERR_WORKSPACE 9   /* workspace / buffer too small       */
#define RNSW_ERR_UNSUPPORTED 10 /* geometry outside the device path  */

/* Tensor layouts. */
#define RNSW_LAYOUT_NHWC 0 /* x (B,H,W,C), w (R,R,C,K), y (B,Ho,Wo,K): rw/layer.py:3 */
#define RNSW_LAYOUT_NCHW 1 /* x (B,C,H,W), w (K,C,R,R) = OIHW, y (B,K,Ho,Wo)        */

typedef struct rnsw_plan rnsw_plan;

/* Build a plan for F(tile_m x tile_m, r x r) over n_res moduli.
 * at: [n_res][M][N], g: [n_res][N][R], bt: [n_res][N][N] symmetric residues
 * (int16, host memory) as produced by reduce_transforms_mod; mrc_inv:
 * [n_res][n_res] with mrc_inv[j][i] = m_i^-1 mod m_j for i < j (host memory).
 * Errors: RNSW_ERR_INVALID (bad modulus / geometry), RNSW_ERR_NOT_COPRIME,
 * RNSW_ERR_SYSTEM (inverse table inconsistent), RNSW_ERR_UNSUPPORTED
 * (N > 24, R > 8, n_res > 4; tiles with N <= 16 and moduli < 4500 run the
 * tensor-core kernels, larger ones the generic CUDA-core kernels), RNSW_ERR_CUDA. */
int rnsw_plan_create(rnsw_plan** out, int tile_m, int r, int n_res, const int32_t* moduli,
                     const int16_t* at, const int16_t* g, const int16_t* bt,
                     const int32_t* mrc_inv);
void rnsw_plan_destroy(rnsw_plan* plan);
/* N (tile side) and the number of int8 limb planes (1 per m < 256, else 2). */
int rnsw_plan_info(const rnsw_plan* plan, int* n, int* n_planes);

/* Buffer sizes in bytes. P = B * ceil(Ho/M) * ceil(Wo/M) tiles. */
size_t rnsw_filter_bytes(const rnsw_plan* plan, int C, int K);
size_t rnsw_v_bytes(const rnsw_plan* plan, int64_t P, int C);
size_t rnsw_m_bytes(const rnsw_plan* plan, int64_t P, int K);
size_t rnsw_workspace_bytes(const rnsw_plan* plan, int B, int H, int W, int C, int K, int pad);

/* Transformed filter bank U = G w G^T mod m_i, in the device GEMM layout
 * [plane][N*N][K][Cp] int8 (Cp = C rounded up to 32/64/128k). */
int rnsw_filter_transform(const rnsw_plan* plan, const int8_t* w, int C, int K, int layout,
                          void* U, size_t U_bytes, void* stream);
/* Import one residue's reference-layout filter transform (N,N,C,K) int16
 * (the dict values of precompute_filter_transforms) into the bank. */
int rnsw_filter_import(const rnsw_plan* plan, int res, const int16_t* u_nnck, int C, int K,
                       void* U, size_t U_bytes, void* stream);

/* Stage 1: V = BT d B mod m_i for every tile and channel -> [plane][N*N][P][Cp]. */
int rnsw_input_transform(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C,
                         int pad, int layout, void* V, size_t V_bytes, void* stream);
/* Small-channel stages 1 + 2 (C <= 4 on a tensor-core plan, e.g. VGG16
 * conv1_1): the split rnsw_conv_forward takes for such layers.  Stage 1
 * writes compact symmetric residues V16[n_res][P][N*N][4] int16
 * (n_res * P * N*N * 8 bytes; same math as rnsw_input_transform,
 * rw/layer.py:278-283); stage 2 forms M = sum_c V U mod m_i on the CUDA cores
 * into the rnsw_winograd_gemm output layout (rw/layer.py:366-372).
 * RNSW_ERR_UNSUPPORTED when C > 4 or the plan is not a tensor-core plan. */
int rnsw_input_transform_compact(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C,
                                 int pad, int layout, void* V16, size_t V16_bytes, void* stream);
int rnsw_small_channel_product(const rnsw_plan* plan, const void* V16, const void* U, int64_t P, int C,
                               int K, void* Mw, size_t Mw_bytes, void* stream);
/* Stage 2: per (residue, position) GEMM on tcgen05 kind::i8, reduced mod m_i
 * -> Winograd-domain product residues, int16, in blocks of 128 tiles:
 * [ceil(P/128)][n_res][N*N][128][Kp] (tile p of block p/128 at row p%128),
 * so each GEMM output tile is written as one contiguous run. */
int rnsw_winograd_gemm(const rnsw_plan* plan, const void* V, const void* U, int64_t P, int C,
                       int K, void* Mw, size_t Mw_bytes, void* stream);
/* Stage 3: Y = AT M A mod m_i, mixed-radix reconstruction, crop/scatter. */
int rnsw_output_transform(const rnsw_plan* plan, const void* Mw, int B, int H, int W, int K,
                          int pad, int layout, int32_t* y, void* stream);
/* Debug view of stage 3 before reconstruction: (n_res, P, K, M, M) int16. */
int rnsw_output_residues(const rnsw_plan* plan, const void* Mw, int64_t P, int K, int16_t* y_res,
                         void* stream);
/* Whole layer: stages 1-3 with a caller-provided workspace. */
int rnsw_conv_forward(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C, int K,
                      int pad, int layout, const void* U, int32_t* y, void* workspace,
                      size_t workspace_bytes, void* stream);

/* rnsw_conv_forward with CUDA events between its stages: the same kernel
 * chain (whatever the plan dispatches to), then a host synchronisation;
 * stage_ms[0..2] = input transform, Winograd product (GEMM or small-channel
 * product), output transform + reconstruction + scatter, in milliseconds.
 * The only synchronising entry point (the reference's `timings` argument). */
int rnsw_conv_forward_timed(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C, int K,
                            int pad, int layout, const void* U, int32_t* y, void* workspace,
                            size_t workspace_bytes, void* stream, float* stage_ms);
/* Overlapping N x N patches of the zero canvas at stride tile_m
 * (rw/layer.py:118-158): x NHWC int8 -> patches
 * (B, ceil(Ho/M), ceil(Wo/M), N, N, C) int8 on the device. */
int rnsw_tile_decompose(const int8_t* x, int B, int H, int W, int C, int tile_m, int r, int pad,
                        int8_t* patches, size_t patches_bytes, void* stream);

/* Whole layer with the VGG16-stack glue fused into the output stage:
 * relu, >> shift, clip to [0,127], optional 2x2 max-pool (even tile_m),
 * written as int8 NHWC (B, Ho[/2], Wo[/2], K) -- the int32 output is never
 * materialised.  Not part of the reference package (BASELINE.json configs
 * 2/4 define the glue); equals rnsw_conv_forward followed by
 * rnsw_requant_pool.  NHWC only; K % 4 == 0; moduli < 4500; `out` 4-byte
 * aligned (RNSW_ERR_INVALID otherwise; 16-byte alignment with K % 16 == 0
 * selects 16-byte stores). */
int rnsw_conv_forward_requant(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C, int K,
                              int pad, const void* U, int shift, int pool, int8_t* out, void* workspace,
                              size_t workspace_bytes, void* stream);
/* The same two whole-layer calls with two caller-created CUDA events
 * (cudaEvent_t, passed as void*) recorded on `stream` after the input
 * transform and after the Winograd product: per-stage device times of the
 * exact kernel chain the untimed call runs (no host synchronisation). */
int rnsw_conv_forward_ev(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C, int K, int pad,
                         int layout, const void* U, int32_t* y, void* workspace, size_t workspace_bytes,
                         void* stream, void* const* events);
int rnsw_conv_forward_requant_ev(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C, int K,
                                 int pad, const void* U, int shift, int pool, int8_t* out, void* workspace,
                                 size_t workspace_bytes, void* stream, void* const* events);
/* Stage 3 with the fused glue (Mw from rnsw_winograd_gemm). */
int rnsw_output_transform_requant(const rnsw_plan* plan, const void* Mw, int B, int H, int W, int K, int pad,
                                  int shift, int pool, int8_t* out, void* stream);

/* Mw8 stage variants (the layout the whole-layer path uses when
 * rnsw_mw8_supported(plan) is 1: F(14x14,3x3) over two 16-bit residues,
 * output transform on tcgen05).  Mw8 holds the same Winograd-domain product
 * as Mw, as y mod m in [0, m) split into low/high byte planes:
 * [ceil(P/128)][n_res][2][N*N][128][Kp] uint8 (rnsw_m_bytes bytes).  The
 * stage calls mirror rnsw_small_channel_product / rnsw_winograd_gemm /
 * rnsw_output_transform / rnsw_output_transform_requant; chaining them gives
 * exactly rnsw_conv_forward(_requant).  RNSW_ERR_UNSUPPORTED for other plans. */
int rnsw_mw8_supported(const rnsw_plan* plan);
int rnsw_small_channel_product_mw8(const rnsw_plan* plan, const void* V16, const void* U, int64_t P, int C,
                                   int K, void* Mw8, size_t Mw8_bytes, void* stream);
int rnsw_winograd_gemm_mw8(const rnsw_plan* plan, const void* V, const void* U, int64_t P, int C, int K,
                           void* Mw8, size_t Mw8_bytes, void* stream);
int rnsw_output_transform_mw8(const rnsw_plan* plan, const void* Mw8, int B, int H, int W, int K, int pad,
                              int layout, int32_t* y, void* stream);
int rnsw_output_transform_requant_mw8(const rnsw_plan* plan, const void* Mw8, int B, int H, int W, int K,
                                      int pad, int shift, int pool, int8_t* out, void* stream);

/* Vectorised MRC of n_res residue arrays ([n_res][count] int16, any congruent
 * representatives) into signed int64. */
int rnsw_mrc_reconstruct(const rnsw_plan* plan, const int16_t* residues, int64_t count,
                         int64_t* out, void* stream);

/* Direct int8 implicit-GEMM convolution on tcgen05, the
 * device counterpart of direct_conv / im2col (rw/layer.py:81-103) for any
 * stride: x NHWC int8 (C % 16 == 0), y NHWC int32, exact.  Weights are
 * packed once by rnsw_direct_pack_weights from (R,R,C,K) (layout 0) or OIHW
 * (layout 1). */
size_t rnsw_direct_weight_bytes(int R, int C, int K);
int rnsw_direct_pack_weights(const int8_t* w, int R, int C, int K, int layout, void* w2, size_t w2_bytes,
                             void* stream);
int rnsw_direct_conv(const int8_t* x, int B, int H, int W, int C, const void* w2, int K, int R, int pad,
                     int stride, int32_t* y, void* stream);

/* Inter-layer glue for the VGG16 stack (not part of the reference package;
 * BASELINE.json config 2/4): relu, >> shift, clip to [0,127], optional 2x2
 * max-pool, NHWC int32 -> NHWC int8. */
int rnsw_requant_pool(const int32_t* y, int B, int H, int W, int C, int shift, int pool,
                      int8_t* out, void* stream);

const char* rnsw_error_string(int code);
/* Human-readable detail of the last error raised on this host thread. */
const char* rnsw_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RNSW_H_ */
