// Internal launch interface between the C ABI (capi.cu) and the kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "plan.h"

namespace rnsw {

// Geometry of one layer call on the device path.
struct Geometry {
  int B, H, W, C, K, pad, layout;
  int Ho, Wo, th, tw;  // output plane, tiles per side
  int64_t P;           // B * th * tw
  int Cp;              // C padded for the tensor-core K dimension
  int Kp;              // K padded to 16
  int bc;              // channel chunk per MMA stage (32 / 64 / 128 bytes)
};

// Mw (K3 -> K4) layout: blocks of 128 tiles, [ceil(P/128)][res][pos][128][Kp]
// int16 residues, so every (tile block, residue, position) output tile of the
// GEMM is one contiguous run of 128*Kp values (its stores stream instead of
// scattering 128 rows over the whole buffer).  rp = res * npos + pos,
// nrp = n_res * npos.
__host__ __device__ inline int64_t mw_offset(int64_t p, int rp, int nrp, int Kp) {
  return (((p >> 7) * nrp + rp) * 128 + (p & 127)) * (int64_t)Kp;
}

// Mw8: the planar variant of Mw that the tcgen05 output transform reads
// (output_umma.cu): 16-bit residues y mod m in [0, m) split into two byte
// planes (limb 0 = low byte, limb 1 = high byte),
// [ceil(P/128)][res][limb][pos][128][Kp] uint8 -- the same size as Mw.
__host__ __device__ inline int64_t mw8_offset(int64_t p, int res, int limb, int pos, int nres, int npos, int Kp) {
  return (((((p >> 7) * nres + res) * 2 + limb) * npos + pos) * 128 + (p & 127)) * (int64_t)Kp;
}

// Mw8 for 8-bit residues (the Kronecker output transform, output_kron.cu):
// y mod m in [0, m) as one byte plane per residue, [ceil(P/128)][res][pos][128][Kp].
__host__ __device__ inline int64_t mw8s_offset(int64_t p, int res, int pos, int nres, int npos, int Kp) {
  return ((((p >> 7) * nres + res) * npos + pos) * 128 + (p & 127)) * (int64_t)Kp;
}

// Host-side mirror of the plan (kept next to the device copy).
struct PlanHost {
  PlanDevice dev;         // host copy of the tables
  PlanDevice* d_plan;     // device copy
  int device;             // CUDA device the tables live on
  // tcgen05 input transform (input_umma.cu): the Kronecker operator
  // kron(BT, BT) mod m per (residue, 128-position block) as shared-memory
  // images of the MMA A operand (K-major, 128B swizzle), one per group.
  uint8_t* d_kr;          // [groups][kr_group_bytes] (nullptr: not built)
  int kr_groups;          // n_res * kr_npb
  int kr_npb;             // 128-position blocks: ceil(N*N / 128)
  int kr_kp;              // K = N*N padded to a multiple of 32
  int kr_khalves;         // 128-byte K chunks per A row: ceil(kr_kp / 128)
  int kr_limbs;           // 1 (m < 256) or 2 (balanced s8 limbs)
  size_t kr_group_bytes;  // kr_limbs * kr_khalves * 16 KB
  int64_t kr_xmax[RNSW_MAX_RES];  // max |Kr d| over positions (|d| <= 128): the accumulator bias floor
  // tcgen05 Kronecker output transform (output_kron.cu), two 16-bit residues:
  // kron(AT, AT) (residue 1 times the mixed-radix factor) per (residue, row
  // block) as four balanced-limb matrices [4][128 rows][kra_kp] int8
  uint8_t* d_kra;
  int kra_npb;
  int kra_kp;
  size_t kra_bytes;
  // ... for 8-bit plans: [rb][res][128 rows][kra8_kp] s8, residue r times W[r][0]
  uint8_t* d_kra8;
  int kra8_npb;
  int kra8_kp;
  size_t kra8_bytes;
};

// Build / release PlanHost::d_kr (input_umma.cu); a plan without it keeps
// the mma.sync input transform.
cudaError_t build_kr_images(PlanHost& plan);
void free_kr_images(PlanHost& plan);
cudaError_t build_kra_images(PlanHost& plan);
cudaError_t build_kra8_images(PlanHost& plan);
void free_kra_images(PlanHost& plan);

cudaError_t launch_filter_transform(const PlanHost& plan, const int8_t* w, int C, int K, int Cp, int layout,
                                    int8_t* U, cudaStream_t s);
cudaError_t launch_filter_import(const PlanHost& plan, int res, const int16_t* u_nnck, int C, int K, int Cp,
                                 int8_t* U, cudaStream_t s);
cudaError_t launch_input_transform(const PlanHost& plan, const Geometry& g, const int8_t* x, int8_t* V,
                                   cudaStream_t s, bool relaxed = false);
// pos_out: 16-bit residues as y mod m in [0, m) instead of symmetric (whole-layer
// path only; the stage API keeps the reference's symmetric residues)
// Tile count of the layer being launched (capi.cu): gates programmatic dependent launch.
void pdl_layer_hint(int64_t P);

// K3 for small P (gemm_t.cu): output channels on the MMA rows, tiles on the
// columns, only the u limb planes of the bank (three accumulators).
bool gemm_t_ok(const PlanDevice& d, int64_t P, int Cp, bool planar, bool pos_out);
cudaError_t launch_winograd_gemm_t(const PlanHost& plan, const int8_t* V, const int8_t* U, int64_t P, int Cp, int K,
                                   int Kp, int16_t* Mw, cudaStream_t s);
cudaError_t launch_winograd_gemm(const PlanHost& plan, const int8_t* V, const int8_t* U, int64_t P, int Cp,
                                 int K, int Kp, int bc, int16_t* Mw, cudaStream_t s, bool pos_out = false,
                                 bool planar = false);
cudaError_t launch_output_transform(const PlanHost& plan, const Geometry& g, const int16_t* Mw, int32_t* y,
                                    int16_t* y_res, cudaStream_t s);
cudaError_t launch_output_transform_tc(const PlanHost& plan, const Geometry& g, const int16_t* Mw, int32_t* y,
                                       int16_t* y_res, cudaStream_t s, int8_t* out8 = nullptr, int shift = 0,
                                       int pool = 0);
bool umma_input_ok(const PlanHost& plan, const Geometry& g);
// relaxed (whole-layer path, 16-bit moduli, C <= 8192): V residues in
// [-m-128, m-128) instead of [-h, h] (see input_umma.cu K1UMode)
cudaError_t launch_input_transform_umma(const PlanHost& plan, const Geometry& g, const int8_t* x, int8_t* V,
                                        cudaStream_t s, bool relaxed = false);
cudaError_t launch_input_transform_tc(const PlanHost& plan, const Geometry& g, const int8_t* x, int8_t* V,
                                      cudaStream_t s);
bool tc_output_ok(const PlanDevice& d);
// tcgen05 output transform (output_umma.cu): F(14x14,3x3) over two 16-bit
// residues; reads Mw8.  mode 0: int32 y (layout g.layout), 1: requant int8,
// 3: requant + 2x2 max-pool int8.
bool umma_output_ok(const PlanDevice& d);
cudaError_t launch_output_transform_umma(const PlanHost& plan, const Geometry& g, const uint8_t* Mw8, int32_t* y,
                                         cudaStream_t s, int8_t* out8 = nullptr, int shift = 0, int pool = 0);
bool force_generic();
// Kronecker output transform (output_kron.cu): mode 0 int32 y, 1 requant int8, 3 requant + pool
bool kron_output_ok(const PlanHost& plan, const Geometry& g, int mode);
cudaError_t launch_output_transform_kron(const PlanHost& plan, const Geometry& g, const uint8_t* Mw8, int32_t* y,
                                         cudaStream_t s, int8_t* out8 = nullptr, int shift = 0, int pool = 0);
// Small-channel path (C <= 4): compact input transform + CUDA-core product (smallc.cu)
bool smallc_ok(const PlanDevice& d, const Geometry& g);
size_t smallc_v16_bytes(const PlanDevice& d, const Geometry& g);
cudaError_t launch_input_transform_compact(const PlanHost& plan, const Geometry& g, const int8_t* x, int16_t* V16,
                                           cudaStream_t s);
cudaError_t launch_smallc_product(const PlanHost& plan, const Geometry& g, const int16_t* V16, const int8_t* U,
                                  int16_t* Mw, cudaStream_t s, bool planar = false);
PFN_cuTensorMapEncodeTiled_v12000 encode_fn();
int num_sms_current();  // SM count of the current device (cached per device)
size_t direct_weight_bytes(int R, int C, int K);
cudaError_t launch_pack_weights(const int8_t* w, int R, int C, int K, int layout, int8_t* w2, cudaStream_t s);
cudaError_t launch_direct_conv(const int8_t* x, int B, int H, int W, int C, const int8_t* w2, int K, int R, int pad,
                               int stride, int32_t* y, cudaStream_t s);
cudaError_t launch_tile_decompose(const int8_t* x, int B, int H, int W, int C, int tile_m, int r, int pad,
                                  int8_t* patches, cudaStream_t s);
cudaError_t launch_mrc(const PlanHost& plan, const int16_t* residues, int64_t count, int64_t* out,
                       cudaStream_t s);
cudaError_t launch_requant_pool(const int32_t* y, int B, int H, int W, int C, int shift, int pool, int8_t* out,
                                cudaStream_t s);

}  // namespace rnsw
