// Direct int8 implicit-GEMM convolution on tcgen05.
//
// The exact counterpart of the reference's direct_conv / im2col
// (rw/layer.py:81-103): y[b,ho,wo,k] = sum_{u,v,c} x[b, s*ho+u-pad, s*wo+v-pad, c]
// * w[u,v,c,k], int8 x int8 -> int32, for any stride s.  It is the GPU
// comparator BASELINE config 5 asks for, the strided path of layer_conv and
// a full-size GPU cross-check.
//
// GEMM view: rows = output pixels, columns = output channels, reduction =
// (u, v, c).  A CTA tile is a TH x TW rectangle of output pixels of one image
// (TH*TW = 128 = the MMA M / TMEM lanes).  For each filter tap (u, v) and
// 128-channel chunk, one 4-D TMA box over NHWC x fetches exactly the im2col
// rows of that tap: box (BC, TW*s, TH*s, 1) with element strides (1, s, s, 1);
// out-of-range coordinates (padding) are zero-filled by the TMA unit.
// Weights are packed once to W2[K][R*R*Cp] (K-major).  Same warp roles as the
// Winograd GEMM: TMA producer, single-thread MMA issuer, TMEM allocator and
// 8 epilogue warps with double-buffered accumulators.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"

namespace rnsw {

namespace {

constexpr int kDM = 128;       // output pixels per tile (TMEM lanes)
constexpr int kDThreads = 384;

struct DirectArgs {
  int B, H, W, C, Cp, K, R, pad, stride, Ho, Wo;
  int th, tw;         // tile rectangle (th * tw == 128)
  int ntile_h, ntile_w, num_kb, nkc, cchunks;
  int64_t total_tiles;
  int32_t* y;
};

template <int BN, int BC>
struct DirectCfg {
  static constexpr int kAB = kDM * BC;
  static constexpr int kBB = BN * BC;
  static constexpr int kStage = kAB + kBB;
  static constexpr int kStagesRaw = (200 * 1024) / kStage;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kStage + 256;
};

template <int BN, int BC>
__global__ void __launch_bounds__(kDThreads, 1)
    direct_conv_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                       DirectArgs args) {
  using Cfg = DirectCfg<BN, BC>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStage);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0), lane = threadIdx.x % 32;  // warp-uniform for the compiler

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto decode = [&](int64_t t, int& b, int& ho0, int& wo0, int& kb) {
    kb = (int)(t % args.num_kb);
    t /= args.num_kb;
    const int twi = (int)(t % args.ntile_w);
    t /= args.ntile_w;
    const int thi = (int)(t % args.ntile_h);
    b = (int)(t / args.ntile_h);
    ho0 = thi * args.th;
    wo0 = twi * args.tw;
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < args.total_tiles; t += gridDim.x) {
        int b, ho0, wo0, kb;
        decode(t, b, ho0, wo0, kb);
        for (int kc = 0; kc < args.nkc; ++kc) {
          const int tap = kc / args.cchunks, cc = kc - tap * args.cchunks;
          const int u = tap / args.R, v = tap - u * args.R;
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], (uint32_t)(Cfg::kAB + Cfg::kBB));
          uint8_t* sa = smem + stage * Cfg::kStage;
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(sa)),
              "l"(reinterpret_cast<uint64_t>(&tmX)), "r"(smem_u32(&full[stage])), "r"(cc * BC),
              "r"(wo0 * args.stride + v - args.pad), "r"(ho0 * args.stride + u - args.pad), "r"(b)
              : "memory");
          const int kcol = tap * args.Cp + cc * BC;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(sa + Cfg::kAB)),
              "l"(reinterpret_cast<uint64_t>(&tmW)), "r"(smem_u32(&full[stage])), "r"(kcol), "r"(kb * BN)
              : "memory");
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8(kDM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int64_t t = blockIdx.x; t < args.total_tiles; t += gridDim.x, ++it) {
        const int as = it & 1;
        mbar_wait(&tempty[as], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem_base + as * BN;
        for (int kc = 0; kc < args.nkc; ++kc) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem + stage * Cfg::kStage);
          const uint32_t b0 = a0 + Cfg::kAB;
#pragma unroll
          for (int k = 0; k < BC / 32; ++k)
            mma_i8(d0, umma_desc_kmajor(a0 + 32 * k, BC), umma_desc_kmajor(b0 + 32 * k, BC), idesc,
                   (kc | k) != 0);
          mma_commit(&empty[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[as]);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3, half = (warp - 4) >> 2;
    constexpr int kHalf = BN / 2;
    constexpr int kBatch = kHalf < 64 ? kHalf : 64;
    int it = 0;
    for (int64_t t = blockIdx.x; t < args.total_tiles; t += gridDim.x, ++it) {
      int b, ho0, wo0, kb;
      decode(t, b, ho0, wo0, kb);
      const int as = it & 1;
      mbar_wait(&tfull[as], (it >> 1) & 1);
      tc_fence_after();
      const int row = q * 32 + lane;  // pixel inside the TH x TW rectangle
      const int ho = ho0 + row / args.tw, wo = wo0 + row % args.tw;
      const bool ok = ho < args.Ho && wo < args.Wo;
      int32_t* yrow = args.y + (((int64_t)b * args.Ho + ho) * args.Wo + wo) * args.K;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + as * BN + half * kHalf;
#pragma unroll 1
      for (int c0 = 0; c0 < kHalf; c0 += kBatch) {
        int32_t v[kBatch / 16][16];
#pragma unroll
        for (int j = 0; j < kBatch / 16; ++j) tmem_ld16(taddr + c0 + 16 * j, v[j]);
        tmem_ld_wait();
        if (c0 + kBatch >= kHalf) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[as]);
        }
#pragma unroll
        for (int j = 0; j < kBatch / 16; ++j) {
          const int col = kb * BN + half * kHalf + c0 + 16 * j;
          if (!ok || col >= args.K) continue;
          if (col + 16 <= args.K && (args.K & 3) == 0) {
            int4* dst = reinterpret_cast<int4*>(yrow + col);
#pragma unroll
            for (int e = 0; e < 4; ++e) dst[e] = make_int4(v[j][4 * e], v[j][4 * e + 1], v[j][4 * e + 2], v[j][4 * e + 3]);
          } else {
            for (int e = 0; e < 16 && col + e < args.K; ++e) yrow[col + e] = v[j][e];
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

// weights (R,R,C,K) or OIHW -> W2[K][R*R*Cp] int8 (zero-padded channels)
__global__ void pack_weights_kernel(const int8_t* __restrict__ w, int R, int C, int Cp, int K, int layout,
                                    int8_t* __restrict__ w2) {
  const int64_t total = (int64_t)K * R * R * Cp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % Cp);
    int64_t r = i / Cp;
    const int tap = (int)(r % (R * R));
    const int k = (int)(r / (R * R));
    const int u = tap / R, v = tap % R;
    int8_t val = 0;
    if (c < C) val = layout == 0 ? w[(((int64_t)u * R + v) * C + c) * K + k] : w[(((int64_t)k * C + c) * R + u) * R + v];
    w2[i] = val;
  }
}

template <int BN, int BC>
cudaError_t run_direct(const DirectArgs& a, const int8_t* x, const int8_t* w2, cudaStream_t s) {
  using Cfg = DirectCfg<BN, BC>;
  auto encode = encode_fn();
  if (encode == nullptr) return cudaErrorInvalidValue;
  CUtensorMap tmX, tmW;
  {
    cuuint64_t dims[4] = {(cuuint64_t)a.C, (cuuint64_t)a.W, (cuuint64_t)a.H, (cuuint64_t)a.B};
    cuuint64_t strides[3] = {(cuuint64_t)a.C, (cuuint64_t)a.W * a.C, (cuuint64_t)a.H * a.W * a.C};
    cuuint32_t box[4] = {(cuuint32_t)BC, (cuuint32_t)(a.tw * a.stride), (cuuint32_t)(a.th * a.stride), 1};
    cuuint32_t es[4] = {1, (cuuint32_t)a.stride, (cuuint32_t)a.stride, 1};
    CUtensorMapSwizzle sw = BC == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : BC == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                                   : CU_TENSOR_MAP_SWIZZLE_32B;
    if (encode(&tmX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(x), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    cuuint64_t wd[2] = {(cuuint64_t)a.R * a.R * a.Cp, (cuuint64_t)a.K};
    cuuint64_t wstr[1] = {(cuuint64_t)a.R * a.R * a.Cp};
    cuuint32_t wbox[2] = {(cuuint32_t)BC, (cuuint32_t)BN};
    cuuint32_t wes[2] = {1, 1};
    if (encode(&tmW, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(w2), wd, wstr, wbox, wes,
               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  auto kern = direct_conv_kernel<BN, BC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = a.total_tiles < sms ? a.total_tiles : sms;
  kern<<<(unsigned)(grid < 1 ? 1 : grid), kDThreads, Cfg::kSmem, s>>>(tmX, tmW, a);
  return cudaGetLastError();
}

template <int BN>
cudaError_t run_direct_bc(const DirectArgs& a, int bc, const int8_t* x, const int8_t* w2, cudaStream_t s) {
  switch (bc) {
    case 32: return run_direct<BN, 32>(a, x, w2, s);
    case 64: return run_direct<BN, 64>(a, x, w2, s);
    default: return run_direct<BN, 128>(a, x, w2, s);
  }
}

}  // namespace

size_t direct_weight_bytes(int R, int C, int K) {
  const int Cp = C <= 32 ? 32 : C <= 64 ? 64 : (C + 127) / 128 * 128;
  return (size_t)K * R * R * Cp;
}

cudaError_t launch_pack_weights(const int8_t* w, int R, int C, int K, int layout, int8_t* w2, cudaStream_t s) {
  const int Cp = C <= 32 ? 32 : C <= 64 ? 64 : (C + 127) / 128 * 128;
  const int64_t total = (int64_t)K * R * R * Cp;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  pack_weights_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(w, R, C, Cp, K, layout, w2);
  return cudaGetLastError();
}

// x NHWC int8 (C % 32 == 0 or C in {32, 64}), w2 from launch_pack_weights, y NHWC int32.
cudaError_t launch_direct_conv(const int8_t* x, int B, int H, int W, int C, const int8_t* w2, int K, int R, int pad,
                               int stride, int32_t* y, cudaStream_t s) {
  DirectArgs a{};
  a.B = B;
  a.H = H;
  a.W = W;
  a.C = C;
  a.Cp = C <= 32 ? 32 : C <= 64 ? 64 : (C + 127) / 128 * 128;
  a.K = K;
  a.R = R;
  a.pad = pad;
  a.stride = stride;
  a.Ho = (H + 2 * pad - R) / stride + 1;
  a.Wo = (W + 2 * pad - R) / stride + 1;
  a.tw = a.Wo <= 8 ? 8 : a.Wo <= 16 ? 16 : 32;
  while (a.tw * stride > 256) a.tw /= 2;
  a.th = kDM / a.tw;
  if (a.th * stride > 256) return cudaErrorInvalidValue;
  a.ntile_h = (a.Ho + a.th - 1) / a.th;
  a.ntile_w = (a.Wo + a.tw - 1) / a.tw;
  const int bc = a.Cp < 128 ? a.Cp : 128;
  a.cchunks = a.Cp / bc;
  a.nkc = R * R * a.cchunks;
  a.y = y;
  const int bn = K <= 64 ? 64 : K <= 128 ? 128 : 256;
  a.num_kb = (K + bn - 1) / bn;
  a.total_tiles = (int64_t)B * a.ntile_h * a.ntile_w * a.num_kb;
  if (bn == 64) return run_direct_bc<64>(a, bc, x, w2, s);
  if (bn == 128) return run_direct_bc<128>(a, bc, x, w2, s);
  return run_direct_bc<256>(a, bc, x, w2, s);
}

}  // namespace rnsw
