// K1 on the 5th-generation tensor cores: V = BT d B mod m for every tile,
// channel and residue (rw/layer.py:278-283, rw/kernel.py:44-47, 21-30),
// written straight into the GEMM operand layout V[plane][pos][P][Cp].
//
// The separable sandwich BT d BT^T is one linear map of the N*N patch:
//     V[(i,j)] = sum_(a,b) Kr[(i,j),(a,b)] d[(a,b)],   Kr = kron(BT, BT) mod m,
// so the whole transform of a tile (all channels at once) is ONE GEMM per
// residue and 128-position block:
//     D[pos, ch] = sum_pix Kr[pos, pix] * patch[pix, ch]      (M=128, N=128, K=N*N)
//   A = Kr limbs: a per-CTA constant, resident in shared memory (K-major,
//       128B swizzle; built on the host into the plan, PlanHost::d_kr);
//   B = the patch, TMA-loaded as a 4-D box (channels x N columns x N rows x 1
//       image) straight from NHWC x: the box IS the MN-major operand (K =
//       pixel rows, N = channels), and TMA's zero fill supplies the conv
//       padding and the canvas extension of tile_decompose (rw/layer.py:118-158);
//   D = s32 in TMEM; 16-bit moduli: two accumulators (Kr = 256 Kr_hi + Kr_lo,
//       balanced s8 limbs), x = 256 D_hi + D_lo, |x| < 2^27.
// The Kronecker form does N*N/(2N) = 8x the MACs of the two-pass separable
// form at N = 16, but it is a single pass: no TMEM round trip between the
// passes, and each output value costs the CUDA cores one reduction and one
// byte split (the mma.sync kernel spent ~165 warp instructions per
// (tile, channel, residue); this one ~8 per value / 32 lanes).  The tensor
// pipe, idle in K1 otherwise, absorbs the extra MACs.
//
// Work: groups g = (residue, position block); CTA b serves group b % G for
// every unit (tile x 128 channels, or a tile PAIR x 64 channels when C = 64:
// the two 64-channel boxes are the two 64-byte MN atoms of one N = 128
// operand), so its Kr image is loaded once.  The G CTAs of a unit run side by
// side and read the same patch (the second to fourth reads hit L2).
// Warp roles (384 threads): 0 TMA producer, 1 MMA issuer, 2 TMEM allocator,
// 4-11 epilogue (lane quadrant x column half): tcgen05.ld -> limb
// recombination -> one exact reduction -> byte planes -> swizzled staging ->
// one TMA bulk tensor store per plane.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace rnsw {

namespace {

constexpr int kUThreads = 384;
constexpr int kGroupRows = 128;  // positions per group (MMA M)
constexpr int kUnitN = 128;      // channels per unit (MMA N): 1 tile x 128 or 2 tiles x 64

struct K1UArgs {
  Geometry g;
  int npos, mout, kp, ksteps, khalves, limbs, groups, npb;
  int tile_stride;      // two-tile: bytes between the two 64-channel patch boxes (one MN atom each)
  int units;            // two-tile: ceil(P / 2); one-tile: P * (Cp / 128)
  int cblocks;          // one-tile: Cp / 128
  int res_of[16];       // group -> residue
  int pb_of[16];        // group -> position block
  int plane_base[RNSW_MAX_RES];
  FastMod fm[RNSW_MAX_RES];
  FastDiv div_img, div_tw, div_cb;
  size_t group_bytes;
};

// Shared-memory budget (bytes): A image, S patch stages, the store staging.
template <int kLimbs>
struct K1UConfig {
  static constexpr int kStageBytes = 256 * 128;  // K <= 256 pixel rows x 128 channel bytes
  static constexpr int kABytes = kLimbs * 2 * 16384;
  static constexpr int kStgBytes = kLimbs * kGroupRows * kUnitN;  // one byte plane per limb
  static constexpr int kStages = (227 * 1024 - 2048 - kABytes - kStgBytes) / kStageBytes > 4
                                     ? 4
                                     : (227 * 1024 - 2048 - kABytes - kStgBytes) / kStageBytes;
  static constexpr int kAccCols = kLimbs * kUnitN;
  static constexpr int kTmemCols = 2 * kAccCols <= 256 ? 256 : 512;
  static constexpr size_t kSmem = 1024 + (size_t)kABytes + (size_t)kStages * kStageBytes + kStgBytes + 256;
  static_assert(kStages >= 2, "shared memory");
};

template <int kLimbs, bool kTwoTiles>
__global__ void __launch_bounds__(kUThreads, 1)
    input_umma_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmV,
                      const uint8_t* __restrict__ kr, K1UArgs args) {
  using Cfg = K1UConfig<kLimbs>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + Cfg::kABytes;
  uint8_t* stg = sB + S * Cfg::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + Cfg::kStgBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int group = (int)(blockIdx.x % args.groups);
  const int u_begin = (int)(blockIdx.x / args.groups), u_step = (int)(gridDim.x / args.groups);
  const int res = args.res_of[group], pb = args.pb_of[group];
  const Geometry& g = args.g;

  // the group's constant A image (kr: built on the host in the final layout)
  {
    const uint4* src = reinterpret_cast<const uint4*>(kr + (size_t)group * args.group_bytes);
    uint4* dst = reinterpret_cast<uint4*>(sA);
    const int n16 = (int)(args.group_bytes / 16);
    for (int i = threadIdx.x; i < n16; i += kUThreads) dst[i] = __ldg(src + i);
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmV);
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
  fence_proxy_async();  // A image (generic stores) -> visible to the MMA (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // unit -> first tile, channel offset
  auto unit_tile = [&](int u, int& p, int& c0) {
    if (kTwoTiles) {
      p = 2 * u;
      c0 = 0;
    } else {
      const int q = (int)fdiv((uint32_t)u, args.div_cb);
      p = q;
      c0 = (u - q * args.cblocks) * 128;
    }
  };
  // tile p -> image and the patch's top-left canvas coordinate (may be
  // negative: TMA fills the padding with zeros)
  auto tile_origin = [&](int p, int& b, int& h0, int& w0) {
    b = (int)fdiv((uint32_t)p, args.div_img);
    const int rem = p - b * (int)args.div_img.d;
    const int ti = (int)fdiv((uint32_t)rem, args.div_tw);
    const int tj = rem - ti * g.tw;
    h0 = ti * args.mout - g.pad;
    w0 = tj * args.mout - g.pad;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      const uint32_t bytes = (uint32_t)(args.npos * 128);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = u_begin; u < args.units; u += u_step) {
        int p, c0;
        unit_tile(u, p, c0);
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], bytes);
        uint8_t* dst = sB + stage * Cfg::kStageBytes;
#pragma unroll
        for (int t = 0; t < (kTwoTiles ? 2 : 1); ++t) {
          // tile p + t; a tile past P reads as zeros (image coordinate B is out of range)
          int b = g.B, h0 = 0, w0 = 0;
          if (p + t < (int)g.P) tile_origin(p + t, b, h0, w0);
          tma_load_4d(dst + t * args.tile_stride, &tmX, &full[stage], c0, w0, h0, b);
        }
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc = idesc_i8x(128, kUnitN, true, true, false, true);  // A K-major, B MN-major
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = u_begin; u < args.units; u += u_step, ++it) {
        const int as = it & 1;
        mbar_wait(&tempty[as], ((it >> 1) & 1) ^ 1);
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t d0 = tmem_base + as * Cfg::kAccCols;
        const uint32_t b_base = smem_u32(sB + stage * Cfg::kStageBytes);
        for (int ks = 0; ks < args.ksteps; ++ks) {
          const uint64_t db = kTwoTiles ? umma_desc_mn_sw64(b_base + ks * 32 * 64, args.tile_stride)
                                        : umma_desc_mn_sw128(b_base + ks * 32 * 128);
#pragma unroll
          for (int l = 0; l < kLimbs; ++l) {
            const uint32_t a_addr = smem_u32(sA) + (l * args.khalves + (ks >> 2)) * 16384 + (ks & 3) * 32;
            mma_i8(d0 + l * kUnitN, umma_desc_kmajor(a_addr, 128), db, idesc, ks > 0 ? 1u : 0u);
          }
        }
        mma_commit(&empty[stage]);
        mma_commit(&tfull[as]);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: 8 warps = 4 lane quadrants x 2 column halves ----------------
    const int q = warp & 3, hh = (warp - 4) >> 2;
    const int row = q * 32 + lane;  // position within the group's block
    const FastMod fm = args.fm[res];
    const int32_t wshift = 128 - fm.h;  // w = v + 128 from r' = v + h
    const int etid = threadIdx.x - 128;
    int it = 0;
    for (int u = u_begin; u < args.units; u += u_step, ++it) {
      int p, c0;
      unit_tile(u, p, c0);
      const int as = it & 1;
      mbar_wait(&tfull[as], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + as * Cfg::kAccCols + hh * 64;
      uint32_t lo[16], hi[16];  // [chunk of 16 channels][word]
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        int32_t a[16], b[16];
        if (kLimbs == 2) {
          tmem_ld16(taddr + ch * 16, a);          // D_hi
          tmem_ld16(taddr + kUnitN + ch * 16, b);  // D_lo
        } else {
          tmem_ld16(taddr + ch * 16, b);
        }
        tmem_ld_wait();
        if (ch == 3) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[as]);
        }
        int32_t w[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int32_t x = kLimbs == 2 ? a[e] * 256 + b[e] : b[e];
          const int32_t r = red_pos_biased(x + fm.off, fm);  // (x + h) mod m in [0, m)
          w[e] = kLimbs == 2 ? r + wshift : r - fm.h;        // 16-bit: w = v + 128; 8-bit: v
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t p01 = __byte_perm((uint32_t)w[4 * e], (uint32_t)w[4 * e + 1], 0x5140);
          const uint32_t p23 = __byte_perm((uint32_t)w[4 * e + 2], (uint32_t)w[4 * e + 3], 0x5140);
          const uint32_t b0 = __byte_perm(p01, p23, 0x5410);
          lo[ch * 4 + e] = kLimbs == 2 ? b0 ^ 0x80808080u : b0;  // low byte of v
          hi[ch * 4 + e] = __byte_perm(p01, p23, 0x7632);         // (v + 128) >> 8
        }
      }
      // staging must be free: the previous unit's bulk store has read it
      if (etid == 0) bulk_wait_read<0>();
      named_bar_sync(1, 256);
      {
#pragma unroll
        for (int pl = 0; pl < kLimbs; ++pl) {
          uint8_t* base = stg + pl * (kGroupRows * kUnitN);
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            const uint32_t* src = pl == 0 ? lo : hi;
            const uint4 v4 = make_uint4(src[ch * 4], src[ch * 4 + 1], src[ch * 4 + 2], src[ch * 4 + 3]);
            uint32_t off;
            if (kTwoTiles) {
              // [pos][tile][64 channels], 64-byte rows, 64B swizzle
              const uint32_t r64 = (uint32_t)(row * 2 + hh);
              off = r64 * 64 + ((((uint32_t)ch) ^ ((r64 >> 1) & 3u)) << 4);
            } else {
              // [pos][128 channels], 128-byte rows, 128B swizzle
              const uint32_t c16 = (uint32_t)(hh * 4 + ch);
              off = (uint32_t)row * 128 + ((c16 ^ ((uint32_t)row & 7u)) << 4);
            }
            *reinterpret_cast<uint4*>(base + off) = v4;
          }
        }
      }
      fence_proxy_async();
      named_bar_sync(1, 256);
      if (etid == 0) {
#pragma unroll
        for (int pl = 0; pl < kLimbs; ++pl)
          tma_store_4d(&tmV, stg + pl * (kGroupRows * kUnitN), c0, p, pb * kGroupRows,
                       args.plane_base[res] + (kLimbs == 2 ? (pl == 0 ? 0 : 1) : 0));
        bulk_commit();
      }
    }
    if (etid == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

int64_t sym_host(int64_t v, int64_t m) {
  v %= m;
  if (v < 0) v += m;
  return v > (m - 1) / 2 ? v - m : v;
}

}  // namespace

cudaError_t build_kr_images(PlanHost& plan) {
  const PlanDevice& d = plan.dev;
  plan.d_kr = nullptr;
  if (!d.fast || d.n > 16 || d.n < 2) return cudaSuccess;
  for (int r = 1; r < d.n_res; ++r)
    if (d.res[r].planes != d.res[0].planes) return cudaSuccess;
  const int N = d.n, npos = N * N;
  plan.kr_limbs = d.res[0].planes;
  plan.kr_npb = (npos + kGroupRows - 1) / kGroupRows;
  plan.kr_groups = d.n_res * plan.kr_npb;
  plan.kr_kp = (npos + 31) / 32 * 32;
  plan.kr_khalves = (plan.kr_kp + 127) / 128;
  plan.kr_group_bytes = (size_t)plan.kr_limbs * plan.kr_khalves * 16384;
  std::vector<uint8_t> img((size_t)plan.kr_groups * plan.kr_group_bytes, 0);
  for (int r = 0; r < d.n_res; ++r) {
    const int64_t m = d.res[r].modulus;
    for (int pbk = 0; pbk < plan.kr_npb; ++pbk) {
      uint8_t* gimg = img.data() + (size_t)(r * plan.kr_npb + pbk) * plan.kr_group_bytes;
      for (int row = 0; row < kGroupRows; ++row) {
        const int pos = pbk * kGroupRows + row;
        if (pos >= npos) break;
        const int i = pos / N, j = pos % N;
        for (int pix = 0; pix < npos; ++pix) {
          const int a = pix / N, b = pix % N;
          const int64_t v = sym_host((int64_t)d.res[r].bt[i * RNSW_MAX_N + a] * d.res[r].bt[j * RNSW_MAX_N + b], m);
          int8_t limb[2];
          if (plan.kr_limbs == 1) {
            limb[0] = (int8_t)v;
          } else {
            const int64_t h = (v + 128 + 256 * 64) / 256 - 64;  // floor((v + 128) / 256)
            limb[0] = (int8_t)h;            // limb 0: high (x 256)
            limb[1] = (int8_t)(v - 256 * h);  // limb 1: low
          }
          const int kh = pix / 128, kb = pix % 128;
          for (int l = 0; l < plan.kr_limbs; ++l) {
            const size_t off = (size_t)(l * plan.kr_khalves + kh) * 16384 + row * 128 +
                               ((((kb >> 4) ^ (row & 7)) << 4) | (kb & 15));
            gimg[off] = (uint8_t)limb[l];
          }
        }
      }
    }
  }
  cudaError_t e = cudaMalloc(&plan.d_kr, img.size());
  if (e != cudaSuccess) {
    plan.d_kr = nullptr;
    return e;
  }
  e = cudaMemcpy(plan.d_kr, img.data(), img.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(plan.d_kr);
    plan.d_kr = nullptr;
  }
  return e;
}

void free_kr_images(PlanHost& plan) {
  if (plan.d_kr) cudaFree(plan.d_kr);
  plan.d_kr = nullptr;
}

bool umma_input_ok(const PlanHost& plan, const Geometry& g) {
  static const bool off = getenv("RNSW_K1_MMA_SYNC") != nullptr;  // A/B switch: the mma.sync kernel
  if (off || force_generic() || plan.d_kr == nullptr || g.layout != 0) return false;
  if (plan.kr_groups > 16) return false;
  return g.C == 64 || (g.C % 128) == 0;
}

cudaError_t launch_input_transform_umma(const PlanHost& plan, const Geometry& g, const int8_t* x, int8_t* V,
                                        cudaStream_t s) {
  const PlanDevice& d = plan.dev;
  const bool two = g.C == 64;
  K1UArgs a{};
  a.g = g;
  a.npos = d.n * d.n;
  a.mout = d.m_out;
  a.tile_stride = (plan.kr_kp * 64 + 1023) / 1024 * 1024;
  a.kp = plan.kr_kp;
  a.ksteps = plan.kr_kp / 32;
  a.khalves = plan.kr_khalves;
  a.limbs = plan.kr_limbs;
  a.groups = plan.kr_groups;
  a.npb = plan.kr_npb;
  a.group_bytes = plan.kr_group_bytes;
  a.cblocks = two ? 1 : g.Cp / 128;
  const int64_t units = two ? (g.P + 1) / 2 : g.P * a.cblocks;
  if (units >= (1ll << 31) || g.P >= (1ll << 31)) return cudaErrorInvalidValue;
  a.units = (int)units;
  for (int gi = 0; gi < a.groups; ++gi) {
    a.res_of[gi] = gi / a.npb;
    a.pb_of[gi] = gi % a.npb;
  }
  for (int r = 0; r < d.n_res; ++r) {
    a.plane_base[r] = d.res[r].plane_base;
    const ResidueTables& t = d.res[r];
    a.fm[r] = FastMod{t.red_mul, t.red_shift, t.red_off, t.modulus, t.half, t.red_negm};
  }
  a.div_img = make_fastdiv((uint32_t)(g.th * g.tw));
  a.div_tw = make_fastdiv((uint32_t)g.tw);
  a.div_cb = make_fastdiv((uint32_t)a.cblocks);

  auto encode = encode_fn();
  if (encode == nullptr) return cudaErrorInvalidValue;
  CUtensorMap tmX, tmV;
  {
    // x NHWC as (C, W, H, B); box = 64 or 128 channels x N x N x 1
    cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.B};
    cuuint64_t strides[3] = {(cuuint64_t)g.C, (cuuint64_t)g.W * g.C, (cuuint64_t)g.H * g.W * g.C};
    cuuint32_t box[4] = {(cuuint32_t)(two ? 64 : 128), (cuuint32_t)d.n, (cuuint32_t)d.n, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (encode(&tmX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(x), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, two ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    // V as (Cp, P, npos, planes); box = channels x tiles x 128 positions x 1 plane
    const int npos = d.n * d.n;
    cuuint64_t dims[4] = {(cuuint64_t)g.Cp, (cuuint64_t)g.P, (cuuint64_t)npos, (cuuint64_t)d.n_planes};
    cuuint64_t strides[3] = {(cuuint64_t)g.Cp, (cuuint64_t)g.P * g.Cp, (cuuint64_t)g.P * g.Cp * npos};
    cuuint32_t box[4] = {(cuuint32_t)(two ? 64 : 128), (cuuint32_t)(two ? 2 : 1), (cuuint32_t)kGroupRows, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (encode(&tmV, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, V, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               two ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int sms = num_sms_current();
  const int per_group = sms / a.groups > 0 ? sms / a.groups : 1;
  int64_t grid = (int64_t)per_group * a.groups;
  const int64_t need = (int64_t)a.units * a.groups;
  if (grid > need) grid = need;
  grid = (grid + a.groups - 1) / a.groups * a.groups;
  auto run = [&](auto kern, size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, kUThreads, smem, s>>>(tmX, tmV, plan.d_kr, a);
    return cudaGetLastError();
  };
  if (plan.kr_limbs == 2)
    return two ? run(input_umma_kernel<2, true>, K1UConfig<2>::kSmem)
               : run(input_umma_kernel<2, false>, K1UConfig<2>::kSmem);
  return two ? run(input_umma_kernel<1, true>, K1UConfig<1>::kSmem)
             : run(input_umma_kernel<1, false>, K1UConfig<1>::kSmem);
}

}  // namespace rnsw
