// K3 for small tile counts (16-bit residues, P <= 48 tiles, <= 80 for C >= 512:
// VGG16 at batch 1, the deep layers at batch <= 64): the per-position modular GEMM of
// rw/layer.py:285-291 / rw/gemm.py:43-97 with the operand roles swapped.
//
// The general GEMM (gemm.cu) puts tiles on the MMA's M = 128 rows: with a
// handful of tiles almost every row is padding, and the layer is bound by
// streaming the four-plane filter bank (u, u' = 256 u mod m, each as two s8
// limbs).  Here the output channels are the M = 128 rows and the tiles the N
// columns (N = P rounded up to 16):
//     D[k, t] = sum_c U[k, c] V[t, c]       per (residue, position, 128 k)
// and only the two limb planes of u are read -- half the bank bytes -- with
// three accumulators
//     D65536 = u_hi v_hi,   D256 = u_hi v_lo + u_lo v_hi,   D1 = u_lo v_lo,
//     y = red(D65536) (65536 mod m) + red(D256) 256 + D1  (mod m)
// (the bounds of epilogue_u2 in gemm.cu: C <= 8192 keeps every partial and
// the recombination below 2^28).  y mod m goes to Mw8 as two byte planes,
// one byte per (tile, channel): a warp writes 32 consecutive channels.
//
// Warps: 0 TMA producer, 1 MMA issuer, 2-5 epilogue (TMEM lane quadrant
// warp & 3; warp 2 also owns the TMEM allocation).  Accumulators are double
// buffered while 2 x 3 x Np <= 512 TMEM columns (Np <= 80), single buffered
// above (Np 96-128: the next unit's MMAs wait for the epilogue's TMEM reads).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace rnsw {
namespace {

constexpr int kTThreads = 192;
constexpr int kTBC = 128;     // channel chunk (bytes) per stage: 128B-swizzled K-major rows

struct GemmTArgs {
  int P, K, Kp, Cp, npos, n_res, nkc, num_kb;
  int64_t units;                  // n_res * npos * num_kb, kb fastest
  int plane_base[RNSW_MAX_RES];   // V limb planes (lo, hi)
  int uplane_base[RNSW_MAX_RES];  // bank planes (0 u_lo, 1 u_hi, 2 u'_lo, 3 u'_hi)
  FastMod fm[RNSW_MAX_RES];
  int32_t r65536[RNSW_MAX_RES];
  uint8_t* mw8;
  FastDiv div_kb, div_pos;
};

template <int NP>
struct GemmTConfig {
  static constexpr int kAPlane = 128 * kTBC;  // one U limb plane: 128 k rows
  static constexpr int kBPlane = NP * kTBC;   // one V limb plane: NP tile rows
  static constexpr int kStage = 2 * kAPlane + 2 * kBPlane;
  static constexpr int kAccCols = 3 * NP;     // D65536 | D256 | D1
  static constexpr int kNB = 2 * kAccCols <= 512 ? 2 : 1;  // accumulator buffers
  static constexpr int kStages = NP <= 80 ? 4 : 3;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kStage + 256;
  static_assert(kNB * kAccCols <= 512, "accumulators exceed TMEM");
  static_assert(kSmem <= 227 * 1024, "stages exceed shared memory");
};

template <int NP>
__global__ void __launch_bounds__(kTThreads, 1)
    winograd_gemm_t_kernel(const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmV,
                           GemmTArgs args) {
  using Cfg = GemmTConfig<NP>;
  constexpr int S = Cfg::kStages;
  constexpr int NB = Cfg::kNB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStage);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0), lane = threadIdx.x % 32;  // warp-uniform for the compiler
  pdl_trigger();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmU);
    tma_prefetch_desc(&tmV);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);  // the four epilogue warps
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();

  // unit u -> (residue, position, 128-channel block kb), kb fastest
  auto unit_coord = [&](int64_t u, int& res, int& pos, int& kb) {
    const uint32_t q = fdiv((uint32_t)u, args.div_kb);
    kb = (int)((uint32_t)u - q * args.div_kb.d);
    const uint32_t r = fdiv(q, args.div_pos);
    pos = (int)(q - r * args.div_pos.d);
    res = (int)r;
  };
  auto stage_a = [&](int s, int l) { return smem + s * Cfg::kStage + l * Cfg::kAPlane; };
  auto stage_b = [&](int s, int l) { return smem + s * Cfg::kStage + 2 * Cfg::kAPlane + l * Cfg::kBPlane; };

  if (warp == 0) {
    // ---------------- TMA producer: lanes 0-3 issue the four boxes of a stage ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t u = blockIdx.x; u < args.units; u += gridDim.x) {
      int res, pos, kb;
      unit_coord(u, res, pos, kb);
      for (int kc = 0; kc < args.nkc; ++kc) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0) mbar_arrive_expect_tx(&full[stage], (uint32_t)Cfg::kStage);
        __syncwarp();
        if (lane < 2)  // u_lo, u_hi (bank planes 0, 1): 128 output channels
          tma_load_3d(stage_a(stage, lane), &tmU, &full[stage], kc * kTBC, kb * 128,
                      (args.uplane_base[res] + lane) * args.npos + pos);
        else if (lane < 4)  // v_lo, v_hi: the tiles (rows >= P zero-filled)
          tma_load_3d(stage_b(stage, lane - 2), &tmV, &full[stage], kc * kTBC, 0,
                      (args.plane_base[res] + lane - 2) * args.npos + pos);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (warp-collective issue) ----------------
    constexpr uint32_t idesc = idesc_i8(128, NP);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int64_t u = blockIdx.x; u < args.units; u += gridDim.x, ++it) {
      const int as = it % NB;
      mbar_wait(&tempty[as], ((it / NB) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d65536 = tmem_base + as * Cfg::kAccCols, d256 = d65536 + NP, d1 = d65536 + 2 * NP;
      for (int kc = 0; kc < args.nkc; ++kc) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t a_lo = smem_u32(stage_a(stage, 0)), a_hi = smem_u32(stage_a(stage, 1));
        const uint32_t b_lo = smem_u32(stage_b(stage, 0)), b_hi = smem_u32(stage_b(stage, 1));
#pragma unroll
        for (int k = 0; k < kTBC / 32; ++k) {
          const uint32_t acc = (kc | k) != 0;
          const uint64_t dal = umma_desc_kmajor(a_lo + 32 * k, kTBC), dah = umma_desc_kmajor(a_hi + 32 * k, kTBC);
          const uint64_t dbl = umma_desc_kmajor(b_lo + 32 * k, kTBC), dbh = umma_desc_kmajor(b_hi + 32 * k, kTBC);
          mma_i8_warp(d65536, dah, dbh, idesc, acc);
          mma_i8_warp(d256, dah, dbl, idesc, acc);
          mma_i8_warp(d256, dal, dbh, idesc, 1u);
          mma_i8_warp(d1, dal, dbl, idesc, acc);
        }
        mma_commit_warp(&empty[stage]);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      mma_commit_warp(&tfull[as]);
    }
  } else {
    // ---------------- epilogue: row k = lane of quadrant warp & 3, columns = tiles ----------------
    const int q = warp & 3;
    const int krow = q * 32 + lane;
    int it = 0;
    for (int64_t u = blockIdx.x; u < args.units; u += gridDim.x, ++it) {
      int res, pos, kb;
      unit_coord(u, res, pos, kb);
      const int as = it % NB;
      mbar_wait(&tfull[as], (it / NB) & 1);
      tc_fence_after();
      const FastMod fm = args.fm[res];
      const int32_t r65536 = args.r65536[res], pb = pos_bias(fm);
      const int k = kb * 128 + krow;
      const bool kok = k < args.Kp;
      uint8_t* lo_plane = args.mw8 + mw8_offset(0, res, 0, pos, args.n_res, args.npos, args.Kp) + k;
      const int64_t plane_step = (int64_t)args.npos * 128 * args.Kp;
      const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + as * Cfg::kAccCols;
#pragma unroll
      for (int t0 = 0; t0 < NP; t0 += 16) {
        int32_t h2[16], h1[16], lo[16];
        tmem_ld16(ta + t0, h2);
        tmem_ld16(ta + NP + t0, h1);
        tmem_ld16(ta + 2 * NP + t0, lo);
        tmem_ld_wait();
        if (t0 + 16 >= NP) {  // every column of this row is in registers
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[as]);
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int t = t0 + e;
          if (kok && t < args.P) {
            const int32_t x = red_fast(h2[e], fm) * r65536 + red_fast(h1[e], fm) * 256 + lo[e];
            const int32_t y = red_pos_biased(x + pb, fm);  // y mod m in [0, m)
            lo_plane[(int64_t)t * args.Kp] = (uint8_t)(y & 255);
            lo_plane[plane_step + (int64_t)t * args.Kp] = (uint8_t)(y >> 8);
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

bool make_tmap_t(CUtensorMap* tm, const void* base, int Cp, int64_t rows, int64_t slabs, int box_rows) {
  auto encode = encode_fn();
  if (encode == nullptr) return false;
  cuuint64_t dims[3] = {(cuuint64_t)Cp, (cuuint64_t)rows, (cuuint64_t)slabs};
  cuuint64_t strides[2] = {(cuuint64_t)Cp, (cuuint64_t)(rows * Cp)};
  cuuint32_t box[3] = {(cuuint32_t)kTBC, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NP>
cudaError_t run_gemm_t(const GemmTArgs& a, const int8_t* V, const int8_t* U, int n_planes, int n_uplanes,
                       cudaStream_t s) {
  using Cfg = GemmTConfig<NP>;
  CUtensorMap tmU, tmV;
  if (!make_tmap_t(&tmU, U, a.Cp, a.K, (int64_t)n_uplanes * a.npos, 128)) return cudaErrorInvalidValue;
  if (!make_tmap_t(&tmV, V, a.Cp, a.P, (int64_t)n_planes * a.npos, NP)) return cudaErrorInvalidValue;
  auto kern = winograd_gemm_t_kernel<NP>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
  if (e != cudaSuccess) return e;
  const int64_t grid = std::min<int64_t>(a.units, num_sms_current());
  return launch_ex(kern, dim3((unsigned)grid), dim3(kTThreads), Cfg::kSmem, s, 1, tmU, tmV, a);
}

}  // namespace

bool gemm_t_ok(const PlanDevice& d, int64_t P, int Cp, bool planar, bool pos_out) {
  // RNSW_GEMM_T=0: never; =N: up to N tiles (at most 128).  Default: up to 48
  // tiles, and up to 80 for C >= 512, where streaming half the filter-bank
  // bytes outweighs the costlier N = 64 / 80 MMAs (conv5 at batch 64: 0.077
  // vs 0.106 ms; conv3 at batch 4, C = 256: 0.037 vs 0.029 ms the other way).
  // At 96-128 tiles (single-buffered accumulators) the tile-row GEMM wins.
  static const char* env = getenv("RNSW_GEMM_T");
  static const int forced = env != nullptr ? std::min(atoi(env), 128) : -1;
  const int max_p = forced >= 0 ? forced : (Cp >= 512 ? 80 : 48);
  if (!planar || !pos_out || P > max_p || Cp % kTBC != 0 || Cp > 8192 || !d.fast) return false;
  for (int r = 0; r < d.n_res; ++r)
    if (d.res[r].planes != 2) return false;
  return true;
}

cudaError_t launch_winograd_gemm_t(const PlanHost& plan, const int8_t* V, const int8_t* U, int64_t P, int Cp, int K,
                                   int Kp, int16_t* Mw, cudaStream_t s) {
  const PlanDevice& d = plan.dev;
  GemmTArgs a{};
  a.P = (int)P;
  a.K = K;
  a.Kp = Kp;
  a.Cp = Cp;
  a.npos = d.n * d.n;
  a.n_res = d.n_res;
  a.nkc = Cp / kTBC;
  a.num_kb = (Kp + 127) / 128;
  a.units = (int64_t)d.n_res * a.npos * a.num_kb;
  a.mw8 = reinterpret_cast<uint8_t*>(Mw);
  for (int r = 0; r < d.n_res; ++r) {
    const ResidueTables& t = d.res[r];
    a.plane_base[r] = t.plane_base;
    a.uplane_base[r] = t.uplane_base;
    a.fm[r] = FastMod{t.red_mul, t.red_shift, t.red_off, t.modulus, t.half, (uint32_t)(-t.modulus)};
    a.r65536[r] = t.r_65536;
  }
  a.div_kb = make_fastdiv((uint32_t)a.num_kb);
  a.div_pos = make_fastdiv((uint32_t)a.npos);
  const int np = d.n_planes, nup = d.n_uplanes;
  if (P <= 16) return run_gemm_t<16>(a, V, U, np, nup, s);
  if (P <= 32) return run_gemm_t<32>(a, V, U, np, nup, s);
  if (P <= 48) return run_gemm_t<48>(a, V, U, np, nup, s);
  if (P <= 64) return run_gemm_t<64>(a, V, U, np, nup, s);
  if (P <= 80) return run_gemm_t<80>(a, V, U, np, nup, s);
  if (P <= 96) return run_gemm_t<96>(a, V, U, np, nup, s);
  return run_gemm_t<128>(a, V, U, np, nup, s);
}

}  // namespace rnsw
