// K4-K6 on tcgen05 in Kronecker form, for two-residue 16-bit plans (tiles up
// to N = 16): the inverse transform of a residue is ONE linear map of the
// N x N Winograd-domain tile,
//     Y_r[(a,b)] = sum_(i,j) KrA_r[(a,b),(i,j)] M_r[(i,j)],  KrA_r = kron(AT_r, AT_r) mod m_r,
// so per (tile, 64 channels) and residue it is one GEMM with M = output
// pixels (a row block of <= 128), N = 64 channels, K = N*N positions
// (rw/kernel.py:50-53), followed by the mixed-radix reconstruction
// (rw/residue.py:180-206), crop/scatter (rw/layer.py:378-388) -- or the fused
// relu / shift / clip / 2x2 max-pool glue.
//
//   A = KrA_r limbs, a per-CTA constant resident in TENSOR memory: with the
//       Winograd-domain product in [0, m) as two byte planes (Mw8: lo, hi <= 16),
//       y = sum KrA (256 hi + lo) = sum (KrA' hi + KrA lo) (mod m), KrA' = 256 KrA
//       mod m, and each of KrA', KrA as balanced s8 limbs: four A matrices,
//       two accumulators  D256 = KrA'_hi hi + KrA_hi lo,  D1 = KrA'_lo hi + KrA_lo lo,
//       y = (256 D256 + D1) mod m, |256 D256 + D1| < 1.7e8 < 2^28;
//   B = the Mw8 planes of one tile, TMA-loaded (64 channels x N*N positions),
//       MN-major 64B swizzle;
//   residue 1's operator carries the mixed-radix factor W = m0^-1 mod m1, so
//       its CTA produces y1 W; the two residues of a row block run on the two
//       CTAs of a cluster, which swap half of their reduced residues through
//       distributed shared memory and each reconstructs 32 of the 64 channels:
//       d1 = (y1 W + y0 (m1 - W)) mod m1,  x = y0 + m0 d1,  signed fold.
// The outputs of a row block (a rectangle of tile rows) leave through one
// TMA bulk tensor store, which also crops edge tiles.
//
// Against the two-pass kernel (output_umma.cu: two TMEM round trips, an
// exact three-byte intermediate, CTA barriers per unit) this spends ~8x the
// tensor MACs -- the tensor pipe has the room -- and per output value only
// one reduction per residue plus the reconstruction on the CUDA cores.
// Warp roles (384 threads): 0 TMA, 1 MMA, 2 TMEM allocator, 3 bulk stores,
// 4-11 epilogue (lane quadrant x channel half); mbarriers link them, cluster-
// scope mbarriers link the two CTAs' residue exchange.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace rnsw {

namespace {

constexpr int kKThreads = 384;
constexpr int kKN = 64;     // channels per unit (MMA N)
constexpr int kKRows = 128;  // output pixels per row block (MMA M)
constexpr int kKStages = 4;
constexpr int kKStageBytes = 2 * 16384;  // two limb planes x <= 256 positions x 64 bytes

struct K4UArgs {
  Geometry g;
  int mout, npos, kp, ksteps, npb, kblocks, units, shift;
  int rb_rows[2], rb_row0[2];
  int limb_stride;      // bytes between the two limb planes of a stage
  FastMod fm[2];
  int32_t bias[2];      // m ceil(2^28 / m): n = x + bias in [0, 2^30)
  uint32_t negw;        // m1 - W (W = m0^-1 mod m1)
  uint32_t m0, signed_bound, dyn;
  FastDiv div_img, div_tw, div_kb;
  size_t a_bytes;       // per (residue, row block): 4 matrices x 128 rows x kp bytes
};

template <int kMode>
struct K4UConfig {
  static constexpr int kStgBytes = kMode == 0 ? kKRows * 32 * 4 : kKRows * 32;  // int32 / int8 staging
  static constexpr size_t kSmem = 1024 + (size_t)kKStages * kKStageBytes + 2 * kKRows * 128 /* ybuf */ +
                                  2 * (size_t)kStgBytes + 256;
};

// tile row block rb, row r (MMA M index) -> output pixel (a_local, b) of the
// block; 2x2 blocks in four consecutive rows when M is even (pooling by
// warp shuffles), row-major otherwise
__host__ __device__ inline void kron_pixel(int r, int M, bool even, int& al, int& b) {
  if (even) {
    const int blk = r >> 2, sub = r & 3, half = M >> 1;
    al = 2 * (blk / half) + (sub >> 1);
    b = 2 * (blk % half) + (sub & 1);
  } else {
    al = r / M;
    b = r % M;
  }
}

template <int kMode>
__global__ void __launch_bounds__(kKThreads, 1)
    output_kron_kernel(const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmO0,
                       const __grid_constant__ CUtensorMap tmO1, const uint8_t* __restrict__ kra, K4UArgs args) {
  using Cfg = K4UConfig<kMode>;
  constexpr int S = kKStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sB = smem;                                // [S][2 limbs][kp rows][64 bytes]
  uint8_t* ybuf = sB + S * kKStageBytes;             // [2][128 rows][64 ch x u16], 16B chunks swizzled
  uint8_t* stg = ybuf + 2 * kKRows * 128;            // [2][staging]
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + 2 * Cfg::kStgBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* yfull = tempty + 2;
  uint64_t* sfull = yfull + 2;
  uint64_t* sempty = sfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + 2);
  // ybuf[b] (here) receives the partner's residues of this CTA's
  // reconstruction channels, pushed with st.async; yfull[b] counts the bytes.
  // Reuse is safe without a return signal: the partner pushes unit it + 2
  // only after its own yfull for it + 1 completed, i.e. after this CTA
  // pushed it + 1, which every thread does after reading ybuf[b] for it.

  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0), lane = threadIdx.x % 32;  // warp-uniform for the compiler
  const int rank = (int)cluster_ctarank();  // = residue
  const int partner = rank ^ 1;
  const int cid = (int)(blockIdx.x >> 1), ncl = (int)(gridDim.x >> 1);
  const int rb = cid % args.npb;
  const int u_begin = cid / args.npb, u_step = ncl / args.npb;
  const Geometry& g = args.g;
  const int M = args.mout;
  const bool even = (M & 1) == 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmM);
    tma_prefetch_desc(rb == 0 ? &tmO0 : &tmO1);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
      mbar_init(&yfull[i], 1);
      mbar_init(&sfull[i], 8);
      mbar_init(&sempty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // the partner arrives on our barriers
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  constexpr uint32_t kAccBase = 256;  // accumulators after the four A matrices (64 columns each)

  const int q = warp & 3, hh = (warp - 4) >> 2;
  if (warp >= 4) {
    // KrA of (this residue, this row block) into TMEM: thread = row, matrices 2hh, 2hh+1
    const int row = q * 32 + lane;
    const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16);
    const uint8_t* src0 = kra + (size_t)(rank * args.npb + rb) * args.a_bytes;
    for (int mi = 2 * hh; mi < 2 * hh + 2; ++mi) {
      const uint4* src = reinterpret_cast<const uint4*>(src0 + ((size_t)mi * kKRows + row) * args.kp);
      for (int c8 = 0; c8 < args.kp / 32; ++c8) {
        const uint4 w0 = __ldg(src + 2 * c8), w1 = __ldg(src + 2 * c8 + 1);
        const uint32_t v[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        tmem_st8(trow + mi * 64 + c8 * 8, v);
      }
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  auto unit_tile = [&](int u, int& p, int& k0) {
    const int pp = (int)fdiv((uint32_t)u, args.div_kb);
    p = pp;
    k0 = (u - pp * args.kblocks) * kKN;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: the two Mw8 planes of this residue ----------------
      int stage = 0;
      uint32_t phase = 0;
      for (int u = u_begin; u < args.units; u += u_step) {
        int p, k0;
        unit_tile(u, p, k0);
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], (uint32_t)(2 * args.npos * kKN));
        uint8_t* dst = sB + stage * kKStageBytes;
        const int L0 = ((p >> 7) * 2 + rank) * 2;
        tma_load_4d(dst, &tmM, &full[stage], k0, p & 127, 0, L0);                           // lo
        tma_load_4d(dst + args.limb_stride, &tmM, &full[stage], k0, p & 127, 0, L0 + 1);    // hi
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (warp-collective) ----------------
    constexpr uint32_t idesc = idesc_i8x(128, kKN, true, false, false, true);  // s8 A (TMEM) x u8 B (MN-major)
    const uint64_t db0 = umma_desc_mn_sw64(smem_u32(sB), 16);
    constexpr uint32_t kBStep = (32 * kKN) >> 4;
    const uint32_t hi_off = (uint32_t)args.limb_stride >> 4;
    const int ksteps = args.ksteps;
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int u = u_begin; u < args.units; u += u_step, ++it) {
      const int as = it & 1;
      mbar_wait(&tempty[as], ((it >> 1) & 1) ^ 1);
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      const uint32_t d256 = tmem_base + kAccBase + as * 128, d1 = d256 + 64;
      const uint64_t dbs = db0 + (uint64_t)(stage * (kKStageBytes >> 4));
      for_ksteps(ksteps, [&](int ks) {
        const uint64_t blo = dbs + (uint64_t)(ks * kBStep), bhi = blo + hi_off;
        const uint32_t a = tmem_base + ks * 8;
        const uint32_t acc = ks > 0 ? 1u : 0u;
        mma_i8_ts_warp(d256, a, bhi, idesc, acc);        // KrA'_hi x hi
        mma_i8_ts_warp(d256, a + 64, blo, idesc, 1u);    // KrA_hi  x lo
        mma_i8_ts_warp(d1, a + 128, bhi, idesc, acc);    // KrA'_lo x hi
        mma_i8_ts_warp(d1, a + 192, blo, idesc, 1u);     // KrA_lo  x lo
      });
      mma_commit_warp(&empty[stage]);
      mma_commit_warp(&tfull[as]);
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {
      // ---------------- bulk stores of the reconstructed outputs ----------------
      const CUtensorMap* tmO = rb == 0 ? &tmO0 : &tmO1;
      const int row0 = args.rb_row0[rb];
      int it = 0;
      for (int u = u_begin; u < args.units; u += u_step, ++it) {
        int p, k0;
        unit_tile(u, p, k0);
        const int sb = it & 1;
        mbar_wait(&sfull[sb], (it >> 1) & 1);
        const int bimg = (int)fdiv((uint32_t)p, args.div_img);
        const int rem = p - bimg * (int)args.div_img.d;
        const int ti = (int)fdiv((uint32_t)rem, args.div_tw);
        const int tj = rem - ti * g.tw;
        const int kc = k0 + rank * 32;
        if (kMode == 3)
          tma_store_4d(tmO, stg + sb * Cfg::kStgBytes, kc, tj * (M / 2), ti * (M / 2) + row0 / 2, bimg);
        else
          tma_store_4d(tmO, stg + sb * Cfg::kStgBytes, kc, tj * M, ti * M + row0, bimg);
        bulk_commit();
        bulk_wait_read<0>();
        mbar_arrive(&sempty[sb]);
      }
      bulk_wait<0>();
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: 8 warps = 4 lane quadrants x 2 channel halves ----------------
    const int row = q * 32 + lane;
    const FastMod fm = args.fm[rank], fm1 = args.fm[1];
    const int32_t bias = args.bias[rank];
    const uint32_t remote_ybase = mapa_shared(smem_u32(ybuf), (uint32_t)partner);
    const uint32_t remote_yfull = mapa_shared(smem_u32(yfull), (uint32_t)partner);
    const int etid = threadIdx.x - 128;
    int al, bcol;
    kron_pixel(row, M, even, al, bcol);
    const bool valid = row < args.rb_rows[rb] * M;
    int it = 0;
    for (int u = u_begin; u < args.units; u += u_step, ++it) {
      const int as = it & 1;
      mbar_wait(&tfull[as], (it >> 1) & 1);
      tc_fence_after();
      // ---- reduce this residue's accumulators: 32 channels of this row ----
      // columns cA = this CTA's reconstruction channels (rank * 32 + hh * 16,
      // kept in registers) and cB = the partner's (published through ybuf):
      // every thread reads back only what the partner's thread (q, hh)
      // wrote, so no CTA barrier is needed around ybuf
      const uint32_t cA = (uint32_t)(rank * 32 + hh * 16), cB = (uint32_t)(partner * 32 + hh * 16);
      const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + kAccBase + as * 128;
      int32_t h0[16], l0[16], h1[16], l1[16];
      tmem_ld16(ta + cA, h0);
      tmem_ld16(ta + 64 + cA, l0);
      tmem_ld16(ta + cB, h1);
      tmem_ld16(ta + 64 + cB, l1);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);
      uint32_t own[8], pub[8];  // 16 residues each, as u16 pairs
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t y0 = (uint32_t)red_pos_biased(h0[2 * e] * 256 + l0[2 * e] + bias, fm);
        const uint32_t y1 = (uint32_t)red_pos_biased(h0[2 * e + 1] * 256 + l0[2 * e + 1] + bias, fm);
        own[e] = y0 | (y1 << 16);
        const uint32_t z0 = (uint32_t)red_pos_biased(h1[2 * e] * 256 + l1[2 * e] + bias, fm);
        const uint32_t z1 = (uint32_t)red_pos_biased(h1[2 * e + 1] * 256 + l1[2 * e + 1] + bias, fm);
        pub[e] = z0 | (z1 << 16);
      }
      // ---- push the partner's channels into its ybuf[b]; ours arrive in ours ----
      const int b = it & 1;
      if (etid == 0) mbar_arrive_expect_tx(&yfull[b], (uint32_t)(kKRows * 32 * 2));
      const uint32_t yrow = (uint32_t)(b * kKRows + row) * 128;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t chunk = (cB >> 3) + c;
        st_async_v4(remote_ybase + yrow + ((chunk ^ ((uint32_t)row & 7u)) << 4),
                    make_uint4(pub[4 * c], pub[4 * c + 1], pub[4 * c + 2], pub[4 * c + 3]), remote_yfull + 8 * b);
      }
      // ---- reconstruct channels cA..cA+15 with the partner's residues of them ----
      mbar_wait(&yfull[b], (it >> 1) & 1);
      uint4 oth[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t chunk = (cA >> 3) + c;
        oth[c] = *reinterpret_cast<const uint4*>(ybuf + yrow + ((chunk ^ ((uint32_t)row & 7u)) << 4));
      }
      const uint32_t* othw = reinterpret_cast<const uint32_t*>(oth);
      const uint32_t* w0 = rank == 0 ? own : othw;
      const uint32_t* w1 = rank == 0 ? othw : own;
      int32_t v[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const uint32_t y0 = (w0[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;   // y0 mod m0
        const uint32_t y1w = (w1[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;  // y1 W mod m1
        const uint32_t d1 = (uint32_t)red_pos_biased((int32_t)(y1w + y0 * args.negw), fm1);
        const uint32_t x = y0 + args.m0 * d1;  // in [0, D)
        if (kMode == 0)
          v[e] = x > args.signed_bound ? (int32_t)(x - args.dyn) : (int32_t)x;
        else if (kMode == 1)
          v[e] = x > args.signed_bound ? 0 : min((int32_t)(x >> args.shift), 127);
        else
          v[e] = x > args.signed_bound ? 0 : (int32_t)x;  // pooled: max first (monotone), shift after
      }
      if (kMode == 3) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          int32_t m2 = max(v[e], __shfl_xor_sync(0xffffffffu, v[e], 1));
          m2 = max(m2, __shfl_xor_sync(0xffffffffu, m2, 2));
          v[e] = min(m2 >> args.shift, 127);
        }
      }
      // ---- staging (layout of the output box) ----
      const int sb = it & 1;
      mbar_wait(&sempty[sb], ((it >> 1) & 1) ^ 1);
      uint8_t* sbuf = stg + sb * Cfg::kStgBytes;
      if (valid) {
        if (kMode == 0) {
          int4* dst = reinterpret_cast<int4*>(sbuf + ((size_t)(al * M + bcol) * 32 + hh * 16) * 4);
#pragma unroll
          for (int c = 0; c < 4; ++c) dst[c] = make_int4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
        } else {
          uint32_t pk[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) pk[c] = pack4_lo(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          if (kMode == 1) {
            *reinterpret_cast<uint4*>(sbuf + (al * M + bcol) * 32 + hh * 16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          } else if ((row & 3) == 0) {
            *reinterpret_cast<uint4*>(sbuf + ((al >> 1) * (M >> 1) + (bcol >> 1)) * 32 + hh * 16) =
                make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfull[sb]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
  cluster_sync();  // the partner may still read our ybuf / arrive on our barriers until here
}


// ---------------------------------------------------------------------------
// 8-bit residues (one s8 limb per constant, one u8 plane per residue): every
// residue of a row block in ONE CTA (A_r = KrA_r W[r][0] mod m_r resident in
// TMEM, 64 columns each; accumulators n_res x 32 columns, double-buffered),
// units of one tile x 32 channels, and the mixed-radix digits folded into the
// reductions: d_j = (acc_j + sum_{i<j} d_i (m_j - W[j][i])) mod m_j.
constexpr int kK8N = 32;

struct K48Args {
  Geometry g;
  int mout, npos, kp, ksteps, npb, kblocks, units, shift, nres;
  int rb_rows[2], rb_row0[2];
  int res_stride;       // bytes between the residues' planes in a stage
  FastMod fm[RNSW_MAX_RES];
  int32_t bias[RNSW_MAX_RES];        // m ceil(2^24 / m)
  uint32_t c[RNSW_MAX_RES][RNSW_MAX_RES];  // m_j - W[j][i], i < j
  uint32_t m[RNSW_MAX_RES];
  uint32_t signed_bound, dyn;
  FastDiv div_img, div_tw, div_kb;
  size_t a_bytes;       // per row block: n_res x 128 rows x kp bytes
};

template <int kMode>
struct K48Config {
  static constexpr int kStages = 6;
  static constexpr int kStageBytes = RNSW_MAX_RES * 8192;  // <= 4 residues x 256 positions x 32 bytes
  static constexpr int kStgBytes = kMode == 0 ? kKRows * 32 * 4 : kKRows * 32;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kStageBytes + 2 * (size_t)kStgBytes + 256;
};

template <int kMode, int kNRes>
__global__ void __launch_bounds__(kKThreads, 1)
    output_kron8_kernel(const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmO0,
                        const __grid_constant__ CUtensorMap tmO1, const uint8_t* __restrict__ kra, K48Args args) {
  using Cfg = K48Config<kMode>;
  constexpr int S = Cfg::kStages;
  constexpr uint32_t kAccBase = kNRes * 64, kAccCols = kNRes * kK8N;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sB = smem;
  uint8_t* stg = sB + S * Cfg::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + 2 * Cfg::kStgBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + 2);

  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0), lane = threadIdx.x % 32;  // warp-uniform for the compiler
  const int rb = (int)(blockIdx.x % args.npb);
  const int u_begin = (int)(blockIdx.x / args.npb), u_step = (int)(gridDim.x / args.npb);
  const Geometry& g = args.g;
  const int M = args.mout;
  const bool even = (M & 1) == 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmM);
    tma_prefetch_desc(rb == 0 ? &tmO0 : &tmO1);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
      mbar_init(&sfull[i], 8);
      mbar_init(&sempty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int q = warp & 3, hh = (warp - 4) >> 2;
  if (warp >= 4) {
    // A_r of this row block into TMEM: thread = row; residues split over hh
    const int row = q * 32 + lane;
    const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16);
    const uint8_t* src0 = kra + (size_t)rb * args.a_bytes;
    for (int r = hh; r < kNRes; r += 2) {
      const uint4* src = reinterpret_cast<const uint4*>(src0 + ((size_t)r * kKRows + row) * args.kp);
      for (int c8 = 0; c8 < args.kp / 32; ++c8) {
        const uint4 w0 = __ldg(src + 2 * c8), w1 = __ldg(src + 2 * c8 + 1);
        const uint32_t v[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        tmem_st8(trow + r * 64 + c8 * 8, v);
      }
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  auto unit_tile = [&](int u, int& p, int& k0) {
    const int pp = (int)fdiv((uint32_t)u, args.div_kb);
    p = pp;
    k0 = (u - pp * args.kblocks) * kK8N;
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = u_begin; u < args.units; u += u_step) {
        int p, k0;
        unit_tile(u, p, k0);
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], (uint32_t)(kNRes * args.npos * kK8N));
        uint8_t* dst = sB + stage * Cfg::kStageBytes;
#pragma unroll
        for (int r = 0; r < kNRes; ++r)
          tma_load_4d(dst + r * args.res_stride, &tmM, &full[stage], k0, p & 127, 0, (p >> 7) * kNRes + r);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_i8x(128, kK8N, true, false, false, true);  // s8 A (TMEM) x u8 B (MN-major)
    const uint64_t db0 = umma_desc_mn_sw32(smem_u32(sB), 16);
    const uint32_t rstep = (uint32_t)args.res_stride >> 4;
    const int ksteps = args.ksteps;
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int u = u_begin; u < args.units; u += u_step, ++it) {
      const int as = it & 1;
      mbar_wait(&tempty[as], ((it >> 1) & 1) ^ 1);
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      const uint32_t d0 = tmem_base + kAccBase + as * kAccCols;
      const uint64_t dbs = db0 + (uint64_t)(stage * (Cfg::kStageBytes >> 4));
      for_ksteps(ksteps, [&](int ks) {
#pragma unroll
        for (int r = 0; r < kNRes; ++r)
          mma_i8_ts_warp(d0 + r * kK8N, tmem_base + r * 64 + ks * 8,
                         dbs + (uint64_t)(r * rstep + ks * ((32 * kK8N) >> 4)), idesc, ks > 0 ? 1u : 0u);
      });
      mma_commit_warp(&empty[stage]);
      mma_commit_warp(&tfull[as]);
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {
      const CUtensorMap* tmO = rb == 0 ? &tmO0 : &tmO1;
      const int row0 = args.rb_row0[rb];
      int it = 0;
      for (int u = u_begin; u < args.units; u += u_step, ++it) {
        int p, k0;
        unit_tile(u, p, k0);
        const int sb = it & 1;
        mbar_wait(&sfull[sb], (it >> 1) & 1);
        const int bimg = (int)fdiv((uint32_t)p, args.div_img);
        const int rem = p - bimg * (int)args.div_img.d;
        const int ti = (int)fdiv((uint32_t)rem, args.div_tw);
        const int tj = rem - ti * g.tw;
        if (kMode == 3)
          tma_store_4d(tmO, stg + sb * Cfg::kStgBytes, k0, tj * (M / 2), ti * (M / 2) + row0 / 2, bimg);
        else
          tma_store_4d(tmO, stg + sb * Cfg::kStgBytes, k0, tj * M, ti * M + row0, bimg);
        bulk_commit();
        bulk_wait_read<0>();
        mbar_arrive(&sempty[sb]);
      }
      bulk_wait<0>();
    }
  } else if (warp >= 4) {
    const int row = q * 32 + lane;
    int al, bcol;
    kron_pixel(row, M, even, al, bcol);
    const bool valid = row < args.rb_rows[rb] * M;
    int it = 0;
    for (int u = u_begin; u < args.units; u += u_step, ++it) {
      const int as = it & 1;
      mbar_wait(&tfull[as], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + kAccBase + as * kAccCols + hh * 16;
      int32_t acc[kNRes][16];
#pragma unroll
      for (int r = 0; r < kNRes; ++r) tmem_ld16(ta + r * kK8N, acc[r]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);
      int32_t v[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        uint32_t d[kNRes];
        uint32_t x = 0, w = 1;
#pragma unroll
        for (int j = 0; j < kNRes; ++j) {
          uint32_t n = (uint32_t)(acc[j][e] + args.bias[j]);
#pragma unroll
          for (int i = 0; i < j; ++i) n += d[i] * args.c[j][i];
          d[j] = (uint32_t)red_pos_biased((int32_t)n, args.fm[j]);
          x += d[j] * w;
          w *= args.m[j];
        }
        if (kMode == 0)
          v[e] = x > args.signed_bound ? (int32_t)(x - args.dyn) : (int32_t)x;
        else if (kMode == 1)
          v[e] = x > args.signed_bound ? 0 : min((int32_t)(x >> args.shift), 127);
        else
          v[e] = x > args.signed_bound ? 0 : (int32_t)x;
      }
      if (kMode == 3) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          int32_t m2 = max(v[e], __shfl_xor_sync(0xffffffffu, v[e], 1));
          m2 = max(m2, __shfl_xor_sync(0xffffffffu, m2, 2));
          v[e] = min(m2 >> args.shift, 127);
        }
      }
      const int sb = it & 1;
      mbar_wait(&sempty[sb], ((it >> 1) & 1) ^ 1);
      uint8_t* sbuf = stg + sb * Cfg::kStgBytes;
      if (valid) {
        if (kMode == 0) {
          int4* dst = reinterpret_cast<int4*>(sbuf + ((size_t)(al * M + bcol) * 32 + hh * 16) * 4);
#pragma unroll
          for (int c = 0; c < 4; ++c) dst[c] = make_int4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
        } else {
          uint32_t pk[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) pk[c] = pack4_lo(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          if (kMode == 1) {
            *reinterpret_cast<uint4*>(sbuf + (al * M + bcol) * 32 + hh * 16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          } else if ((row & 3) == 0) {
            *reinterpret_cast<uint4*>(sbuf + ((al >> 1) * (M >> 1) + (bcol >> 1)) * 32 + hh * 16) =
                make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfull[sb]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

int64_t symh(int64_t v, int64_t m) {
  v %= m;
  if (v < 0) v += m;
  return v > (m - 1) / 2 ? v - m : v;
}

}  // namespace

// Row blocks of a tile for the Kronecker output transform: whole tile rows,
// <= 128 pixels, an even number of rows (2x2 pooling stays inside a block).
static void kron_blocks(int M, int& npb, int rows[2], int row0[2]) {
  if (M * M <= kKRows) {
    npb = 1;
    rows[0] = M;
    row0[0] = 0;
    rows[1] = 0;
    row0[1] = M;
    return;
  }
  int r = kKRows / M;
  r &= ~1;
  npb = 2;
  rows[0] = r;
  row0[0] = 0;
  rows[1] = M - r;
  row0[1] = r;
}

cudaError_t build_kra_images(PlanHost& plan) {
  const PlanDevice& d = plan.dev;
  plan.d_kra = nullptr;
  if (!d.fast || d.n > 16 || d.n_res != 2 || d.res[0].planes != 2 || d.res[1].planes != 2) return cudaSuccess;
  const int N = d.n, M = d.m_out, npos = N * N;
  int npb, rows[2], row0[2];
  kron_blocks(M, npb, rows, row0);
  if (npb > 2 || rows[1] > kKRows / M) return cudaSuccess;
  plan.kra_npb = npb;
  plan.kra_kp = (npos + 31) / 32 * 32;
  plan.kra_bytes = (size_t)4 * kKRows * plan.kra_kp;
  std::vector<uint8_t> img((size_t)2 * npb * plan.kra_bytes, 0);
  const bool even = (M & 1) == 0;
  for (int r = 0; r < 2; ++r) {
    const int64_t m = d.res[r].modulus;
    const int64_t w = r == 0 ? 1 : d.mrc_w[1][0];
    for (int rb = 0; rb < npb; ++rb) {
      uint8_t* gimg = img.data() + (size_t)(r * npb + rb) * plan.kra_bytes;
      for (int row = 0; row < rows[rb] * M; ++row) {
        int al, b;
        kron_pixel(row, M, even, al, b);
        const int a = row0[rb] + al;
        for (int pos = 0; pos < npos; ++pos) {
          const int i = pos / N, j = pos % N;
          const int64_t v = symh((int64_t)d.res[r].at[a * RNSW_MAX_N + i] * d.res[r].at[b * RNSW_MAX_N + j] % m * w, m);
          const int64_t vp = symh(v * 256, m);
          auto hi = [](int64_t c) { return (c + 128 + 256 * 64) / 256 - 64; };  // floor((c + 128) / 256)
          const int8_t limbs[4] = {(int8_t)hi(vp), (int8_t)hi(v), (int8_t)(vp - 256 * hi(vp)),
                                   (int8_t)(v - 256 * hi(v))};
          for (int mi = 0; mi < 4; ++mi)
            gimg[((size_t)mi * kKRows + row) * plan.kra_kp + pos] = (uint8_t)limbs[mi];
        }
      }
    }
  }
  cudaError_t e = cudaMalloc(&plan.d_kra, img.size());
  if (e != cudaSuccess) {
    plan.d_kra = nullptr;
    return e;
  }
  e = cudaMemcpy(plan.d_kra, img.data(), img.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(plan.d_kra);
    plan.d_kra = nullptr;
  }
  return e;
}

void free_kra_images(PlanHost& plan) {
  if (plan.d_kra) cudaFree(plan.d_kra);
  plan.d_kra = nullptr;
  if (plan.d_kra8) cudaFree(plan.d_kra8);
  plan.d_kra8 = nullptr;
}

// 8-bit plans: A_r = kron(AT_r, AT_r) W[r][0] mod m_r (W[0][0] = 1), one s8
// matrix per residue and row block, [rb][res][128 rows][kp].
cudaError_t build_kra8_images(PlanHost& plan) {
  const PlanDevice& d = plan.dev;
  plan.d_kra8 = nullptr;
  if (!d.fast || d.n > 16 || d.n_res < 1 || d.n_res > 4) return cudaSuccess;
  for (int r = 0; r < d.n_res; ++r)
    if (d.res[r].planes != 1) return cudaSuccess;
  const int N = d.n, M = d.m_out, npos = N * N;
  int npb, rows[2], row0[2];
  kron_blocks(M, npb, rows, row0);
  plan.kra8_npb = npb;
  plan.kra8_kp = (npos + 31) / 32 * 32;
  plan.kra8_bytes = (size_t)d.n_res * kKRows * plan.kra8_kp;
  std::vector<uint8_t> img((size_t)npb * plan.kra8_bytes, 0);
  const bool even = (M & 1) == 0;
  for (int rb = 0; rb < npb; ++rb)
    for (int r = 0; r < d.n_res; ++r) {
      const int64_t m = d.res[r].modulus;
      const int64_t w = r == 0 ? 1 : d.mrc_w[r][0];
      uint8_t* gimg = img.data() + (size_t)rb * plan.kra8_bytes + (size_t)r * kKRows * plan.kra8_kp;
      for (int row = 0; row < rows[rb] * M; ++row) {
        int al, b;
        kron_pixel(row, M, even, al, b);
        const int a = row0[rb] + al;
        for (int pos = 0; pos < npos; ++pos) {
          const int i = pos / N, j = pos % N;
          const int64_t v =
              symh((int64_t)d.res[r].at[a * RNSW_MAX_N + i] * d.res[r].at[b * RNSW_MAX_N + j] % m * w, m);
          gimg[(size_t)row * plan.kra8_kp + pos] = (uint8_t)(int8_t)v;
        }
      }
    }
  cudaError_t e = cudaMalloc(&plan.d_kra8, img.size());
  if (e != cudaSuccess) {
    plan.d_kra8 = nullptr;
    return e;
  }
  e = cudaMemcpy(plan.d_kra8, img.data(), img.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(plan.d_kra8);
    plan.d_kra8 = nullptr;
  }
  return e;
}

bool kron8_output_ok(const PlanHost& plan, const Geometry& g, int mode) {
  static const bool off = getenv("RNSW_K4_TWO_PASS") != nullptr;
  if (off || force_generic() || plan.d_kra8 == nullptr) return false;
  if (smallc_ok(plan.dev, g)) return false;  // the C <= 4 product writes the int16 layout
  if (mode == 0) return g.layout == 0 && (g.K % 4) == 0;
  return (g.K % 16) == 0;
}

bool kron_output_ok(const PlanHost& plan, const Geometry& g, int mode) {
  static const bool off = getenv("RNSW_K4_TWO_PASS") != nullptr;  // A/B switch: the two-pass kernels
  static const bool force = getenv("RNSW_K4_KRON") != nullptr;    // A/B switch: also for F(14x14, 3x3)
  if (kron8_output_ok(plan, g, mode)) return true;
  if (off || force_generic() || plan.d_kra == nullptr) return false;
  // F(14x14, 3x3): the two-pass tcgen05 kernel (output_umma.cu) is faster --
  // per output value it folds the residue reductions into the mixed-radix
  // digits (two reductions instead of three) and wastes fewer MMA rows (196
  // pixels need 256 Kronecker rows)
  if (umma_output_ok(plan.dev) && !force) return false;
  if (mode == 0) return g.layout == 0 && (g.K % 4) == 0;
  return (g.K % 16) == 0;
}

static cudaError_t launch_kron8(const PlanHost& plan, const Geometry& g, const uint8_t* Mw8, int32_t* y,
                                cudaStream_t s, int8_t* out8, int shift, int pool);

cudaError_t launch_output_transform_kron(const PlanHost& plan, const Geometry& g, const uint8_t* Mw8, int32_t* y,
                                         cudaStream_t s, int8_t* out8, int shift, int pool) {
  const PlanDevice& d = plan.dev;
  if (plan.d_kra8 != nullptr) return launch_kron8(plan, g, Mw8, y, s, out8, shift, pool);
  K4UArgs a{};
  a.g = g;
  a.mout = d.m_out;
  a.npos = d.n * d.n;
  a.kp = plan.kra_kp;
  a.ksteps = a.kp / 32;
  kron_blocks(d.m_out, a.npb, a.rb_rows, a.rb_row0);
  a.kblocks = (g.K + kKN - 1) / kKN;
  const int64_t units = g.P * a.kblocks;
  if (units >= (1ll << 31) || g.P >= (1ll << 31)) return cudaErrorInvalidValue;
  a.units = (int)units;
  a.shift = shift;
  a.limb_stride = (a.kp * kKN + 1023) / 1024 * 1024;
  for (int r = 0; r < 2; ++r) {
    const ResidueTables& t = d.res[r];
    a.fm[r] = FastMod{t.red_mul, t.red_shift, t.red_off, t.modulus, t.half, t.red_negm};
    a.bias[r] = (int32_t)(t.modulus * (((1ll << 28) + t.modulus - 1) / t.modulus));
  }
  a.negw = (uint32_t)(d.res[1].modulus - d.mrc_w[1][0]);
  a.m0 = (uint32_t)d.res[0].modulus;
  a.signed_bound = (uint32_t)d.signed_bound;
  a.dyn = (uint32_t)d.dynamic_range;
  a.div_img = make_fastdiv((uint32_t)(g.th * g.tw));
  a.div_tw = make_fastdiv((uint32_t)g.tw);
  a.div_kb = make_fastdiv((uint32_t)a.kblocks);
  a.a_bytes = plan.kra_bytes;

  auto encode = encode_fn();
  if (encode == nullptr) return cudaErrorInvalidValue;
  const int64_t num_pb = (g.P + 127) / 128;
  CUtensorMap tmM, tmO0, tmO1;
  {
    // Mw8 as (Kp, 128 tiles, npos, L = (pb * 2 + res) * 2 + limb); box = 64 channels x 1 tile x npos x 1
    cuuint64_t dims[4] = {(cuuint64_t)g.Kp, 128, (cuuint64_t)a.npos, (cuuint64_t)(num_pb * 4)};
    cuuint64_t strides[3] = {(cuuint64_t)g.Kp, (cuuint64_t)g.Kp * 128, (cuuint64_t)g.Kp * 128 * a.npos};
    cuuint32_t box[4] = {(cuuint32_t)kKN, 1, (cuuint32_t)a.npos, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (encode(&tmM, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(Mw8), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int mode = out8 == nullptr ? 0 : (pool ? 3 : 1);
  {
    // output NHWC as (K, Wo', Ho', B); box = 32 channels x tile columns x block rows x 1
    const int esz = mode == 0 ? 4 : 1;
    const int Wo = mode == 3 ? g.Wo / 2 : g.Wo, Ho = mode == 3 ? g.Ho / 2 : g.Ho;
    const int bw = mode == 3 ? d.m_out / 2 : d.m_out;
    void* base = mode == 0 ? static_cast<void*>(y) : static_cast<void*>(out8);
    cuuint64_t dims[4] = {(cuuint64_t)g.K, (cuuint64_t)Wo, (cuuint64_t)Ho, (cuuint64_t)g.B};
    cuuint64_t strides[3] = {(cuuint64_t)g.K * esz, (cuuint64_t)Wo * g.K * esz, (cuuint64_t)Ho * Wo * g.K * esz};
    cuuint32_t es[4] = {1, 1, 1, 1};
    for (int rb = 0; rb < a.npb; ++rb) {
      const int bh = mode == 3 ? a.rb_rows[rb] / 2 : a.rb_rows[rb];
      cuuint32_t box[4] = {32, (cuuint32_t)bw, (cuuint32_t)bh, 1};
      if (encode(rb == 0 ? &tmO0 : &tmO1, mode == 0 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 4,
                 base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
    if (a.npb == 1) tmO1 = tmO0;
  }
  const int sms = num_sms_current();
  int ncl = sms / 2;
  ncl = ncl / a.npb * a.npb;
  const int64_t need = (int64_t)a.units * a.npb;
  if (ncl > need) ncl = (int)need;
  if (ncl < a.npb) ncl = a.npb;
  auto run = [&](auto kern, size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * ncl));
    cfg.blockDim = dim3(kKThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, tmM, tmO0, tmO1, (const uint8_t*)plan.d_kra, a);
  };
  if (mode == 0) return run(output_kron_kernel<0>, K4UConfig<0>::kSmem);
  if (mode == 1) return run(output_kron_kernel<1>, K4UConfig<1>::kSmem);
  return run(output_kron_kernel<3>, K4UConfig<3>::kSmem);
}

static cudaError_t launch_kron8(const PlanHost& plan, const Geometry& g, const uint8_t* Mw8, int32_t* y,
                                cudaStream_t s, int8_t* out8, int shift, int pool) {
  const PlanDevice& d = plan.dev;
  K48Args a{};
  a.g = g;
  a.mout = d.m_out;
  a.npos = d.n * d.n;
  a.kp = plan.kra8_kp;
  a.ksteps = a.kp / 32;
  a.nres = d.n_res;
  kron_blocks(d.m_out, a.npb, a.rb_rows, a.rb_row0);
  a.kblocks = (g.K + kK8N - 1) / kK8N;
  const int64_t units = g.P * a.kblocks;
  if (units >= (1ll << 31) || g.P >= (1ll << 31)) return cudaErrorInvalidValue;
  a.units = (int)units;
  a.shift = shift;
  a.res_stride = (a.kp * kK8N + 1023) / 1024 * 1024;
  for (int j = 0; j < d.n_res; ++j) {
    const ResidueTables& t = d.res[j];
    a.fm[j] = FastMod{t.red_mul, t.red_shift, t.red_off, t.modulus, t.half, t.red_negm};
    a.bias[j] = (int32_t)(t.modulus * (((1ll << 24) + t.modulus - 1) / t.modulus));
    a.m[j] = (uint32_t)t.modulus;
    for (int i = 0; i < j; ++i) a.c[j][i] = (uint32_t)((t.modulus - d.mrc_w[j][i]) % t.modulus);
  }
  a.signed_bound = (uint32_t)d.signed_bound;
  a.dyn = (uint32_t)d.dynamic_range;
  a.div_img = make_fastdiv((uint32_t)(g.th * g.tw));
  a.div_tw = make_fastdiv((uint32_t)g.tw);
  a.div_kb = make_fastdiv((uint32_t)a.kblocks);
  a.a_bytes = plan.kra8_bytes;

  auto encode = encode_fn();
  if (encode == nullptr) return cudaErrorInvalidValue;
  const int64_t num_pb = (g.P + 127) / 128;
  CUtensorMap tmM, tmO0, tmO1;
  {
    // 8-bit Mw8 as (Kp, 128 tiles, npos, pb * n_res + res); box = 32 channels x 1 x npos x 1
    cuuint64_t dims[4] = {(cuuint64_t)g.Kp, 128, (cuuint64_t)a.npos, (cuuint64_t)(num_pb * d.n_res)};
    cuuint64_t strides[3] = {(cuuint64_t)g.Kp, (cuuint64_t)g.Kp * 128, (cuuint64_t)g.Kp * 128 * a.npos};
    cuuint32_t box[4] = {(cuuint32_t)kK8N, 1, (cuuint32_t)a.npos, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (encode(&tmM, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(Mw8), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int mode = out8 == nullptr ? 0 : (pool ? 3 : 1);
  {
    const int esz = mode == 0 ? 4 : 1;
    const int Wo = mode == 3 ? g.Wo / 2 : g.Wo, Ho = mode == 3 ? g.Ho / 2 : g.Ho;
    const int bw = mode == 3 ? d.m_out / 2 : d.m_out;
    void* base = mode == 0 ? static_cast<void*>(y) : static_cast<void*>(out8);
    cuuint64_t dims[4] = {(cuuint64_t)g.K, (cuuint64_t)Wo, (cuuint64_t)Ho, (cuuint64_t)g.B};
    cuuint64_t strides[3] = {(cuuint64_t)g.K * esz, (cuuint64_t)Wo * g.K * esz, (cuuint64_t)Ho * Wo * g.K * esz};
    cuuint32_t es[4] = {1, 1, 1, 1};
    for (int rb = 0; rb < a.npb; ++rb) {
      const int bh = mode == 3 ? a.rb_rows[rb] / 2 : a.rb_rows[rb];
      cuuint32_t box[4] = {32, (cuuint32_t)bw, (cuuint32_t)bh, 1};
      if (encode(rb == 0 ? &tmO0 : &tmO1, mode == 0 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 4,
                 base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
    if (a.npb == 1) tmO1 = tmO0;
  }
  const int sms = num_sms_current();
  int64_t grid = sms / a.npb * a.npb;
  const int64_t need = (int64_t)a.units * a.npb;
  if (grid > need) grid = need;
  if (grid < a.npb) grid = a.npb;
  auto run = [&](auto kern, size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, kKThreads, smem, s>>>(tmM, tmO0, tmO1, (const uint8_t*)plan.d_kra8, a);
    return cudaGetLastError();
  };
#define RNSW_K48(NR)                                                                       \
  if (d.n_res == NR) {                                                                     \
    if (mode == 0) return run(output_kron8_kernel<0, NR>, K48Config<0>::kSmem);             \
    if (mode == 1) return run(output_kron8_kernel<1, NR>, K48Config<1>::kSmem);             \
    return run(output_kron8_kernel<3, NR>, K48Config<3>::kSmem);                            \
  }
  RNSW_K48(1)
  RNSW_K48(2)
  RNSW_K48(3)
  RNSW_K48(4)
#undef RNSW_K48
  return cudaErrorInvalidValue;
}

}  // namespace rnsw
