// K3: the Winograd-domain contraction on the 5th-generation tensor cores.
//
// For every residue r and transform position pos the reference computes
//     acc[pos] = (V[pos] (P x C)  @  U[pos] (C x K))  mod m_r
// with int32 accumulation reduced every accumulation_chunk(m) channels
// (rw/layer.py:251-263, 285-291; rw/gemm.py:43-97).  Here one persistent,
// warp-specialised kernel runs all (residue, position, P-block, K-block)
// tiles:
//   warp 0      TMA producer: V and U limb planes -> 128B/64B/32B-swizzled smem
//   warp 1      MMA issuer:   tcgen05.mma.cta_group::1.kind::i8, s32 in TMEM
//   warp 2      TMEM allocator
//   warps 4-11  epilogue:     tcgen05.ld -> limb recombination -> mod m -> int16
//                             -> swizzled smem staging -> TMA bulk tensor store
// TMEM holds two accumulator sets so the epilogue of tile i overlaps the
// MMAs of tile i+1.  16-bit plans with >= 2 tile blocks run as CTA pairs
// (clusters of 2) that multicast the filter-bank planes (see the kernel).
// Output: Mw in blocks of 128 tiles (kernels.h mw_offset).
//
// 16-bit moduli: V residues are two s8 planes v = 256*v_hi + v_lo; the
// filter bank holds the limbs of u and of u' = 256*u mod m.  Then
//     v*u = v_hi*256*u + v_lo*u  ==  v_hi*u' + v_lo*u               (mod m)
//         == 256*(v_hi*u'_hi + v_lo*u_hi) + (v_hi*u'_lo + v_lo*u_lo)
// so each k-step issues 2 MMAs of N = 2*BN ([u'_hi;u'_lo] and [u_hi;u_lo]
// stacked in smem) into the adjacent accumulators [A256 | A1]; the epilogue
// recombines 256*A256 + A1 (< 2^28 for C <= 512) with a single exact
// reduction.  |acc| <= C * 128^2 < 2^31 for C <= 131071 (host-checked).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

// 1: the whole-layer 16-bit epilogue is software-pipelined by 16-column chunks
#ifndef RNSW_GEMM_EPI_PIPE
#define RNSW_GEMM_EPI_PIPE 1
#endif


namespace rnsw {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

namespace {

constexpr int kBlockM = 128;  // tiles (P) per MMA tile: TMEM lanes
constexpr int kThreads = 384;  // warps 0-3 producer/MMA/alloc/idle, 4-11 epilogue

struct GemmArgs {
  int64_t P;
  int K, Kp, Cp, npos, n_res;
  int num_pb, num_kb, nkc;
  int64_t total_tiles;
  int planes[RNSW_MAX_RES];
  int plane_base[RNSW_MAX_RES];   // V planes
  int uplane_base[RNSW_MAX_RES];  // filter-bank planes (4 per 16-bit residue)
  int modulus[RNSW_MAX_RES];
  float inv_m[RNSW_MAX_RES];
  int r256[RNSW_MAX_RES];
  int r65536[RNSW_MAX_RES];
  FastMod fm[RNSW_MAX_RES];
  int fast;   // exact division-free reductions apply (plan.fast and C <= 8192)
  int fast2;  // additionally C <= 512: 256*A256 + A1 needs a single reduction
  int pos_out;  // fast2 16-bit residues written as y mod m in [0, m) (the output
                // transform's limb split accepts it; saves the symmetric shift)
  int16_t* Mw;
  int64_t mw8_plane;  // bytes between the two limb planes of one (tile block, residue, position) (Mw8)
  int planar;  // pos_out residues as two byte planes (Mw8, kernels.h) for the tcgen05 output transform
  FastDiv div_kb, div_pb, div_pos;  // work-tile index decomposition (total_tiles < 2^31)
};

// work tile t -> (kb fastest, pb, pos, res) without 64-bit divisions
struct TileCoord {
  int kb, pb, pos, res;
};
RNSW_DEV TileCoord tile_coord(uint32_t t, const GemmArgs& a) {
  TileCoord c;
  uint32_t q = fdiv(t, a.div_kb);
  c.kb = (int)(t - q * a.div_kb.d);
  t = q;
  q = fdiv(t, a.div_pb);
  c.pb = (int)(t - q * a.div_pb.d);
  t = q;
  q = fdiv(t, a.div_pos);
  c.pos = (int)(t - q * a.div_pos.d);
  c.res = (int)q;
  return c;
}

// MAXPL: 1 = 8-bit residues (one plane each side); 2 = 16-bit residues with
// the four-plane filter bank (u, u' = 256 u mod m: two accumulators); 3 =
// 16-bit residues reading only the u planes of the bank (three accumulators
// A65536 | A256 | A1, four N = BN MMAs per k-step): half the filter-bank
// bytes, for the layers whose bank stream dominates (small P).
template <int BN, int MAXPL>
struct GemmTraits {
  static constexpr int kAccCols = (MAXPL == 1 ? 1 : MAXPL == 2 ? 2 : 3) * BN;  // TMEM columns per accumulator set
  static constexpr int kTmemCols = (2 * kAccCols <= 32) ? 32
                                   : (2 * kAccCols <= 64) ? 64
                                   : (2 * kAccCols <= 128) ? 128
                                   : (2 * kAccCols <= 256) ? 256 : 512;
  static_assert(2 * kAccCols <= 512, "accumulators exceed TMEM");
};

constexpr int a_planes(int maxpl) { return maxpl == 1 ? 1 : 2; }
constexpr int b_planes(int maxpl) { return maxpl == 1 ? 1 : (maxpl == 2 ? 4 : 2); }

template <int BC>
constexpr int stage_bytes(int bn, int maxpl) {
  // A: V planes (1 or 2); B: filter-bank planes (1, 4, or 2)
  return a_planes(maxpl) * kBlockM * BC + b_planes(maxpl) * bn * BC;
}

template <int BN, int BC, int MAXPL, bool TS = true, int SB = 1, bool CG2 = false>
struct GemmConfig {
  // CG2 (CTA pair, cta_group::2): each CTA stages its two V planes and two of
  // the four filter planes (its N half of both MMAs' B operands)
  static constexpr int kStageBytes = CG2 ? 2 * kBlockM * BC + 2 * BN * BC : stage_bytes<BC>(BN, MAXPL);
  // BN <= 128: the epilogue stages each output tile in shared memory (int16,
  // 128B-swizzled boxes of 64 columns) and writes it with TMA bulk tensor
  // stores; per-thread 16-byte stores of 128 scattered rows were the GEMM's
  // bottleneck (profiles/r01_gemm_*).  BN = 256 (8-bit) keeps direct stores.
  static constexpr bool kTmaStore = TS && BN <= 128;
  // SB staging tiles: with 2, tile i's bulk store drains while tile i+1 is
  // staged (chosen when a work tile has few K chunks, so the operand stages
  // it costs matter less)
  static constexpr int kStoreTile = kBlockM * BN * 2;
  static constexpr int kStoreBufs = SB;
  static constexpr int kStoreBytes = kTmaStore ? kStoreBufs * kStoreTile : 0;
  static constexpr int kStagesRaw = (224 * 1024 - kStoreBytes) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kAPlaneBytes = kBlockM * BC;
  static constexpr int kBPlaneBytes = BN * BC;
  static constexpr size_t kSmemBytes =
      1024 /*align slack*/ + (size_t)kStages * kStageBytes + kStoreBytes + 256 /*barriers*/;
};

// one output row (tile) of 16 int16 residues into the staging tile: box
// col / 64, 128-byte rows, 16-byte chunk c at c ^ (row & 7) (TMA SWIZZLE_128B)
RNSW_DEV void sts16_swz(uint8_t* stg, int row, int col, const int32_t (&r)[16]) {
  uint32_t w[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) w[e] = __byte_perm((uint32_t)r[2 * e], (uint32_t)r[2 * e + 1], 0x5410);
  uint8_t* box = stg + (col >> 6) * (kBlockM * 128) + row * 128;
  const int c = (col & 63) >> 3;
  *reinterpret_cast<uint4*>(box + (((c) ^ (row & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
  *reinterpret_cast<uint4*>(box + (((c + 1) ^ (row & 7)) << 4)) = make_uint4(w[4], w[5], w[6], w[7]);
}

// Planar variant (Mw8): the low and high bytes of 16 residues [0, m) into
// the two plane tiles of the staging buffer (BN-byte rows; 128B swizzle for
// BN = 128, 64B swizzle for BN = 64, matching the store tensor map).
template <int BN>
RNSW_DEV void sts8x2_swz(uint8_t* stg, int row, int col, const int32_t (&r)[16]) {
  uint32_t lo[4], hi[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t a = __byte_perm((uint32_t)r[4 * e], (uint32_t)r[4 * e + 1], 0x5140);
    const uint32_t b = __byte_perm((uint32_t)r[4 * e + 2], (uint32_t)r[4 * e + 3], 0x5140);
    lo[e] = __byte_perm(a, b, 0x5410);
    hi[e] = __byte_perm(a, b, 0x7632);
  }
  uint32_t off = row * BN + col;
  off = BN == 128 ? swz128(off) : (off ^ (((off >> 7) & 3u) << 4));
  *reinterpret_cast<uint4*>(stg + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  *reinterpret_cast<uint4*>(stg + kBlockM * BN + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
}

// 8-bit residues [0, m) as ONE byte plane (the 8-bit Mw8, kernels.h mw8s_offset).
template <int BN>
RNSW_DEV void sts8_swz(uint8_t* stg, int row, int col, const int32_t (&r)[16]) {
  uint32_t w[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) w[e] = pack4_lo(r[4 * e], r[4 * e + 1], r[4 * e + 2], r[4 * e + 3]);
  uint32_t off = row * BN + col;
  off = BN == 128 ? swz128(off) : (off ^ (((off >> 7) & 3u) << 4));
  *reinterpret_cast<uint4*>(stg + off) = make_uint4(w[0], w[1], w[2], w[3]);
}

RNSW_DEV void store8x2(uint8_t* lo_row, uint8_t* hi_row, const int32_t (&r)[16]) {
  uint32_t lo[4], hi[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t a = __byte_perm((uint32_t)r[4 * e], (uint32_t)r[4 * e + 1], 0x5140);
    const uint32_t b = __byte_perm((uint32_t)r[4 * e + 2], (uint32_t)r[4 * e + 3], 0x5140);
    lo[e] = __byte_perm(a, b, 0x5410);
    hi[e] = __byte_perm(a, b, 0x7632);
  }
  *reinterpret_cast<uint4*>(lo_row) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  *reinterpret_cast<uint4*>(hi_row) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
}

// Epilogue helpers.  Each thread owns one accumulator row (tile p) and a
// half of the BN columns.  All TMEM loads of a batch are issued before a
// single wait; the accumulator is released (tempty arrive) as soon as the
// last batch has landed in registers, so the next tile's MMAs overlap the
// reductions and stores.

RNSW_DEV int32_t reduce_generic(int32_t v, const GemmArgs& a, int res) {
  return sym_mod(v, a.modulus[res], a.inv_m[res]);
}

RNSW_DEV void store16(int16_t* dst, const int32_t (&r)[16]) {
  int16_t o[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) o[e] = (int16_t)r[e];
  int4* d = reinterpret_cast<int4*>(dst);
  d[0] = *reinterpret_cast<const int4*>(&o[0]);
  d[1] = *reinterpret_cast<const int4*>(&o[8]);
}

// remote != 0: the barrier lives in the CTA pair's leader (its shared::cluster address)
RNSW_DEV void release_acc(uint64_t* bar, int lane, uint32_t remote = 0) {
  tc_fence_before();
  __syncwarp();
  if (lane == 0) {
    if (remote != 0)
      mbar_arrive_remote(remote);
    else
      mbar_arrive(bar);
  }
}

// 16-bit residues: two accumulators (A256, A1) per column.
template <int BN, int ACC_COLS>
RNSW_DEV void epilogue_limbs(const GemmArgs& a, int res, uint32_t taddr, int16_t* out_row, uint8_t* out8, int col0,
                             bool row_ok, uint64_t* tempty, int lane, uint8_t* stg, int srow, int scol0,
                             uint32_t trem = 0) {
  constexpr int kHalf = BN / 2;
  constexpr int kBatch = kHalf < 32 ? kHalf : 32;  // 2 x 32 registers in flight
  const FastMod fm = a.fm[res];
  if (RNSW_GEMM_EPI_PIPE && a.fast2 && a.pos_out && a.planar && stg != nullptr && kHalf % 16 == 0) {
    // the whole-layer (VGG16) path, software-pipelined by 16-column chunks:
    // the next chunk's TMEM loads fly while this one is reduced and staged
    constexpr int kN = kHalf / 16;
    const int32_t pb = pos_bias(fm);
    int32_t buf[2][2][16];
    tmem_ld16(taddr, buf[0][0]);
    tmem_ld16(taddr + BN, buf[0][1]);
    tmem_ld_wait();
    if (kN == 1) release_acc(tempty, lane, trem);
#pragma unroll
    for (int j = 0; j < kN; ++j) {
      if (j + 1 < kN) {
        tmem_ld16(taddr + 16 * (j + 1), buf[(j + 1) & 1][0]);
        tmem_ld16(taddr + BN + 16 * (j + 1), buf[(j + 1) & 1][1]);
      }
      int32_t r[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) r[e] = red_pos_biased(buf[j & 1][0][e] * 256 + buf[j & 1][1][e] + pb, fm);
      sts8x2_swz<BN>(stg, srow, scol0 + 16 * j, r);
      if (j + 1 < kN) {
        tmem_ld_wait();
        if (j + 2 == kN) release_acc(tempty, lane, trem);  // every column of this thread is in registers
      }
    }
    return;
  }
#pragma unroll 1
  for (int c0 = 0; c0 < kHalf; c0 += kBatch) {
    int32_t hi[kBatch / 16][16], lo[kBatch / 16][16];
#pragma unroll
    for (int j = 0; j < kBatch / 16; ++j) {
      tmem_ld16(taddr + c0 + 16 * j, hi[j]);
      tmem_ld16(taddr + BN + c0 + 16 * j, lo[j]);
    }
    tmem_ld_wait();
    if (c0 + kBatch >= kHalf) release_acc(tempty, lane, trem);
#pragma unroll
    for (int j = 0; j < kBatch / 16; ++j) {
      int32_t r[16];
      if (a.fast2) {
        // C <= 512, m < 4500: |256*A256 + A1| <= 512*(9*9+128*9)*256 + 512*(9*128+128*128) < 2^28
        if (a.pos_out) {
          const int32_t pb = pos_bias(fm);
#pragma unroll
          for (int e = 0; e < 16; ++e) r[e] = red_pos_biased(hi[j][e] * 256 + lo[j][e] + pb, fm);
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) r[e] = red_fast(hi[j][e] * 256 + lo[j][e], fm);
        }
      } else if (a.fast) {
#pragma unroll
        for (int e = 0; e < 16; ++e) r[e] = red_fast(red_fast(hi[j][e], fm) * 256 + lo[j][e], fm);
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e)
          r[e] = reduce_generic(reduce_generic(hi[j][e], a, res) * 256 + reduce_generic(lo[j][e], a, res), a, res);
      }
      const int col = col0 + c0 + 16 * j;
      if (a.planar && !(a.fast2 && a.pos_out)) {
        // Mw8 holds y mod m in [0, m): lift the symmetric representatives
#pragma unroll
        for (int e = 0; e < 16; ++e) r[e] += r[e] < 0 ? fm.m : 0;
      }
      if (a.planar) {
        if (stg != nullptr)
          sts8x2_swz<BN>(stg, srow, scol0 + c0 + 16 * j, r);
        else if (row_ok && col < a.Kp)
          store8x2(out8 + col, out8 + a.mw8_plane + col, r);
      } else if (stg != nullptr) {
        sts16_swz(stg, srow, scol0 + c0 + 16 * j, r);
      } else if (row_ok && col < a.Kp) {
        store16(out_row + col, r);
      }
    }
  }
}

// 16-bit residues from the two-plane bank (MAXPL 3): three accumulators
// [A65536 | A256 | A1] per column, y = 65536 A65536 + 256 A256 + A1 (mod m).
// |A65536| <= C 17*9, |A256| <= C (17*128 + 128*9), |A1| <= C 128^2 (V limbs of
// relaxed residues, input_umma.cu), so for C <= 8192 each partial and the
// recombination red(A65536) r65536 + red(A256) 256 + A1 stay below 2^28.
template <int BN>
RNSW_DEV void epilogue_u2(const GemmArgs& a, int res, uint32_t taddr, int16_t* out_row, uint8_t* out8, int col0,
                          bool row_ok, uint64_t* tempty, int lane, uint8_t* stg, int srow, int scol0,
                             uint32_t trem = 0) {
  constexpr int kHalf = BN / 2;
  constexpr int kBatch = kHalf < 16 ? kHalf : 16;
  const FastMod fm = a.fm[res];
  const int32_t r65536 = a.r65536[res];
  const int32_t pb = pos_bias(fm);
#pragma unroll 1
  for (int c0 = 0; c0 < kHalf; c0 += kBatch) {
    int32_t h2[16], h1[16], lo[16];
    tmem_ld16(taddr + c0, h2);
    tmem_ld16(taddr + BN + c0, h1);
    tmem_ld16(taddr + 2 * BN + c0, lo);
    tmem_ld_wait();
    if (c0 + kBatch >= kHalf) release_acc(tempty, lane, trem);
    int32_t r[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int32_t t = red_fast(h2[e], fm) * r65536 + red_fast(h1[e], fm) * 256 + lo[e];
      r[e] = a.pos_out ? red_pos_biased(t + pb, fm) : red_fast(t, fm);
    }
    const int col = col0 + c0;
    if (a.planar) {
      if (!a.pos_out) {
#pragma unroll
        for (int e = 0; e < 16; ++e) r[e] += r[e] < 0 ? fm.m : 0;
      }
      if (stg != nullptr)
        sts8x2_swz<BN>(stg, srow, scol0 + c0, r);
      else if (row_ok && col < a.Kp)
        store8x2(out8 + col, out8 + a.mw8_plane + col, r);
    } else if (stg != nullptr) {
      sts16_swz(stg, srow, scol0 + c0, r);
    } else if (row_ok && col < a.Kp) {
      store16(out_row + col, r);
    }
  }
}

// 8-bit residues: one accumulator per column.
template <int BN>
RNSW_DEV void epilogue_single(const GemmArgs& a, int res, uint32_t taddr, int16_t* out_row, uint8_t* out8, int col0,
                              bool row_ok, uint64_t* tempty, int lane, uint8_t* stg, int srow, int scol0,
                             uint32_t trem = 0) {
  constexpr int kHalf = BN / 2;
  constexpr int kBatch = kHalf < 64 ? kHalf : 64;
  const FastMod fm = a.fm[res];
  if (RNSW_GEMM_EPI_PIPE && a.fast && a.planar && stg != nullptr && kHalf % 32 == 0) {
    // 8-bit whole-layer path, software-pipelined by 32-column chunks (two
    // x16 loads in flight while the previous 32 columns are reduced)
    constexpr int kN = kHalf / 32;
    int32_t buf[2][2][16];
    tmem_ld16(taddr, buf[0][0]);
    tmem_ld16(taddr + 16, buf[0][1]);
    tmem_ld_wait();
    if (kN == 1) release_acc(tempty, lane, trem);
#pragma unroll
    for (int j = 0; j < kN; ++j) {
      if (j + 1 < kN) {
        tmem_ld16(taddr + 32 * (j + 1), buf[(j + 1) & 1][0]);
        tmem_ld16(taddr + 32 * (j + 1) + 16, buf[(j + 1) & 1][1]);
      }
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        int32_t r[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          r[e] = red_fast(buf[j & 1][hf][e], fm);
          r[e] += r[e] < 0 ? fm.m : 0;  // one byte plane of y mod m in [0, m)
        }
        sts8_swz<BN>(stg, srow, scol0 + 32 * j + 16 * hf, r);
      }
      if (j + 1 < kN) {
        tmem_ld_wait();
        if (j + 2 == kN) release_acc(tempty, lane, trem);
      }
    }
    return;
  }
#pragma unroll 1
  for (int c0 = 0; c0 < kHalf; c0 += kBatch) {
    int32_t v[kBatch / 16][16];
#pragma unroll
    for (int j = 0; j < kBatch / 16; ++j) tmem_ld16(taddr + c0 + 16 * j, v[j]);
    tmem_ld_wait();
    if (c0 + kBatch >= kHalf) release_acc(tempty, lane, trem);
#pragma unroll
    for (int j = 0; j < kBatch / 16; ++j) {
      int32_t r[16];
      if (a.fast) {
#pragma unroll
        for (int e = 0; e < 16; ++e) r[e] = red_fast(v[j][e], fm);
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) r[e] = reduce_generic(v[j][e], a, res);
      }
      const int col = col0 + c0 + 16 * j;
      if (a.planar) {
        // one byte plane of y mod m in [0, m)
#pragma unroll
        for (int e = 0; e < 16; ++e) r[e] += r[e] < 0 ? fm.m : 0;
        if (stg != nullptr) {
          sts8_swz<BN>(stg, srow, scol0 + c0 + 16 * j, r);
        } else if (row_ok && col < a.Kp) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) w[e] = pack4_lo(r[4 * e], r[4 * e + 1], r[4 * e + 2], r[4 * e + 3]);
          *reinterpret_cast<uint4*>(out8 + col) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      } else if (stg != nullptr) {
        sts16_swz(stg, srow, scol0 + c0 + 16 * j, r);
      } else if (row_ok && col < a.Kp) {
        store16(out_row + col, r);
      }
    }
  }
}

// MC = 2: a cluster of two CTAs works on tile pairs (pb, pb+1) of the same
// (residue, position, kb).  Each CTA TMA-loads its own V tile and half of
// the filter-bank planes, multicast into both CTAs' stage, so the filter
// bytes moved from L2 per MMA halve (the deep layers are bound by L2 -> SM
// operand traffic, not by the tensor pipe: profiles/r01_gemm_*).  A stage is
// refilled only after both CTAs' MMAs released it (empty barriers count 2,
// MMA commits multicast to the pair).
// MC = 3 (16-bit plans): the same tile pairs as one cta_group::2 MMA of
// M = 256 -- each CTA stages its own V tile and only its N half of the filter
// planes (u'_hi, u_hi on the even CTA, u'_lo, u_lo on the odd one), loads
// complete on the even CTA's barrier, the even CTA issues, commits multicast
// to both, and both CTAs' epilogues release the accumulators to the even CTA.
template <int BN, int BC, int MAXPL, int MC, bool TS, int SB>
__global__ void __launch_bounds__(kThreads, 1)
    winograd_gemm_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmU,
                         const __grid_constant__ CUtensorMap tmM, GemmArgs args) {
  constexpr bool CG2 = MC == 3;
  constexpr int CS = MC == 1 ? 1 : 2;  // CTAs per cluster
  static_assert(!CG2 || MAXPL == 2, "CTA-pair MMAs: 16-bit plans only");
  pdl_trigger();
  using Cfg = GemmConfig<BN, BC, MAXPL, TS, SB, CG2>;
  using Tr = GemmTraits<BN, MAXPL>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + S * Cfg::kStageBytes;  // output staging tile (kTmaStore)
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + Cfg::kStoreBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);  // warp-uniform for the compiler (role branches, MMA operands in uniform registers)
  const int lane = threadIdx.x % 32;
  const int rank = CS == 2 ? (int)cluster_ctarank() : 0;
  // work units: (kb fastest, pb group of CS tiles, pos, res); this CTA takes
  // pb = CS * unit_pb + rank of every unit of its cluster
  const int64_t u_begin = blockIdx.x / CS, u_step = gridDim.x / CS;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmU);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], MC == 2 ? 2 : 1);  // CG2: the leader's multicast commit
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], CG2 ? 16 : 8);  // CG2: both CTAs' epilogue warps
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    if (CG2)
      tmem_alloc_2sm<Tr::kTmemCols>(tmem_slot);
    else
      tmem_alloc<Tr::kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if (CS == 2)
    cluster_sync();  // the peer multicasts / completes into this CTA's stages and barriers
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // V (and the Mw buffer's previous readers) from the previous kernels

  auto stage_a = [&](int s, int pl) { return smem + s * Cfg::kStageBytes + pl * Cfg::kAPlaneBytes; };
  auto stage_b = [&](int s, int pl) {
    return smem + s * Cfg::kStageBytes + a_planes(MAXPL) * Cfg::kAPlaneBytes + pl * Cfg::kBPlaneBytes;
  };  // B smem slots, 16-bit: [0] u'_hi, [1] u'_lo, [2] u_hi, [3] u_lo (bank plane b -> slot 3 - b),
     // so slots 0-1 and 2-3 are each one 2*BN-row K-major operand; 8-bit: [0] u
  // MAXPL 3: [0] u_hi, [1] u_lo (bank planes 1, 0)
  auto bslot = [&](int b, int pl) { return (MAXPL == 2 && pl == 2) ? 3 - b : (MAXPL == 3 ? 1 - b : b); };
  const uint32_t lead_bar0 = CG2 ? mapa_shared(smem_u32(&full[0]), 0) : 0u;  // the leader's full[0]

  if (warp == 0) {
    // ---------------- TMA producer (whole warp) ----------------
    // lane 0 arms the stage barrier, then lane j issues load j of the chunk
    // (A planes, then this CTA's filter planes), so the chunk's 4-6 TMA
    // instructions go out together instead of back to back from one thread
    int stage = 0;
    uint32_t phase = 0;
#ifdef RNSW_GEMM_NOLOAD
    int nfill = 0;
#endif
    for (int64_t t = u_begin; t < args.total_tiles; t += u_step) {
      const TileCoord tc = tile_coord((uint32_t)t, args);
      const int kb = tc.kb, pb = CS * tc.pb + rank, pos = tc.pos, res = tc.res;
      const int pl = args.planes[res];
      const int upl = MAXPL == 3 ? 2 : (pl == 2 ? 4 : 1);
      const int nb = MC == 2 ? 2 : (CG2 ? 2 : upl);  // filter planes this CTA loads
      const int b0 = MC == 2 ? 2 * rank : 0;          // first of them (MC = 2)
      // CG2: the leader's barrier counts both CTAs' A planes and filter halves
      const uint32_t bytes = CG2 ? (uint32_t)(2 * (pl * Cfg::kAPlaneBytes + 2 * Cfg::kBPlaneBytes))
                                 : (uint32_t)(pl * Cfg::kAPlaneBytes + upl * Cfg::kBPlaneBytes);
      for (int kc = 0; kc < args.nkc; ++kc) {
        mbar_wait(&empty[stage], phase ^ 1);
#ifdef RNSW_GEMM_NOLOAD  // diagnostic: after two rounds of the ring, stages are reused without loads
        if (++nfill > 2 * S) {
          if (lane == 0) mbar_arrive(&full[stage]);
          __syncwarp();
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
          continue;
        }
#endif
        if (lane == 0 && (!CG2 || rank == 0)) mbar_arrive_expect_tx(&full[stage], bytes);
        __syncwarp();
        if (CG2) {
          // bank planes 0 u_lo, 1 u_hi, 2 u'_lo, 3 u'_hi; slot 0 = this CTA's N half
          // of [u'_hi ; u'_lo] (MMA 1), slot 1 = its half of [u_hi ; u_lo] (MMA 2)
          const uint32_t lb = lead_bar0 + (uint32_t)stage * 8u;
          if (lane < 2) {
            tma_load_3d_2sm(stage_a(stage, lane), &tmV, lb, kc * BC, pb * kBlockM,
                            (args.plane_base[res] + lane) * args.npos + pos);
          } else if (lane < 4) {
            const int slot = lane - 2, b = (slot == 0 ? 3 : 1) - rank;
            tma_load_3d_2sm(stage_b(stage, slot), &tmU, lb, kc * BC, kb * BN,
                            (args.uplane_base[res] + b) * args.npos + pos);
          }
        } else if (lane < pl) {
          tma_load_3d(stage_a(stage, lane), &tmV, &full[stage], kc * BC, pb * kBlockM,
                      (args.plane_base[res] + lane) * args.npos + pos);
        } else if (lane < pl + nb) {
          const int b = b0 + lane - pl;
          if (MC == 2)
            tma_load_3d_mc(stage_b(stage, bslot(b, pl)), &tmU, &full[stage], kc * BC, kb * BN,
                           (args.uplane_base[res] + b) * args.npos + pos, (uint16_t)0x3);
          else
            tma_load_3d(stage_b(stage, bslot(b, pl)), &tmU, &full[stage], kc * BC, kb * BN,
                        (args.uplane_base[res] + b) * args.npos + pos);
        }
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (!CG2 || rank == 0) {
      // ---------------- MMA issuer (warp-collective: every lane runs the loop, one elected lane
      // issues; the operands are warp-uniform and stay in uniform registers) ----------------
      constexpr uint32_t idesc = idesc_i8(kBlockM, BN);
      constexpr uint32_t idesc2 = idesc_i8(CG2 ? 2 * kBlockM : kBlockM, 2 * BN);  // 16-bit: [A256 | A1] in one MMA
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
#ifdef RNSW_GEMM_PROF
      long long g_te = 0, g_f = 0, g_is = 0, g_0 = clock64(), g_mma = 0, g_cm = 0, g_tc = 0;
#endif
      for (int64_t t = u_begin; t < args.total_tiles; t += u_step, ++it) {
#ifdef RNSW_GEMM_PROF
        long long g0 = clock64();
#endif
        const int res = tile_coord((uint32_t)t, args).res;
        const int pl = args.planes[res];
        const int as = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
#ifdef RNSW_GEMM_PROF
        long long g1 = clock64();
        g_tc += g1 - g0;
#endif
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
#ifdef RNSW_GEMM_PROF
        g_te += clock64() - g1;
#endif
        const uint32_t d0 = tmem_base + as * Tr::kAccCols;
        for (int kc = 0; kc < args.nkc; ++kc) {
#ifdef RNSW_GEMM_PROF
          long long g2 = clock64();
#endif
          mbar_wait(&full[stage], phase);
          tc_fence_after();
#ifdef RNSW_GEMM_PROF
          long long g3 = clock64();
          g_f += g3 - g2;
          g_mma += BC / 32 * ((MAXPL == 1 || pl == 1) ? 1 : (MAXPL == 3 ? 4 : 2));
#endif
          const uint32_t a0 = smem_u32(stage_a(stage, 0));
          const uint32_t b0 = smem_u32(stage_b(stage, 0));
          // one branch per stage, then a branch-free unrolled MMA sequence
          // (a runtime test between consecutive MMAs costs tensor throughput)
          if (CG2) {
#pragma unroll
            for (int k = 0; k < BC / 32; ++k) {
              // M = 256 over the pair; B = the two CTAs' N halves at the same offsets
              const uint32_t acc = (kc | k) != 0;
              const uint64_t da_lo = umma_desc_kmajor(a0 + 32 * k, BC);
              const uint64_t da_hi = umma_desc_kmajor(a0 + Cfg::kAPlaneBytes + 32 * k, BC);
              const uint64_t db_p = umma_desc_kmajor(b0 + 32 * k, BC);                      // u'_hi | u'_lo half
              const uint64_t db_u = umma_desc_kmajor(b0 + Cfg::kBPlaneBytes + 32 * k, BC);  // u_hi | u_lo half
              mma_i8_warp_2sm(d0, da_hi, db_p, idesc2, acc);
              mma_i8_warp_2sm(d0, da_lo, db_u, idesc2, 1u);
            }
          } else if (MAXPL == 1 || pl == 1) {
#pragma unroll
            for (int k = 0; k < BC / 32; ++k)
              mma_i8_warp(d0, umma_desc_kmajor(a0 + 32 * k, BC), umma_desc_kmajor(b0 + 32 * k, BC), idesc,
                     (kc | k) != 0);
          } else if (MAXPL == 3) {
#pragma unroll
            for (int k = 0; k < BC / 32; ++k) {
              // v u = 65536 v_hi u_hi + 256 (v_hi u_lo + v_lo u_hi) + v_lo u_lo
              const uint32_t acc = (kc | k) != 0;
              const uint64_t da_lo = umma_desc_kmajor(a0 + 32 * k, BC);
              const uint64_t da_hi = umma_desc_kmajor(a0 + Cfg::kAPlaneBytes + 32 * k, BC);
              const uint64_t db_hi = umma_desc_kmajor(b0 + 32 * k, BC);                      // slot 0: u_hi
              const uint64_t db_ul = umma_desc_kmajor(b0 + Cfg::kBPlaneBytes + 32 * k, BC);   // slot 1: u_lo
              mma_i8_warp(d0, da_hi, db_hi, idesc, acc);
              mma_i8_warp(d0 + BN, da_hi, db_ul, idesc, acc);
              mma_i8_warp(d0 + BN, da_lo, db_hi, idesc, 1u);
              mma_i8_warp(d0 + 2 * BN, da_lo, db_ul, idesc, acc);
            }
          } else {
#pragma unroll
            for (int k = 0; k < BC / 32; ++k) {
              // v*u = 256*(v_hi*u'_hi + v_lo*u_hi) + (v_hi*u'_lo + v_lo*u_lo): the
              // accumulator columns [A256 | A1] take N = 2*BN rows of B at once
              const uint32_t acc = (kc | k) != 0;
              const uint64_t da_lo = umma_desc_kmajor(a0 + 32 * k, BC);
              const uint64_t da_hi = umma_desc_kmajor(a0 + Cfg::kAPlaneBytes + 32 * k, BC);
              const uint64_t db_p = umma_desc_kmajor(b0 + 32 * k, BC);                         // [u'_hi ; u'_lo]
              const uint64_t db_u = umma_desc_kmajor(b0 + 2 * Cfg::kBPlaneBytes + 32 * k, BC);  // [u_hi ; u_lo]
              mma_i8_warp(d0, da_hi, db_p, idesc2, acc);
              mma_i8_warp(d0, da_lo, db_u, idesc2, 1u);
            }
          }
          if (CG2)
            mma_commit_warp_2sm(&empty[stage]);
          else if (MC == 2)
            mma_commit_warp_mc(&empty[stage], (uint16_t)0x3);
          else
            mma_commit_warp(&empty[stage]);
#ifdef RNSW_GEMM_PROF
          g_is += clock64() - g3;
#endif
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
#ifdef RNSW_GEMM_PROF
        long long g4 = clock64();
#endif
        if (CG2)
          mma_commit_warp_2sm(&tfull[as]);
        else
          mma_commit_warp(&tfull[as]);
#ifdef RNSW_GEMM_PROF
        g_cm += clock64() - g4;
#endif
      }
#ifdef RNSW_GEMM_PROF
      if (lane == 0 && blockIdx.x < 2 && it > 0) printf("GEMMPROF2 cta %d tile_coord %lld commit %lld\n", blockIdx.x, g_tc, g_cm);
#endif
#ifdef RNSW_GEMM_PROF
      if (lane == 0 && blockIdx.x < 2 && it > 0)
        printf("GEMMPROF cta %d BN %d BC %d tiles %d mmas %lld total %lld wait_tempty %lld wait_full %lld issue %lld (cyc/mma %.1f)\n",
               blockIdx.x, BN, BC, it, g_mma, clock64() - g_0, g_te, g_f, g_is, (double)(clock64() - g_0) / g_mma);
#endif
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: 8 warps = 4 TMEM lane quadrants x 2 column halves ----------------
    const int q = warp & 3;                 // TMEM lane quadrant this warp may access
    const int half = (warp - 4) >> 2;       // column half of the accumulator tile
    constexpr int kHalf = BN / 2;
    int it = 0;
    for (int64_t t = u_begin; t < args.total_tiles; t += u_step, ++it) {
      const TileCoord tc = tile_coord((uint32_t)t, args);
      const int kb = tc.kb, pb = CS * tc.pb + rank, pos = tc.pos, res = tc.res;
      const int pl = args.planes[res];
      const int as = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      // CG2: the accumulators are released to the leader CTA's barrier
      const uint32_t rel_remote = CG2 ? mapa_shared(smem_u32(&tempty[as]), 0) : 0u;
      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
#ifdef RNSW_GEMM_NOEPI  // diagnostic: hand the accumulator straight back (no reads, no stores)
      release_acc(&tempty[as], lane, CG2 ? rel_remote : 0u);
      continue;
#endif
      const int64_t p = (int64_t)pb * kBlockM + q * 32 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + as * Tr::kAccCols + half * kHalf;
      int16_t* out_row = args.Mw + mw_offset(p, res * args.npos + pos, args.n_res * args.npos, args.Kp);
      const int col0 = kb * BN + half * kHalf;
      const bool row_ok = p < args.P;
      const bool quad_live = (int64_t)pb * kBlockM + q * 32 < args.P;
      if (Cfg::kTmaStore) {
        // the previous tile's bulk store must have read the staging tile
        // the store that last used this staging tile has read it
        if (warp == 4 && lane == 0) {
          if (Cfg::kStoreBufs == 2)
            bulk_wait_read<1>();
          else
            bulk_wait_read<0>();
        }
        named_bar_sync(1, 256);
      }
      uint8_t* stg_b = stg + (Cfg::kStoreBufs == 2 ? (it & 1) * Cfg::kStoreTile : 0);
      uint8_t* stg_t = Cfg::kTmaStore ? stg_b : nullptr;
      if (!quad_live) {
        // every row of this warp's lane quadrant is past the last tile (small
        // or ragged P): nothing to reduce, just free the accumulator
        release_acc(&tempty[as], lane, CG2 ? rel_remote : 0u);
      } else if (MAXPL == 3) {
        uint8_t* out8 = reinterpret_cast<uint8_t*>(args.Mw) +
                        mw8_offset(p, res, 0, pos, args.n_res, args.npos, args.Kp);
        epilogue_u2<BN>(args, res, taddr, out_row, out8, col0, row_ok, &tempty[as], lane, stg_t, q * 32 + lane,
                        half * kHalf);
      } else if (MAXPL == 2 && pl == 2) {
        uint8_t* out8 = reinterpret_cast<uint8_t*>(args.Mw) +
                        mw8_offset(p, res, 0, pos, args.n_res, args.npos, args.Kp);
        epilogue_limbs<BN, Tr::kAccCols>(args, res, taddr, out_row, out8, col0, row_ok, &tempty[as], lane, stg_t,
                                         q * 32 + lane, half * kHalf, CG2 ? rel_remote : 0u);
      } else {
        uint8_t* out8 = reinterpret_cast<uint8_t*>(args.Mw) + mw8s_offset(p, res, pos, args.n_res, args.npos, args.Kp);
        epilogue_single<BN>(args, res, taddr, out_row, out8, col0, row_ok, &tempty[as], lane, stg_t, q * 32 + lane,
                            half * kHalf);
      }
      if (Cfg::kTmaStore) {
        fence_proxy_async();  // staging writes -> visible to the bulk-copy engine
        named_bar_sync(1, 256);
        if (warp == 4 && lane == 0) {
          if (args.planar) {
            // both limb planes of the tile: slabs (pb * n_res + res) * 2 + {0, 1};
            // 8-bit residues: the one plane, slab pb * n_res + res
            tma_store_3d(&tmM, stg_b, kb * BN, pos * kBlockM, (pb * args.n_res + res) * (MAXPL == 1 ? 1 : 2));
          } else {
            const int row0 = (int)(((int64_t)pb * args.n_res * args.npos + res * args.npos + pos) * kBlockM);
#pragma unroll
            for (int bx = 0; bx < (BN + 63) / 64; ++bx)
              tma_store_2d(&tmM, stg_b + bx * (kBlockM * 128), kb * BN + 64 * bx, row0);
          }
          bulk_commit();
        }
      }
    }
    if (Cfg::kTmaStore && warp == 4 && lane == 0) bulk_wait<0>();  // stores complete before exit
  }

  tc_fence_before();
  if (CG2)
    cluster_sync();  // the pair's MMAs and both CTAs' TMEM reads are done
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (CG2)
      tmem_dealloc_2sm<Tr::kTmemCols>(tmem_base);
    else
      tmem_dealloc<Tr::kTmemCols>(tmem_base);
  }
  if (MC == 2) cluster_sync();  // no CTA leaves while its peer may still signal it
}

// ---------------------------------------------------------------------------
// Host side: tensor maps and dispatch.

// Mw as a 2-D int16 array [rows][Kp] (blocked layout rows), box 64 x 128,
// 128B swizzle: the epilogue's bulk store target.
bool make_tmap_mw(CUtensorMap* tm, const void* base, int Kp, int64_t rows) {
  auto encode = encode_fn();
  if (encode == nullptr) return false;
  cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)Kp * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)kBlockM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Mw8 as a 2-D uint8 array [rows][Kp] (rows = limb-plane rows), box BN x 128.
// Mw8 as [slab = (pb * n_res + res) * 2 + limb][pos * 128 + t][Kp]; one box =
// both limb planes of an output tile (BN x 128 rows x 2), one store per tile.
bool make_tmap_mw8_store(CUtensorMap* tm, const void* base, int Kp, int64_t rows, int bn, int npos, int planes = 2) {
  auto encode = encode_fn();
  if (encode == nullptr) return false;
  const int64_t slab_rows = (int64_t)npos * kBlockM;
  cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)slab_rows, (cuuint64_t)(rows / slab_rows)};
  cuuint64_t strides[2] = {(cuuint64_t)Kp, (cuuint64_t)(slab_rows * Kp)};
  cuuint32_t box[3] = {(cuuint32_t)bn, (cuuint32_t)kBlockM, (cuuint32_t)planes};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, bn == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3-D view [slabs][rows][Cp] of int8 limb planes; box = (bc bytes, box_rows, 1).
bool make_tmap(CUtensorMap* tm, const void* base, int Cp, int64_t rows, int64_t slabs, int bc, int box_rows) {
  auto encode = encode_fn();
  if (encode == nullptr) return false;
  cuuint64_t dims[3] = {(cuuint64_t)Cp, (cuuint64_t)rows, (cuuint64_t)slabs};
  cuuint64_t strides[2] = {(cuuint64_t)Cp, (cuuint64_t)(rows * Cp)};
  cuuint32_t box[3] = {(cuuint32_t)bc, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMapSwizzle sw = bc == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : bc == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                     : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

// SM count of the current device, cached per device id (plans are per device,
// and one process may drive several GPUs).
int num_sms_current() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
  if (dev >= 64) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }
  if (cache[dev] == 0) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n;
  }
  return cache[dev];
}

namespace {

template <int BN, int BC, int MAXPL, int MC, bool TS, int SB>
cudaError_t run_gemm(const GemmArgs& a, const int8_t* V, const int8_t* U, int n_planes, int n_uplanes,
                     cudaStream_t s) {
  using Cfg = GemmConfig<BN, BC, MAXPL, TS, SB, MC == 3>;
  constexpr int CS = MC == 1 ? 1 : 2;  // CTAs per cluster
  CUtensorMap tmV, tmU;
  if (!make_tmap(&tmV, V, a.Cp, a.P, (int64_t)n_planes * a.npos, BC, kBlockM)) return cudaErrorInvalidValue;
  if (!make_tmap(&tmU, U, a.Cp, a.K, (int64_t)n_uplanes * a.npos, BC, BN)) return cudaErrorInvalidValue;
  CUtensorMap tmM;
  const int64_t mw_rows = (a.P + kBlockM - 1) / kBlockM * (int64_t)a.n_res * a.npos * kBlockM;
  if (a.planar) {
    const int out_planes = MAXPL == 1 ? 1 : 2;
    if (!make_tmap_mw8_store(&tmM, a.Mw, a.Kp, mw_rows * out_planes, BN, a.npos, out_planes))
      return cudaErrorInvalidValue;
  } else if (!make_tmap_mw(&tmM, a.Mw, a.Kp, mw_rows)) {
    return cudaErrorInvalidValue;
  }
  auto kern = winograd_gemm_kernel<BN, BC, MAXPL, MC, TS, SB>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  const int num_sms = num_sms_current();
  int64_t grid = a.total_tiles * CS < num_sms ? a.total_tiles * CS : num_sms;
  grid = grid / CS * CS;
  if (grid < CS) grid = CS;
  return launch_ex(kern, dim3((unsigned)grid), dim3(kThreads), Cfg::kSmemBytes, s, CS, tmV, tmU, tmM, a);
}

template <int BN, int MAXPL, int MC, bool TS>
cudaError_t run_gemm_bc_ts(const GemmArgs& a, int bc, const int8_t* V, const int8_t* U, int n_planes,
                           int n_uplanes, cudaStream_t s) {
  // two staging tiles also for CTA pairs with 64-byte chunks (C = 256: -2 to
  // -3%; with 128-byte chunks the stages they cost hurt, +20%)
  if (TS && (a.nkc <= 2 || (MC == 3 && bc == 64))) {
    switch (bc) {
      case 32: return run_gemm<BN, 32, MAXPL, MC, TS, 2>(a, V, U, n_planes, n_uplanes, s);
      case 64: return run_gemm<BN, 64, MAXPL, MC, TS, 2>(a, V, U, n_planes, n_uplanes, s);
      default: return run_gemm<BN, 128, MAXPL, MC, TS, 2>(a, V, U, n_planes, n_uplanes, s);
    }
  }
  switch (bc) {
    case 32: return run_gemm<BN, 32, MAXPL, MC, TS, 1>(a, V, U, n_planes, n_uplanes, s);
    case 64: return run_gemm<BN, 64, MAXPL, MC, TS, 1>(a, V, U, n_planes, n_uplanes, s);
    default: return run_gemm<BN, 128, MAXPL, MC, TS, 1>(a, V, U, n_planes, n_uplanes, s);
  }
}

// Bulk-store epilogue unless the last tile block is mostly empty (small
// batches): a bulk store writes all 128 rows of a block, the per-thread
// epilogue only the live ones.
template <int BN, int MAXPL, int MC = 1>
cudaError_t run_gemm_bc(const GemmArgs& a, int bc, const int8_t* V, const int8_t* U, int n_planes, int n_uplanes,
                        cudaStream_t s) {
  const int64_t dead_rows = (int64_t)a.num_pb * kBlockM - a.P;
  if (dead_rows * 8 <= a.P) return run_gemm_bc_ts<BN, MAXPL, MC, true>(a, bc, V, U, n_planes, n_uplanes, s);
  return run_gemm_bc_ts<BN, MAXPL, MC, false>(a, bc, V, U, n_planes, n_uplanes, s);
}

}  // namespace

cudaError_t launch_winograd_gemm(const PlanHost& plan, const int8_t* V, const int8_t* U, int64_t P, int Cp, int K,
                                 int Kp, int bc, int16_t* Mw, cudaStream_t s, bool pos_out, bool planar) {
  const PlanDevice& d = plan.dev;
  // a handful of tiles: the transposed GEMM (channels on the MMA rows, half the bank bytes)
  if (gemm_t_ok(d, P, Cp, planar, pos_out)) return launch_winograd_gemm_t(plan, V, U, P, Cp, K, Kp, Mw, s);
  GemmArgs a{};
  a.P = P;
  a.K = K;
  a.Kp = Kp;
  a.Cp = Cp;
  a.npos = d.n * d.n;
  a.n_res = d.n_res;
  a.nkc = Cp / bc;
  a.Mw = Mw;
  a.pos_out = pos_out ? 1 : 0;
  a.planar = planar ? 1 : 0;
  a.mw8_plane = (int64_t)a.npos * kBlockM * Kp;
  int maxpl = 1;
  for (int r = 0; r < d.n_res; ++r) {
    a.planes[r] = d.res[r].planes;
    a.plane_base[r] = d.res[r].plane_base;
    a.uplane_base[r] = d.res[r].uplane_base;
    a.modulus[r] = d.res[r].modulus;
    a.inv_m[r] = d.res[r].inv_m;
    a.r256[r] = d.res[r].r_256;
    a.r65536[r] = d.res[r].r_65536;
    const ResidueTables& t = d.res[r];
    a.fm[r] = FastMod{t.red_mul, t.red_shift, t.red_off, t.modulus, t.half, (uint32_t)(-t.modulus)};
    if (d.res[r].planes > maxpl) maxpl = d.res[r].planes;
  }
  a.fast = (d.fast && Cp <= 8192) ? 1 : 0;
  a.fast2 = (a.fast && Cp <= 512) ? 1 : 0;
  // 16-bit: 2 accumulators per set -> BN up to 128 with double-buffered TMEM;
  // the channel chunk drops to 64 bytes so 4 pipeline stages fit (A 2 planes +
  // B 4 planes per stage)
  int bn;
  if (maxpl == 2) bn = Kp <= 64 ? 64 : 128;
  else bn = Kp <= 64 ? 64 : ((Kp <= 128 || planar) ? 128 : 256);
  // CTA-pair (cta_group::2) GEMMs with C >= 512 keep 128-byte channel chunks
  // (3 stages of 64 KB: conv4_2 -6%, conv5 -2%); C = 256 is faster with
  // 64-byte chunks (6 stages; +10% with 128)
  static const char* cg2_env0 = getenv("RNSW_GEMM_CG2");
  const bool cg2_planned = (cg2_env0 != nullptr ? atoi(cg2_env0) != 0 : Cp >= 128) && (P + kBlockM - 1) / kBlockM >= 2 &&
                           getenv("RNSW_GEMM_NO_MC") == nullptr;
  static const int bc128_min = getenv("RNSW_GEMM_BC128_MIN") ? atoi(getenv("RNSW_GEMM_BC128_MIN")) : 512;  // A/B switch
  const bool cg2_bc128 = cg2_planned && Cp >= bc128_min && Cp % 128 == 0;
  if (maxpl == 2 && bc > 64 && !cg2_bc128) {
    bc = 64;
    a.nkc = Cp / bc;
  }
  a.num_pb = (int)((P + kBlockM - 1) / kBlockM);
  a.num_kb = (Kp + bn - 1) / bn;
  a.total_tiles = (int64_t)d.n_res * a.npos * a.num_pb * a.num_kb;
  if (a.total_tiles >= (1ll << 31)) return cudaErrorInvalidValue;  // FastDiv range
  a.div_kb = make_fastdiv((uint32_t)a.num_kb);
  a.div_pb = make_fastdiv((uint32_t)a.num_pb);
  a.div_pos = make_fastdiv((uint32_t)a.npos);
  const int np = d.n_planes, nup = d.n_uplanes;
  bool all16 = true;
  for (int r = 0; r < d.n_res; ++r) all16 = all16 && d.res[r].planes == 2;
  static const bool no_mc = getenv("RNSW_GEMM_NO_MC") != nullptr;  // A/B switch
  // CTA pairs as cta_group::2 MMAs of M = 256 (each CTA stages half of the
  // filter planes) for C >= 128, where the operand stream bounds the GEMM
  // (VGG16 conv4_2: -15%, conv3_2: -5%; since the warp-collective issue also
  // conv3_1: -15%, conv2_2: -7%); multicast pairs for C = 64 (cta_group::2:
  // +6% on conv1_2).  RNSW_GEMM_CG2=0/1 forces either.
  static const char* cg2_env = getenv("RNSW_GEMM_CG2");
  const bool cg2 = cg2_env != nullptr ? atoi(cg2_env) != 0 : Cp >= 128;
  // RNSW_GEMM_U2=1: the two-plane-bank variant (MAXPL 3) for every 16-bit
  // layer, =2: where the bank stream dominates (4 K C >= 2 P C + 4 P K).  Off
  // by default: on B200 it measured slower even at batch 1 (0.83 vs 0.63 ms
  // for the VGG16 GEMMs) -- four N = 64 MMAs per k-step cost 1.5x the tensor
  // time per output column of two N = 256 ones, and at small P the 128-row
  // MMAs are mostly padding, so halving the bank bytes does not pay.
  static const int u2_mode = getenv("RNSW_GEMM_U2") ? atoi(getenv("RNSW_GEMM_U2")) : 0;
  if (maxpl == 2 && all16 && a.fast && u2_mode != 0) {
    const double bank4 = 4.0 * Kp * Cp, act = (double)P * (2.0 * Cp + 4.0 * Kp);
    const bool u2 = u2_mode == 1 || bank4 >= act;
    if (u2) {
      bn = 64;
      a.num_kb = (Kp + bn - 1) / bn;
      a.total_tiles = (int64_t)d.n_res * a.npos * a.num_pb * a.num_kb;
      if (a.total_tiles >= (1ll << 31)) return cudaErrorInvalidValue;
      a.div_kb = make_fastdiv((uint32_t)a.num_kb);
      return run_gemm_bc<64, 3>(a, bc, V, U, np, nup, s);
    }
  }
  if (maxpl == 2 && all16 && (a.num_pb >= 4 || (cg2 && a.num_pb >= 2)) && !no_mc) {
    // CTA pairs over (pb, pb+1) with the filter planes multicast (see the kernel);
    // with only 2-3 tile blocks the pair's lockstep costs more than the shared
    // filter bytes save (VGG16 conv5 at batch 256: -10% without pairs)
    const int num_pbu = (a.num_pb + 1) / 2;
    a.total_tiles = (int64_t)d.n_res * a.npos * num_pbu * a.num_kb;
    a.div_pb = make_fastdiv((uint32_t)num_pbu);
    if (cg2) {
      if (bn == 64) return run_gemm_bc<64, 2, 3>(a, bc, V, U, np, nup, s);
      return run_gemm_bc<128, 2, 3>(a, bc, V, U, np, nup, s);
    }
    if (bn == 64) return run_gemm_bc<64, 2, 2>(a, bc, V, U, np, nup, s);
    return run_gemm_bc<128, 2, 2>(a, bc, V, U, np, nup, s);
  }
  if (maxpl == 2) {
    if (bn == 64) return run_gemm_bc<64, 2>(a, bc, V, U, np, nup, s);
    return run_gemm_bc<128, 2>(a, bc, V, U, np, nup, s);
  }
  if (bn == 64) return run_gemm_bc<64, 1>(a, bc, V, U, np, nup, s);
  if (bn == 128) return run_gemm_bc<128, 1>(a, bc, V, U, np, nup, s);
  return run_gemm_bc<256, 1>(a, bc, V, U, np, nup, s);
}

}  // namespace rnsw
