// K1 on the 5th-generation tensor cores: V = BT d B mod m for every tile,
// channel and residue (rw/layer.py:278-283, rw/kernel.py:44-47, 21-30),
// written straight into the GEMM operand layout V[plane][pos][P][Cp].
//
// The separable sandwich BT d BT^T is one linear map of the N*N patch:
//     V[(i,j)] = sum_(a,b) Kr[(i,j),(a,b)] d[(a,b)],   Kr = kron(BT, BT) mod m,
// so the whole transform of a tile (all channels at once) is ONE GEMM per
// residue and 128-position block:
//     D[pos, ch] = sum_pix Kr[pos, pix] * patch[pix, ch]      (M=128, N=64, K=N*N)
//   A = Kr limbs: a per-CTA constant, resident in TENSOR memory (K-major, four
//       int8 per column; written once with tcgen05.st), so the MMA reads only
//       B from shared memory;
//   B = the patch, TMA-loaded as a 4-D box (64 channels x N columns x N rows
//       x 1 image) straight from NHWC x: the box IS the MN-major operand (K =
//       pixel rows, N = channels, 64B swizzle), and TMA's zero fill supplies
//       the conv padding and the canvas extension of tile_decompose
//       (rw/layer.py:118-158);
//   D = s32 in TMEM; 16-bit moduli: two accumulators (Kr = 256 Kr_hi + Kr_lo,
//       balanced s8 limbs), x = 256 D_hi + D_lo, |x| < 2^27.
// The Kronecker form does N*N/(2N) = 8x the MACs of the two-pass separable
// form at N = 16, but it is a single pass: no TMEM round trip between the
// passes, and each output value costs the CUDA cores three instructions plus
// a byte split (the mma.sync kernel spent ~165 warp instructions per
// (tile, channel, residue)).  The tensor pipe, idle in K1 otherwise, absorbs
// the extra MACs.
//
// Work: groups g = (residue, position block); CTA b serves group b % G for
// every unit (one tile x 64 channels), so its Kr operand is loaded once.
// The G CTAs of a unit run side by side and read the same patch (the second
// to fourth reads hit L2).  Warp roles (384 threads): 0 TMA producer, 1 MMA
// issuer, 2 TMEM allocator, 3 bulk stores, 4-11 epilogue (lane quadrant x
// column half): tcgen05.ld -> limb recombination -> one reduction -> byte
// planes -> swizzled staging; mbarriers (no CTA barriers) link the roles.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.h"

// Diagnostic builds only (tools/variant_build.sh -DRNSW_K1_DIAG=n): 1 = no
// staging stores / bulk stores, 2 = no conversion, 3 = one MMA per unit, 4 = tile-major V.
#ifndef RNSW_K1_DIAG
#define RNSW_K1_DIAG 0
#endif
// 9 = no TMEM loads in the epilogue, 10 = 9 without stores
#define RNSW_K1_ONE_MMA (RNSW_K1_DIAG == 3 || (RNSW_K1_DIAG >= 5 && RNSW_K1_DIAG <= 8))
#define RNSW_K1_NO_STORE (RNSW_K1_DIAG == 1 || (RNSW_K1_DIAG >= 5 && RNSW_K1_DIAG <= 8) || RNSW_K1_DIAG >= 10)
// 11 = no staging / bulk stores; each epilogue lane writes its 64 bytes straight to global (wrong layout)
// 12 = no staging writes (the bulk stores still run, on stale staging)
#define RNSW_K1_NO_TMEM_LD (RNSW_K1_DIAG == 9 || RNSW_K1_DIAG == 10)
#ifndef RNSW_K1_DEFER
#define RNSW_K1_DEFER 1
#endif
// 1 (default): the tile-pair staging rows under the 128B swizzle (conflict-free
// stores); 0: plain rows (measured 17% slower)
#ifndef RNSW_K1_STG_SWZ
#define RNSW_K1_STG_SWZ 1
#endif
#ifndef RNSW_K1_STAGES
#define RNSW_K1_STAGES 8
#endif
#ifndef RNSW_K1_STAGES8
#define RNSW_K1_STAGES8 4
#endif
#ifndef RNSW_K1_NSTG
#define RNSW_K1_NSTG 2
#endif
#ifndef RNSW_K1_EPI_PIPE
#define RNSW_K1_EPI_PIPE 0
#endif
// 1: the accumulator bias is added in the epilogue (one IADD per value)
// instead of by two bias MMAs per unit (11% of the unit's tensor work) --
// measured 7% slower on conv1_2 than the bias MMAs, so off
#ifndef RNSW_K1_EPI_BIAS
#define RNSW_K1_EPI_BIAS 0
#endif

namespace rnsw {

namespace {

constexpr int kGroupRows = 128;  // positions per group (MMA M)
constexpr int kUnitN = 64;       // channels per unit (MMA N)
// epilogue warps: 16 (4 lane quadrants x 4 column quarters of 16 channels)
// or 8 (x 2 column halves of 32); more warps hide the TMEM-load / reduction
// latency of the epilogue, which paces the MMA warp through tempty
#ifndef RNSW_K1_EPI_WARPS
#define RNSW_K1_EPI_WARPS 8
#endif
constexpr int kEpiWarps = RNSW_K1_EPI_WARPS;
constexpr int kEpiCols = kUnitN / (kEpiWarps / 4);  // channels per epilogue warp
constexpr int kUThreads = 128 + 32 * kEpiWarps;

struct K1UArgs {
  Geometry g;
  int npos, mout, kp, ksteps, limbs, groups, npb;
  int units;            // P * (Cp / 64)
  int cblocks;          // Cp / 64
  int res_of[16];       // group -> residue
  int pb_of[16];        // group -> position block
  int plane_base[RNSW_MAX_RES];
  FastMod fm[RNSW_MAX_RES];
  uint32_t mul0[RNSW_MAX_RES];    // ceil(2^32 / m): quotient estimate (kRel16)
  int32_t bias_s1[RNSW_MAX_RES];  // 16-bit: bias = 127 (256 S1 + S2), see K1UMode
  int32_t bias_s2[RNSW_MAX_RES];
  FastDiv div_img, div_tw, div_cb;
  size_t group_bytes;   // [limb][128 rows][kp] plain bytes per group
  uint8_t* v_raw;       // diagnostic 11 only
  int pair128;          // Cp == 64 and P even: a unit pair's two tiles are one 128-byte V row
};

// Output modes.  For 16-bit moduli each unit's accumulators start from a
// bias made by one extra K = 32 MMA per limb with constant operands (A =
// 127 everywhere, B rows beta_k with sum beta = S1 resp. S2), so D_hi / D_lo
// come out as x + 127 (256 S1 + S2) and the epilogue's reduction is three
// instructions per value; S1, S2 are chosen on the host so the bias is a
// multiple of m plus the offset the mode needs and exceeds the largest |x|:
//   kSym8  (8-bit moduli): v = symmetric residue in [-h, h], one s8 plane;
//          no bias MMA: n = x + off (off = h mod m): v = (n - h) - floor(n/m) m.
//   kSym16 (16-bit, stage API): v symmetric, planes lo = byte0(v + 128) ^ 0x80,
//          hi = (v + 128) >> 8 (the reference's residues, bit for bit).
//   kRel16 (16-bit, whole-layer path): w = n - q m with q = umulhi(n, ceil(2^32/m))
//          -- floor(n/m) or one more, no shift -- so v = w - 128 lies in
//          [-m-128, m-128) instead of [-h, h]: any representative is exact
//          for the GEMM, whose single reduction still holds (limb hi in
//          [-17, 16]: 256 A256 + A1 <= 512 (17*9 + 128*9) 256 + 512 (17*128 +
//          128*128) < 1.9e8 < 2^28 for C <= 512; capi uses it for C <= 8192).
enum K1UMode { kSym8 = 0, kSym16 = 1, kRel16 = 2 };

// TMEM columns: [accumulator buffers 2 x limbs x 64 | Kr limbs x kp/4 | bias A 8]
template <int kLimbs>
struct K1UConfig {
  static constexpr int kStageBytes = 256 * kUnitN;  // K <= 256 pixel rows x 64 channel bytes
  // 8-bit plans: 4 stages, so two CTAs (256 TMEM columns each) fit per SM --
  // their small layers are latency-bound (BASELINE configs 1, 3, 5)
  static constexpr int kStages = kLimbs == 1 ? RNSW_K1_STAGES8 : RNSW_K1_STAGES;
  static constexpr int kNStg = RNSW_K1_NSTG;  // staging buffers (unit pairs in flight to the bulk stores)
  // staging per unit PAIR (two tiles x 64 channels, or one tile x 128): the
  // bulk stores then write 128-byte rows instead of 64-byte ones
  static constexpr int kStgBytes = kLimbs * kGroupRows * 2 * kUnitN;
  static constexpr int kBiasBytes = kLimbs == 2 ? 2 * 32 * kUnitN : 0;
  static constexpr int kAccCols = kLimbs * kUnitN;
  static constexpr int kACol = 2 * kAccCols;          // Kr limb l at kACol + l * 64 (kp <= 256)
  static constexpr int kBiasCol = kACol + kLimbs * 64;
  static constexpr int kTmemCols = kLimbs == 2 ? 512 : 256;
  static_assert(kBiasCol + 8 <= kTmemCols, "TMEM");
  static constexpr size_t kSmem =
      1024 + (size_t)kStages * kStageBytes + kNStg * (size_t)kStgBytes + kBiasBytes + 256;
};

// One unit's MMAs (16-bit plans, one CTA per group) from ONE asm block: one
// elect.sync, the two bias MMAs, kKs K-steps x two limbs, both commits; every
// operand is a base register plus a literal, so the issuing warp spends ~4
// uniform-datapath instructions per MMA (a separate block per MMA re-elected
// and moved each descriptor through R2UR: ~10 instructions per 32-cycle MMA).
// B descriptors: the patch stage / bias tiles, MN-major, 64B swizzle; the
// start-address field advances by 128 (2 KB) per K-step.
#define K1_MMA_TS(D, A) "@e tcgen05.mma.cta_group::1.kind::i8 [" D "], [" A "], db, %7, po;\n\t"
#define K1_KSTEP(KS)                                                         \
  "add.u32 a, %1, " #KS " * 8;\n\tadd.u32 bl, %3, " #KS " * 128;\n\t"         \
  "mov.b64 db, {bl, %4};\n\t" K1_MMA_TS("%0", "a")                            \
  "add.u32 a, %1, 64 + " #KS " * 8;\n\t" K1_MMA_TS("t", "a")
#define K1_UNIT_HEAD                                                                              \
  "{\n\t.reg .pred e, pz, po;\n\t.reg .b32 t, a, bl;\n\t.reg .b64 db;\n\t"                          \
  "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 pz, 0, 0;\n\tsetp.eq.b32 po, 0, 0;\n\t"               \
  "add.u32 t, %0, 64;\n\t"                                                                          \
  "mov.b64 db, {%5, %4};\n\t@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%2], db, %7, pz;\n\t"       \
  "mov.b64 db, {%6, %4};\n\t@e tcgen05.mma.cta_group::1.kind::i8 [t], [%2], db, %7, pz;\n\t"
#define K1_UNIT_TAIL                                                                              \
  "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n\t"             \
  "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%9];\n\t}"
#define K1_UNIT_ASM(STEPS)                                                                                  \
  asm volatile(K1_UNIT_HEAD STEPS K1_UNIT_TAIL ::"r"(d0), "r"(ta), "r"(bias_col), "r"(db_lo), "r"(db_hi),  \
               "r"(dbh_lo), "r"(dbl_lo), "r"(idesc), "r"(bar_empty), "r"(bar_tfull)                        \
               : "memory")
#define K1_S1 K1_KSTEP(0)
#define K1_S2 K1_S1 K1_KSTEP(1)
#define K1_S3 K1_S2 K1_KSTEP(2)
#define K1_S4 K1_S3 K1_KSTEP(3)
#define K1_S5 K1_S4 K1_KSTEP(4)
#define K1_S6 K1_S5 K1_KSTEP(5)
#define K1_S7 K1_S6 K1_KSTEP(6)
#define K1_S8 K1_S7 K1_KSTEP(7)
// (one instance per K-step count: a jump table in front of the block made the
// compiler treat the warp as possibly diverged and re-elect per MMA)
template <int kKs>
RNSW_DEV void k1_issue_unit16(uint32_t d0, uint32_t ta, uint32_t bias_col, uint32_t db_lo, uint32_t db_hi,
                              uint32_t dbh_lo, uint32_t dbl_lo, uint32_t idesc, uint32_t bar_empty,
                              uint32_t bar_tfull) {
  __syncwarp();  // converged: the compiler then keeps the block's operands in uniform registers
  if constexpr (kKs == 8) K1_UNIT_ASM(K1_S8);
  else if constexpr (kKs == 7) K1_UNIT_ASM(K1_S7);
  else if constexpr (kKs == 6) K1_UNIT_ASM(K1_S6);
  else if constexpr (kKs == 5) K1_UNIT_ASM(K1_S5);
  else if constexpr (kKs == 4) K1_UNIT_ASM(K1_S4);
  else if constexpr (kKs == 3) K1_UNIT_ASM(K1_S3);
  else if constexpr (kKs == 2) K1_UNIT_ASM(K1_S2);
  else K1_UNIT_ASM(K1_S1);
}

// kPair: a 2-CTA cluster serves both 128-position blocks of a residue (N*N >
// 128): one cta_group::2 MMA of M = 256 per K-step and limb, A = each CTA's
// block of Kr in its own TMEM, B = the patch split by channels (32 per CTA),
// so each SM loads and the tensor core reads half of the patch per unit.
template <int kMode, bool kPair>
__global__ void __launch_bounds__(kUThreads, 1)
    input_umma_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmV,
                      const __grid_constant__ CUtensorMap tmV2, const uint8_t* __restrict__ kr, K1UArgs args) {
  constexpr int kLimbs = kMode == kSym8 ? 1 : 2;
  constexpr int kBN = kPair ? kUnitN / 2 : kUnitN;  // patch channels (B columns) in this CTA's shared memory
  pdl_trigger();
  using Cfg = K1UConfig<kLimbs>;
  constexpr int S = Cfg::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned, derived from the shared array so stores stay STS
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sB = smem;                          // [S][256 rows][64 bytes]
  uint8_t* stg = sB + S * Cfg::kStageBytes;    // [2][plane][128 rows][64 bytes]
  uint8_t* sBias = stg + Cfg::kNStg * Cfg::kStgBytes;   // [B_hi | B_lo] 32 rows x 64 bytes each
  uint64_t* full = reinterpret_cast<uint64_t*>(sBias + Cfg::kBiasBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;   // staging buffer written by the 8 epilogue warps
  uint64_t* sempty = sfull + Cfg::kNStg;   // staging buffer read by its bulk store
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + Cfg::kNStg);

  // the warp index through a shuffle: the compiler then treats the role branches (and everything
  // computed inside them) as warp-uniform and keeps the MMA operands in uniform registers
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0), lane = threadIdx.x % 32;
  const uint32_t crank = kPair ? cluster_ctarank() : 0u;
  const int cid = kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // cluster (or CTA) id
  const int ncl = kPair ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int group = cid % args.groups;
  // units come in pairs (2k, 2k+1): two consecutive tiles when Cp = 64, else
  // two consecutive 64-channel blocks of one tile (Cp is a multiple of 128)
  const int pr_begin = cid / args.groups, pr_step = ncl / args.groups;
  const int npairs = (args.units + 1) / 2;
#define RNSW_FOR_UNITS(u)                                              \
  for (int pr_ = pr_begin; pr_ < npairs; pr_ += pr_step)               \
    for (int h_ = 0, u = 2 * pr_; h_ < 2 && u < args.units; ++h_, ++u)
  const int res = args.res_of[group], pb = kPair ? (int)crank : args.pb_of[group];
  const int kr_group = kPair ? res * args.npb + pb : group;  // Kr image of (residue, position block)
  const Geometry& g = args.g;
  const FastMod fm = args.fm[res];

  if (kLimbs == 2) {
    // bias B operands: row k of B_hi = beta_k (sum S1), of B_lo = gamma_k
    // (sum S2); uniform rows, so the swizzle is moot
    const int s1 = args.bias_s1[res], s2 = args.bias_s2[res];
    for (int i = threadIdx.x; i < 2 * 32 * kBN / 4; i += kUThreads) {
      const int k = (i % (32 * kBN / 4)) / (kBN / 4), sum = i < 32 * kBN / 4 ? s1 : s2;
      const int beta = sum / 32 + (k < (sum % 32) ? 1 : 0);
      reinterpret_cast<uint32_t*>(sBias)[i] = (uint32_t)(uint8_t)(int8_t)beta * 0x01010101u;
    }
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(args.cblocks == 1 ? &tmV : &tmV2);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kPair ? 2 * kEpiWarps : kEpiWarps);  // kPair: both CTAs' epilogue warps
    }
    for (int i = 0; i < Cfg::kNStg; ++i) {
      mbar_init(&sfull[i], 2 * kEpiWarps);  // epilogue warps x 2 units of a pair
      mbar_init(&sempty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    if (kPair)
      tmem_alloc_2sm<Cfg::kTmemCols>(tmem_slot);
    else
      tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  }
  fence_proxy_async();  // bias operands (generic stores) -> visible to the MMA (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // epilogue thread geometry: lane quadrant q, column block hh (kEpiCols channels)
  const int q = warp & 3, hh = (warp - 4) >> 2;
  if (warp >= 4) {
    // the group's Kr operand into TMEM: thread = row (position), limb hh
    // (8-bit: one limb, written by hh = 0), kp/4 columns of four K bytes
    const int row = q * 32 + lane;
    const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16);
    if (hh < kLimbs) {
      const uint4* src = reinterpret_cast<const uint4*>(kr + (size_t)kr_group * args.group_bytes +
                                                        ((size_t)hh * kGroupRows + row) * args.kp);
      // 8 columns = 32 K bytes per store; four stores' loads in flight together
      // (one dependent load per store made this prologue ~8 L2 latencies long)
      const int n8 = args.kp / 32;
      for (int c8 = 0; c8 < n8; c8 += 4) {
        uint4 w[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) w[e] = c8 + (e >> 1) < n8 ? __ldg(src + 2 * c8 + e) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (c8 + e >= n8) break;
          const uint32_t v[8] = {w[2 * e].x, w[2 * e].y, w[2 * e].z, w[2 * e].w,
                                 w[2 * e + 1].x, w[2 * e + 1].y, w[2 * e + 1].z, w[2 * e + 1].w};
          tmem_st8(trow + Cfg::kACol + hh * 64 + (c8 + e) * 8, v);
        }
      }
    }
    if (kLimbs == 2 && hh == 0) {
      const uint32_t v[8] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                             0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
      tmem_st8(trow + Cfg::kBiasCol, v);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  if (kPair)
    cluster_sync();  // both CTAs' Kr in TMEM and barriers initialised before the pair's first MMA / remote arrival
  else
    __syncthreads();
  tc_fence_after();
  pdl_wait();  // the previous kernel's activations (and its use of V) are complete from here on

  // unit -> tile, channel offset
  auto unit_tile = [&](int u, int& p, int& c0) {
    const int qq = (int)fdiv((uint32_t)u, args.div_cb);
    p = qq;
    c0 = (u - qq * args.cblocks) * kUnitN;
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

#ifdef RNSW_K1_MMA_ONLY
  if (warp != 1) {
  } else
#endif
  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      const uint32_t bytes = (uint32_t)(args.npos * kBN);
      int stage = 0;
      uint32_t phase = 0;
      RNSW_FOR_UNITS(u) {
        int p, c0, b, h0, w0;
        unit_tile(u, p, c0);
        tile_origin(p, b, h0, w0);
        mbar_wait(&empty[stage], phase ^ 1);
#ifdef RNSW_K1_NOLOAD
        if (u >= 2 * S * pr_step) {  // diagnostic: the first units load, later ones reuse the stale stages
          mbar_arrive(&full[stage]);
        } else
#endif
        if (kPair) {
          // this CTA's 32 channels; the bytes of both halves complete on the leader's barrier
          if (crank == 0) mbar_arrive_expect_tx(&full[stage], 2 * bytes);
          tma_load_4d_2sm(sB + stage * Cfg::kStageBytes, &tmX, mapa_shared(smem_u32(&full[stage]), 0),
                          c0 + (int)crank * kBN, w0, h0, b);
        } else {
          mbar_arrive_expect_tx(&full[stage], bytes);
          tma_load_4d(sB + stage * Cfg::kStageBytes, &tmX, &full[stage], c0, w0, h0, b);
        }
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && (!kPair || crank == 0)) {
    // ---------------- MMA issuer (warp-collective: descriptors stay uniform) ----------------
    // kPair: M = 256 over the CTA pair, N = 64 split 32 + 32 (32B-swizzled halves)
    constexpr uint32_t idesc = idesc_i8x(kPair ? 256 : 128, kUnitN, true, true, false, true);  // A K-major (TMEM), B MN-major
    // descriptors advance by adding the byte offset / 16 to the start-address field
    const uint64_t db0 = kPair ? umma_desc_mn_sw32(smem_u32(sB), 1024) : umma_desc_mn_sw64(smem_u32(sB), 16);
    const uint64_t dbh = kPair ? umma_desc_mn_sw32(smem_u32(sBias), 1024) : umma_desc_mn_sw64(smem_u32(sBias), 16);
    const uint64_t dbl = kPair ? umma_desc_mn_sw32(smem_u32(sBias + 32 * kBN), 1024)
                               : umma_desc_mn_sw64(smem_u32(sBias + 32 * kBN), 16);
    constexpr uint32_t kBStep = (32 * kBN) >> 4;  // one K-step of the patch
    auto mma_ts = [&](uint32_t d, uint32_t a, uint64_t bd, uint32_t id, uint32_t acc) {
      if (kPair)
        mma_i8_ts_warp_2sm(d, a, bd, id, acc);
      else
        mma_i8_ts_warp(d, a, bd, id, acc);
    };
    constexpr uint32_t kStageStep = Cfg::kStageBytes >> 4;
    const uint32_t ta = tmem_base + Cfg::kACol;
    const int ksteps = args.ksteps;
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
#ifdef RNSW_K1_PROBE
    if (!kPair) {  // diagnostic: the bare MMA sequence on this kernel's operands, timed
      long long p0 = clock64();
      for (int pu = 0; pu < 2000; ++pu) {
        const uint32_t d0 = tmem_base + (pu & 1) * Cfg::kAccCols;
        const uint64_t db_stage = db0 + (uint64_t)((pu & 7) * kStageStep);
        mma_i8_ts_warp(d0, tmem_base + Cfg::kBiasCol, dbh, idesc, 0u);
        mma_i8_ts_warp(d0 + kUnitN, tmem_base + Cfg::kBiasCol, dbl, idesc, 0u);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint64_t db = db_stage + (uint64_t)(ks * kBStep);
          mma_i8_ts_warp(d0, ta + ks * 8, db, idesc, 1u);
          mma_i8_ts_warp(d0 + kUnitN, ta + 64 + ks * 8, db, idesc, 1u);
        }
      }
      mma_commit_warp(&tfull[0]);
      mbar_wait(&tfull[0], 0);
      long long p1 = clock64();
      if (lane == 0 && blockIdx.x < 2) printf("K1PROBE cta %d %lld cycles per unit\n", blockIdx.x, (p1 - p0) / 2000);
    }
#endif
#ifdef RNSW_K1_PROF
    long long c_te = 0, c_f = 0, c_is = 0, c_0 = clock64();
#endif
    RNSW_FOR_UNITS(u) {
      const int as = it & 1;
#ifdef RNSW_K1_PROF
      long long c1 = clock64();
#endif
#ifdef RNSW_K1_NOWAIT
      if (it < RNSW_K1_NOWAIT)
#endif
      mbar_wait(&tempty[as], ((it >> 1) & 1) ^ 1);  // kPair: releases from both CTAs
#ifdef RNSW_K1_PROF
      long long c2 = clock64();
#endif
#ifdef RNSW_K1_NOWAIT
      if (it < RNSW_K1_NOWAIT)
#endif
      mbar_wait(&full[stage], phase);
      tc_fence_after();
#ifdef RNSW_K1_PROF
      long long c3 = clock64();
      c_te += c2 - c1;
      c_f += c3 - c2;
#endif
      const uint32_t d0 = tmem_base + as * Cfg::kAccCols;
      const uint64_t db_stage = db0 + (uint64_t)(stage * kStageStep);
#if !defined(RNSW_K1_PROF) && !RNSW_K1_EPI_BIAS && !RNSW_K1_ONE_MMA && !defined(RNSW_K1_OLD_ISSUE)
      if constexpr (kLimbs == 2 && !kPair) {
        if (ksteps == 8 || ksteps == 4) {  // N*N = 256 (F(14,3), the VGG16 plan) / 128-position blocks of N = 12
          if (ksteps == 8)
            k1_issue_unit16<8>(d0, ta, tmem_base + Cfg::kBiasCol, (uint32_t)db_stage, (uint32_t)(db0 >> 32),
                               (uint32_t)dbh, (uint32_t)dbl, idesc, smem_u32(&empty[stage]), smem_u32(&tfull[as]));
          else
            k1_issue_unit16<4>(d0, ta, tmem_base + Cfg::kBiasCol, (uint32_t)db_stage, (uint32_t)(db0 >> 32),
                               (uint32_t)dbh, (uint32_t)dbl, idesc, smem_u32(&empty[stage]), smem_u32(&tfull[as]));
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
          ++it;
          continue;
        }
      }
#endif
      if (kLimbs == 2 && !RNSW_K1_EPI_BIAS) {  // the bias: D_hi = 127 S1, D_lo = 127 S2 (overwrites the buffer)
        mma_ts(d0, tmem_base + Cfg::kBiasCol, dbh, idesc, 0u);
        mma_ts(d0 + kUnitN, tmem_base + Cfg::kBiasCol, dbl, idesc, 0u);
      }
#ifdef RNSW_K1_PROF
      long long tsk[9];
#endif
      auto kstep = [&](int ks) {
#ifdef RNSW_K1_PROF
        tsk[ks] = clock64();
#endif
        const uint64_t db = db_stage + (uint64_t)(ks * kBStep);
        const uint32_t acc = ((kLimbs == 2 && !RNSW_K1_EPI_BIAS) || ks > 0) ? 1u : 0u;
        mma_ts(d0, ta + ks * 8, db, idesc, acc);
        if (kLimbs == 2) mma_ts(d0 + kUnitN, ta + 64 + ks * 8, db, idesc, acc);
      };
      for_ksteps(RNSW_K1_ONE_MMA ? 1 : ksteps, kstep);  // branch-free unrolled MMA sequence
#ifdef RNSW_K1_PROF
      tsk[8] = clock64();
      if (lane == 0 && blockIdx.x == 0 && (it == 1000 || it == 1001 || it == 1500))
        printf("K1MMA it %d issue deltas %lld %lld %lld %lld %lld %lld %lld %lld | from start of unit %lld\n", it,
               tsk[1] - tsk[0], tsk[2] - tsk[1], tsk[3] - tsk[2], tsk[4] - tsk[3], tsk[5] - tsk[4], tsk[6] - tsk[5],
               tsk[7] - tsk[6], tsk[8] - tsk[7], tsk[0] - c3);
#endif
      if (kPair) {
        mma_commit_warp_2sm(&empty[stage]);
        mma_commit_warp_2sm(&tfull[as]);
      } else {
        mma_commit_warp(&empty[stage]);
        mma_commit_warp(&tfull[as]);
      }
#ifdef RNSW_K1_PROF
      c_is += clock64() - c3;
#endif
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
      ++it;
    }
#ifdef RNSW_K1_PROF
    if (lane == 0 && blockIdx.x < 4)
      printf("K1PROF cta %d units %d total %lld wait_tempty %lld wait_full %lld issue %lld (per unit: %lld %lld %lld %lld)\n",
             blockIdx.x, it, clock64() - c_0, c_te, c_f, c_is, (clock64() - c_0) / it, c_te / it, c_f / it, c_is / it);
#endif
  } else if (warp == 3) {
    if (lane == 0) {
      // ---------------- bulk stores of the staged V rows (one per unit pair) ----------------
      const bool two = args.cblocks == 1;
      int jt = 0;
      for (int pr = pr_begin; pr < npairs; pr += pr_step, ++jt) {
        int p, c0;
        unit_tile(2 * pr, p, c0);
        const int sb = jt % Cfg::kNStg;
        const uint32_t sph = (uint32_t)(jt / Cfg::kNStg) & 1u;
        mbar_wait(&sfull[sb], sph);
        uint8_t* sbuf = stg + sb * Cfg::kStgBytes;
#pragma unroll
        for (int pl = 0; pl < (RNSW_K1_NO_STORE ? 0 : kLimbs); ++pl)
          tma_store_4d(two ? &tmV : &tmV2, sbuf + pl * (kGroupRows * 2 * kUnitN), c0,
                       (two && args.pair128) ? (p >> 1) : p, pb * kGroupRows, args.plane_base[res] + pl);
        bulk_commit();
        bulk_wait_read<0>();  // the staging buffer may be rewritten
        mbar_arrive(&sempty[sb]);
      }
      bulk_wait<0>();
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: 8 warps = 4 lane quadrants x 2 channel halves ----------------
    const int row = q * 32 + lane;  // position within the group's block
    const uint32_t mul0 = args.mul0[res];
    const int32_t ebias = RNSW_K1_EPI_BIAS ? 127 * (256 * args.bias_s1[res] + args.bias_s2[res]) : 0;
    auto convert = [&](const int32_t (&a)[16], const int32_t (&b)[16], uint32_t* lo, uint32_t* hi) {
      int32_t w[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        if (kMode == kRel16) {
          const uint32_t n = (uint32_t)(a[e] * 256 + b[e] + ebias);  // x + bias, bias = 128 (mod m)
          w[e] = (int32_t)(__umulhi(n, mul0) * fm.negm + n);  // = x + 128 (mod m), in [-m, m)
        } else if (kMode == kSym16) {
          const int32_t r = red_pos_biased(a[e] * 256 + b[e] + ebias, fm);  // (x + h) mod m
          w[e] = r + (128 - fm.h);                                  // v + 128
        } else {
          const uint32_t n = (uint32_t)(b[e] + fm.off);  // x + off, off = h (mod m)
          const uint32_t qq = __umulhi(n, fm.mul) >> fm.shift;
          w[e] = (int32_t)(qq * fm.negm + (n - (uint32_t)fm.h));  // v in [-h, h]
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t p01 = __byte_perm((uint32_t)w[4 * e], (uint32_t)w[4 * e + 1], 0x5140);
        const uint32_t p23 = __byte_perm((uint32_t)w[4 * e + 2], (uint32_t)w[4 * e + 3], 0x5140);
        const uint32_t b0 = __byte_perm(p01, p23, 0x5410);
        lo[e] = kLimbs == 2 ? b0 ^ 0x80808080u : b0;  // low byte of v
        hi[e] = __byte_perm(p01, p23, 0x7632);         // (v + 128) >> 8
      }
    };
    const bool two = args.cblocks == 1;
    int it = 0, jt = -1;
    // deferred staging hand-off (RNSW_K1_DEFER): a unit's fence.proxy.async +
    // sfull arrive happen after the next unit's TMEM loads and conversion, so
    // the warp does not stall on its own st.shared completing
    int pend_sb = -1, pend_extra = 0;
    auto hand_off = [&]() {
      if (pend_sb < 0) return;
      fence_proxy_async();  // staging writes -> visible to the bulk-copy engine
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&sfull[pend_sb]);
        if (pend_extra) mbar_arrive(&sfull[pend_sb]);  // a lone last unit
      }
      pend_sb = -1;
    };
#ifdef RNSW_K1_PROF
    long long e_tf = 0, e_se = 0, e_0 = clock64();
#endif
    RNSW_FOR_UNITS(u) {
      if (h_ == 0) ++jt;
      const int as = it & 1;
#ifdef RNSW_K1_PROF
      long long e1 = clock64();
#endif
      mbar_wait(&tfull[as], (it >> 1) & 1);
      tc_fence_after();
#ifdef RNSW_K1_PROF
      e_tf += clock64() - e1;
#endif
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + as * Cfg::kAccCols + hh * kEpiCols;
      uint32_t lo[8], hi[8];  // [chunk of 16 channels][word]
      int32_t a0[16], b0[16], a1[16], b1[16];
#if RNSW_K1_NO_TMEM_LD  // diagnostic: no TMEM reads in the epilogue (MMA pipeline alone)
#pragma unroll
      for (int e = 0; e < 16; ++e) a0[e] = b0[e] = a1[e] = b1[e] = e + it;
      if (false)
#endif
      // (RNSW_K1_EPI_PIPE: the second 16-channel chunk's loads fly while the
      // first chunk is converted; the buffer is released after the second wait)
      constexpr bool kPipe = RNSW_K1_EPI_PIPE && kEpiCols == 32 && !RNSW_K1_NO_TMEM_LD &&
                             RNSW_K1_DIAG != 2 && RNSW_K1_DIAG != 6;
      if (kLimbs == 2) {
        tmem_ld16(taddr, a0);
        tmem_ld16(taddr + kUnitN, b0);
        if (kEpiCols == 32) {
          if (kPipe) tmem_ld_wait();
          tmem_ld16(taddr + 16, a1);
          tmem_ld16(taddr + kUnitN + 16, b1);
        }
      } else {
        tmem_ld16(taddr, b0);
        if (kEpiCols == 32) {
          if (kPipe) tmem_ld_wait();
          tmem_ld16(taddr + 16, b1);
        }
      }
      if (kPipe) convert(a0, b0, lo, hi);
      tmem_ld_wait();
      // hand the buffer back to the MMA warp (kPair: the leader CTA's barrier)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (kPair)
          mbar_arrive_remote(mapa_shared(smem_u32(&tempty[as]), 0));
        else
          mbar_arrive(&tempty[as]);
      }
      if (RNSW_K1_DIAG != 2 && RNSW_K1_DIAG != 6) {
        if (!kPipe) convert(a0, b0, lo, hi);
        if (kEpiCols == 32) convert(a1, b1, lo + 4, hi + 4);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) lo[e] = hi[e] = (uint32_t)(a0[e] ^ b1[e]);
      }
      // the pair's staging buffer must be free: its previous bulk store has read it
      const int sb = jt % Cfg::kNStg;
      const uint32_t sph = (uint32_t)(jt / Cfg::kNStg) & 1u;
      if (RNSW_K1_DEFER) hand_off();  // the previous unit's staging, now surely written
#ifdef RNSW_K1_PROF
      long long e2 = clock64();
#endif
      if (h_ == 0) mbar_wait(&sempty[sb], sph ^ 1u);
#ifdef RNSW_K1_PROF
      e_se += clock64() - e2;
#endif
      uint8_t* sbuf = stg + sb * Cfg::kStgBytes;
#if RNSW_K1_DIAG == 11
      {
        uint4* dst = reinterpret_cast<uint4*>(args.v_raw + (((size_t)u * 8 + (warp - 4)) * 32 + lane) * 64);
        dst[0] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        dst[1] = make_uint4(lo[4], lo[5], lo[6], lo[7]);
        dst[2] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        dst[3] = make_uint4(hi[4], hi[5], hi[6], hi[7]);
      }
#endif
#pragma unroll
      for (int pl = 0; pl < ((RNSW_K1_NO_STORE || RNSW_K1_DIAG == 12) ? 0 : kLimbs); ++pl) {
        uint8_t* base = sbuf + pl * (kGroupRows * 2 * kUnitN);
#pragma unroll
        for (int ch = 0; ch < kEpiCols / 16; ++ch) {
          const uint32_t* src = pl == 0 ? lo : hi;
          const uint4 v4 = make_uint4(src[ch * 4], src[ch * 4 + 1], src[ch * 4 + 2], src[ch * 4 + 3]);
          uint32_t off;
          if (two && args.pair128) {
            // [pos][tiles 2k, 2k+1][64 channels] as one 128-byte row under the
            // 128B swizzle: the 32 positions of a warp spread over all 32
            // banks (64-byte rows under the 64B swizzle put them on 4 chunk
            // columns, 8-way conflicts)
            const uint32_t c16 = (uint32_t)(h_ * 4 + hh * (kEpiCols / 16) + ch);
            off = (uint32_t)row * 128 + (RNSW_K1_STG_SWZ ? ((c16 ^ ((uint32_t)row & 7u)) << 4) : (c16 << 4));
          } else if (two) {
            // odd P: [pos][tile h_][64 channels], 64-byte rows, 64B swizzle (chunk ^= (row >> 1) & 3)
            const uint32_t r64 = (uint32_t)(row * 2 + h_), c16 = (uint32_t)(hh * (kEpiCols / 16) + ch);
            off = r64 * 64 + ((c16 ^ ((r64 >> 1) & 3u)) << 4);
          } else {
            // [pos][128 channels of blocks h_]: 128-byte rows, 128B swizzle (chunk ^= row & 7)
            const uint32_t c16 = (uint32_t)(h_ * 4 + hh * (kEpiCols / 16) + ch);
            off = (uint32_t)row * 128 + ((c16 ^ ((uint32_t)row & 7u)) << 4);
          }
          *reinterpret_cast<uint4*>(base + off) = v4;
        }
      }
      pend_sb = sb;
      pend_extra = (h_ == 0 && u + 1 >= args.units) ? 1 : 0;
      if (!RNSW_K1_DEFER) hand_off();
      ++it;
    }
    hand_off();  // the last unit's
#ifdef RNSW_K1_PROF
    if (lane == 0 && blockIdx.x < 4 && (warp == 4 || warp == 11))
      printf("K1PROF cta %d epi warp %d units %d total %lld wait_tfull %lld wait_sempty %lld (per unit %lld %lld %lld)\n",
             blockIdx.x, warp, it, clock64() - e_0, e_tf, e_se, (clock64() - e_0) / it, e_tf / it, e_se / it);
#endif
  }
  tc_fence_before();
  if (kPair)
    cluster_sync();  // the pair's last MMAs and TMEM reads are done in both CTAs
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (kPair)
      tmem_dealloc_2sm<Cfg::kTmemCols>(tmem_base);
    else
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
  plan.kr_group_bytes = (size_t)plan.kr_limbs * kGroupRows * plan.kr_kp;
  std::vector<uint8_t> img((size_t)plan.kr_groups * plan.kr_group_bytes, 0);
  for (int r = 0; r < RNSW_MAX_RES; ++r) plan.kr_xmax[r] = 0;
  for (int r = 0; r < d.n_res; ++r) {
    const int64_t m = d.res[r].modulus;
    for (int pbk = 0; pbk < plan.kr_npb; ++pbk) {
      uint8_t* gimg = img.data() + (size_t)(r * plan.kr_npb + pbk) * plan.kr_group_bytes;
      for (int row = 0; row < kGroupRows; ++row) {
        const int pos = pbk * kGroupRows + row;
        if (pos >= npos) break;
        const int i = pos / N, j = pos % N;
        int64_t xrow = 0;
        for (int pix = 0; pix < npos; ++pix) {
          const int a = pix / N, b = pix % N;
          const int64_t v = sym_host((int64_t)d.res[r].bt[i * RNSW_MAX_N + a] * d.res[r].bt[j * RNSW_MAX_N + b], m);
          int8_t limb[2];
          if (plan.kr_limbs == 1) {
            limb[0] = (int8_t)v;
            xrow += 128 * (v < 0 ? -v : v);
          } else {
            const int64_t h = (v + 128 + 256 * 64) / 256 - 64;  // floor((v + 128) / 256)
            limb[0] = (int8_t)h;            // limb 0: high (x 256)
            limb[1] = (int8_t)(v - 256 * h);  // limb 1: low
            xrow += 128 * (256 * (h < 0 ? -h : h) + (limb[1] < 0 ? -limb[1] : limb[1]));
          }
          for (int l = 0; l < plan.kr_limbs; ++l)
            gimg[((size_t)l * kGroupRows + row) * plan.kr_kp + pix] = (uint8_t)limb[l];
        }
        if (xrow > plan.kr_xmax[r]) plan.kr_xmax[r] = xrow;
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
  return g.C % 64 == 0;
}

cudaError_t launch_input_transform_umma(const PlanHost& plan, const Geometry& g, const int8_t* x, int8_t* V,
                                        cudaStream_t s, bool relaxed) {
  const PlanDevice& d = plan.dev;
  K1UArgs a{};
  a.g = g;
  a.npos = d.n * d.n;
  a.mout = d.m_out;
  a.kp = plan.kr_kp;
  a.ksteps = plan.kr_kp / 32;
  a.limbs = plan.kr_limbs;
  // CTA pairs (cta_group::2) when a residue has two 128-position blocks
  // (opt-in, RNSW_K1_PAIR=1: measured equal or slower -- K1 is not bound by
  // its patch reads)
  static const bool want_pair = getenv("RNSW_K1_PAIR") != nullptr;
  const bool pair = want_pair && plan.kr_npb == 2;
  a.groups = pair ? d.n_res : plan.kr_groups;
  a.npb = plan.kr_npb;
  a.group_bytes = plan.kr_group_bytes;
  a.v_raw = reinterpret_cast<uint8_t*>(V);
  a.cblocks = g.Cp / kUnitN;
  const int64_t units = g.P * a.cblocks;
  if (units >= (1ll << 31) || g.P >= (1ll << 31)) return cudaErrorInvalidValue;
  a.units = (int)units;
  for (int gi = 0; gi < a.groups; ++gi) {
    a.res_of[gi] = pair ? gi : gi / a.npb;
    a.pb_of[gi] = pair ? 0 : gi % a.npb;  // pair: the CTA's rank in its cluster
  }
  for (int r = 0; r < d.n_res; ++r) {
    a.plane_base[r] = d.res[r].plane_base;
    const ResidueTables& t = d.res[r];
    a.fm[r] = FastMod{t.red_mul, t.red_shift, t.red_off, t.modulus, t.half, t.red_negm};
    a.mul0[r] = (uint32_t)(((1ull << 32) + t.modulus - 1) / t.modulus);
    if (plan.kr_limbs == 2) {
      // bias = 127 T with T = 256 S1 + S2, T >= xmax / 127 and bias = target
      // (mod m): target h (kSym16: n mod m = (x + h) mod m) or 128 (kRel16)
      const int64_t m = t.modulus, target = relaxed ? 128 : t.half;
      int64_t inv127 = 1;
      while ((127 * inv127) % m != 1) ++inv127;
      const int64_t want = target * inv127 % m;
      const int64_t t0 = (plan.kr_xmax[r] + 126) / 127;
      const int64_t T = t0 + ((want - t0) % m + m) % m;
      if ((T >> 8) > 4064 || 127 * T + plan.kr_xmax[r] >= (1ll << 30)) return cudaErrorInvalidValue;
      a.bias_s1[r] = (int32_t)(T >> 8);
      a.bias_s2[r] = (int32_t)(T & 255);
    }
  }
  a.div_img = make_fastdiv((uint32_t)(g.th * g.tw));
  a.div_tw = make_fastdiv((uint32_t)g.tw);
  a.div_cb = make_fastdiv((uint32_t)a.cblocks);

  auto encode = encode_fn();
  if (encode == nullptr) return cudaErrorInvalidValue;
  CUtensorMap tmX, tmV;
  {
    // x NHWC as (C, W, H, B); box = 64 channels x N x N x 1 (pair: 32 channels per CTA, 32B swizzle)
    cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.B};
    cuuint64_t strides[3] = {(cuuint64_t)g.C, (cuuint64_t)g.W * g.C, (cuuint64_t)g.H * g.W * g.C};
    cuuint32_t box[4] = {(cuuint32_t)(pair ? kUnitN / 2 : kUnitN), (cuuint32_t)d.n, (cuuint32_t)d.n, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (encode(&tmX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(x), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, pair ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  CUtensorMap tmV2;
  {
    // V as (Cp, P, npos, planes); a unit pair's box = 64 channels x 2 tiles x
    // 128 positions x 1 plane (Cp = 64: with P even one 128-byte row per
    // position, 128B swizzle; odd P 64B swizzle) or 128 channels x 1 tile x
    // 128 positions x 1 plane (128B swizzle)
    const int npos = d.n * d.n;
    cuuint64_t dims[4] = {(cuuint64_t)g.Cp, (cuuint64_t)g.P, (cuuint64_t)npos, (cuuint64_t)d.n_planes};
#if RNSW_K1_DIAG == 4
    // diagnostic: tile-major V (positions of a tile contiguous) -- wrong for the GEMM, write-locality probe
    cuuint64_t strides[3] = {(cuuint64_t)npos * g.Cp, (cuuint64_t)g.Cp, (cuuint64_t)g.P * g.Cp * npos};
#else
    cuuint64_t strides[3] = {(cuuint64_t)g.Cp, (cuuint64_t)g.P * g.Cp, (cuuint64_t)g.P * g.Cp * npos};
#endif
    cuuint32_t es[4] = {1, 1, 1, 1};
    a.pair128 = (g.Cp == 64 && (g.P & 1) == 0) ? 1 : 0;
    if (a.pair128) {
      // tile pairs as 128-byte rows: (2 Cp, P / 2, npos, planes)
      cuuint64_t dims2[4] = {(cuuint64_t)(2 * g.Cp), (cuuint64_t)(g.P / 2), (cuuint64_t)npos, (cuuint64_t)d.n_planes};
#if RNSW_K1_DIAG == 4
      cuuint64_t strides2[3] = {(cuuint64_t)(2 * g.Cp) * npos, (cuuint64_t)(2 * g.Cp), (cuuint64_t)g.P * g.Cp * npos};
#else
      cuuint64_t strides2[3] = {(cuuint64_t)(2 * g.Cp), (cuuint64_t)g.P * g.Cp, (cuuint64_t)g.P * g.Cp * npos};
#endif
      cuuint32_t boxp[4] = {(cuuint32_t)(2 * kUnitN), 1, (cuuint32_t)kGroupRows, 1};
      if (encode(&tmV, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, V, dims2, strides2, boxp, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 RNSW_K1_STG_SWZ ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    } else {
      cuuint32_t box[4] = {(cuuint32_t)kUnitN, 2, (cuuint32_t)kGroupRows, 1};
      if (encode(&tmV, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, V, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
    cuuint32_t box2[4] = {(cuuint32_t)(2 * kUnitN), 1, (cuuint32_t)kGroupRows, 1};
    if (g.Cp >= 128 && encode(&tmV2, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, V, dims, strides, box2, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    if (g.Cp < 128) tmV2 = tmV;
  }
  // one CTA (or CTA pair) per SM (pair) spread evenly over the groups
  const int sms = num_sms_current();
  // co-resident CTAs per SM: 2 for the 8-bit plans when their shared memory fits twice
  const size_t smem_need = plan.kr_limbs == 2 ? K1UConfig<2>::kSmem : K1UConfig<1>::kSmem;
  const int per_sm = (!pair && plan.kr_limbs == 1 && 2 * (smem_need + 1024) <= 228 * 1024) ? 2 : 1;
  const int slots = pair ? sms / 2 : sms * per_sm;
  const int per_group = slots / a.groups > 0 ? slots / a.groups : 1;
  int64_t grid = (int64_t)per_group * a.groups;
  const int64_t need = (int64_t)((a.units + 1) / 2) * a.groups;
  if (grid > need) grid = need;
  grid = (grid + a.groups - 1) / a.groups * a.groups;
  auto run = [&](auto kern, size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return launch_ex(kern, dim3((unsigned)(pair ? 2 * grid : grid)), dim3(kUThreads), smem, s, pair ? 2 : 1, tmX, tmV,
                     tmV2, (const uint8_t*)plan.d_kr, a);
  };
  if (pair) {
    if (plan.kr_limbs == 2)
      return relaxed ? run(input_umma_kernel<kRel16, true>, K1UConfig<2>::kSmem)
                     : run(input_umma_kernel<kSym16, true>, K1UConfig<2>::kSmem);
    return run(input_umma_kernel<kSym8, true>, K1UConfig<1>::kSmem);
  }
  if (plan.kr_limbs == 2)
    return relaxed ? run(input_umma_kernel<kRel16, false>, K1UConfig<2>::kSmem)
                   : run(input_umma_kernel<kSym16, false>, K1UConfig<2>::kSmem);
  return run(input_umma_kernel<kSym8, false>, K1UConfig<1>::kSmem);
}

}  // namespace rnsw
