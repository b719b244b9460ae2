// K4-K6 on the 5th-generation tensor cores for F(14x14, 3x3) over two 16-bit
// residues (BASELINE configs 2 and 4): inverse Winograd transform
// Y = AT M A mod m for both residues, mixed-radix reconstruction and
// crop/scatter -- or the fused relu / shift / clip / 2x2 max-pool glue -- in
// one kernel (rw/kernel.py:50-53, rw/residue.py:180-206, rw/layer.py:374-388).
//
// Persistent CTAs (two per SM, 8 warps, 256 TMEM columns each) over work
// units of one tile x 32 output channels.
// The GEMM (or the small-channel product) leaves y mod m in [0, m) as two
// byte planes (Mw8, kernels.h), so both transform passes are tcgen05
// kind::i8 MMAs with M = 128, N = 32, K = 32 and the CUDA cores only
// recombine limbs, reduce and reconstruct:
//
//   pass 1  rows (j, k) = 4 columns j x 32 channels k, K = (limb, i):
//           A1 = Mat[i][j] limbs, TMA-loaded MN-major (32B swizzle) straight
//           from Mw8; B1 = [256 AT mod m | AT] limbs; D1 = [A256 | A1] per a.
//           z[a] = 256 A256 + A1 = sum_i AT[a][i] Mat[i][j] (mod m) is kept
//           exact (|z| < 2^23, plan z3) and written back as three bytes
//           z0, z1 (u8) and z2 (s8) into
//   pass 2  rows (k, a) = 8 channels x 16 rows a, K = (limb, j):
//           A2 = z limbs (MN-major, one 16-byte chunk per (thread, limb)),
//           B2 = limbs of AT W, 256 AT W and 65536 AT W mod m (W = the
//           mixed-radix factor of the residue), plus constant K rows that
//           add a multiple of m as the reduction bias; D2 = [A256 | A1] per
//           b.  y = 256 A256 + A1 reduces once to the mixed-radix digit.
//
// Per unit: 2 TMA boxes (one per residue), 8 + 16 MMAs issued from one asm
// block per pass, two TMEM round trips; every column group of pass 1 and every
// channel block of pass 2 commits to its own mbarrier, so each epilogue starts
// on the first block while the rest of the batch runs; the next unit's boxes
// load during this unit's epilogues.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace rnsw {
namespace {

// Waits for the MMA batches: with RNSW_K4_SLEEP=ns the waiting warps suspend
// in mbarrier.try_wait (woken when the phase completes) instead of spinning,
// leaving issue slots to the co-resident CTA
#ifndef RNSW_K4_EPI2_PIPE
#define RNSW_K4_EPI2_PIPE 1
#endif
#ifndef RNSW_K4_EARLY_P1
#define RNSW_K4_EARLY_P1 1
#endif
#ifndef RNSW_K4_EARLY_P1_ALL
#define RNSW_K4_EARLY_P1_ALL 0
#endif
#ifndef RNSW_K4_SLEEP
#define RNSW_K4_SLEEP 0
#endif
// 1: every pair of pass-1 MMAs (one column group of both residues) and every
// channel block of pass 2 commits to its own mbarrier, so an epilogue starts on
// the first block while the rest of the batch still runs (0: two commits per
// batch, one per warp group)
#ifndef RNSW_K4_FINE
#define RNSW_K4_FINE 1
#endif
#if RNSW_K4_SLEEP
#define K4_WAIT(b, ph) mbar_wait_sleep(b, ph, RNSW_K4_SLEEP)
#else
#define K4_WAIT(b, ph) mbar_wait(b, ph)
#endif

constexpr int kKB = 32;     // output channels per work unit
constexpr int kThr = 256;   // 8 warps: TMEM lane quadrant q = warp & 3, half h = warp >> 2
constexpr int kOpBytes = 4096;  // one MMA A operand: 32 K rows x 128 bytes
constexpr int kOffA1 = 0;                         // [res][g]          8 x 4 KB
constexpr int kOffA2 = kOffA1 + 8 * kOpBytes;     // [res][mb][step]  16 x 4 KB
constexpr int kOffB1 = kOffA2 + 16 * kOpBytes;    // [res]             2 x 1 KB
constexpr int kOffB2 = kOffB1 + 2 * 1024;         // [res][step]       4 x 1 KB
constexpr int kOffOut = kOffB2 + 4 * 1024;        // output staging
constexpr int kPixB = 48;   // staged bytes per pixel, int8 modes (16-byte aligned rows for 16-byte stores)
constexpr int kPixW = 33;   // staged words per pixel (int32 mode)
// Staging of the int8 tile when it leaves through one TMA bulk tensor store
// (kTma): dense 32-byte pixels, every staged byte at a per-thread base plus a
// literal.  Pooled (7 x 7): no swizzle (rows 224 bytes apart: the 7 storing
// lanes of a warp meet 2-way).  Unpooled (14 x 14): 32B swizzle (16-byte chunk
// ^= pixel bit 2; dense rows would put a warp's 16 rows a into two banks); the
// swizzle bit of pixel (a, b) is bit 2 of (6 a mod 8) + b, so each thread
// keeps four bases -- plain / flipped chunk, for columns whose bit agrees or
// disagrees between even and odd rows -- and picks one per column at compile
// time.
// The int32 mode stages its 196 x 33-word tile in the A1 region (32 KB, free
// once pass 1 has completed): the next unit's Mw8 boxes are then requested
// after the stores instead of during the epilogues, and in exchange two CTAs
// fit per SM like in the int8 modes (a separate 26 KB staging tile allowed one).
constexpr int out_bytes(int mode) { return mode == 0 ? 0 : (mode == 1 ? 196 * kPixB : 49 * kPixB); }
constexpr int out_off(int mode) { return mode == 0 ? kOffA1 : kOffOut; }
constexpr int smem_bytes(int mode) { return 1024 + kOffOut + ((out_bytes(mode) + 15) & ~15) + 128; }
static_assert(196 * kPixW * 4 <= 8 * kOpBytes, "the int32 tile must fit the A1 region");

// The MMA batches of a pass are issued from ONE asm block: one elect.sync,
// every descriptor = the (1024-byte aligned) shared-memory base in descriptor
// units plus a literal, so the issuing warp spends a few instructions per MMA
// (separate per-MMA blocks rebuilt both 64-bit descriptors from the address
// and re-elected each time: ~17 instructions per MMA on the critical warp).
#define K4_OFF_A1 0
#define K4_OFF_A2 32768
#define K4_OFF_B1 98304
#define K4_OFF_B2 100352
static_assert(K4_OFF_A1 == kOffA1 && K4_OFF_A2 == kOffA2 && K4_OFF_B1 == kOffB1 && K4_OFF_B2 == kOffB2, "asm offsets");
#define K4_STR2(x) #x
#define K4_STR(x) K4_STR2(x)
// D columns, A byte offset / LBO field / high word, B byte offset, idesc operand, accumulate predicate
#define K4_MMA(DCOL, AOFF, ALBO, AHI, BOFF, ID, ACCP)                           \
  "add.u32 t, %0, " K4_STR(DCOL) ";\n\t"                                        \
  "add.u32 al, %1, " K4_STR((((AOFF) >> 4) + ((ALBO) << 16))) ";\n\t"           \
  "add.u32 bl, %1, " K4_STR((((BOFF) >> 4) + (1 << 16))) ";\n\t"                \
  "mov.b64 da, {al, " K4_STR(AHI) "};\n\t"                                      \
  "mov.b64 db, {bl, 0xC0004010};\n\t"                                           \
  "@e tcgen05.mma.cta_group::1.kind::i8 [t], da, db, " ID ", " ACCP ";\n\t"
#define K4_COMMIT(BAR) "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [" BAR "];\n\t"
#define K4_COMMIT_AT(BASE, I) "add.u32 ba, " BASE ", " #I " * 8;\n\t" K4_COMMIT("ba")
// pass 1, v = res * 4 + gg: A1 + v * 4 KB (MN-major, 32B swizzle, LBO 1 KB), B1 + res * 1 KB
#define K4_P1(V) K4_MMA((V) * 32, K4_OFF_A1 + (V) * 4096, 64, 0xC0004010, K4_OFF_B1 + ((V) >> 2) * 1024, "%2", "pz")
// pass 2, v = res * 4 + mb: A2 + v * 8 KB (MN-major, 128B swizzle; step 1 at + 4 KB), B2 + res * 2 KB (+ 1 KB)
#define K4_P2(V)                                                                                              \
  K4_MMA((V) * 32, K4_OFF_A2 + (V) * 8192, 1, 0x40004040, K4_OFF_B2 + ((V) >> 2) * 2048, "%2", "pz")           \
  K4_MMA((V) * 32, K4_OFF_A2 + (V) * 8192 + 4096, 1, 0x40004040, K4_OFF_B2 + ((V) >> 2) * 2048 + 1024, "%3", "po")
#define K4_ASM_HEAD                                                                                   \
  "{\n\t.reg .pred e, pz, po;\n\t.reg .b32 t, al, bl, ba;\n\t.reg .b64 da, db;\n\t"                        \
  "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 pz, 0, 0;\n\tsetp.eq.b32 po, 0, 0;\n\t"

struct UArgs {
  Geometry g;
  int8_t* out8;
  int32_t* y;
  int shift;
  int vec16;           // int8 output: K % 16 == 0 and out8 16-byte aligned -> 16-byte stores
  int tma_out;         // int8 NHWC output through a TMA bulk tensor store of the staged tile (needs vec16)
  int kblocks;
  int64_t units;       // P * kblocks work units (tile, 32-channel block)
  int32_t negw10;      // -W[1][0] (kept opaque to the compiler: one IMAD per digit)
  uint32_t mul0;       // ceil(2^32 / m0): quotient estimate of the first digit
  FastDiv div_img, div_tw, div_kb;
};

// Persistent: two CTAs per SM (each 256 TMEM columns, shared by the pass-1
// and pass-2 accumulators) walk the work units u = (tile p, channel block
// kb); while one CTA waits for its MMAs the other runs its epilogues.  The
// Mw8 boxes of the next unit load during the current unit's epilogues.
// (A single 16-warp CTA per SM that overlaps pass 1 of the next unit with
// epilogue 2 in separate TMEM halves measured 25% slower: every warp then
// waits on the same pass-2 completion and barriers.)
template <int kMode, bool kTma>
__global__ void __launch_bounds__(kThr, 2)
    output_umma_kernel(const PlanDevice* __restrict__ plan, const __grid_constant__ CUtensorMap tm,
                       const __grid_constant__ CUtensorMap tmo, UArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned, derived from the shared array so stores stay STS
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kOffOut + ((out_bytes(kMode) + 15) & ~15));
  uint64_t* bar_tfree = bar + 3;  // RNSW_K4_EARLY_P1: every warp has read its pass-2 accumulators
  uint64_t* bar_p1 = bar + 4;     // RNSW_K4_FINE: pass 1, column group gg of both residues complete
  uint64_t* bar_p2 = bar + 8;     // RNSW_K4_FINE: pass 2, channel block mbi of warp group h complete (index 2 mbi + h)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 12);
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;  // warp-uniform for the compiler
  const int q = warp & 3, h = warp >> 2;
  const Geometry& g = args.g;
  pdl_trigger();
  // staged bytes (int8 modes): this thread's rows (k, a) start at st_base; a
  // pixel is kPix bytes, the second channel block of the warp group 8 further
  constexpr int kPix = kTma ? 32 : kPixB;
  uint8_t* st_base;
  uint8_t* st_e[2];  // unpooled kTma: columns b with b % 4 < 2, swizzle bit = bit2(b) ^ s
  uint8_t* st_f[2];  //                columns b with b % 4 >= 2
  {
    const int a = lane & 15, kl0 = 16 * h + 2 * q + (lane >> 4);
    const int row = kMode == 3 ? (a >> 1) * 7 * kPix : a * 14 * kPix;
    st_base = smem + kOffOut + row + kl0;
    // bit 2 of (14 a + b) = bit2(b) ^ [a % 4 == 2]          for even a
    //                     = bit2(b + 2) ^ [a % 4 == 1]      for odd a
    const int flip = (a & 1) ? ((a & 3) == 1) : ((a & 3) == 2);
    st_e[0] = st_base + 16 * (flip ? 1 - 2 * h : 0);  // chunk bit of kl0 is h: kl0 ^ 16
    st_e[1] = st_base + 16 * (flip ? 0 : 1 - 2 * h);
    st_f[0] = (a & 1) ? st_e[1] : st_e[0];  // bit2(b + 2) = !bit2(b) for b % 4 >= 2
    st_f[1] = (a & 1) ? st_e[0] : st_e[1];
  }
  // address of column b of this thread's row, channel block mbi (unpooled)
  auto st_col = [&](int mbi, int b) -> uint8_t* {
    if constexpr (kTma && kMode == 1) {
      const int s = (b >> 2) & 1;
      return ((b & 3) < 2 ? st_e[s] : st_f[s]) + mbi * 8 + b * 32;
    } else {
      return st_base + mbi * 8 + b * kPix;
    }
  };
  constexpr int kStoreTid = 192;  // issues (and waits for) the bulk tensor stores: not the MMA warp

  if (tid == 0) {
    tma_prefetch_desc(&tm);
    mbar_init(&bar[0], 1);  // Mw8 boxes landed
    mbar_init(&bar[1], 1);  // MMA batch for warps 0-3 complete
    mbar_init(&bar[2], 1);  // MMA batch for warps 4-7 complete (implies bar[1]: commits track all prior MMAs)
    mbar_init(bar_tfree, kThr / 32);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&bar_p1[i], 1);
      mbar_init(&bar_p2[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(tslot);

  // Constant B operands (K-major, 32-byte rows, 32B swizzle): built on the
  // host into the plan (capi.cu build_umma_b), 6 KB copied once per CTA
  for (int idx = tid; idx < 6144 / 16; idx += kThr)
    reinterpret_cast<uint4*>(smem + kOffB1)[idx] = __ldg(reinterpret_cast<const uint4*>(plan->umma_b) + idx);
  const FastMod fm0 = fast_mod_of(plan->res[0]), fm1 = fast_mod_of(plan->res[1]);
  // the constant 127 in K rows 16..31 of every step-1 A2 operand (see B2)
  for (int idx = tid; idx < 8 * 512; idx += kThr) {
    const int u = idx >> 9, w = idx & 511;  // 512 words = rows 16..31 of buffer u
    *reinterpret_cast<uint32_t*>(smem + kOffA2 + (u * 2 + 1) * kOpBytes + 2048 + 4 * w) = 0x7F7F7F7Fu;
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  pdl_wait();  // Mw8 and the output buffer's previous users

  const int32_t negw10 = args.negw10;
  const uint32_t mul0 = args.mul0;
  const uint32_t m0 = (uint32_t)fm0.m;
  const uint32_t signed_bound = (uint32_t)plan->signed_bound, dyn_range = (uint32_t)plan->dynamic_range;
  constexpr uint32_t kIdP1 = idesc_i8x(128, 32, false, true, true, false);   // u8 MN-major x s8
  constexpr uint32_t kIdP2s = idesc_i8x(128, 32, true, true, true, false);   // s8 MN-major x s8
  uint8_t* A1 = smem + kOffA1;
  uint8_t* A2 = smem + kOffA2;
  const uint32_t dbase = (smem_u32(smem) >> 4) & 0x3FFF;  // descriptor start-address field of the operand area
  const uint32_t bar1_addr = smem_u32(RNSW_K4_FINE ? &bar_p1[0] : &bar[1]);
  const uint32_t bar2_addr = smem_u32(RNSW_K4_FINE ? &bar_p2[0] : &bar[2]);

  // unit -> (tile p, channel offset k0); kb fastest
  auto unit_p = [&](int64_t u) { return (int)fdiv((uint32_t)u, args.div_kb); };
  auto issue_load = [&](int64_t u) {
    const int p = unit_p(u), k0 = (int)(u - (int64_t)p * args.kblocks) * kKB;
    mbar_arrive_expect_tx(&bar[0], 8 * kOpBytes);
    const int L0 = (p >> 7) * 4;  // (pb * n_res + res) * 2 + limb, n_res = 2
#pragma unroll
    for (int res = 0; res < 2; ++res)  // one box per residue: all 16 columns j (4 KB per column group)
      tma_load_5d(A1 + res * 4 * kOpBytes, &tm, &bar[0], k0, 0, L0 + 2 * res, 0, p & 127);
  };
  const int64_t u_step = gridDim.x;
  // each MMA batch is committed in two halves, one per warp group (h), so the
  // first group starts its epilogue while the second half still runs
  uint32_t ph_tma = 0, ph_mma = 0, ph_tfree = 0, ph1 = 0, ph2 = 0;
  uint64_t* my_bar = &bar[1 + h];
  (void)ph_mma;
  (void)my_bar;
  auto issue_p1 = [&]() {  // warp 0: pass 1 into the 256 TMEM columns once the boxes landed
    mbar_wait(&bar[0], ph_tma);
    ph_tma ^= 1;
    tc_fence_after();
    // v = res * 4 + gg; residue h feeds warp group h
#if RNSW_K4_FINE
    asm volatile(K4_ASM_HEAD K4_P1(0) K4_P1(4) K4_COMMIT_AT("%4", 0) K4_P1(1) K4_P1(5) K4_COMMIT_AT("%4", 1) K4_P1(2)
                     K4_P1(6) K4_COMMIT_AT("%4", 2) K4_P1(3) K4_P1(7) K4_COMMIT_AT("%4", 3) "}" ::"r"(tbase),
                 "r"(dbase), "r"(kIdP1), "r"(kIdP2s), "r"(bar1_addr), "r"(bar2_addr)
                 : "memory");
#else
    asm volatile(K4_ASM_HEAD K4_P1(0) K4_P1(1) K4_P1(2) K4_P1(3) K4_COMMIT("%4") K4_P1(4) K4_P1(5) K4_P1(6) K4_P1(7)
                     K4_COMMIT("%5") "}" ::"r"(tbase),
                 "r"(dbase), "r"(kIdP1), "r"(kIdP2s), "r"(bar1_addr), "r"(bar2_addr)
                 : "memory");
#endif
  };
  if (warp == 0 && (int64_t)blockIdx.x < args.units) {
    if (lane == 0) issue_load(blockIdx.x);
    __syncwarp();
    issue_p1();
  }

#ifdef RNSW_K4_PROF
  long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pt0 = clock64();
  int pn = 0;
#define K4T(i) { long long _c = clock64(); pc[i] += _c - pl_; pl_ = _c; }
#else
#define K4T(i)
#endif
  for (int64_t u = blockIdx.x; u < args.units; u += u_step) {
#ifdef RNSW_K4_PROF
    long long pl_ = clock64();
    ++pn;
#endif
    const int p = unit_p(u), k0 = (int)(u - (int64_t)p * args.kblocks) * kKB;
    // ---- pass 1 (issued before the previous unit's stores) ----
#if RNSW_K4_FINE
    // column group gg of this unit's pass 1 (both residues) has completed
    auto wait_p1 = [&](int gg) {
      K4_WAIT(&bar_p1[gg], ph1);
      tc_fence_after();
      // the last group's barrier means all of pass 1 is done: A1 is free
      if (gg == 3 && kMode != 0 && tid == kThr / 2 && u + u_step < args.units) issue_load(u + u_step);  // lands during the epilogues
    };
    wait_p1(0);
    K4T(0)
#else
    auto wait_p1 = [&](int) {};
    K4_WAIT(my_bar, ph_mma);
    K4T(0)
    ph_mma ^= 1;
    tc_fence_after();
    // the second group's barrier means all of pass 1 is done: A1 is free
    if (kMode != 0 && tid == kThr / 2 && u + u_step < args.units) issue_load(u + u_step);  // lands during the epilogues
#endif

    // ---- epilogue 1: warp (q, h): columns j = 4 gg + q of residue h, lane = channel ----
    {
      uint8_t* a2 = A2 + (h * 4 + (lane >> 3)) * 2 * kOpBytes;
      const uint32_t chunk = (uint32_t)(lane & 7) << 4;
      // column group gg: z -> three byte limbs -> A2 (the TMEM loads of the
      // next group are in flight meanwhile: two register sets, one wait each)
      auto body = [&](int gg, const int32_t (&hi)[16], const int32_t (&lo)[16]) {
        const int j = 4 * gg + q;
        int32_t z[16];
#pragma unroll
        for (int a = 0; a < 14; ++a) z[a] = hi[a] * 256 + lo[a];
        z[14] = z[15] = 0;  // rows a >= 14 of AT are zero; their pass-2 rows are discarded
        uint32_t w0[4], w1[4], w2[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t t01 = __byte_perm(z[4 * c], z[4 * c + 1], 0x5140);
          const uint32_t t23 = __byte_perm(z[4 * c + 2], z[4 * c + 3], 0x5140);
          w0[c] = __byte_perm(t01, t23, 0x5410);
          w1[c] = __byte_perm(t01, t23, 0x7632);
          w2[c] = __byte_perm(__byte_perm(z[4 * c], z[4 * c + 1], 0x0062),
                              __byte_perm(z[4 * c + 2], z[4 * c + 3], 0x0062), 0x5410);
        }
        *reinterpret_cast<uint4*>(a2 + swz128(j * 128 + chunk)) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
        *reinterpret_cast<uint4*>(a2 + swz128((16 + j) * 128 + chunk)) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
        *reinterpret_cast<uint4*>(a2 + kOpBytes + swz128(j * 128 + chunk)) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
      };
      const uint32_t ta = tbase + ((uint32_t)(32 * q) << 16) + h * 4 * 32;
#if RNSW_K4_EPI1_ALLLD
      {  // all eight TMEM loads in flight, one wait
        int32_t hv[4][16], lv[4][16];
#pragma unroll
        for (int gg = 0; gg < 4; ++gg) {
          tmem_ld16(ta + 32 * gg, hv[gg]);
          tmem_ld16(ta + 32 * gg + 16, lv[gg]);
        }
        tmem_ld_wait();
#pragma unroll
        for (int gg = 0; gg < 4; ++gg) body(gg, hv[gg], lv[gg]);
      }
      static_assert(!RNSW_K4_FINE, "RNSW_K4_EPI1_ALLLD needs RNSW_K4_FINE=0");
#else
      int32_t hA[16], lA[16], hB[16], lB[16];
      tmem_ld16(ta, hA);
      tmem_ld16(ta + 16, lA);
      tmem_ld_wait();
      wait_p1(1);
      tmem_ld16(ta + 32, hB);
      tmem_ld16(ta + 48, lB);
      body(0, hA, lA);
      tmem_ld_wait();
      wait_p1(2);
      tmem_ld16(ta + 64, hA);
      tmem_ld16(ta + 80, lA);
      body(1, hB, lB);
      tmem_ld_wait();
      wait_p1(3);
      tmem_ld16(ta + 96, hB);
      tmem_ld16(ta + 112, lB);
      body(2, hA, lA);
      tmem_ld_wait();
      body(3, hB, lB);
#endif
      ph1 ^= 1;
    }
    K4T(1)
    if (kTma && tid == kStoreTid) bulk_wait_read<0>();  // the previous tile's bulk stores have read the staging
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    K4T(2)

    // ---- pass 2 into the same columns (pass 1 has been read) ----
    if (warp == 0) {
      tc_fence_after();
#if RNSW_K4_FINE
      // each warp group's first channel block (both residues) first, then the second blocks
      asm volatile(K4_ASM_HEAD K4_P2(0) K4_P2(4) K4_COMMIT_AT("%5", 0) K4_P2(2) K4_P2(6) K4_COMMIT_AT("%5", 1) K4_P2(1)
                       K4_P2(5) K4_COMMIT_AT("%5", 2) K4_P2(3) K4_P2(7) K4_COMMIT_AT("%5", 3) "}" ::"r"(tbase),
                   "r"(dbase), "r"(kIdP1), "r"(kIdP2s), "r"(bar1_addr), "r"(bar2_addr)
                   : "memory");
#else
      // channel blocks mb 0, 1 of both residues (warps 0-3) first, then mb 2, 3
      asm volatile(K4_ASM_HEAD K4_P2(0) K4_P2(1) K4_P2(4) K4_P2(5) K4_COMMIT("%4") K4_P2(2) K4_P2(3) K4_P2(6) K4_P2(7)
                       K4_COMMIT("%5") "}" ::"r"(tbase),
                   "r"(dbase), "r"(kIdP1), "r"(kIdP2s), "r"(bar1_addr), "r"(bar2_addr)
                   : "memory");
#endif
    }
    K4T(3)
#if RNSW_K4_FINE
    // channel block mbi of this warp group (both residues) has completed
    auto wait_p2 = [&](int mbi) {
      K4_WAIT(&bar_p2[2 * mbi + h], ph2);
      tc_fence_after();
    };
    wait_p2(0);
    if (!RNSW_K4_EPI2_PIPE) wait_p2(1);
#else
    auto wait_p2 = [&](int) {};
    K4_WAIT(my_bar, ph_mma);
    ph_mma ^= 1;
    tc_fence_after();
#endif
    K4T(4)

    // ---- epilogue 2: lane row (k, a) = (2q + lane/16, lane % 16) of channel blocks mb = 2h, 2h+1 ----
    const int b_img = (int)fdiv((uint32_t)p, args.div_img);
    const int rem = p - b_img * (int)args.div_img.d;
    const int ti = (int)fdiv((uint32_t)rem, args.div_tw);
    const int tj = rem - ti * g.tw;
    {
      const int a = lane & 15, kk8 = 2 * q + (lane >> 4);
      // one channel block mbi of this warp group (mode 1 unrolls both blocks:
      // 2-3% faster; the pooled and int32 modes would spill at 128 registers)
      auto epi2_block = [&](const int mbi) {
      const int mb = 2 * h + mbi, kl = mb * 8 + kk8;
      int32_t h0[16], l0[16], h1[16], l1[16];
      const uint32_t ta = tbase + ((uint32_t)(32 * q) << 16) + mb * 32;
      tmem_ld16(ta, h0);
      tmem_ld16(ta + 16, l0);
      tmem_ld16(ta + 128, h1);
      tmem_ld16(ta + 144, l1);
      tmem_ld_wait();
      int32_t qv[14];
#pragma unroll
      for (int b = 0; b < 14; ++b) {
        // mixed-radix digits (rw/residue.py:195-206): d0 = y0 mod m0,
        // d1 = (y1 - d0) m0^-1 mod m1 (the factor rides in B2 of residue 1);
        // the MMA added the bias, both sums are already non-negative.
        // d0 may be any representative in [-m0, m0): its quotient
        // umulhi(n, ceil(2^32 / m0)) is floor(n / m0) or one more (no shift).
        // Then x = d0 + m0 d1 in [-m0, D) is still the right value mod D,
        // and x < 0 is a (small) negative output, folded by the signed test.
        const int32_t n0 = h0[b] * 256 + l0[b];
        const int32_t d0 = (int32_t)(__umulhi((uint32_t)n0, mul0) * fm0.negm + (uint32_t)n0);
        const int32_t d1 = red_pos_biased(d0 * negw10 + (h1[b] * 256 + l1[b]), fm1);
        const uint32_t x = (uint32_t)d0 + m0 * (uint32_t)d1;
        const bool neg = x > signed_bound;  // unsigned: also every x < 0
        if constexpr (kMode == 0)
          qv[b] = (int32_t)((int32_t)x > (int32_t)signed_bound ? x - dyn_range : x);
        else if constexpr (kMode == 1)
          qv[b] = neg ? 0 : min((int32_t)(x >> args.shift), 127);
        else
          qv[b] = neg ? 0 : (int32_t)x;  // shift and clip after the max (monotone)
      }
      if constexpr (kMode == 3) {
#pragma unroll
        for (int c = 0; c < 7; ++c) {
          int32_t m2 = max(qv[2 * c], qv[2 * c + 1]);
          m2 = max(m2, __shfl_xor_sync(0xffffffffu, m2, 1));  // rows a, a ^ 1
          m2 = min(m2 >> args.shift, 127);
          if ((a & 1) == 0 && a < 14) st_base[mbi * 8 + c * kPix] = (uint8_t)m2;
        }
      } else if constexpr (kMode == 1) {
        if (a < 14) {
#pragma unroll
          for (int b = 0; b < 14; ++b) *st_col(mbi, b) = (uint8_t)qv[b];
        }
      } else {
        int32_t* ys = reinterpret_cast<int32_t*>(smem + out_off(0));
        if (a < 14) {
#pragma unroll
          for (int b = 0; b < 14; ++b) ys[(a * 14 + b) * kPixW + kl] = qv[b];
        }
      }
      };
#if RNSW_K4_EPI2_PIPE
      // software-pipelined by half blocks: columns 8 hf .. 8 hf + 7 of one
      // channel block are reduced while the next half's TMEM loads fly (two
      // 32-register sets, the same peak as one 16-column block)
      auto emit = [&](int mbi, int hf, const int32_t (&H0)[8], const int32_t (&L0)[8], const int32_t (&H1)[8],
                      const int32_t (&L1)[8]) {
        const int mb = 2 * h + mbi, kl = mb * 8 + kk8;
        constexpr int kNb = 8;
        int32_t qv[kNb];
#pragma unroll
        for (int e = 0; e < kNb; ++e) {
          const int32_t n0 = H0[e] * 256 + L0[e];
          const int32_t d0 = (int32_t)(__umulhi((uint32_t)n0, mul0) * fm0.negm + (uint32_t)n0);
          const int32_t d1 = red_pos_biased(d0 * negw10 + (H1[e] * 256 + L1[e]), fm1);
          const uint32_t x = (uint32_t)d0 + m0 * (uint32_t)d1;
          const bool neg = x > signed_bound;
          if constexpr (kMode == 0)
            qv[e] = (int32_t)((int32_t)x > (int32_t)signed_bound ? x - dyn_range : x);
          else if constexpr (kMode == 1)
            qv[e] = neg ? 0 : min((int32_t)(x >> args.shift), 127);
          else
            qv[e] = neg ? 0 : (int32_t)x;
        }
        const int nb = hf == 0 ? 8 : 6;  // columns b = 8 hf + e < 14
        if constexpr (kMode == 3) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (2 * c >= nb) break;
            int32_t m2 = max(qv[2 * c], qv[2 * c + 1]);
            m2 = max(m2, __shfl_xor_sync(0xffffffffu, m2, 1));  // rows a, a ^ 1
            m2 = min(m2 >> args.shift, 127);
            if ((a & 1) == 0 && a < 14) st_base[mbi * 8 + (4 * hf + c) * kPix] = (uint8_t)m2;
          }
        } else if constexpr (kMode == 1) {
          if (a < 14) {
#pragma unroll
            for (int e = 0; e < kNb; ++e)
              if (e < nb) *st_col(mbi, 8 * hf + e) = (uint8_t)qv[e];
          }
        } else {
          int32_t* ys = reinterpret_cast<int32_t*>(smem + out_off(0));
          if (a < 14) {
#pragma unroll
            for (int e = 0; e < kNb; ++e)
              if (e < nb) ys[(a * 14 + 8 * hf + e) * kPixW + kl] = qv[e];
          }
        }
      };
      auto load = [&](int mbi, int hf, int32_t (&H0)[8], int32_t (&L0)[8], int32_t (&H1)[8], int32_t (&L1)[8]) {
        const uint32_t ta = tbase + ((uint32_t)(32 * q) << 16) + (2 * h + mbi) * 32 + 8 * hf;
        tmem_ld8(ta, H0);
        tmem_ld8(ta + 16, L0);
        tmem_ld8(ta + 128, H1);
        tmem_ld8(ta + 144, L1);
      };
      int32_t aH0[8], aL0[8], aH1[8], aL1[8], bH0[8], bL0[8], bH1[8], bL1[8];
      load(0, 0, aH0, aL0, aH1, aL1);
      tmem_ld_wait();
      load(0, 1, bH0, bL0, bH1, bL1);
      emit(0, 0, aH0, aL0, aH1, aL1);
      tmem_ld_wait();
      wait_p2(1);
      load(1, 0, aH0, aL0, aH1, aL1);
      emit(0, 1, bH0, bL0, bH1, bL1);
      tmem_ld_wait();
      load(1, 1, bH0, bL0, bH1, bL1);
      emit(1, 0, aH0, aL0, aH1, aL1);
      tmem_ld_wait();
      if (RNSW_K4_EARLY_P1 && (kMode == 3 || (RNSW_K4_EARLY_P1_ALL && kMode != 0))) {
        // (pooled mode only: -1 to -2% there, +2% on the unpooled layers)
        // this warp's TMEM reads are done: once all are, warp 0 issues the
        // next unit's pass 1 over the same columns (it then overlaps the
        // rest of epilogue 2 and the stores, not only the stores)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_tfree);
        if (warp == 0 && u + u_step < args.units) {
          mbar_wait(bar_tfree, ph_tfree);
          tc_fence_after();
          issue_p1();
        }
        ph_tfree ^= 1;
      }
      emit(1, 1, bH0, bL0, bH1, bL1);
      (void)epi2_block;
#else
      if constexpr (kMode == 1) {
        epi2_block(0);
        epi2_block(1);
      } else {
#pragma unroll 1
        for (int mbi = 0; mbi < 2; ++mbi) epi2_block(mbi);
      }
#endif
    }
    ph2 ^= 1;
    K4T(5)
    if (kTma) fence_proxy_async();  // staging writes -> visible to the bulk stores
    tc_fence_before();
    __syncthreads();  // staging complete; pass-2 accumulators read
    K4T(6)
    if (kMode != 0 && !(RNSW_K4_EARLY_P1 && RNSW_K4_EPI2_PIPE && (kMode == 3 || (RNSW_K4_EARLY_P1_ALL && kMode != 0))) && warp == 0 &&
        u + u_step < args.units) {
      tc_fence_after();
      issue_p1();  // the next unit's pass 1 overlaps these stores
    }

    // ---- stores ----
    if constexpr (kTma) {
      // one bulk tensor store of the staged tile (clipped at the image edges
      // and at K); the staging is rewritten only after the next epilogue 1,
      // by when the storing thread has waited for the read
      constexpr int side = kMode == 3 ? 7 : 14;
      if (tid == kStoreTid) {
        tma_store_4d(&tmo, smem + kOffOut, k0, tj * side, ti * side, b_img);
        bulk_commit();
      }
    } else if constexpr (kMode == 0) {
      const int32_t* ys = reinterpret_cast<const int32_t*>(smem + out_off(0));
      if (g.layout == 0) {
        for (int idx = tid; idx < 196 * kKB; idx += kThr) {
          const int px = idx >> 5, c = idx & 31, a = px / 14, b = px - a * 14;
          const int ho = ti * 14 + a, wo = tj * 14 + b;
          if (ho < g.Ho && wo < g.Wo && k0 + c < g.K)
            args.y[(((int64_t)b_img * g.Ho + ho) * g.Wo + wo) * g.K + k0 + c] = ys[px * kPixW + c];
        }
      } else {
        for (int idx = tid; idx < 196 * kKB; idx += kThr) {
          const int c = idx / 196, px = idx - c * 196, a = px / 14, b = px - a * 14;
          const int ho = ti * 14 + a, wo = tj * 14 + b;
          if (ho < g.Ho && wo < g.Wo && k0 + c < g.K)
            args.y[(((int64_t)b_img * g.K + k0 + c) * g.Ho + ho) * g.Wo + wo] = ys[px * kPixW + c];
        }
      }
    } else if (args.vec16) {
      // 16-byte words (K % 16 == 0 and a 16-byte aligned output buffer)
      constexpr int side = kMode == 3 ? 7 : 14;
      const int Ho = kMode == 3 ? g.Ho / 2 : g.Ho, Wo = kMode == 3 ? g.Wo / 2 : g.Wo;
      for (int idx = tid; idx < side * side * (kKB / 16); idx += kThr) {
        const int wq = idx & 1, px = idx >> 1, a = px / side, b = px - a * side;
        const int ho = ti * side + a, wo = tj * side + b;
        if (ho >= Ho || wo >= Wo || k0 + 16 * wq >= g.K) continue;
        const uint4 word = *reinterpret_cast<const uint4*>(smem + kOffOut + px * kPixB + 16 * wq);
        *reinterpret_cast<uint4*>(args.out8 + (((int64_t)b_img * Ho + ho) * Wo + wo) * g.K + k0 + 16 * wq) = word;
      }
    } else {
      constexpr int side = kMode == 3 ? 7 : 14;
      const int Ho = kMode == 3 ? g.Ho / 2 : g.Ho, Wo = kMode == 3 ? g.Wo / 2 : g.Wo;
      for (int idx = tid; idx < side * side * (kKB / 4); idx += kThr) {
        const int wq = idx & 7, px = idx >> 3, a = px / side, b = px - a * side;
        const int ho = ti * side + a, wo = tj * side + b;
        if (ho >= Ho || wo >= Wo || k0 + 4 * wq >= g.K) continue;
        const uint32_t word = *reinterpret_cast<const uint32_t*>(smem + kOffOut + px * kPixB + 4 * wq);
        *reinterpret_cast<uint32_t*>(args.out8 + (((int64_t)b_img * Ho + ho) * Wo + wo) * g.K + k0 + 4 * wq) = word;
      }
    }
    if constexpr (kMode == 0) {
      // the staged tile (in A1) has been read by every thread: the async proxy may overwrite it
      fence_proxy_async();
      __syncthreads();
      if (warp == 0 && u + u_step < args.units) {
        if (lane == 0) issue_load(u + u_step);
        __syncwarp();
        tc_fence_after();
        issue_p1();  // waits for the boxes; the other CTA of the SM computes meanwhile
      }
    }
    K4T(7)
  }

  if (kTma && tid == kStoreTid) bulk_wait<0>();
#ifdef RNSW_K4_PROF
  if (lane == 0 && blockIdx.x < 2 && (warp == 0 || warp == 1 || warp == 4) && pn > 0)
    printf("K4PROF cta %d warp %d units %d per-unit cycles: total %lld | wait_p1 %lld epi1 %lld bar1 %lld p2issue %lld wait_p2 %lld epi2 %lld bar2 %lld stores+p1issue %lld\n",
           blockIdx.x, warp, pn, (clock64() - pt0) / pn, pc[0] / pn, pc[1] / pn, pc[2] / pn, pc[3] / pn, pc[4] / pn,
           pc[5] / pn, pc[6] / pn, pc[7] / pn);
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tbase);
  }
}

// Mw8 as a 5-D tensor (k, i, L = (pb * n_res + res) * 2 + limb, j, t); one
// box = 32 channels x 16 rows i x 2 limbs x 4 columns j x 1 tile lands in
// shared memory as [j][limb][i][32 channels]: per column j a 32 B-swizzled
// MN atom of K = 32 rows (limb, i), the 4 atoms 1 KB apart -- an MN-major
// M = 128 (j, k), K = 32 operand.  (With the 128B swizzle TMA would pad
// each 32-byte box row to 128 bytes.)
bool make_tmap_mw8(CUtensorMap* tm, const void* base, int Kp, int64_t num_pb, int nres) {
  auto encode = encode_fn();
  if (encode == nullptr) return false;
  cuuint64_t dims[5] = {(cuuint64_t)Kp, 16, (cuuint64_t)(num_pb * nres * 2), 16, 128};
  cuuint64_t strides[4] = {(cuuint64_t)Kp * 128 * 16, (cuuint64_t)Kp * 128 * 256, (cuuint64_t)Kp * 128,
                           (cuuint64_t)Kp};
  cuuint32_t box[5] = {32, 16, 2, 16, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, const_cast<void*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

bool umma_output_ok(const PlanDevice& d) {
  static const bool off = getenv("RNSW_K4_MMA_SYNC") != nullptr;  // A/B switch: the mma.sync kernel
  return !off && !force_generic() && d.fast && d.n == 16 && d.m_out == 14 && d.n_res == 2 &&
         d.res[0].planes == 2 && d.res[1].planes == 2 && d.z3;
}

cudaError_t launch_output_transform_umma(const PlanHost& plan, const Geometry& g, const uint8_t* Mw8, int32_t* y,
                                         cudaStream_t s, int8_t* out8, int shift, int pool) {
  if (g.P >= (1ll << 31)) return cudaErrorInvalidValue;
  const int64_t num_pb = (g.P + 127) / 128;
  CUtensorMap tm;
  if (!make_tmap_mw8(&tm, Mw8, g.Kp, num_pb, 2)) return cudaErrorInvalidValue;
  UArgs a{};
  a.g = g;
  a.out8 = out8;
  a.y = y;
  a.shift = shift;
  a.vec16 = out8 != nullptr && (g.K & 15) == 0 && (reinterpret_cast<uintptr_t>(out8) & 15) == 0;
  // int8 NHWC output: one TMA bulk tensor store per tile (RNSW_K4_STG_STORES=1: the per-thread stores)
  static const bool stg_stores = getenv("RNSW_K4_STG_STORES") != nullptr;
  CUtensorMap tmo;
  memset(&tmo, 0, sizeof(tmo));
  a.tma_out = 0;
  if (a.vec16 && !stg_stores) {
    const bool pooled = pool != 0;
    const int oh = pooled ? g.Ho / 2 : g.Ho, ow = pooled ? g.Wo / 2 : g.Wo, side = pooled ? 7 : 14;
    auto encode = encode_fn();
    if (encode != nullptr) {
      cuuint64_t dims[4] = {(cuuint64_t)g.K, (cuuint64_t)ow, (cuuint64_t)oh, (cuuint64_t)g.B};
      cuuint64_t strides[3] = {(cuuint64_t)g.K, (cuuint64_t)ow * g.K, (cuuint64_t)oh * ow * g.K};
      cuuint32_t box[4] = {(cuuint32_t)kKB, (cuuint32_t)side, (cuuint32_t)side, 1};
      cuuint32_t es[4] = {1, 1, 1, 1};
      a.tma_out = encode(&tmo, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, out8, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, pooled ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_32B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS ? 1 : 0;
    }
  }
  a.kblocks = (g.K + kKB - 1) / kKB;
  a.units = g.P * a.kblocks;
  if (a.units >= (1ll << 31)) return cudaErrorInvalidValue;  // FastDiv range
  a.negw10 = -plan.dev.mrc_w[1][0];
  a.mul0 = (uint32_t)(((1ull << 32) + plan.dev.res[0].modulus - 1) / plan.dev.res[0].modulus);
  a.div_img = make_fastdiv((uint32_t)(g.th * g.tw));
  a.div_tw = make_fastdiv((uint32_t)g.tw);
  a.div_kb = make_fastdiv((uint32_t)a.kblocks);
  const int num_sms = num_sms_current();
  const int mode = out8 == nullptr ? 0 : (pool ? 3 : 1);
  auto launch = [&](auto kern, int smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    // persistent grid: as many CTAs as are co-resident -- 2 per SM in every
    // mode (launch bounds; the shared-memory footprint is checked below)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    const int per_sm = (228 * 1024) / (smem + 1024) >= 2 ? 2 : 1;
    const unsigned grid = (unsigned)std::min<int64_t>(a.units, (int64_t)per_sm * num_sms);
    return launch_ex(kern, dim3(grid), dim3(kThr), (size_t)smem, s, 1, (const PlanDevice*)plan.d_plan, tm, tmo, a);
  };
  if (mode == 0) return launch(output_umma_kernel<0, false>, smem_bytes(0));
  if (mode == 1)
    return a.tma_out ? launch(output_umma_kernel<1, true>, smem_bytes(1)) : launch(output_umma_kernel<1, false>, smem_bytes(1));
  return a.tma_out ? launch(output_umma_kernel<3, true>, smem_bytes(3)) : launch(output_umma_kernel<3, false>, smem_bytes(3));
}

}  // namespace rnsw
