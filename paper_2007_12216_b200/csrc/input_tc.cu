// K1 on the tensor cores: V = BT d B mod m for every tile, channel and
// residue (rw/layer.py:278-283, rw/kernel.py:44-47, 21-30), written straight
// into the GEMM operand layout V[plane][pos][P][Cp].
//
// CTA = one tile p x 64 channels; each warp owns 16 channels.  A lane loads
// 16 channels of 4 patch pixels (two 16-byte rows per n-tile), and 4x4 byte
// transposes (PRMT) turn them into mma.sync B fragments, so the patch never
// touches shared memory:
//   pass 1  T^T = BT * D^T    (A = BT constants, B = patch bytes)
//   pass 2  V^T = T^T * BT^T  (A = pass-1 C registers with the contraction
//                              index permuted onto the k-slots, B = BT^T)
// 16-bit moduli: pass 1 keeps T exact (|T| < 2^23) as three byte limbs
// T = 65536 T2 + 256 T1 + T0 instead of reducing it, and pass 2 multiplies
// them by BT, BT' = 256 BT and BT'' = 65536 BT (mod m), each in two limbs,
// into two accumulators (256 * acc256 + acc1).  The output limbs come from
// w = v + 128: hi = w >> 8 and lo = (w & 255) ^ 0x80.
// Each lane ends up holding 8 transform positions x 16 channels, i.e. one
// 16-byte row segment of V per position and plane, stored with one vector
// store.  16-bit moduli: BT is split into two s8 limbs (see below); every
// exact int32 sum stays below 2^28 (m < 4500), so one division-free
// reduction per output value suffices.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"

namespace rnsw {
namespace {

constexpr int kCTAChannels = 64;


// 4x4 byte transpose: in[e] = 4 channels of pixel e -> out[q] = channel q of pixels 0..3.
RNSW_DEV void transpose4x4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&o)[4]) {
  const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w2, w3, 0x5140);
  const uint32_t t2 = __byte_perm(w0, w1, 0x7362), t3 = __byte_perm(w2, w3, 0x7362);
  o[0] = __byte_perm(t0, t1, 0x5410);
  o[1] = __byte_perm(t0, t1, 0x7632);
  o[2] = __byte_perm(t2, t3, 0x5410);
  o[3] = __byte_perm(t2, t3, 0x7632);
}

RNSW_DEV uint32_t word_of(const uint4& v, int u) { return u == 0 ? v.x : u == 1 ? v.y : u == 2 ? v.z : v.w; }

// kCompact (C <= 4, the small-channel path of smallc.cu): each warp owns one
// tile and writes its 4 channels as symmetric int16 residues to
// V16[res][P][pos][4] instead of the GEMM limb planes.
// Non-compact output: the CTA's V rows of one residue are staged in shared
// memory as OWT[plane][pos][64 channels] (64-byte rows, 16-byte chunks XOR
// (pos >> 1) & 3 = TMA SWIZZLE_64B) and written by one TMA bulk tensor store
// per plane (one 64-byte segment per position) instead of 16-byte stores
// from four warps.  The finished 4-channel words leave registers after each
// u, keeping the kernel at 4 CTAs per SM.
// kFull: NHWC with C % 64 == 0 -- 16-byte patch loads, every channel real
// (no channel-loop exits, no masked limb flips), as a separate instance.
template <int kPL, bool kCompact, bool kFull = false>
__global__ void __launch_bounds__(128, 4) input_transform_tc_kernel(const PlanDevice* __restrict__ plan, Geometry g,
                                                                 const int8_t* __restrict__ x,
                                                                 int8_t* __restrict__ V,
                                                                 const __grid_constant__ CUtensorMap tmVout) {
  __shared__ int32_t BT16[RNSW_MAX_RES * 256];
  __shared__ __align__(1024) uint32_t OWT[2][256][16];
  pdl_trigger();
  pdl_wait();  // the previous kernel's activations / its use of V
  const int N = plan->n, M = plan->m_out, npos = N * N, nres = plan->n_res;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
  const int ncb = (g.Cp + kCTAChannels - 1) / kCTAChannels;
  // channel blocks of one tile are adjacent in launch order
  const int64_t p = kCompact ? (int64_t)blockIdx.x * 4 + warp : blockIdx.x / ncb;
  const int c_base = kCompact ? 0 : (int)(blockIdx.x % ncb) * kCTAChannels + warp * 16;
  for (int idx = tid; idx < nres * 256; idx += blockDim.x) {
    const int r = idx >> 8, a = (idx >> 4) & 15, b = idx & 15;
    BT16[idx] = (a < N && b < N) ? plan->res[r].bt[a * RNSW_MAX_N + b] : 0;
  }
  __syncthreads();
  if (kCompact && p >= g.P) return;
  // non-compact: every warp stays for the CTA barriers of the bulk stores;
  // warps past C compute nothing (their channel loop breaks at once) and
  // stage zero rows; chunks past Cp are clipped by the store
  const int b_img = (int)(p / (g.th * g.tw));
  const int ti = (int)((p / g.tw) % g.th);
  const int tj = (int)(p % g.tw);

  // ---- patch: raw[ni][e] = channels c_base..+15 of pixel (a = g + 8 ni, b = 4t + e)
  uint4 raw[2][4];
  const bool vec = kFull || (g.layout == 0 && (g.C & 15) == 0);
#pragma unroll
  for (int ni = 0; ni < 2; ++ni)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int a = gq + 8 * ni, bcol = 4 * tq + e;
      const int h = ti * M + a - g.pad, w = tj * M + bcol - g.pad;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (a < N && bcol < N && h >= 0 && h < g.H && w >= 0 && w < g.W && c_base < g.C) {
        if (vec) {
          v = __ldg(reinterpret_cast<const uint4*>(x + (((int64_t)b_img * g.H + h) * g.W + w) * g.C + c_base));
        } else {
          uint32_t wd[4] = {0, 0, 0, 0};
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int c = c_base + q;
            if (c < g.C) {
              const int64_t xi = g.layout == 0 ? (((int64_t)b_img * g.H + h) * g.W + w) * g.C + c
                                               : (((int64_t)b_img * g.C + c) * g.H + h) * g.W + w;
              wd[q >> 2] |= (uint32_t)(uint8_t)x[xi] << (8 * (q & 3));
            }
          }
          v = make_uint4(wd[0], wd[1], wd[2], wd[3]);
        }
      }
      raw[ni][e] = v;
    }

  for (int r = 0; r < nres; ++r) {
    const ResidueTables& tb = plan->res[r];
    const FastMod fm = fast_mod_of(tb);
    const int32_t pbias = pos_bias(fm);  // -> representative in [0, m)
    const int32_t sbias = fm.off;        // -> [0, m) shifted by h: subtract h for the symmetric residue
    constexpr int planes = kPL;
    const int32_t* bt = BT16 + r * 256;
    // pass-1 A: BT rows j = g / g+8, columns b = 4t..4t+3
    int32_t av[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      av[e] = bt[gq * 16 + 4 * tq + e];
      av[4 + e] = bt[(gq + 8) * 16 + 4 * tq + e];
    }
    const uint32_t alo0 = pack4_lo(av[0], av[1], av[2], av[3]);
    const uint32_t alo1 = pack4_lo(av[4], av[5], av[6], av[7]);
    const uint32_t ahi0 = pack4_lo(limb_hi(av[0]), limb_hi(av[1]), limb_hi(av[2]), limb_hi(av[3]));
    const uint32_t ahi1 = pack4_lo(limb_hi(av[4]), limb_hi(av[5]), limb_hi(av[6]), limb_hi(av[7]));
    // pass-2 B: column i = g + 8 ni, k-slot e <-> a = {2t, 2t+1, 8+2t, 9+2t}[e]
    // BT, BT' = 256 BT and BT'' = 65536 BT (mod m) (16-bit: 2 accumulators)
    uint32_t blo[2], bhi[2], bplo[2], bphi[2], bpplo[2], bpphi[2];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const int i = gq + 8 * ni;
      const int32_t v0 = bt[i * 16 + 2 * tq], v1 = bt[i * 16 + 2 * tq + 1];
      const int32_t v2 = bt[i * 16 + 8 + 2 * tq], v3 = bt[i * 16 + 9 + 2 * tq];
      blo[ni] = pack4_lo(v0, v1, v2, v3);
      bhi[ni] = pack4_lo(limb_hi(v0), limb_hi(v1), limb_hi(v2), limb_hi(v3));
      if (planes == 2) {
        const int32_t w0 = red_fast(v0 * 256, fm), w1 = red_fast(v1 * 256, fm);
        const int32_t w2 = red_fast(v2 * 256, fm), w3 = red_fast(v3 * 256, fm);
        bplo[ni] = pack4_lo(w0, w1, w2, w3);
        bphi[ni] = pack4_lo(limb_hi(w0), limb_hi(w1), limb_hi(w2), limb_hi(w3));
        const int32_t x0 = red_fast(w0 * 256, fm), x1 = red_fast(w1 * 256, fm);
        const int32_t x2 = red_fast(w2 * 256, fm), x3 = red_fast(w3 * 256, fm);
        bpplo[ni] = pack4_lo(x0, x1, x2, x3);
        bpphi[ni] = pack4_lo(limb_hi(x0), limb_hi(x1), limb_hi(x2), limb_hi(x3));
      }
    }

    uint32_t outw[2][8];     // [plane][position slot] word of 4 channels (this u)
    uint32_t outc[8][2];     // kCompact: [position slot][channel pair] int16 x 2
#pragma unroll
    for (int s = 0; s < 8; ++s) outc[s][0] = outc[s][1] = 0u;
#pragma unroll
    for (int u = 0; u < (kCompact ? 1 : 4); ++u) {
      uint32_t din[2][4];
      transpose4x4(word_of(raw[0][0], u), word_of(raw[0][1], u), word_of(raw[0][2], u), word_of(raw[0][3], u),
                   din[0]);
      transpose4x4(word_of(raw[1][0], u), word_of(raw[1][1], u), word_of(raw[1][2], u), word_of(raw[1][3], u),
                   din[1]);
#pragma unroll
      for (int s = 0; s < 8; ++s) outw[0][s] = outw[1][s] = 0u;
      // channels of this word: a rolled loop (unrolled by 2 in the full-channel
      // instance, measured best) keeps the kernel inside the instruction
      // cache -- the fully unrolled body missed in L0/L1.5
      constexpr int kQUnroll = kFull ? 2 : 1;
#pragma unroll kQUnroll
      for (int q = 0; q < 4; ++q) {
        if (!kFull && c_base + 4 * u + q >= g.C) break;  // padding channels stay 0
        const uint32_t dq0 = q == 0 ? din[0][0] : q == 1 ? din[0][1] : q == 2 ? din[0][2] : din[0][3];
        const uint32_t dq1 = q == 0 ? din[1][0] : q == 1 ? din[1][1] : q == 2 ? din[1][2] : din[1][3];
        const uint32_t bsel = (0x3210u & ~(0xFu << (4 * q))) | (0x4u << (4 * q));  // insert byte 0 at byte q
        const uint32_t bsel1 = (0x3210u & ~(0xFu << (4 * q))) | (0x5u << (4 * q)); // insert byte 1 at byte q
        int32_t v[2][4];
        if (planes == 2) {
          // pass 1: T exact, as byte limbs (see the header)
          int32_t t[2][4];
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) {
            int32_t hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
            imma_ss(hi, ahi0, ahi1, ni ? dq1 : dq0);
            imma_ss(lo, alo0, alo1, ni ? dq1 : dq0);
#pragma unroll
            for (int e = 0; e < 4; ++e) t[ni][e] = hi[e] * 256 + lo[e];
          }
          // pass 2: A rows j = g / g+8, k-slots = {2t, 2t+1, 8+2t, 9+2t}
          // bytes 0 and 1 share their first byte-pairing step
          const uint32_t pa = __byte_perm(t[0][0], t[0][1], 0x5140), qa = __byte_perm(t[1][0], t[1][1], 0x5140);
          const uint32_t pb = __byte_perm(t[0][2], t[0][3], 0x5140), qb = __byte_perm(t[1][2], t[1][3], 0x5140);
          const uint32_t t0a = __byte_perm(pa, qa, 0x5410), t1a = __byte_perm(pa, qa, 0x7632);
          const uint32_t t0b = __byte_perm(pb, qb, 0x5410), t1b = __byte_perm(pb, qb, 0x7632);
          const uint32_t t2a = pack4_byte<2>(t[0][0], t[0][1], t[1][0], t[1][1]);
          const uint32_t t2b = pack4_byte<2>(t[0][2], t[0][3], t[1][2], t[1][3]);
          // kCompact wants v itself, the limb planes w = v + 128
          const int32_t vshift = kCompact ? -fm.h : 128 - fm.h;
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) {
            int32_t a256[4] = {0, 0, 0, 0}, a1[4] = {sbias, sbias, sbias, sbias};
            imma_ss(a256, t2a, t2b, bpphi[ni]);
            imma_us(a256, t1a, t1b, bphi[ni]);
            imma_us(a256, t0a, t0b, bhi[ni]);
            imma_ss(a1, t2a, t2b, bpplo[ni]);
            imma_us(a1, t1a, t1b, bplo[ni]);
            imma_us(a1, t0a, t0b, blo[ni]);
            // |256 a256 + a1| < 2^25
#pragma unroll
            for (int e = 0; e < 4; ++e) v[ni][e] = red_pos_biased(a256[e] * 256 + a1[e], fm) + vshift;
          }
        } else {
          // pass 1 -> T in [0, m): the reduction bias rides in the accumulator
          int32_t t[2][4];
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) {
            int32_t acc[4] = {pbias, pbias, pbias, pbias};
            imma_ss(acc, alo0, alo1, ni ? dq1 : dq0);
#pragma unroll
            for (int e = 0; e < 4; ++e) t[ni][e] = red_pos_biased(acc[e], fm);
          }
          // pass 2: T in [0, m < 256) is one u8 limb
          const uint32_t tlo0 = pack4_lo(t[0][0], t[0][1], t[1][0], t[1][1]);
          const uint32_t tlo1 = pack4_lo(t[0][2], t[0][3], t[1][2], t[1][3]);
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) {
            int32_t acc[4] = {sbias, sbias, sbias, sbias};
            imma_us(acc, tlo0, tlo1, blo[ni]);
#pragma unroll
            for (int e = 0; e < 4; ++e) v[ni][e] = red_pos_biased(acc[e], fm) - fm.h;
          }
        }
        if constexpr (kCompact) {
          const uint32_t hsel = (q & 1) ? 0x5410u : 0x3254u;  // int16 into the high / low half
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            const uint32_t val = (uint32_t)v[s >> 2][s & 3];
            if (q < 2) outc[s][0] = __byte_perm(outc[s][0], val, hsel);
            else outc[s][1] = __byte_perm(outc[s][1], val, hsel);
          }
        } else {
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            const int32_t val = v[s >> 2][s & 3];  // 16-bit: w = v + 128
            outw[0][s] = __byte_perm(outw[0][s], (uint32_t)val, bsel);
            if (planes == 2) outw[1][s] = __byte_perm(outw[1][s], (uint32_t)val, bsel1);  // byte 1 = w >> 8
          }
        }
      }
      if constexpr (!kCompact) {
        if (planes == 2) {
          // low limb = (w & 255) ^ 0x80, on the real channels only
          const int nv = kFull ? 4 : min(max(g.C - (c_base + 4 * u), 0), 4);
          const uint32_t flip = nv >= 4 ? 0x80808080u : (0x80808080u & ((1u << (8 * nv)) - 1u));
#pragma unroll
          for (int s = 0; s < 8; ++s) outw[0][s] ^= flip;
        }
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const int e = s & 3, ni = s >> 2;
          const int j = gq + 8 * (e >> 1), i = 8 * ni + 2 * tq + (e & 1);
          const int pos = i * N + j;
          if (i >= N || j >= N) continue;
          const int w = (((warp ^ (pos >> 1)) & 3) << 2) + u;  // 64B swizzle of chunk `warp`
          OWT[0][pos][w] = outw[0][s];
          if (planes == 2) OWT[1][pos][w] = outw[1][s];
        }
      }
    }
    if constexpr (kCompact) {
      // slot s = 4 ni + e: row j = g + 8 (e >> 1), column i = 8 ni + 2t + (e & 1)
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int e = s & 3, ni = s >> 2;
        const int j = gq + 8 * (e >> 1), i = 8 * ni + 2 * tq + (e & 1);
        if (i >= N || j >= N) continue;
        *reinterpret_cast<uint2*>(V + ((((int64_t)r * g.P + p) * npos + i * N + j) << 3)) =
            make_uint2(outc[s][0], outc[s][1]);
      }
    } else {
      fence_proxy_async();  // staging writes -> visible to the bulk-copy engine
      __syncthreads();
      if (tid == 0) {
        for (int pl = 0; pl < planes; ++pl)
          tma_store_3d(&tmVout, &OWT[pl][0][0], (int)(blockIdx.x % ncb) * kCTAChannels, (int)p,
                       (tb.plane_base + pl) * npos);
        bulk_commit();
        bulk_wait_read<0>();  // OWT is rewritten by the next residue
      }
      __syncthreads();
    }
  }
}

}  // namespace

cudaError_t launch_input_transform_tc(const PlanHost& plan, const Geometry& g, const int8_t* x, int8_t* V,
                                      cudaStream_t s) {
  dim3 grid((unsigned)(g.P * ((g.Cp + kCTAChannels - 1) / kCTAChannels)));
  // V as [n_planes * npos][P][Cp] bytes; box = 64 channels x 1 tile x npos positions
  const int npos = plan.dev.n * plan.dev.n;
  auto encode = encode_fn();
  if (encode == nullptr) return cudaErrorInvalidValue;
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)g.Cp, (cuuint64_t)g.P, (cuuint64_t)plan.dev.n_planes * npos};
  cuuint64_t strides[2] = {(cuuint64_t)g.Cp, (cuuint64_t)g.P * g.Cp};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)npos};
  cuuint32_t estr[3] = {1, 1, 1};
  if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, V, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const bool full = g.layout == 0 && (g.C & 63) == 0;
  cudaError_t e;
  if (plan.dev.res[0].planes == 2) {
    if (full)
      e = launch_ex(input_transform_tc_kernel<2, false, true>, dim3(grid), dim3(128), 0, s, 1, (const PlanDevice*)plan.d_plan, g, x, V, tm);
    else
      e = launch_ex(input_transform_tc_kernel<2, false, false>, dim3(grid), dim3(128), 0, s, 1, (const PlanDevice*)plan.d_plan, g, x, V, tm);
  } else {
    if (full)
      e = launch_ex(input_transform_tc_kernel<1, false, true>, dim3(grid), dim3(128), 0, s, 1, (const PlanDevice*)plan.d_plan, g, x, V, tm);
    else
      e = launch_ex(input_transform_tc_kernel<1, false, false>, dim3(grid), dim3(128), 0, s, 1, (const PlanDevice*)plan.d_plan, g, x, V, tm);
  }
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_input_transform_compact(const PlanHost& plan, const Geometry& g, const int8_t* x, int16_t* V16,
                                           cudaStream_t s) {
  if (g.C > 4) return cudaErrorInvalidValue;
  dim3 grid((unsigned)((g.P + 3) / 4));
  int8_t* V = reinterpret_cast<int8_t*>(V16);
  CUtensorMap unused{};
  cudaError_t e;
  if (plan.dev.res[0].planes == 2)
    e = launch_ex(input_transform_tc_kernel<2, true>, dim3(grid), dim3(128), 0, s, 1, (const PlanDevice*)plan.d_plan, g, x, V, unused);
  else
    e = launch_ex(input_transform_tc_kernel<1, true>, dim3(grid), dim3(128), 0, s, 1, (const PlanDevice*)plan.d_plan, g, x, V, unused);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace rnsw
