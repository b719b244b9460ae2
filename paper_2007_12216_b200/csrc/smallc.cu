// Small-channel layers (C <= 4, e.g. VGG16 conv1_1 with C = 3): the
// Winograd-domain product M = sum_c V[c] * U[c][k] mod m (rw/layer.py:366-372,
// rw/gemm.py:91-97) on the CUDA cores.
//
// A tensor-core GEMM would pad the 3-channel contraction to K = 32 and
// stream 10x more V than the layer has, so for C <= 4 the input transform
// writes compact int16 residues V16[res][P][pos][4] (input_tc.cu, kCompact)
// and this kernel forms the product directly into the output transform's
// input layout Mw (blocked, kernels.h mw_offset).  Each thread keeps the filter residues
// of one (residue, position, 8 output channels) in registers for a run of
// tiles: per tile it loads 8 bytes of V16 (shared by 8 threads), does
// 4 x 8 exact int32 products and 8 division-free reductions, and stores one
// 16-byte row segment of Mw.
#include "common.cuh"
#include "kernels.h"

#ifndef RNSW_SMALLC_MINB
#define RNSW_SMALLC_MINB 4  // C = 3 planar: 64 registers, 4 CTAs (32 warps) per SM to cover the V16 load latency (-7% vs 77 registers, 3 CTAs)
#endif
#ifndef RNSW_SMALLC_AHEAD
#define RNSW_SMALLC_AHEAD 8
#endif

namespace rnsw {
namespace {

// kPL == 2 (16-bit moduli): Mw holds y mod m in [0, m), which the output
// transform's limb split accepts (its bound analysis covers [0, m)).
// kPL == 1: symmetric residues (the s8 fragments of the output transform).
// kPlanar (16-bit only): write Mw8, the two byte planes the tcgen05 output
// transform reads (kernels.h mw8_offset).
// kC3: C == 3 (VGG16 conv1_1), the zero fourth channel is skipped.
template <int kPL, bool kPlanar = false, bool kC3 = false>
__global__ void __launch_bounds__(256, kC3 ? RNSW_SMALLC_MINB : 2) smallc_product_kernel(const PlanDevice* __restrict__ plan, int P, int K,
                                                             int Kp, int Cp, const int16_t* __restrict__ V16,
                                                             const int8_t* __restrict__ U, int16_t* __restrict__ Mw,
                                                             int tiles_per_cta) {
  pdl_trigger();
  const int N = plan->n, npos = N * N, nres = plan->n_res;
  const int kgroups = Kp >> 3;
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= npos * kgroups) return;
  const int pos = slot / kgroups, kg = slot - pos * kgroups;
  const int r = blockIdx.y;
  const ResidueTables& t = plan->res[r];
  const FastMod fm = fast_mod_of(t);

  // filter residues u[k][c] = lo + 256 hi from the bank's limb planes
  // [plane][pos][K][Cp] (transforms.cu store_uplanes)
  const int64_t plane_stride = (int64_t)npos * K * Cp;
  int32_t u[8][4];
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const int k = kg * 8 + kk;
    // channels 0..3 of one (plane, pos, k) row are 4 contiguous bytes (Cp >= 32)
    uint32_t lo4 = 0, hi4 = 0;
    if (k < K) {
      const int8_t* b = U + (int64_t)t.uplane_base * plane_stride + ((int64_t)pos * K + k) * Cp;
      lo4 = __ldg(reinterpret_cast<const uint32_t*>(b));
      if (kPL == 2) hi4 = __ldg(reinterpret_cast<const uint32_t*>(b + plane_stride));
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int32_t lo = (int32_t)(lo4 << (24 - 8 * c)) >> 24, hi = (int32_t)(hi4 << (24 - 8 * c)) >> 24;
      u[kk][c] = kPL == 2 ? lo + 256 * hi : lo;
    }
  }
  const int32_t bias = kPL == 2 ? pos_bias(fm) : fm.off;
  pdl_wait();  // V16 from the input transform
  const int p_begin = blockIdx.z * tiles_per_cta, p_end = min(P, p_begin + tiles_per_cta);
  const uint2* src = reinterpret_cast<const uint2*>(V16) + ((int64_t)r * P + p_begin) * npos + pos;
  const int rp = r * npos + pos, nrp = nres * npos;
  // V16 rows of 8 tiles are loaded together ahead of their products
  constexpr int kAhead = RNSW_SMALLC_AHEAD;
  uint8_t* out8 = nullptr;  // Mw8 row of the current tile (advances by Kp within a block of 128 tiles)
  for (int p0 = p_begin; p0 < p_end; p0 += kAhead) {
    uint2 wv[kAhead];
#pragma unroll
    for (int i = 0; i < kAhead; ++i)
      wv[i] = p0 + i < p_end ? __ldg(src + (int64_t)(p0 - p_begin + i) * npos) : make_uint2(0, 0);
#pragma unroll
    for (int i = 0; i < kAhead; ++i) {
      const int p = p0 + i;
      if (p >= p_end) break;
      const uint2 w = wv[i];
      const int32_t v0 = (int32_t)(w.x << 16) >> 16, v1 = (int32_t)w.x >> 16;
      const int32_t v2 = (int32_t)(w.y << 16) >> 16, v3 = (int32_t)w.y >> 16;
      uint32_t o[4];
      int32_t yv[8];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        int32_t y[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int kk = 2 * h + e;
          // |sum| <= 4 h^2 < 2^28 for m < 4500
          const int32_t n =
              kC3 ? bias + v0 * u[kk][0] + v1 * u[kk][1] + v2 * u[kk][2]
                  : bias + v0 * u[kk][0] + v1 * u[kk][1] + v2 * u[kk][2] + v3 * u[kk][3];
          y[e] = kPL == 2 ? red_pos_biased(n, fm) : red_pos_biased(n, fm) - fm.h;
          yv[kk] = y[e];
        }
        o[h] = __byte_perm((uint32_t)y[0], (uint32_t)y[1], 0x5410);
      }
      if constexpr (kPlanar) {
        if (p == p_begin || (p & 127) == 0)
          out8 = reinterpret_cast<uint8_t*>(Mw) + mw8_offset(p, r, 0, pos, nres, npos, Kp) + 8 * kg;
        else
          out8 += Kp;
        uint8_t* base = out8;
        const uint32_t a0 = __byte_perm((uint32_t)yv[0], (uint32_t)yv[1], 0x5140);
        const uint32_t a1 = __byte_perm((uint32_t)yv[2], (uint32_t)yv[3], 0x5140);
        const uint32_t a2 = __byte_perm((uint32_t)yv[4], (uint32_t)yv[5], 0x5140);
        const uint32_t a3 = __byte_perm((uint32_t)yv[6], (uint32_t)yv[7], 0x5140);
        *reinterpret_cast<uint2*>(base) = make_uint2(__byte_perm(a0, a1, 0x5410), __byte_perm(a2, a3, 0x5410));
        *reinterpret_cast<uint2*>(base + (int64_t)npos * 128 * Kp) =
            make_uint2(__byte_perm(a0, a1, 0x7632), __byte_perm(a2, a3, 0x7632));
      } else {
        *(reinterpret_cast<uint4*>(Mw + mw_offset(p, rp, nrp, Kp)) + kg) = make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
  }
}

}  // namespace

bool smallc_ok(const PlanDevice& d, const Geometry& g) { return g.C <= 4 && tc_output_ok(d); }

size_t smallc_v16_bytes(const PlanDevice& d, const Geometry& g) {
  return (size_t)d.n_res * g.P * d.n * d.n * 4 * sizeof(int16_t);
}

cudaError_t launch_smallc_product(const PlanHost& plan, const Geometry& g, const int16_t* V16, const int8_t* U,
                                  int16_t* Mw, cudaStream_t s, bool planar) {
  const PlanDevice& d = plan.dev;
  const int npos = d.n * d.n, slots = npos * (g.Kp / 8);
  const int bx = (slots + 255) / 256;
  // about 4 CTAs per SM in total, each amortising its register-held filter
  // residues over up to 64 tiles (also at batch 1)
  const int64_t per_tile = (int64_t)bx * d.n_res;
  const int tpc = (int)std::max<int64_t>(1, std::min<int64_t>(64, g.P * per_tile / (148 * 4)));
  dim3 grid(bx, d.n_res, (unsigned)((g.P + tpc - 1) / tpc));
  cudaError_t e;
  if (d.res[0].planes == 2 && planar && g.C == 3)
    e = launch_ex(smallc_product_kernel<2, true, true>, grid, dim3(256), 0, s, 1, (const PlanDevice*)plan.d_plan, (int)g.P, g.K, g.Kp, g.Cp, V16, U, Mw, tpc);
  else if (d.res[0].planes == 2 && planar)
    e = launch_ex(smallc_product_kernel<2, true>, grid, dim3(256), 0, s, 1, (const PlanDevice*)plan.d_plan, (int)g.P, g.K, g.Kp, g.Cp, V16, U, Mw, tpc);
  else if (d.res[0].planes == 2)
    e = launch_ex(smallc_product_kernel<2>, grid, dim3(256), 0, s, 1, (const PlanDevice*)plan.d_plan, (int)g.P, g.K, g.Kp, g.Cp, V16, U, Mw, tpc);
  else
    e = launch_ex(smallc_product_kernel<1>, grid, dim3(256), 0, s, 1, (const PlanDevice*)plan.d_plan, (int)g.P, g.K, g.Kp, g.Cp, V16, U, Mw, tpc);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace rnsw
