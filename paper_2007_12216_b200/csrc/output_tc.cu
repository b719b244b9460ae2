// K4-K6 on the tensor cores: inverse Winograd transform Y = AT M A mod m for
// every residue, mixed-radix reconstruction and crop/scatter, in one kernel
// (rw/kernel.py:50-53, rw/residue.py:180-206, rw/layer.py:374-388).
//
// CTA = one tile p x 32 output channels, 4 warps x 8 channels.  The GEMM
// output Mw[p][res][pos][k] (int16 residues) is staged through shared memory
// transposed to [res][k][pos] so each warp can feed one channel's 16x16
// transform-domain tile straight into mma.sync fragments:
//   pass 1  Z^T = AT * Mat^T      (A = AT constants, B = Mat^T from smem)
//   pass 2  Y^T = Z^T * AT^T      (A = pass-1 C registers, no shuffles: the
//                                  contraction index i is permuted so the C
//                                  fragment columns land on the A k-slots)
// 16-bit moduli use two s8 limbs on each side (4 MMAs per product, 3
// accumulators) whose exact int32 recombination stays below 2^28 for
// m < 6000, so each value needs a single division-free reduction.
#include "common.cuh"
#include "kernels.h"

namespace rnsw {
namespace {

constexpr int kKB = 32;       // output channels per CTA
constexpr int kRowS = 258;    // int16 per staged row (516 B: conflict-free transposed stores)

struct ResConst {
  FastMod fm;
  int planes;
};

__global__ void __launch_bounds__(128) output_transform_tc_kernel(const PlanDevice* __restrict__ plan, Geometry g,
                                                                  const int16_t* __restrict__ Mw,
                                                                  int32_t* __restrict__ y,
                                                                  int16_t* __restrict__ y_res) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int N = plan->n, M = plan->m_out, npos = N * N, nres = plan->n_res;
  int16_t* S = reinterpret_cast<int16_t*>(smem_raw);  // [nres][kKB][kRowS]
  const int s_bytes = (nres * kKB * kRowS * 2 + 15) & ~15;
  int32_t* AT16 = reinterpret_cast<int32_t*>(smem_raw + s_bytes);  // [nres][16][16], zero padded
  int32_t* O = AT16 + nres * 256;                                   // [M*M][kKB]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
  const int64_t p = blockIdx.x;
  const int k0 = blockIdx.y * kKB;

  for (int idx = tid; idx < nres * 256; idx += blockDim.x) {
    const int r = idx >> 8, a = (idx >> 4) & 15, j = idx & 15;
    AT16[idx] = (a < M && j < N) ? plan->res[r].at[a * RNSW_MAX_N + j] : 0;
  }
  if (N < 16) {
    for (int idx = tid; idx < nres * kKB * kRowS / 2; idx += blockDim.x) reinterpret_cast<int32_t*>(S)[idx] = 0;
    __syncthreads();
  }
  // stage: 16 B (8 channels) per load, 4 loads per (res, pos) row segment
  for (int idx = tid; idx < nres * npos * 4; idx += blockDim.x) {
    const int kc = idx & 3, rp = idx >> 2;
    const int r = rp / npos, pos = rp - r * npos;
    const int i = pos / N, j = pos - i * N;
    int4 v = make_int4(0, 0, 0, 0);
    if (k0 + 8 * kc < g.Kp)
      v = __ldg(reinterpret_cast<const int4*>(Mw + ((p * nres + r) * npos + pos) * (int64_t)g.Kp + k0 + 8 * kc));
    const int16_t* e = reinterpret_cast<const int16_t*>(&v);
    int16_t* dst = S + (r * kKB + 8 * kc) * kRowS + 16 * i + j;
#pragma unroll
    for (int q = 0; q < 8; ++q) dst[q * kRowS] = e[q];
  }
  __syncthreads();

  ResConst rc[RNSW_MAX_RES];
#pragma unroll
  for (int r = 0; r < RNSW_MAX_RES; ++r)
    if (r < nres) rc[r] = ResConst{fast_mod_of(plan->res[r]), plan->res[r].planes};

  const int b_lo = gq, b_hi = gq + 8;  // pass-2 C rows = output column offset b
  for (int kk = 0; kk < kKB / 4; ++kk) {
    const int k = warp * (kKB / 4) + kk;
    int32_t yv[RNSW_MAX_RES][8];
#pragma unroll
    for (int r = 0; r < RNSW_MAX_RES; ++r) {
      if (r >= nres) break;
      const int32_t* at = AT16 + r * 256;
      const int16_t* row = S + (r * kKB + k) * kRowS;
      const FastMod fm = rc[r].fm;
      // constant fragments: pass-1 A = AT rows b, cols j = 4t..4t+3;
      // pass-2 B: column a, k-slot e <-> i = {2t, 2t+1, 8+2t, 9+2t}[e]
      int32_t a1v[8], b2v[2][4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a1v[e] = at[gq * 16 + 4 * tq + e];
        a1v[4 + e] = at[(gq + 8) * 16 + 4 * tq + e];
      }
#pragma unroll
      for (int na = 0; na < 2; ++na) {
        const int a = gq + 8 * na;
        b2v[na][0] = at[a * 16 + 2 * tq];
        b2v[na][1] = at[a * 16 + 2 * tq + 1];
        b2v[na][2] = at[a * 16 + 8 + 2 * tq];
        b2v[na][3] = at[a * 16 + 9 + 2 * tq];
      }
      int32_t z[2][4];
      if (rc[r].planes == 2) {
        const uint32_t alo0 = pack4_lo(a1v[0], a1v[1], a1v[2], a1v[3]);
        const uint32_t alo1 = pack4_lo(a1v[4], a1v[5], a1v[6], a1v[7]);
        const uint32_t ahi0 = pack4_lo(limb_hi(a1v[0]), limb_hi(a1v[1]), limb_hi(a1v[2]), limb_hi(a1v[3]));
        const uint32_t ahi1 = pack4_lo(limb_hi(a1v[4]), limb_hi(a1v[5]), limb_hi(a1v[6]), limb_hi(a1v[7]));
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          const int i = gq + 8 * ni;
          const uint32_t w0 = *reinterpret_cast<const uint32_t*>(row + 16 * i + 4 * tq);
          const uint32_t w1 = *reinterpret_cast<const uint32_t*>(row + 16 * i + 4 * tq + 2);
          const uint32_t blo = __byte_perm(w0, w1, 0x6420);  // u8 low bytes
          const uint32_t bhi = __byte_perm(w0, w1, 0x7531);  // s8 high bytes
          int32_t hh[4] = {0, 0, 0, 0}, cr[4] = {0, 0, 0, 0}, ll[4] = {0, 0, 0, 0};
          imma_ss(hh, ahi0, ahi1, bhi);
          imma_su(cr, ahi0, ahi1, blo);
          imma_ss(cr, alo0, alo1, bhi);
          imma_su(ll, alo0, alo1, blo);
#pragma unroll
          for (int e = 0; e < 4; ++e) z[ni][e] = red_fast(hh[e] * 65536 + cr[e] * 256 + ll[e], fm);
        }
      } else {
        const uint32_t a0 = pack4_lo(a1v[0], a1v[1], a1v[2], a1v[3]);
        const uint32_t a1 = pack4_lo(a1v[4], a1v[5], a1v[6], a1v[7]);
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          const int i = gq + 8 * ni;
          const uint32_t w0 = *reinterpret_cast<const uint32_t*>(row + 16 * i + 4 * tq);
          const uint32_t w1 = *reinterpret_cast<const uint32_t*>(row + 16 * i + 4 * tq + 2);
          const uint32_t b = __byte_perm(w0, w1, 0x6420);  // residues fit s8
          int32_t acc[4] = {0, 0, 0, 0};
          imma_ss(acc, a0, a1, b);
#pragma unroll
          for (int e = 0; e < 4; ++e) z[ni][e] = red_fast(acc[e], fm);
        }
      }
      // pass 2: A = Z^T (rows b = g / g+8; k-slots <- columns i of pass 1)
      if (rc[r].planes == 2) {
        const uint32_t zlo0 = pack4_lo(z[0][0], z[0][1], z[1][0], z[1][1]);
        const uint32_t zlo1 = pack4_lo(z[0][2], z[0][3], z[1][2], z[1][3]);
        const uint32_t zhi0 = pack4_lo(limb_hi(z[0][0]), limb_hi(z[0][1]), limb_hi(z[1][0]), limb_hi(z[1][1]));
        const uint32_t zhi1 = pack4_lo(limb_hi(z[0][2]), limb_hi(z[0][3]), limb_hi(z[1][2]), limb_hi(z[1][3]));
#pragma unroll
        for (int na = 0; na < 2; ++na) {
          const uint32_t blo = pack4_lo(b2v[na][0], b2v[na][1], b2v[na][2], b2v[na][3]);
          const uint32_t bhi = pack4_lo(limb_hi(b2v[na][0]), limb_hi(b2v[na][1]), limb_hi(b2v[na][2]),
                                        limb_hi(b2v[na][3]));
          int32_t hh[4] = {0, 0, 0, 0}, cr[4] = {0, 0, 0, 0}, ll[4] = {0, 0, 0, 0};
          imma_ss(hh, zhi0, zhi1, bhi);
          imma_ss(cr, zhi0, zhi1, blo);
          imma_ss(cr, zlo0, zlo1, bhi);
          imma_ss(ll, zlo0, zlo1, blo);
#pragma unroll
          for (int e = 0; e < 4; ++e) yv[r][4 * na + e] = red_fast(hh[e] * 65536 + cr[e] * 256 + ll[e], fm);
        }
      } else {
        const uint32_t za0 = pack4_lo(z[0][0], z[0][1], z[1][0], z[1][1]);
        const uint32_t za1 = pack4_lo(z[0][2], z[0][3], z[1][2], z[1][3]);
#pragma unroll
        for (int na = 0; na < 2; ++na) {
          const uint32_t b = pack4_lo(b2v[na][0], b2v[na][1], b2v[na][2], b2v[na][3]);
          int32_t acc[4] = {0, 0, 0, 0};
          imma_ss(acc, za0, za1, b);
#pragma unroll
          for (int e = 0; e < 4; ++e) yv[r][4 * na + e] = red_fast(acc[e], fm);
        }
      }
    }
    // yv[r][4*na + e]: a = 8*na + 2t + (e & 1), b = g + 8*(e >> 1)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int a = 8 * (q >> 2) + 2 * tq + (q & 1);
      const int b = (q & 2) ? b_hi : b_lo;
      if (a >= M || b >= M) continue;
      if (y_res != nullptr) {
        if (k0 + k < g.K) {
#pragma unroll
          for (int r = 0; r < RNSW_MAX_RES; ++r)
            if (r < nres) y_res[(((int64_t)r * g.P + p) * g.K + k0 + k) * M * M + a * M + b] = (int16_t)yv[r][q];
        }
        continue;
      }
      // mixed-radix reconstruction (rw/residue.py:195-206), exact in int32 for D < 2^31
      int32_t d[RNSW_MAX_RES];
      int32_t t0 = yv[0][q];
      d[0] = t0 < 0 ? t0 + rc[0].fm.m : t0;
      uint32_t x = (uint32_t)d[0], radix = (uint32_t)rc[0].fm.m;
#pragma unroll
      for (int j = 1; j < RNSW_MAX_RES; ++j) {
        if (j >= nres) break;
        int32_t t = yv[j][q];
        for (int i2 = 0; i2 < j; ++i2) t = red_fast((t - d[i2]) * (int32_t)plan->mrc_inv[j][i2], rc[j].fm);
        d[j] = t < 0 ? t + rc[j].fm.m : t;
        x += radix * (uint32_t)d[j];
        radix *= (uint32_t)rc[j].fm.m;
      }
      int64_t v = (int64_t)x;
      if (v > plan->signed_bound) v -= plan->dynamic_range;
      O[(a * M + b) * kKB + k] = (int32_t)v;
    }
  }
  if (y_res != nullptr) return;
  __syncthreads();

  const int b_img = (int)(p / (g.th * g.tw));
  const int ti = (int)((p / g.tw) % g.th);
  const int tj = (int)(p % g.tw);
  const int kvalid = min(kKB, g.K - k0);
  if (g.layout == 0 && (g.K & 3) == 0) {
    // NHWC: each pixel's 32 channels are 128 contiguous bytes
    for (int idx = tid; idx < M * M * (kKB / 4); idx += blockDim.x) {
      const int kq = idx % (kKB / 4), pix = idx / (kKB / 4);
      const int a = pix / M, bcol = pix - a * M;
      const int ho = ti * M + a, wo = tj * M + bcol;
      if (ho >= g.Ho || wo >= g.Wo || 4 * kq >= kvalid) continue;
      const int4 v = *reinterpret_cast<const int4*>(O + pix * kKB + 4 * kq);
      *reinterpret_cast<int4*>(y + (((int64_t)b_img * g.Ho + ho) * g.Wo + wo) * g.K + k0 + 4 * kq) = v;
    }
  } else {
    for (int idx = tid; idx < M * M * kKB; idx += blockDim.x) {
      int k, pix;
      if (g.layout == 0) {
        k = idx % kKB;
        pix = idx / kKB;
      } else {
        pix = idx % (M * M);
        k = idx / (M * M);
      }
      const int a = pix / M, bcol = pix - a * M;
      const int ho = ti * M + a, wo = tj * M + bcol;
      if (ho >= g.Ho || wo >= g.Wo || k >= kvalid) continue;
      const int64_t yi = g.layout == 0 ? (((int64_t)b_img * g.Ho + ho) * g.Wo + wo) * g.K + k0 + k
                                       : (((int64_t)b_img * g.K + k0 + k) * g.Ho + ho) * g.Wo + wo;
      y[yi] = O[pix * kKB + k];
    }
  }
}

}  // namespace

size_t output_tc_smem(const PlanDevice& d) {
  return (size_t)((d.n_res * kKB * kRowS * 2 + 15) & ~15) + d.n_res * 256 * 4 + (size_t)d.m_out * d.m_out * kKB * 4;
}

cudaError_t launch_output_transform_tc(const PlanHost& plan, const Geometry& g, const int16_t* Mw, int32_t* y,
                                       int16_t* y_res, cudaStream_t s) {
  const size_t smem = output_tc_smem(plan.dev);
  static int attr_done = 0;
  if (!attr_done) {
    cudaFuncSetAttribute(output_transform_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr_done = 1;
  }
  dim3 grid((unsigned)g.P, (g.K + kKB - 1) / kKB);
  output_transform_tc_kernel<<<grid, 128, smem, s>>>(plan.d_plan, g, Mw, y, y_res);
  return cudaGetLastError();
}

}  // namespace rnsw
