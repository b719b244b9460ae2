// Memory-bound stages of the RNS-Winograd layer on sm_100a:
//   K2 filter transform   U = G g G^T mod m      (rw/kernel.py:38-41)
//   K1 input transform    V = BT d B mod m        (rw/kernel.py:44-47)
//   K4-K6 output stage    Y = AT M A mod m, MRC, crop/scatter
//                         (rw/kernel.py:50-53, rw/residue.py:180-206,
//                          rw/layer.py:374-388)
// plus the standalone MRC and the VGG inter-layer glue.
//
// Device layouts (all int8 limb planes are s8, see residue.planes_for_modulus):
//   U  [plane][pos][K][Cp]      pos = i*N + j of the N x N transform domain
//   V  [plane][pos][P][Cp]      P = B*th*tw tiles, tile p = (b*th + ti)*tw + tj
//   Mw [P/128][res][pos][128][Kp] int16  GEMM output, symmetric residues
//                                          (blocked layout, kernels.h mw_offset)
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace rnsw {

namespace {

constexpr int kChanBlock = 32;  // channels per CTA in K1 / output channels in K4

// Filter-bank planes of one residue: v itself (1 plane) for m < 256; for
// 16-bit moduli the limbs of v and of v' = 256*v mod m (4 planes), so the
// GEMM can form v_x*v_w with two accumulators (see gemm.cu).
RNSW_DEV void store_uplanes(int8_t* base, int64_t plane_stride, const ResidueTables& t, int32_t v) {
  if (t.uplanes == 1) {
    base[0] = (int8_t)v;
    return;
  }
  int8_t lo, hi;
  split_limbs(v, lo, hi);
  base[0] = lo;
  base[plane_stride] = hi;
  split_limbs(sym_mod(v * 256, t.modulus, t.inv_m), lo, hi);
  base[2 * plane_stride] = lo;
  base[3 * plane_stride] = hi;
}

// Write one symmetric residue as its limb plane(s).
RNSW_DEV void store_planes(int8_t* base, int64_t plane_stride, int planes, int32_t v) {
  if (planes == 1) {
    base[0] = (int8_t)v;
  } else {
    int8_t lo, hi;
    split_limbs(v, lo, hi);
    base[0] = lo;
    base[plane_stride] = hi;
  }
}

// ---------------------------------------------------------------------------
// K2: filter transform.  One thread per (c, k); loops over residues.
__global__ void filter_transform_kernel(const PlanDevice* __restrict__ plan, const int8_t* __restrict__ w, int C,
                                        int K, int Cp, int layout, int8_t* __restrict__ U) {
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int k = blockIdx.y * 8 + threadIdx.y;
  if (c >= Cp || k >= K) return;
  const int N = plan->n, R = plan->r, npos = N * N;
  int32_t g[RNSW_MAX_R * RNSW_MAX_R];
  for (int u = 0; u < R; ++u)
    for (int v = 0; v < R; ++v) {
      int32_t val = 0;
      if (c < C) {
        int64_t idx = layout == 0 ? ((int64_t)(u * R + v) * C + c) * K + k : (((int64_t)k * C + c) * R + u) * R + v;
        val = w[idx];
      }
      g[u * R + v] = val;
    }
  for (int r = 0; r < plan->n_res; ++r) {
    const ResidueTables& t = plan->res[r];
    const int32_t m = t.modulus;
    const float inv = t.inv_m;
    int32_t tg[RNSW_MAX_N * RNSW_MAX_R];  // (G g) mod m, N x R
    for (int i = 0; i < N; ++i)
      for (int v = 0; v < R; ++v) {
        int32_t s = 0;
        for (int u = 0; u < R; ++u) s += t.g[i * RNSW_MAX_R + u] * g[u * R + v];
        tg[i * R + v] = sym_mod(s, m, inv);
      }
    const int64_t plane_stride = (int64_t)npos * K * Cp;
    int8_t* ubase = U + (int64_t)t.uplane_base * plane_stride + (int64_t)k * Cp + c;
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        int32_t s = 0;
        for (int v = 0; v < R; ++v) s += tg[i * R + v] * t.g[j * RNSW_MAX_R + v];
        store_uplanes(ubase + (int64_t)(i * N + j) * K * Cp, plane_stride, t, sym_mod(s, m, inv));
      }
  }
}

// Reference-layout (N,N,C,K) residues of one modulus -> device filter bank.
__global__ void filter_import_kernel(const PlanDevice* __restrict__ plan, int res, const int16_t* __restrict__ src,
                                     int C, int K, int Cp, int8_t* __restrict__ U) {
  const int N = plan->n, npos = N * N;
  const int64_t total = (int64_t)npos * K * Cp;
  const ResidueTables& t = plan->res[res];
  const int64_t plane_stride = total;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(idx % Cp);
    const int64_t rest = idx / Cp;
    const int k = (int)(rest % K);
    const int pos = (int)(rest / K);
    int32_t v = c < C ? sym_mod(src[((int64_t)pos * C + c) * K + k], t.modulus, t.inv_m) : 0;
    store_uplanes(U + (int64_t)t.uplane_base * plane_stride + idx, plane_stride, t, v);
  }
}

// ---------------------------------------------------------------------------
// K1: input transform.  CTA = (tile p, 32-channel block).  The N x N patch is
// gathered with zero fill (conv padding + right/bottom canvas extension of
// tile_decompose, rw/layer.py:118-158), then BT d B is applied per residue in
// two separable passes with a symmetric reduction after each
// (rw/kernel.py:21-30).
__global__ void __launch_bounds__(256) input_transform_kernel(const PlanDevice* __restrict__ plan, Geometry g,
                                                              const int8_t* __restrict__ x, int8_t* __restrict__ V) {
  extern __shared__ int32_t smem[];
  const int N = plan->n, M = plan->m_out, npos = N * N;
  int32_t* D = smem;                          // [a][b][c]
  int32_t* T = D + npos * kChanBlock;         // [a][j][c]
  int32_t* BT = T + npos * kChanBlock;        // [res][N][N]
  const int tid = threadIdx.x;
  const int64_t p = blockIdx.x;
  const int c0 = blockIdx.y * kChanBlock;
  const int b = (int)(p / (g.th * g.tw));
  const int ti = (int)((p / g.tw) % g.th);
  const int tj = (int)(p % g.tw);

  for (int idx = tid; idx < plan->n_res * npos; idx += blockDim.x) {
    const int r = idx / npos, e = idx % npos;
    BT[idx] = plan->res[r].bt[(e / N) * RNSW_MAX_N + e % N];
  }
  for (int idx = tid; idx < npos * kChanBlock; idx += blockDim.x) {
    const int c = idx % kChanBlock, ab = idx / kChanBlock;
    const int h = ti * M + ab / N - g.pad, w = tj * M + ab % N - g.pad;
    int32_t v = 0;
    if (h >= 0 && h < g.H && w >= 0 && w < g.W && c0 + c < g.C) {
      const int64_t xi = g.layout == 0 ? (((int64_t)b * g.H + h) * g.W + w) * g.C + c0 + c
                                       : (((int64_t)b * g.C + c0 + c) * g.H + h) * g.W + w;
      v = x[xi];
    }
    D[idx] = v;
  }
  __syncthreads();

  const int64_t plane_stride = (int64_t)npos * g.P * g.Cp;
  for (int r = 0; r < plan->n_res; ++r) {
    const ResidueTables& t = plan->res[r];
    const int32_t m = t.modulus;
    const float inv = t.inv_m;
    const int32_t* bt = BT + r * npos;
    // pass 1: T[a][j] = sum_b D[a][b] * BT[j][b]
    for (int idx = tid; idx < npos * kChanBlock; idx += blockDim.x) {
      const int c = idx % kChanBlock, aj = idx / kChanBlock;
      const int a = aj / N, j = aj % N;
      int32_t s = 0;
      for (int bb = 0; bb < N; ++bb) s += D[(a * N + bb) * kChanBlock + c] * bt[j * N + bb];
      T[idx] = sym_mod(s, m, inv);
    }
    __syncthreads();
    // pass 2: V[i][j] = sum_a BT[i][a] * T[a][j]
    for (int idx = tid; idx < npos * kChanBlock; idx += blockDim.x) {
      const int c = idx % kChanBlock, ij = idx / kChanBlock;
      const int i = ij / N, j = ij % N;
      int32_t s = 0;
      for (int a = 0; a < N; ++a) s += bt[i * N + a] * T[(a * N + j) * kChanBlock + c];
      int8_t* dst = V + ((int64_t)t.plane_base * npos + ij) * g.P * g.Cp + p * g.Cp + c0 + c;
      store_planes(dst, plane_stride, t.planes, sym_mod(s, m, inv));
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K4-K6: output transform + MRC + scatter.  CTA = (tile p, 32 output channels).
__global__ void __launch_bounds__(256) output_transform_kernel(const PlanDevice* __restrict__ plan, Geometry g,
                                                               const int16_t* __restrict__ Mw,
                                                               int32_t* __restrict__ y, int16_t* __restrict__ y_res,
                                                               int kChanBlock) {
  extern __shared__ int32_t smem[];
  const int N = plan->n, M = plan->m_out, npos = N * N, nres = plan->n_res;
  int32_t* S = smem;                           // [res][pos][k]
  int32_t* Z = S + nres * npos * kChanBlock;   // [i][b][k]  (N x M)
  int32_t* Y = Z + N * M * kChanBlock;         // [res][a*M+b][k]
  int32_t* AT = Y + nres * M * M * kChanBlock; // [res][M][N]
  const int tid = threadIdx.x;
  const int64_t p = blockIdx.x;
  const int k0 = blockIdx.y * kChanBlock;

  for (int idx = tid; idx < nres * M * N; idx += blockDim.x) {
    const int r = idx / (M * N), e = idx % (M * N);
    AT[idx] = plan->res[r].at[(e / N) * RNSW_MAX_N + e % N];
  }
  for (int idx = tid; idx < nres * npos * kChanBlock; idx += blockDim.x) {
    const int k = idx % kChanBlock, rp = idx / kChanBlock;
    S[idx] = (k0 + k < g.Kp) ? (int32_t)Mw[mw_offset(p, rp, nres * npos, g.Kp) + k0 + k] : 0;
  }
  __syncthreads();

  for (int r = 0; r < nres; ++r) {
    const int32_t m = plan->res[r].modulus;
    const float inv = plan->res[r].inv_m;
    const int32_t* at = AT + r * M * N;
    const int32_t* s_r = S + r * npos * kChanBlock;
    for (int idx = tid; idx < N * M * kChanBlock; idx += blockDim.x) {
      const int k = idx % kChanBlock, ib = idx / kChanBlock;
      const int i = ib / M, bcol = ib % M;
      int32_t s = 0;
      for (int j = 0; j < N; ++j) s += s_r[(i * N + j) * kChanBlock + k] * at[bcol * N + j];
      Z[idx] = sym_mod(s, m, inv);
    }
    __syncthreads();
    for (int idx = tid; idx < M * M * kChanBlock; idx += blockDim.x) {
      const int k = idx % kChanBlock, ab = idx / kChanBlock;
      const int a = ab / M, bcol = ab % M;
      int32_t s = 0;
      for (int i = 0; i < N; ++i) s += at[a * N + i] * Z[(i * M + bcol) * kChanBlock + k];
      Y[r * M * M * kChanBlock + idx] = sym_mod(s, m, inv);
    }
    __syncthreads();
  }

  const int b = (int)(p / (g.th * g.tw));
  const int ti = (int)((p / g.tw) % g.th);
  const int tj = (int)(p % g.tw);
  for (int idx = tid; idx < M * M * kChanBlock; idx += blockDim.x) {
    const int k = idx % kChanBlock, ab = idx / kChanBlock;
    const int a = ab / M, bcol = ab % M;
    if (k0 + k >= g.K) continue;
    if (y_res != nullptr) {
      for (int r = 0; r < nres; ++r)
        y_res[(((int64_t)r * g.P + p) * g.K + k0 + k) * M * M + ab] = (int16_t)Y[r * M * M * kChanBlock + idx];
      continue;
    }
    const int ho = ti * M + a, wo = tj * M + bcol;
    if (ho >= g.Ho || wo >= g.Wo) continue;
    // mixed-radix digits (rw/residue.py:195-206)
    int64_t d[RNSW_MAX_RES];
    for (int j = 0; j < nres; ++j) {
      const int64_t mj = plan->res[j].modulus;
      int64_t t = ((int64_t)Y[j * M * M * kChanBlock + idx] % mj + mj) % mj;
      for (int i = 0; i < j; ++i) t = (((t - d[i]) * plan->mrc_inv[j][i]) % mj + mj) % mj;
      d[j] = t;
    }
    int64_t v = d[nres - 1];
    for (int j = nres - 2; j >= 0; --j) v = v * plan->res[j].modulus + d[j];
    if (v > plan->signed_bound) v -= plan->dynamic_range;
    const int64_t yi = g.layout == 0 ? (((int64_t)b * g.Ho + ho) * g.Wo + wo) * g.K + k0 + k
                                     : (((int64_t)b * g.K + k0 + k) * g.Ho + ho) * g.Wo + wo;
    y[yi] = (int32_t)v;
  }
}

__global__ void mrc_kernel(const PlanDevice* __restrict__ plan, const int16_t* __restrict__ res, int64_t count,
                           int64_t* __restrict__ out) {
  const int nres = plan->n_res;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t d[RNSW_MAX_RES];
    for (int j = 0; j < nres; ++j) {
      const int64_t mj = plan->res[j].modulus;
      int64_t t = ((int64_t)res[(int64_t)j * count + e] % mj + mj) % mj;
      for (int i = 0; i < j; ++i) t = (((t - d[i]) * plan->mrc_inv[j][i]) % mj + mj) % mj;
      d[j] = t;
    }
    int64_t v = d[nres - 1];
    for (int j = nres - 2; j >= 0; --j) v = v * plan->res[j].modulus + d[j];
    if (v > plan->signed_bound) v -= plan->dynamic_range;
    out[e] = v;
  }
}

// relu -> >> shift -> clip [0,127] -> optional 2x2 max-pool (floor), NHWC.
__global__ void requant_pool_kernel(const int32_t* __restrict__ y, int B, int H, int W, int C, int shift, int pool,
                                    int8_t* __restrict__ out) {
  const int Ho = pool ? H / 2 : H, Wo = pool ? W / 2 : W;
  const int64_t total = (int64_t)B * Ho * Wo * C;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % C);
    int64_t r = e / C;
    const int wo = (int)(r % Wo);
    r /= Wo;
    const int ho = (int)(r % Ho);
    const int b = (int)(r / Ho);
    int32_t v;
    if (pool) {
      const int64_t base = (((int64_t)b * H + 2 * ho) * W + 2 * wo) * C + c;
      v = max(max(y[base], y[base + C]), max(y[base + (int64_t)W * C], y[base + (int64_t)W * C + C]));
    } else {
      v = y[(((int64_t)b * H + ho) * W + wo) * C + c];
    }
    v = v > 0 ? (v >> shift) : 0;
    out[e] = (int8_t)(v > 127 ? 127 : v);
  }
}


// Vectorised glue for C % 4 == 0: four channels per thread (int4 loads,
// one 32-bit store of four int8).
__global__ void requant_pool_vec4_kernel(const int4* __restrict__ y, int B, int H, int W, int C4, int shift,
                                         int pool, uint32_t* __restrict__ out) {
  const int Ho = pool ? H / 2 : H, Wo = pool ? W / 2 : W;
  const int64_t total = (int64_t)B * Ho * Wo * C4;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c4 = (int)(e % C4);
    int64_t r = e / C4;
    const int wo = (int)(r % Wo);
    r /= Wo;
    const int ho = (int)(r % Ho);
    const int b = (int)(r / Ho);
    int4 v;
    if (pool) {
      const int64_t base = (((int64_t)b * H + 2 * ho) * W + 2 * wo) * C4 + c4;
      const int4 a0 = __ldg(y + base), a1 = __ldg(y + base + C4);
      const int4 a2 = __ldg(y + base + (int64_t)W * C4), a3 = __ldg(y + base + (int64_t)W * C4 + C4);
      v.x = max(max(a0.x, a1.x), max(a2.x, a3.x));
      v.y = max(max(a0.y, a1.y), max(a2.y, a3.y));
      v.z = max(max(a0.z, a1.z), max(a2.z, a3.z));
      v.w = max(max(a0.w, a1.w), max(a2.w, a3.w));
    } else {
      v = __ldg(y + (((int64_t)b * H + ho) * W + wo) * C4 + c4);
    }
    auto q = [shift](int32_t t) -> uint32_t { return (uint32_t)min(t > 0 ? t >> shift : 0, 127); };
    out[e] = q(v.x) | (q(v.y) << 8) | (q(v.z) << 16) | (q(v.w) << 24);
  }
}

// tile_decompose (rw/layer.py:118-158): overlapping N x N patches at stride
// tile_m of the zero canvas (input at offset pad, zero-extended right and
// bottom), patches[b][ti][tj][a][c2][ch].  Not on the layer path (K1 reads the
// canvas through its own addressing); this is the public API counterpart.
__global__ void tile_decompose_kernel(const int8_t* __restrict__ x, int B, int H, int W, int C, int M, int N,
                                      int pad, int th, int tw, int8_t* __restrict__ out) {
  const int64_t total = (int64_t)B * th * tw * N * N * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int c = (int)(t % C);
    t /= C;
    const int bb = (int)(t % N);
    t /= N;
    const int a = (int)(t % N);
    t /= N;
    const int tj = (int)(t % tw);
    t /= tw;
    const int ti = (int)(t % th);
    const int b = (int)(t / th);
    const int h = ti * M + a - pad, w = tj * M + bb - pad;
    out[i] = (h >= 0 && h < H && w >= 0 && w < W) ? x[(((int64_t)b * H + h) * W + w) * C + c] : (int8_t)0;
  }
}

}  // namespace

// RNSW_FORCE_GENERIC=1 routes every stage to the generic CUDA-core kernels
// (test hook for the cross-check of the two paths).
bool force_generic() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RNSW_FORCE_GENERIC");
    v = (e != nullptr && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// The tensor-core output kernel is instantiated for uniform limb planes:
// 1-2 residues of 16-bit moduli or 1-4 residues of 8-bit moduli.
bool tc_output_ok(const PlanDevice& d) {
  if (!d.fast || d.n > 16) return false;
  for (int r = 1; r < d.n_res; ++r)
    if (d.res[r].planes != d.res[0].planes) return false;
  return d.res[0].planes == 1 || d.n_res <= 2;
}

namespace {

int grid_for(int64_t total, int threads) {
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 32) blocks = 148 * 32;
  return blocks < 1 ? 1 : (int)blocks;
}

}  // namespace

cudaError_t launch_filter_transform(const PlanHost& plan, const int8_t* w, int C, int K, int Cp, int layout,
                                    int8_t* U, cudaStream_t s) {
  dim3 block(32, 8);
  dim3 grid((Cp + 31) / 32, (K + 7) / 8);
  filter_transform_kernel<<<grid, block, 0, s>>>(plan.d_plan, w, C, K, Cp, layout, U);
  return cudaGetLastError();
}

cudaError_t launch_filter_import(const PlanHost& plan, int res, const int16_t* u_nnck, int C, int K, int Cp,
                                 int8_t* U, cudaStream_t s) {
  const int64_t total = (int64_t)plan.dev.n * plan.dev.n * K * Cp;
  filter_import_kernel<<<grid_for(total, 256), 256, 0, s>>>(plan.d_plan, res, u_nnck, C, K, Cp, U);
  return cudaGetLastError();
}

cudaError_t launch_input_transform(const PlanHost& plan, const Geometry& g, const int8_t* x, int8_t* V,
                                   cudaStream_t s, bool relaxed) {
  if (tc_output_ok(plan.dev) && !force_generic()) {
    if (umma_input_ok(plan, g))
      return launch_input_transform_umma(plan, g, x, V, s, relaxed && plan.kr_limbs == 2 && g.C <= 8192);
    return launch_input_transform_tc(plan, g, x, V, s);
  }
  const int npos = plan.dev.n * plan.dev.n;
  const size_t smem = (size_t)(2 * npos * kChanBlock + plan.dev.n_res * npos) * sizeof(int32_t);
  // the >48 KB opt-in is per device: set it on every launch (cheap host call)
  cudaError_t e = cudaFuncSetAttribute(input_transform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)g.P, g.Cp / kChanBlock);
  input_transform_kernel<<<grid, 256, smem, s>>>(plan.d_plan, g, x, V);
  return cudaGetLastError();
}

cudaError_t launch_output_transform(const PlanHost& plan, const Geometry& g, const int16_t* Mw, int32_t* y,
                                    int16_t* y_res, cudaStream_t s) {
  if (tc_output_ok(plan.dev) && !force_generic()) return launch_output_transform_tc(plan, g, Mw, y, y_res, s);
  const int N = plan.dev.n, M = plan.dev.m_out, nres = plan.dev.n_res;
  int kcb = kChanBlock;
  auto smem_for = [&](int cb) {
    return (size_t)(nres * N * N * cb + N * M * cb + nres * M * M * cb + nres * M * N) * sizeof(int32_t);
  };
  while (kcb > 4 && smem_for(kcb) > 200 * 1024) kcb /= 2;  // large tiles / many residues
  const size_t smem = smem_for(kcb);
  cudaError_t e = cudaFuncSetAttribute(output_transform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       220 * 1024);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)g.P, (g.K + kcb - 1) / kcb);
  output_transform_kernel<<<grid, 256, smem, s>>>(plan.d_plan, g, Mw, y, y_res, kcb);
  return cudaGetLastError();
}

cudaError_t launch_tile_decompose(const int8_t* x, int B, int H, int W, int C, int tile_m, int r, int pad,
                                  int8_t* patches, cudaStream_t s) {
  const int Ho = H + 2 * pad - r + 1, Wo = W + 2 * pad - r + 1;
  const int th = (Ho + tile_m - 1) / tile_m, tw = (Wo + tile_m - 1) / tile_m, n = tile_m + r - 1;
  const int64_t total = (int64_t)B * th * tw * n * n * C;
  tile_decompose_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, B, H, W, C, tile_m, n, pad, th, tw, patches);
  return cudaGetLastError();
}

cudaError_t launch_mrc(const PlanHost& plan, const int16_t* residues, int64_t count, int64_t* out, cudaStream_t s) {
  mrc_kernel<<<grid_for(count, 256), 256, 0, s>>>(plan.d_plan, residues, count, out);
  return cudaGetLastError();
}

cudaError_t launch_requant_pool(const int32_t* y, int B, int H, int W, int C, int shift, int pool, int8_t* out,
                                cudaStream_t s) {
  const int64_t total = (int64_t)B * (pool ? H / 2 : H) * (pool ? W / 2 : W) * C;
  if ((C & 3) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 3) == 0) {
    requant_pool_vec4_kernel<<<grid_for(total / 4, 256), 256, 0, s>>>(reinterpret_cast<const int4*>(y), B, H, W,
                                                                      C / 4, shift, pool,
                                                                      reinterpret_cast<uint32_t*>(out));
    return cudaGetLastError();
  }
  requant_pool_kernel<<<grid_for(total, 256), 256, 0, s>>>(y, B, H, W, C, shift, pool, out);
  return cudaGetLastError();
}

}  // namespace rnsw
