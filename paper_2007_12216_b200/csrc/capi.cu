// C ABI entry points (include/rnsw.h): plan construction, argument checking,
// buffer sizing and stage orchestration.  Every entry point validates its
// arguments on the host before any device work, mirroring the reference's
// "raise before doing work" behaviour (rw/layer.py:321-359), and reports
// failures as codes that the Python layer maps onto the reference's
// exception classes (paper_2007_12216_b200/errors.py).
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "../../include/rnsw.h"
#include "kernels.h"

struct rnsw_plan {
  rnsw::PlanHost host;
};

// Programmatic dependent launch for the layer kernels (declared in
// common.cuh) when the layer is small: its kernels are short and launch /
// prologue latency matters (VGG16 batch 1: -8%, batch 32: -1.6%); at batch
// 256 it measured +3 to +4.5% when the 65536-tile layers take part and
// -0.4% up to 16384 tiles.  The layer entry points record the tile count
// (pdl_layer_hint); RNSW_PDL=0 disables it, RNSW_PDL=N sets the tile limit
// (default 16384).
namespace {
thread_local int64_t g_pdl_tiles = 0;
}
namespace rnsw {
void pdl_layer_hint(int64_t P) { g_pdl_tiles = P; }
}  // namespace rnsw
bool pdl_enabled() {
  static const int64_t max_tiles = [] {
    const char* e = getenv("RNSW_PDL");
    return e == nullptr ? (int64_t)16384 : (int64_t)atoll(e) * (atoll(e) == 1 ? 16384 : 1);
  }();
  return g_pdl_tiles > 0 && g_pdl_tiles <= max_tiles;
}

namespace {

thread_local char g_last_error[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(RNSW_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return a < 0 ? -a : a;
}

int32_t sym(int64_t x, int32_t m) {
  int64_t r = x % m;
  if (r < 0) r += m;
  if (r > (m - 1) / 2) r -= m;
  return (int32_t)r;
}

int64_t round_up(int64_t x, int64_t q) { return (x + q - 1) / q * q; }

int padded_channels(int C) {
  if (C <= 32) return 32;
  if (C <= 64) return 64;
  return (int)round_up(C, 128);
}

int check_plan(const rnsw_plan* plan) {
  if (plan == nullptr) return fail(RNSW_ERR_INVALID, "null plan");
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(RNSW_ERR_CUDA, "cudaGetDevice failed");
  if (dev != plan->host.device)
    return fail(RNSW_ERR_UNSUPPORTED, "plan was created on device %d, current device is %d", plan->host.device, dev);
  return RNSW_OK;
}

int make_geometry(const rnsw_plan* plan, int B, int H, int W, int C, int K, int pad, int layout, rnsw::Geometry* g) {
  const PlanDevice& d = plan->host.dev;
  if (B < 1 || H < 1 || W < 1 || C < 1 || K < 1 || pad < 0)
    return fail(RNSW_ERR_SHAPE, "bad layer geometry B=%d H=%d W=%d C=%d K=%d pad=%d", B, H, W, C, K, pad);
  if (layout != RNSW_LAYOUT_NHWC && layout != RNSW_LAYOUT_NCHW) return fail(RNSW_ERR_INVALID, "bad layout %d", layout);
  g->B = B;
  g->H = H;
  g->W = W;
  g->C = C;
  g->K = K;
  g->pad = pad;
  g->layout = layout;
  g->Ho = H + 2 * pad - d.r + 1;
  g->Wo = W + 2 * pad - d.r + 1;
  if (g->Ho < 1 || g->Wo < 1) return fail(RNSW_ERR_SHAPE, "padded input smaller than the filter");
  g->th = (g->Ho + d.m_out - 1) / d.m_out;
  g->tw = (g->Wo + d.m_out - 1) / d.m_out;
  g->P = (int64_t)B * g->th * g->tw;
  rnsw::pdl_layer_hint(g->P);
  // s32 accumulators must stay below 2^31: per channel at most 128 * 128
  // (8-bit residues) or, for 16-bit residues, |v_hi u'_lo + v_lo u_lo| <=
  // 9 * 128 + 128 * 128 = 17536 (limbs of symmetric residues, gemm.cu)
  bool wide = false;
  for (int i = 0; i < d.n_res; ++i) wide = wide || d.res[i].planes == 2;
  if ((int64_t)C * (wide ? 17536 : 128 * 128) > 2147483647LL)
    return fail(RNSW_ERR_OVERFLOW, "C=%d channels can overflow the int32 tensor-core accumulator", C);
  if (g->P > 2147483647LL) return fail(RNSW_ERR_UNSUPPORTED, "too many tiles (%lld)", (long long)g->P);
  g->Cp = padded_channels(C);
  g->Kp = (int)round_up(K, 16);
  g->bc = g->Cp < 128 ? g->Cp : 128;
  return RNSW_OK;
}

size_t v_bytes(const PlanDevice& d, int64_t P, int Cp) { return (size_t)d.n_planes * d.n * d.n * P * Cp; }
size_t m_bytes(const PlanDevice& d, int64_t P, int Kp) {  // blocked layout (kernels.h mw_offset)
  return (size_t)((P + 127) / 128) * 128 * d.n_res * d.n * d.n * Kp * sizeof(int16_t);
}

}  // namespace

namespace {
// Host copy of the output_umma.cu constant operands (see PlanDevice::umma_b):
// B1[res] rows n = (acc, a) x K slots (limb, i) hold the balanced limbs of
// AT (limb 0) and 256 AT mod m (limb 1); B2[res][0] rows (acc, b) x (z0 | z1, j)
// the limbs of ATW and 256 ATW, B2[res][1] (z2, j) those of 65536 ATW, then
// 16 bias slots whose 127-weighted sum is 127 X, X = m ceil(360000 / m): for
// every m < 4500 it exceeds the most negative pass-2 input (pass-2 sum
// >= -16 h (255 + 255 + 128) > -2.3e7, digit term d0 W[1][0] > -m0 m1 > -2.03e7)
// and keeps the largest below 2^30.
// ATW = AT W[1][0] for residue 1 (the mixed-radix factor), AT for residue 0.
void build_umma_b(PlanDevice& d) {
  auto sym = [](int64_t v, int64_t m) {
    v %= m;
    if (v < 0) v += m;
    return v > (m - 1) / 2 ? v - m : v;
  };
  auto limb = [](int64_t c, int acc) {
    const int64_t hi = (c + 128 + 256 * 64) / 256 - 64;  // floor((c + 128) / 256)
    return (int8_t)(acc == 0 ? hi : c - 256 * hi);
  };
  auto swz = [](uint32_t off) { return off ^ (((off >> 7) & 1u) << 4); };
  memset(d.umma_b, 0, sizeof(d.umma_b));
  for (int res = 0; res < 2; ++res) {
    const int64_t m = d.res[res].modulus;
    for (int n = 0; n < 32; ++n)
      for (int kap = 0; kap < 32; ++kap) {
        const int acc = n >> 4, a = n & 15, lb = kap >> 4, i = kap & 15;
        const int64_t at = a < 14 ? d.res[res].at[a * RNSW_MAX_N + i] : 0;
        d.umma_b[res * 1024 + swz(n * 32 + kap)] = (uint8_t)limb(lb == 0 ? at : sym(at * 256, m), acc);
      }
    for (int step = 0; step < 2; ++step)
      for (int n = 0; n < 32; ++n)
        for (int kap = 0; kap < 32; ++kap) {
          const int acc = n >> 4, b = n & 15, j = kap & 15;
          int8_t v = 0;
          if (step == 1 && kap >= 16) {
            const int64_t X = m * ((360000 + m - 1) / m);
            const int64_t S = acc == 0 ? (X >> 8) : (X & 255), sl = kap - 16;
            v = (int8_t)(S / 16 + (sl < S % 16 ? 1 : 0));
          } else if (b < 14 && (step == 0 || kap < 16)) {
            int64_t c = d.res[res].at[b * RNSW_MAX_N + j];
            if (res) c = sym(c * d.mrc_w[1][0], m);
            const int shifts = step == 1 ? 2 : (kap >> 4);
            for (int t = 0; t < shifts; ++t) c = sym(c * 256, m);
            v = limb(c, acc);
          }
          d.umma_b[2048 + (res * 2 + step) * 1024 + swz(n * 32 + kap)] = (uint8_t)v;
        }
  }
}
}  // namespace

extern "C" {

const char* rnsw_error_string(int code) {
  switch (code) {
    case RNSW_OK: return "ok";
    case RNSW_ERR_INVALID: return "invalid argument";
    case RNSW_ERR_SHAPE: return "shape mismatch";
    case RNSW_ERR_STRIDE: return "unsupported stride";
    case RNSW_ERR_RANGE: return "dynamic range exceeded";
    case RNSW_ERR_NOT_COPRIME: return "moduli not coprime";
    case RNSW_ERR_OVERFLOW: return "accumulator overflow risk";
    case RNSW_ERR_SYSTEM: return "residue system mismatch";
    case RNSW_ERR_CUDA: return "CUDA error";
    case RNSW_ERR_WORKSPACE: return "buffer too small";
    case RNSW_ERR_UNSUPPORTED: return "unsupported on the device path";
    default: return "unknown error";
  }
}

const char* rnsw_last_error(void) { return g_last_error; }

int rnsw_plan_create(rnsw_plan** out, int tile_m, int r, int n_res, const int32_t* moduli, const int16_t* at,
                     const int16_t* g, const int16_t* bt, const int32_t* mrc_inv) {
  if (out == nullptr || moduli == nullptr || at == nullptr || g == nullptr || bt == nullptr || mrc_inv == nullptr)
    return fail(RNSW_ERR_INVALID, "null argument");
  *out = nullptr;
  if (tile_m < 1 || r < 1) return fail(RNSW_ERR_INVALID, "need tile_m >= 1 and r >= 1");
  const int n = tile_m + r - 1;
  if (n < 2) return fail(RNSW_ERR_INVALID, "tile_m + r - 1 must be at least 2");
  if (n > RNSW_MAX_N || r > RNSW_MAX_R)
    return fail(RNSW_ERR_UNSUPPORTED, "F(%d,%d): tile side %d exceeds the device limit %d", tile_m, r, n, RNSW_MAX_N);
  // (tensor-core transform kernels need N <= 16; larger tiles use the generic kernels)
  if (n_res < 1 || n_res > RNSW_MAX_RES)
    return fail(RNSW_ERR_UNSUPPORTED, "%d moduli: the device path takes 1..%d", n_res, RNSW_MAX_RES);
  for (int i = 0; i < n_res; ++i) {
    const int m = moduli[i];
    if (m < 3 || m % 2 == 0 || m > 32767) return fail(RNSW_ERR_INVALID, "modulus must be odd and in [3, 32767], got %d", m);
    for (int j = 0; j < i; ++j)
      if (gcd64(m, moduli[j]) != 1)
        return fail(RNSW_ERR_NOT_COPRIME, "moduli %d and %d share factor %lld", moduli[j], m, (long long)gcd64(m, moduli[j]));
  }
  rnsw_plan* plan = new (std::nothrow) rnsw_plan();
  if (plan == nullptr) return fail(RNSW_ERR_INVALID, "out of host memory");
  PlanDevice& d = plan->host.dev;
  memset(&d, 0, sizeof(d));
  d.m_out = tile_m;
  d.r = r;
  d.n = n;
  d.n_res = n_res;
  d.dynamic_range = 1;
  int plane = 0, uplane = 0;
  for (int i = 0; i < n_res; ++i) {
    ResidueTables& t = d.res[i];
    const int m = moduli[i];
    const int half = (m - 1) / 2;
    t.modulus = m;
    t.planes = m < 256 ? 1 : 2;
    t.plane_base = plane;
    plane += t.planes;
    t.uplanes = m < 256 ? 1 : 4;
    t.uplane_base = uplane;
    uplane += t.uplanes;
    t.inv_m = 1.0f / (float)m;
    t.r_256 = sym(256, m);
    t.r_65536 = sym(65536, m);
    t.half = half;
    {
      int sh = 0;
      while ((2 << sh) <= m) ++sh;  // sh = floor(log2 m)
      const unsigned __int128 num = (unsigned __int128)1 << (32 + sh);
      t.red_mul = (uint32_t)((num + m - 1) / m);
      t.red_shift = sh;
      const int64_t L = ((1LL << 28) + m - 1) / m;
      t.red_off = (int32_t)(half + m * L);
      t.red_negm = (uint32_t)(-(int64_t)m);
    }
    auto load = [&](const int16_t* src, int rows, int cols, int stride, int32_t* dst) -> bool {
      for (int a = 0; a < rows; ++a)
        for (int b = 0; b < cols; ++b) {
          const int v = src[(size_t)i * rows * cols + a * cols + b];
          if (v < -half || v > half) return false;
          dst[a * stride + b] = v;
        }
      return true;
    };
    if (!load(at, tile_m, n, RNSW_MAX_N, t.at) || !load(g, n, r, RNSW_MAX_R, t.g) || !load(bt, n, n, RNSW_MAX_N, t.bt)) {
      delete plan;
      return fail(RNSW_ERR_INVALID, "transform entries for modulus %d are not symmetric residues", m);
    }
    d.dynamic_range *= m;
  }
  d.n_planes = plane;
  d.n_uplanes = uplane;
  {
    bool fast = d.dynamic_range < (1LL << 31);
    for (int i = 0; i < n_res; ++i) fast = fast && moduli[i] < 4500;  // keeps every limb recombination below 2^28
    d.fast = fast ? 1 : 0;
  }
  {
    // K4's unreduced pass 1 (output_tc.cu, output_umma.cu): the sum over j of
    // AT'[a][j] hi + AT[a][j] lo, AT' = 256 AT mod m, with hi, lo the bytes of
    // y mod m in [0, m) (hi <= (m-1) >> 8, lo <= 255), must fit
    // three bytes as a signed value for every row a of every 16-bit residue
    bool z3 = true;
    for (int i = 0; i < n_res; ++i) {
      const ResidueTables& t = d.res[i];
      if (t.planes != 2) continue;
      const int64_t hi_max = (t.modulus - 1) >> 8;  // high byte of y mod m in [0, m)
      for (int a = 0; a < tile_m; ++a) {
        int64_t bound = 0;
        for (int j = 0; j < n; ++j) {
          const int64_t v = t.at[a * RNSW_MAX_N + j];
          const int64_t vp = sym(v * 256, t.modulus);
          bound += hi_max * (vp < 0 ? -vp : vp) + 255 * (v < 0 ? -v : v);
        }
        z3 = z3 && bound < (1 << 23);
      }
    }
    d.z3 = z3 ? 1 : 0;
  }
  d.signed_bound = (d.dynamic_range - 1) / 2;
  for (int j = 0; j < n_res; ++j)
    for (int i = 0; i < j; ++i) {
      const int64_t inv = mrc_inv[j * n_res + i];
      if (((int64_t)moduli[i] * inv % moduli[j] + moduli[j]) % moduli[j] != 1) {
        delete plan;
        return fail(RNSW_ERR_SYSTEM, "mrc_inv[%d][%d]=%lld is not %d^-1 mod %d", j, i, (long long)inv, moduli[i],
                    moduli[j]);
      }
      d.mrc_inv[j][i] = inv;
    }
  for (int j = 0; j < n_res; ++j)
    for (int i = j - 1; i >= 0; --i) {
      const int64_t mj = moduli[j], next = i == j - 1 ? 1 : d.mrc_w[j][i + 1];
      d.mrc_w[j][i] = (int32_t)(((next * (d.mrc_inv[j][i] % mj)) % mj + mj) % mj);
    }
  if (n == 16 && tile_m == 14 && n_res == 2 && d.res[0].planes == 2 && d.res[1].planes == 2) build_umma_b(d);
  cudaError_t e = cudaGetDevice(&plan->host.device);
  if (e == cudaSuccess) e = cudaMalloc(&plan->host.d_plan, sizeof(PlanDevice));
  if (e == cudaSuccess) e = cudaMemcpy(plan->host.d_plan, &d, sizeof(d), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = rnsw::build_kr_images(plan->host);
  if (e == cudaSuccess) e = rnsw::build_kra_images(plan->host);
  if (e == cudaSuccess) e = rnsw::build_kra8_images(plan->host);
  if (e != cudaSuccess) {
    if (plan->host.d_plan) cudaFree(plan->host.d_plan);
    rnsw::free_kr_images(plan->host);
    rnsw::free_kra_images(plan->host);
    delete plan;
    return cuda_fail(e, "rnsw_plan_create");
  }
  *out = plan;
  return RNSW_OK;
}

void rnsw_plan_destroy(rnsw_plan* plan) {
  if (plan == nullptr) return;
  if (plan->host.d_plan) cudaFree(plan->host.d_plan);
  rnsw::free_kr_images(plan->host);
  rnsw::free_kra_images(plan->host);
  delete plan;
}

int rnsw_plan_info(const rnsw_plan* plan, int* n, int* n_planes) {
  if (plan == nullptr) return fail(RNSW_ERR_INVALID, "null plan");
  if (n) *n = plan->host.dev.n;
  if (n_planes) *n_planes = plan->host.dev.n_planes;
  return RNSW_OK;
}

size_t rnsw_filter_bytes(const rnsw_plan* plan, int C, int K) {
  if (plan == nullptr || C < 1 || K < 1) return 0;
  const PlanDevice& d = plan->host.dev;
  return (size_t)d.n_uplanes * d.n * d.n * K * padded_channels(C);
}

size_t rnsw_v_bytes(const rnsw_plan* plan, int64_t P, int C) {
  if (plan == nullptr || P < 1 || C < 1) return 0;
  return v_bytes(plan->host.dev, P, padded_channels(C));
}

size_t rnsw_m_bytes(const rnsw_plan* plan, int64_t P, int K) {
  if (plan == nullptr || P < 1 || K < 1) return 0;
  return m_bytes(plan->host.dev, P, (int)round_up(K, 16));
}

size_t rnsw_workspace_bytes(const rnsw_plan* plan, int B, int H, int W, int C, int K, int pad) {
  if (plan == nullptr) return 0;
  rnsw::Geometry g;
  if (make_geometry(plan, B, H, W, C, K, pad, RNSW_LAYOUT_NHWC, &g) != RNSW_OK) return 0;
  return round_up(v_bytes(plan->host.dev, g.P, g.Cp), 256) + m_bytes(plan->host.dev, g.P, g.Kp);
}

int rnsw_filter_transform(const rnsw_plan* plan, const int8_t* w, int C, int K, int layout, void* U, size_t U_bytes,
                          void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (w == nullptr || U == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (C < 1 || K < 1) return fail(RNSW_ERR_SHAPE, "bad filter shape C=%d K=%d", C, K);
  if (layout != RNSW_LAYOUT_NHWC && layout != RNSW_LAYOUT_NCHW) return fail(RNSW_ERR_INVALID, "bad layout %d", layout);
  if (U_bytes < rnsw_filter_bytes(plan, C, K)) return fail(RNSW_ERR_WORKSPACE, "filter bank buffer too small");
  cudaError_t e = rnsw::launch_filter_transform(plan->host, w, C, K, padded_channels(C), layout,
                                                static_cast<int8_t*>(U), (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "filter_transform");
}

int rnsw_filter_import(const rnsw_plan* plan, int res, const int16_t* u_nnck, int C, int K, void* U, size_t U_bytes,
                       void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (u_nnck == nullptr || U == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (res < 0 || res >= plan->host.dev.n_res) return fail(RNSW_ERR_SYSTEM, "residue index %d out of range", res);
  if (U_bytes < rnsw_filter_bytes(plan, C, K)) return fail(RNSW_ERR_WORKSPACE, "filter bank buffer too small");
  cudaError_t e = rnsw::launch_filter_import(plan->host, res, u_nnck, C, K, padded_channels(C),
                                             static_cast<int8_t*>(U), (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "filter_import");
}

int rnsw_input_transform(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C, int pad, int layout,
                         void* V, size_t V_bytes, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (x == nullptr || V == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  rnsw::Geometry g;
  if (int rc = make_geometry(plan, B, H, W, C, 1, pad, layout, &g)) return rc;
  if (V_bytes < v_bytes(plan->host.dev, g.P, g.Cp)) return fail(RNSW_ERR_WORKSPACE, "V buffer too small");
  cudaError_t e = rnsw::launch_input_transform(plan->host, g, x, static_cast<int8_t*>(V), (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "input_transform");
}

int rnsw_input_transform_compact(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C, int pad,
                                 int layout, void* V16, size_t V16_bytes, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (x == nullptr || V16 == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  rnsw::Geometry g;
  if (int rc = make_geometry(plan, B, H, W, C, 1, pad, layout, &g)) return rc;
  if (!rnsw::smallc_ok(plan->host.dev, g))
    return fail(RNSW_ERR_UNSUPPORTED, "compact transform needs C <= 4 and a tensor-core plan (C=%d)", C);
  if (V16_bytes < rnsw::smallc_v16_bytes(plan->host.dev, g)) return fail(RNSW_ERR_WORKSPACE, "V16 buffer too small");
  cudaError_t e = rnsw::launch_input_transform_compact(plan->host, g, x, static_cast<int16_t*>(V16),
                                                       (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "input_transform_compact");
}

int rnsw_small_channel_product(const rnsw_plan* plan, const void* V16, const void* U, int64_t P, int C, int K,
                               void* Mw, size_t Mw_bytes, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (V16 == nullptr || U == nullptr || Mw == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (P < 1 || P > 2147483647LL || C < 1 || K < 1) return fail(RNSW_ERR_SHAPE, "bad product shape P=%lld C=%d K=%d",
                                                          (long long)P, C, K);
  rnsw::Geometry g{};
  g.P = P;
  rnsw::pdl_layer_hint(P);
  g.C = C;
  g.K = K;
  g.Cp = padded_channels(C);
  g.Kp = (int)round_up(K, 16);
  if (!rnsw::smallc_ok(plan->host.dev, g))
    return fail(RNSW_ERR_UNSUPPORTED, "small-channel product needs C <= 4 and a tensor-core plan (C=%d)", C);
  if (Mw_bytes < m_bytes(plan->host.dev, P, g.Kp)) return fail(RNSW_ERR_WORKSPACE, "Mw buffer too small");
  cudaError_t e = rnsw::launch_smallc_product(plan->host, g, static_cast<const int16_t*>(V16),
                                              static_cast<const int8_t*>(U), static_cast<int16_t*>(Mw),
                                              (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "small_channel_product");
}

int rnsw_winograd_gemm(const rnsw_plan* plan, const void* V, const void* U, int64_t P, int C, int K, void* Mw,
                       size_t Mw_bytes, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (V == nullptr || U == nullptr || Mw == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (P < 1 || C < 1 || K < 1) return fail(RNSW_ERR_SHAPE, "bad GEMM shape P=%lld C=%d K=%d", (long long)P, C, K);
  rnsw::pdl_layer_hint(P);
  if ((int64_t)C * 128 * 128 > 2147483647LL) return fail(RNSW_ERR_OVERFLOW, "C=%d can overflow int32", C);
  const int Cp = padded_channels(C), Kp = (int)round_up(K, 16);
  if (Mw_bytes < m_bytes(plan->host.dev, P, Kp)) return fail(RNSW_ERR_WORKSPACE, "Mw buffer too small");
  cudaError_t e = rnsw::launch_winograd_gemm(plan->host, static_cast<const int8_t*>(V), static_cast<const int8_t*>(U),
                                             P, Cp, K, Kp, Cp < 128 ? Cp : 128, static_cast<int16_t*>(Mw),
                                             (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "winograd_gemm");
}

int rnsw_output_transform(const rnsw_plan* plan, const void* Mw, int B, int H, int W, int K, int pad, int layout,
                          int32_t* y, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (Mw == nullptr || y == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  rnsw::Geometry g;
  if (int rc = make_geometry(plan, B, H, W, 1, K, pad, layout, &g)) return rc;
  cudaError_t e = rnsw::launch_output_transform(plan->host, g, static_cast<const int16_t*>(Mw), y, nullptr,
                                                (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "output_transform");
}

int rnsw_output_residues(const rnsw_plan* plan, const void* Mw, int64_t P, int K, int16_t* y_res, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (Mw == nullptr || y_res == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (P < 1 || K < 1) return fail(RNSW_ERR_SHAPE, "bad shape");
  const PlanDevice& d = plan->host.dev;
  rnsw::Geometry g{};
  g.B = 1;
  g.K = K;
  g.Kp = (int)round_up(K, 16);
  g.P = P;
  g.th = 1;
  g.tw = (int)P;  // one row of tiles: only p matters for the residue view
  g.Ho = d.m_out;
  g.Wo = (int)(P * d.m_out);
  cudaError_t e = rnsw::launch_output_transform(plan->host, g, static_cast<const int16_t*>(Mw), nullptr, y_res,
                                                (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "output_residues");
}

namespace {
// K1 + K3 of a whole-layer call: the tensor-core GEMM path, or for C <= 4
// the compact transform + CUDA-core product (smallc.cu), into Mw.
// planar: leave Mw8 (the byte planes the tcgen05 output transform reads).
// ev (optional): events recorded after K1 (ev[0]) and after K3 (ev[1]).
int transform_and_product(const rnsw_plan* plan, const rnsw::Geometry& g, const int8_t* x, const void* U, int8_t* V,
                          int16_t* Mw, cudaStream_t s, bool planar = false, cudaEvent_t* ev = nullptr) {
  cudaError_t e;
  if (rnsw::smallc_ok(plan->host.dev, g) && !rnsw::force_generic()) {
    int16_t* V16 = reinterpret_cast<int16_t*>(V);
    e = rnsw::launch_input_transform_compact(plan->host, g, x, V16, s);
    if (e != cudaSuccess) return cuda_fail(e, "input_transform_compact");
    if (ev) cudaEventRecord(ev[0], s);
    e = rnsw::launch_smallc_product(plan->host, g, V16, static_cast<const int8_t*>(U), Mw, s, planar);
    if (ev) cudaEventRecord(ev[1], s);
    return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "smallc_product");
  }
  // whole-layer path: the GEMM accepts any representative of V (relaxed K1)
  e = rnsw::launch_input_transform(plan->host, g, x, V, s, true);
  if (e != cudaSuccess) return cuda_fail(e, "input_transform");
  if (ev) cudaEventRecord(ev[0], s);
  e = rnsw::launch_winograd_gemm(plan->host, V, static_cast<const int8_t*>(U), g.P, g.Cp, g.K, g.Kp, g.bc, Mw, s,
                                 rnsw::tc_output_ok(plan->host.dev) && !rnsw::force_generic(), planar);
  if (ev) cudaEventRecord(ev[1], s);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "winograd_gemm");
}

// One whole layer: the dispatch rnsw_conv_forward runs (and, with ev, the
// same chain with events between the stages: rnsw_conv_forward_timed).
int conv_forward_impl(const rnsw_plan* plan, const rnsw::Geometry& g, const int8_t* x, const void* U, int32_t* y,
                      void* workspace, size_t workspace_bytes, cudaStream_t s, cudaEvent_t* ev) {
  const PlanDevice& d = plan->host.dev;
  const size_t vb = round_up(v_bytes(d, g.P, g.Cp), 256);
  const size_t mb = m_bytes(d, g.P, g.Kp);
  if (workspace_bytes < vb + mb) return fail(RNSW_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, vb + mb);
  int8_t* V = static_cast<int8_t*>(workspace);
  int16_t* Mw = reinterpret_cast<int16_t*>(static_cast<uint8_t*>(workspace) + vb);
  if (rnsw::kron_output_ok(plan->host, g, 0)) {
    if (int rc = transform_and_product(plan, g, x, U, V, Mw, s, true, ev)) return rc;
    cudaError_t e = rnsw::launch_output_transform_kron(plan->host, g, reinterpret_cast<const uint8_t*>(Mw), y, s);
    return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "output_transform_kron");
  }
  if (rnsw::umma_output_ok(d)) {
    if (int rc = transform_and_product(plan, g, x, U, V, Mw, s, true, ev)) return rc;
    cudaError_t e = rnsw::launch_output_transform_umma(plan->host, g, reinterpret_cast<const uint8_t*>(Mw), y, s);
    return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "output_transform_umma");
  }
  if (int rc = transform_and_product(plan, g, x, U, V, Mw, s, false, ev)) return rc;
  cudaError_t e = rnsw::launch_output_transform(plan->host, g, Mw, y, nullptr, s);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "output_transform");
}
}  // namespace

int rnsw_conv_forward(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C, int K, int pad, int layout,
                      const void* U, int32_t* y, void* workspace, size_t workspace_bytes, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (x == nullptr || U == nullptr || y == nullptr || workspace == nullptr)
    return fail(RNSW_ERR_INVALID, "null buffer");
  rnsw::Geometry g;
  if (int rc = make_geometry(plan, B, H, W, C, K, pad, layout, &g)) return rc;
  return conv_forward_impl(plan, g, x, U, y, workspace, workspace_bytes, (cudaStream_t)stream, nullptr);
}

int rnsw_conv_forward_timed(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C, int K, int pad,
                            int layout, const void* U, int32_t* y, void* workspace, size_t workspace_bytes,
                            void* stream, float* stage_ms) {
  if (int rc = check_plan(plan)) return rc;
  if (x == nullptr || U == nullptr || y == nullptr || workspace == nullptr || stage_ms == nullptr)
    return fail(RNSW_ERR_INVALID, "null buffer");
  rnsw::Geometry g;
  if (int rc = make_geometry(plan, B, H, W, C, K, pad, layout, &g)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaEventCreate(&ev[i]);
  int rc = RNSW_OK;
  if (e != cudaSuccess) {
    rc = cuda_fail(e, "cudaEventCreate");
  } else {
    cudaEventRecord(ev[0], s);
    rc = conv_forward_impl(plan, g, x, U, y, workspace, workspace_bytes, s, ev + 1);
    if (rc == RNSW_OK) {
      cudaEventRecord(ev[3], s);
      e = cudaEventSynchronize(ev[3]);
      for (int i = 0; i < 3 && e == cudaSuccess; ++i) e = cudaEventElapsedTime(&stage_ms[i], ev[i], ev[i + 1]);
      if (e != cudaSuccess) rc = cuda_fail(e, "stage timing");
    }
  }
  for (int i = 0; i < 4; ++i)
    if (ev[i]) cudaEventDestroy(ev[i]);
  return rc;
}

int rnsw_tile_decompose(const int8_t* x, int B, int H, int W, int C, int tile_m, int r, int pad, int8_t* patches,
                        size_t patches_bytes, void* stream) {
  if (x == nullptr || patches == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (B < 1 || H < 1 || W < 1 || C < 1 || tile_m < 1 || r < 1 || pad < 0)
    return fail(RNSW_ERR_SHAPE, "bad tiling geometry");
  const int Ho = H + 2 * pad - r + 1, Wo = W + 2 * pad - r + 1;
  if (Ho < 1 || Wo < 1) return fail(RNSW_ERR_SHAPE, "padded input smaller than the filter");
  const int th = (Ho + tile_m - 1) / tile_m, tw = (Wo + tile_m - 1) / tile_m, n = tile_m + r - 1;
  const size_t need = (size_t)B * th * tw * n * n * C;
  if (patches_bytes < need) return fail(RNSW_ERR_WORKSPACE, "patch buffer %zu < %zu bytes", patches_bytes, need);
  cudaError_t e = rnsw::launch_tile_decompose(x, B, H, W, C, tile_m, r, pad, patches, (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "tile_decompose");
}

namespace {
int requant_impl(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C, int K, int pad, const void* U,
                 int shift, int pool, int8_t* out, void* workspace, size_t workspace_bytes, cudaStream_t s,
                 cudaEvent_t* ev) {
  if (int rc = check_plan(plan)) return rc;
  if (x == nullptr || U == nullptr || out == nullptr || workspace == nullptr)
    return fail(RNSW_ERR_INVALID, "null buffer");
  if (shift < 0 || shift > 31) return fail(RNSW_ERR_INVALID, "shift must be in [0, 31]");
  if (!rnsw::tc_output_ok(plan->host.dev))
    return fail(RNSW_ERR_UNSUPPORTED, "fused requantisation needs the tensor-core transform path (moduli < 4500)");
  if ((K & 3) != 0) return fail(RNSW_ERR_UNSUPPORTED, "fused requantisation needs K %% 4 == 0");
  if ((reinterpret_cast<uintptr_t>(out) & 3) != 0) return fail(RNSW_ERR_INVALID, "out must be 4-byte aligned");
  if (pool && (plan->host.dev.m_out & 1)) return fail(RNSW_ERR_UNSUPPORTED, "fused 2x2 pooling needs an even tile_m");
  rnsw::Geometry g;
  if (int rc = make_geometry(plan, B, H, W, C, K, pad, RNSW_LAYOUT_NHWC, &g)) return rc;
  if (pool && (g.Ho < 2 || g.Wo < 2)) return fail(RNSW_ERR_SHAPE, "pooling needs Ho, Wo >= 2");
  const PlanDevice& d = plan->host.dev;
  const size_t vb = round_up(v_bytes(d, g.P, g.Cp), 256);
  const size_t mb = m_bytes(d, g.P, g.Kp);
  if (workspace_bytes < vb + mb) return fail(RNSW_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, vb + mb);
  int8_t* V = static_cast<int8_t*>(workspace);
  int16_t* Mw = reinterpret_cast<int16_t*>(static_cast<uint8_t*>(workspace) + vb);
  if (rnsw::kron_output_ok(plan->host, g, pool ? 3 : 1)) {
    if (int rc = transform_and_product(plan, g, x, U, V, Mw, s, true, ev)) return rc;
    cudaError_t e = rnsw::launch_output_transform_kron(plan->host, g, reinterpret_cast<const uint8_t*>(Mw), nullptr, s,
                                                       out, shift, pool);
    return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "output_transform_requant_kron");
  }
  if (rnsw::umma_output_ok(d)) {
    if (int rc = transform_and_product(plan, g, x, U, V, Mw, s, true, ev)) return rc;
    cudaError_t e = rnsw::launch_output_transform_umma(plan->host, g, reinterpret_cast<const uint8_t*>(Mw), nullptr, s,
                                                       out, shift, pool);
    return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "output_transform_requant_umma");
  }
  if (int rc = transform_and_product(plan, g, x, U, V, Mw, s, false, ev)) return rc;
  cudaError_t e = rnsw::launch_output_transform_tc(plan->host, g, Mw, nullptr, nullptr, s, out, shift, pool);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "output_transform_requant");
}
}  // namespace

int rnsw_conv_forward_requant(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C, int K, int pad,
                              const void* U, int shift, int pool, int8_t* out, void* workspace,
                              size_t workspace_bytes, void* stream) {
  return requant_impl(plan, x, B, H, W, C, K, pad, U, shift, pool, out, workspace, workspace_bytes,
                      (cudaStream_t)stream, nullptr);
}

int rnsw_conv_forward_requant_ev(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C, int K, int pad,
                                 const void* U, int shift, int pool, int8_t* out, void* workspace,
                                 size_t workspace_bytes, void* stream, void* const* events) {
  if (events == nullptr || events[0] == nullptr || events[1] == nullptr) return fail(RNSW_ERR_INVALID, "null event");
  cudaEvent_t ev[2] = {(cudaEvent_t)events[0], (cudaEvent_t)events[1]};
  return requant_impl(plan, x, B, H, W, C, K, pad, U, shift, pool, out, workspace, workspace_bytes,
                      (cudaStream_t)stream, ev);
}

int rnsw_conv_forward_ev(const rnsw_plan* plan, const int8_t* x, int B, int H, int W, int C, int K, int pad,
                         int layout, const void* U, int32_t* y, void* workspace, size_t workspace_bytes, void* stream,
                         void* const* events) {
  if (int rc = check_plan(plan)) return rc;
  if (x == nullptr || U == nullptr || y == nullptr || workspace == nullptr)
    return fail(RNSW_ERR_INVALID, "null buffer");
  if (events == nullptr || events[0] == nullptr || events[1] == nullptr) return fail(RNSW_ERR_INVALID, "null event");
  rnsw::Geometry g;
  if (int rc = make_geometry(plan, B, H, W, C, K, pad, layout, &g)) return rc;
  cudaEvent_t ev[2] = {(cudaEvent_t)events[0], (cudaEvent_t)events[1]};
  return conv_forward_impl(plan, g, x, U, y, workspace, workspace_bytes, (cudaStream_t)stream, ev);
}

int rnsw_output_transform_requant(const rnsw_plan* plan, const void* Mw, int B, int H, int W, int K, int pad,
                                  int shift, int pool, int8_t* out, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (Mw == nullptr || out == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (!rnsw::tc_output_ok(plan->host.dev) || (K & 3) != 0 || (pool && (plan->host.dev.m_out & 1)))
    return fail(RNSW_ERR_UNSUPPORTED, "fused requantisation not available for this plan/geometry");
  if ((reinterpret_cast<uintptr_t>(out) & 3) != 0) return fail(RNSW_ERR_INVALID, "out must be 4-byte aligned");
  rnsw::Geometry g;
  if (int rc = make_geometry(plan, B, H, W, 1, K, pad, RNSW_LAYOUT_NHWC, &g)) return rc;
  cudaError_t e = rnsw::launch_output_transform_tc(plan->host, g, static_cast<const int16_t*>(Mw), nullptr, nullptr,
                                                   (cudaStream_t)stream, out, shift, pool);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "output_transform_requant");
}

int rnsw_mw8_supported(const rnsw_plan* plan) {
  if (check_plan(plan)) return 0;
  return rnsw::umma_output_ok(plan->host.dev) ? 1 : 0;
}

int rnsw_small_channel_product_mw8(const rnsw_plan* plan, const void* V16, const void* U, int64_t P, int C, int K,
                                   void* Mw8, size_t Mw8_bytes, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (!rnsw::umma_output_ok(plan->host.dev)) return fail(RNSW_ERR_UNSUPPORTED, "plan does not use the Mw8 layout");
  if (V16 == nullptr || U == nullptr || Mw8 == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (P < 1 || P > 2147483647LL || C < 1 || K < 1) return fail(RNSW_ERR_SHAPE, "bad product shape P=%lld C=%d K=%d",
                                                          (long long)P, C, K);
  rnsw::Geometry g{};
  g.P = P;
  g.C = C;
  g.K = K;
  g.Cp = padded_channels(C);
  g.Kp = (int)round_up(K, 16);
  if (!rnsw::smallc_ok(plan->host.dev, g))
    return fail(RNSW_ERR_UNSUPPORTED, "small-channel product needs C <= 4 (C=%d)", C);
  if (Mw8_bytes < m_bytes(plan->host.dev, P, g.Kp)) return fail(RNSW_ERR_WORKSPACE, "Mw8 buffer too small");
  cudaError_t e = rnsw::launch_smallc_product(plan->host, g, static_cast<const int16_t*>(V16),
                                              static_cast<const int8_t*>(U), static_cast<int16_t*>(Mw8),
                                              (cudaStream_t)stream, true);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "small_channel_product_mw8");
}

int rnsw_winograd_gemm_mw8(const rnsw_plan* plan, const void* V, const void* U, int64_t P, int C, int K, void* Mw8,
                           size_t Mw8_bytes, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (!rnsw::umma_output_ok(plan->host.dev)) return fail(RNSW_ERR_UNSUPPORTED, "plan does not use the Mw8 layout");
  if (V == nullptr || U == nullptr || Mw8 == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (P < 1 || C < 1 || K < 1) return fail(RNSW_ERR_SHAPE, "bad GEMM shape P=%lld C=%d K=%d", (long long)P, C, K);
  if ((int64_t)C * 128 * 128 > 2147483647LL) return fail(RNSW_ERR_OVERFLOW, "C=%d can overflow int32", C);
  const int Cp = padded_channels(C), Kp = (int)round_up(K, 16);
  if (Mw8_bytes < m_bytes(plan->host.dev, P, Kp)) return fail(RNSW_ERR_WORKSPACE, "Mw8 buffer too small");
  cudaError_t e = rnsw::launch_winograd_gemm(plan->host, static_cast<const int8_t*>(V), static_cast<const int8_t*>(U),
                                             P, Cp, K, Kp, Cp < 128 ? Cp : 128, static_cast<int16_t*>(Mw8),
                                             (cudaStream_t)stream, true, true);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "winograd_gemm_mw8");
}

int rnsw_output_transform_mw8(const rnsw_plan* plan, const void* Mw8, int B, int H, int W, int K, int pad, int layout,
                              int32_t* y, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (!rnsw::umma_output_ok(plan->host.dev)) return fail(RNSW_ERR_UNSUPPORTED, "plan does not use the Mw8 layout");
  if (Mw8 == nullptr || y == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  rnsw::Geometry g;
  if (int rc = make_geometry(plan, B, H, W, 1, K, pad, layout, &g)) return rc;
  cudaError_t e = rnsw::launch_output_transform_umma(plan->host, g, static_cast<const uint8_t*>(Mw8), y,
                                                     (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "output_transform_mw8");
}

int rnsw_output_transform_requant_mw8(const rnsw_plan* plan, const void* Mw8, int B, int H, int W, int K, int pad,
                                      int shift, int pool, int8_t* out, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (!rnsw::umma_output_ok(plan->host.dev)) return fail(RNSW_ERR_UNSUPPORTED, "plan does not use the Mw8 layout");
  if (Mw8 == nullptr || out == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (shift < 0 || shift > 31) return fail(RNSW_ERR_INVALID, "shift must be in [0, 31]");
  if ((K & 3) != 0) return fail(RNSW_ERR_UNSUPPORTED, "fused requantisation needs K %% 4 == 0");
  if ((reinterpret_cast<uintptr_t>(out) & 3) != 0) return fail(RNSW_ERR_INVALID, "out must be 4-byte aligned");
  rnsw::Geometry g;
  if (int rc = make_geometry(plan, B, H, W, 1, K, pad, RNSW_LAYOUT_NHWC, &g)) return rc;
  if (pool && (g.Ho < 2 || g.Wo < 2)) return fail(RNSW_ERR_SHAPE, "pooling needs Ho, Wo >= 2");
  cudaError_t e = rnsw::launch_output_transform_umma(plan->host, g, static_cast<const uint8_t*>(Mw8), nullptr,
                                                     (cudaStream_t)stream, out, shift, pool);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "output_transform_requant_mw8");
}

size_t rnsw_direct_weight_bytes(int R, int C, int K) {
  if (R < 1 || C < 1 || K < 1) return 0;
  return rnsw::direct_weight_bytes(R, C, K);
}

int rnsw_direct_pack_weights(const int8_t* w, int R, int C, int K, int layout, void* w2, size_t w2_bytes,
                             void* stream) {
  if (w == nullptr || w2 == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (R < 1 || C < 1 || K < 1) return fail(RNSW_ERR_SHAPE, "bad filter shape");
  if (layout != RNSW_LAYOUT_NHWC && layout != RNSW_LAYOUT_NCHW) return fail(RNSW_ERR_INVALID, "bad layout %d", layout);
  if (w2_bytes < rnsw::direct_weight_bytes(R, C, K)) return fail(RNSW_ERR_WORKSPACE, "packed weight buffer too small");
  cudaError_t e = rnsw::launch_pack_weights(w, R, C, K, layout, static_cast<int8_t*>(w2), (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "direct_pack_weights");
}

int rnsw_direct_conv(const int8_t* x, int B, int H, int W, int C, const void* w2, int K, int R, int pad, int stride,
                     int32_t* y, void* stream) {
  if (x == nullptr || w2 == nullptr || y == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (B < 1 || H < 1 || W < 1 || C < 1 || K < 1 || R < 1 || pad < 0 || stride < 1)
    return fail(RNSW_ERR_SHAPE, "bad direct conv geometry");
  if (C % 16 != 0) return fail(RNSW_ERR_UNSUPPORTED, "direct conv needs C %% 16 == 0 (TMA row alignment), got %d", C);
  if ((int64_t)R * R * C * 128 * 128 > 2147483647LL)
    return fail(RNSW_ERR_OVERFLOW, "R*R*C = %d can overflow the int32 accumulator", R * R * C);
  const int Ho = (H + 2 * pad - R) / stride + 1, Wo = (W + 2 * pad - R) / stride + 1;
  if (H + 2 * pad < R || W + 2 * pad < R || Ho < 1 || Wo < 1) return fail(RNSW_ERR_SHAPE, "padded input smaller than the filter");
  if (stride > 16) return fail(RNSW_ERR_UNSUPPORTED, "stride %d too large for the TMA box", stride);
  cudaError_t e = rnsw::launch_direct_conv(x, B, H, W, C, static_cast<const int8_t*>(w2), K, R, pad, stride, y,
                                           (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "direct_conv");
}

int rnsw_mrc_reconstruct(const rnsw_plan* plan, const int16_t* residues, int64_t count, int64_t* out, void* stream) {
  if (int rc = check_plan(plan)) return rc;
  if (residues == nullptr || out == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (count < 0) return fail(RNSW_ERR_SHAPE, "negative count");
  if (count == 0) return RNSW_OK;
  cudaError_t e = rnsw::launch_mrc(plan->host, residues, count, out, (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "mrc_reconstruct");
}

int rnsw_requant_pool(const int32_t* y, int B, int H, int W, int C, int shift, int pool, int8_t* out, void* stream) {
  if (y == nullptr || out == nullptr) return fail(RNSW_ERR_INVALID, "null buffer");
  if (B < 1 || H < 1 || W < 1 || C < 1 || shift < 0 || shift > 31) return fail(RNSW_ERR_SHAPE, "bad requant shape");
  if (pool && (H < 2 || W < 2)) return fail(RNSW_ERR_SHAPE, "pooling needs H, W >= 2");
  cudaError_t e = rnsw::launch_requant_pool(y, B, H, W, C, shift, pool, out, (cudaStream_t)stream);
  return e == cudaSuccess ? RNSW_OK : cuda_fail(e, "requant_pool");
}

}  // extern "C"
