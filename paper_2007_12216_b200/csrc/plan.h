// Internal plan layout shared by the host entry points and the kernels.
#pragma once
#include <cstdint>

#define RNSW_MAX_RES 4   // residues per system
#define RNSW_MAX_N 24    // tile side N = M + R - 1 (tensor-core transforms: N <= 16)
#define RNSW_MAX_R 8     // filter side

// Constant tables one residue needs on the device, as int32 so kernels can
// load them straight into shared memory.
struct ResidueTables {
  int32_t modulus;
  int32_t planes;      // 1: |v| <= 127 fits s8; 2: balanced hi/lo s8 limbs
  int32_t plane_base;  // first limb-plane index of this residue in V
  int32_t uplanes;     // filter-bank planes: 1, or 4 = {U lo, U hi, U' lo, U' hi} with U' = 256*U mod m
  int32_t uplane_base; // first plane of this residue in the filter bank U
  float inv_m;         // 1.0f / modulus
  int32_t r_256;       // 256 mod m (symmetric)
  int32_t r_65536;     // 65536 mod m (symmetric)
  // Exact division-free symmetric reduction for |x| < 2^28 (see red_fast in
  // common.cuh): n = x + red_off in [0, 2^30), floor(n/m) = umulhi(n, red_mul) >> red_shift.
  uint32_t red_mul;
  int32_t red_shift;
  int32_t red_off;
  // (uint32)(-m), stored rather than derived so the compiler keeps
  // q*negm + n as one IMAD instead of negating q and multiplying by m
  uint32_t red_negm;
  int32_t half;        // (m - 1) / 2
  int32_t at[RNSW_MAX_N * RNSW_MAX_N];  // AT (M x N), row-major, stride N
  int32_t bt[RNSW_MAX_N * RNSW_MAX_N];  // BT (N x N)
  int32_t g[RNSW_MAX_N * RNSW_MAX_R];   // G  (N x R), stride R
};

struct PlanDevice {
  int32_t m_out;  // M (outputs per tile side)
  int32_t r;      // R
  int32_t n;      // N = M + R - 1
  int32_t n_res;
  int32_t n_planes;  // total limb planes over all residues (V)
  int32_t n_uplanes; // total filter-bank planes over all residues (U)
  int32_t fast;      // 1: tensor-core transform kernels apply (all m < 4500, D < 2^31)
  int32_t z3;        // 1: K4 pass-1 sums of every 16-bit residue fit 24-bit signed (three-limb pass 2)
  int64_t dynamic_range;
  int64_t signed_bound;
  int64_t mrc_inv[RNSW_MAX_RES][RNSW_MAX_RES];  // m_i^-1 mod m_j, i < j
  // Expanded mixed-radix weights: digit d_j = y_j*W[j][0] - sum_{i<j} d_i*W[j][i]
  // (mod m_j), W[j][i] = prod_{k=i}^{j-1} m_k^-1 mod m_j, in [0, m_j).
  int32_t mrc_w[RNSW_MAX_RES][RNSW_MAX_RES];
  ResidueTables res[RNSW_MAX_RES];
  // Constant B operands of the tcgen05 output transform (output_umma.cu),
  // built on the host for F(14x14,3x3) plans over two 16-bit residues:
  // B1[res] (1 KB each) then B2[res][step] (1 KB each), 32-byte rows,
  // 32B-swizzled s8.
  alignas(16) uint8_t umma_b[6144];
};
