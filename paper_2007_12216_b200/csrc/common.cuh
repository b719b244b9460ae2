// Shared device helpers for the RNS-Winograd sm_100a kernels:
//  * exact symmetric modular reduction (no integer division),
//  * limb split of 16-bit residues into two s8 planes,
//  * thin inline-PTX wrappers for mbarrier / TMA / tcgen05.
#pragma once
#include <cstdint>
#include <utility>

#include <cuda_runtime.h>

#include "plan.h"

#define RNSW_DEV __device__ __forceinline__

// ---- programmatic dependent launch (PDL) ----
// Every kernel of the layer chain lets its successor launch early
// (pdl_trigger, first thing) and waits for its predecessor's results
// (pdl_wait) after a prologue that touches only constants (TMEM allocation,
// barrier setup, plan / operator tables), so a successor's prologue overlaps
// its predecessor's tail.  Without the launch attribute both are no-ops.
RNSW_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
RNSW_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Host: launch with the PDL attribute (unless RNSW_PDL=0) and an optional
// cluster dimension.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster,
                             Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = (unsigned)cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// Modular arithmetic.  Residues are kept in the symmetric range
// [-(m-1)/2, (m-1)/2] of an odd modulus m (rw/residue.py:25-33); every stage
// of the reference reduces into that range after each product
// (rw/kernel.py:21-30, rw/gemm.py:91-97).

// Exact symmetric reduction of any int32 x.  Two float quotient estimates:
// the first brings |x| below ~2^9 + m, the second is then exact because x/m
// can never sit on a .5 tie for odd m.
RNSW_DEV int32_t sym_mod(int32_t x, int32_t m, float inv_m) {
  int32_t q = __float2int_rn(__int2float_rn(x) * inv_m);
  int32_t r = x - q * m;
  q = __float2int_rn(__int2float_rn(r) * inv_m);
  r -= q * m;
  return r;
}

// Symmetric reduction for |x| < 2^22 using only FMA/ALU-pipe float ops.
// x + 1.5*2^23 is exact in fp32 for |x| < 2^22, rint via the same magic.
// The quotient estimate can be off by one near a half-way point, so a
// final compare/select folds r back into [-(m-1)/2, (m-1)/2].
RNSW_DEV int32_t sym_mod_small(int32_t x, float m, float inv_m) {
  const float magic = 12582912.0f;  // 1.5 * 2^23
  float f = __int_as_float(x + 0x4B400000) - magic;
  float q = __fadd_rn(__fmul_rn(f, inv_m), magic) - magic;
  float r = __fmaf_rn(-q, m, f);
  const float half = 0.5f * m;
  r = r > half ? r - m : r;
  r = r < -half ? r + m : r;
  return __float_as_int(r + magic) - 0x4B400000;
}

// Exact symmetric reduction for |x| < 2^28 without division: with
// s = floor(log2 m), mul = ceil(2^(32+s) / m) and n = x + h + m*ceil(2^28/m)
// in [0, 2^30), floor(n/m) = umulhi(n, mul) >> s exactly (the rounding error
// n*(mul*m - 2^(32+s)) / (m*2^(32+s)) stays below 1/(2m)).  Then
// n - floor(n/m)*m - h is x's representative in [-h, h].
struct FastMod {
  uint32_t mul;
  int32_t shift, off, m, h;
  uint32_t negm;  // (uint32)(-m): n - q*m as one IMAD q*negm + n
};

RNSW_DEV FastMod fast_mod_of(const ResidueTables& t) {
  return FastMod{t.red_mul, t.red_shift, t.red_off, t.modulus, t.half, t.red_negm};
}

RNSW_DEV int32_t red_fast(int32_t x, const FastMod& f) {
  const uint32_t n = (uint32_t)(x + f.off);
  const uint32_t q = __umulhi(n, f.mul) >> f.shift;
  return (int32_t)(q * f.negm + n) - f.h;
}

// Non-negative representative in [0, m) of n - f.off + (f.off - f.h)... i.e.
// red_pos_biased(n) = (x mod m) when n = x + m*L with L = ceil(2^28/m) (see
// pos_bias).  The bias can be pre-loaded into an MMA accumulator so the
// reduction is IMAD.HI + SHF + IMAD only.
RNSW_DEV int32_t pos_bias(const FastMod& f) { return f.off - f.h; }

RNSW_DEV int32_t red_pos_biased(int32_t n, const FastMod& f) {
  const uint32_t q = __umulhi((uint32_t)n, f.mul) >> f.shift;
  return (int32_t)(q * f.negm + (uint32_t)n);
}

RNSW_DEV int32_t red_pos(int32_t x, const FastMod& f) { return red_pos_biased(x + pos_bias(f), f); }

// Same result as red_pos_biased, computed as n - q*m (IMAD with a negated
// quotient); ptxas schedules the output transform better with this form.
RNSW_DEV int32_t red_pos_biased_sub(int32_t n, const FastMod& f) {
  const uint32_t q = __umulhi((uint32_t)n, f.mul) >> f.shift;
  return (int32_t)((uint32_t)n - q * (uint32_t)f.m);
}

// Exact unsigned division by a runtime constant d for n < 2^31:
// s = floor(log2 d), mul = ceil(2^(32+s) / d) as a 33-bit value (mul_hi:mul_lo);
// floor(n/d) = (umulhi(n, mul_lo) + (mul_hi ? n : 0)) >> s.  The rounding
// error n*(mul*d - 2^(32+s)) / (d*2^(32+s)) < n / 2^(32+s) < 1/d.
struct FastDiv {
  uint32_t mul_lo, mul_hi, shift, d;
};

inline FastDiv make_fastdiv(uint32_t d) {
  uint32_t s = 0;
  while ((2ull << s) <= d) ++s;
  const unsigned long long num = 1ull << (32 + s);
  const unsigned long long mul = (num + d - 1) / d;  // <= 2^32
  return FastDiv{(uint32_t)mul, (uint32_t)(mul >> 32), s, d};
}

RNSW_DEV uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return (__umulhi(n, f.mul_lo) + (f.mul_hi ? n : 0u)) >> f.shift;
}

// 64-bit exact symmetric reduction (used for the mixed-radix digits).
RNSW_DEV int64_t sym_mod64(int64_t x, int64_t m) {
  int64_t r = x % m;
  if (r > (m - 1) / 2) r -= m;
  if (r < -(m - 1) / 2) r += m;
  return r;
}

// Balanced two-limb split of a residue v with |v| <= 16383:
// v = 256*hi + lo, lo = sign-extended low byte in [-128,127], hi in [-64,64].
RNSW_DEV void split_limbs(int32_t v, int8_t& lo, int8_t& hi) {
  lo = (int8_t)(v & 0xFF);
  hi = (int8_t)((v - (int32_t)lo) >> 8);
}

// ---------------------------------------------------------------------------
// PTX wrappers (sm_100a).

RNSW_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

RNSW_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

RNSW_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

RNSW_DEV void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

RNSW_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

RNSW_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

RNSW_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t"
      "}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// Same wait with a suspend-time hint: the thread sleeps in try_wait (up to
// `ns` nanoseconds per attempt, woken when the phase completes) instead of
// re-issuing it in a tight loop -- waiting epilogue warps then leave their
// issue slots to the warps that have work.
RNSW_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns = 20000) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITS_%=;\n\t"
      "}" ::"r"(addr),
      "r"(parity), "r"(ns)
      : "memory");
}

RNSW_DEV void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}

RNSW_DEV void tma_load_3d(void* dst, const void* desc, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

RNSW_DEV void tma_load_5d(void* dst, const void* desc, uint64_t* bar, int c0, int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

RNSW_DEV void tma_load_4d(void* dst, const void* desc, uint64_t* bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// Bulk tensor store smem -> global (bulk-group completion).
RNSW_DEV void tma_store_2d(const void* desc, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(desc)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
RNSW_DEV void tma_store_3d(const void* desc, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(desc)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
RNSW_DEV void tma_store_4d(const void* desc, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(desc)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
RNSW_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N bulk groups still read their shared-memory source
template <int N>
RNSW_DEV void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
RNSW_DEV void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
RNSW_DEV void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// The same load delivered to every CTA of the cluster in ctaMask (same smem
// offset, each CTA's mbarrier at the same offset receives the bytes).
RNSW_DEV void tma_load_3d_mc(void* dst, const void* desc, uint64_t* bar, int c0, int c1, int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}

RNSW_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// Shared-memory address of the same variable in CTA `rank` of the cluster
// (distributed shared memory).
RNSW_DEV uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// Arrive (release, cluster scope) on an mbarrier of another CTA of the cluster.
RNSW_DEV void mbar_arrive_cluster(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
// Arrive on an mbarrier of another CTA of the cluster with the default
// (.release.cta) semantics, as CUTLASS's ClusterBarrier does: enough for
// handing TMEM back across a CTA pair (the tcgen05 fences order the TMEM
// accesses), without the cluster-scope release / acquire cost.
RNSW_DEV void mbar_arrive_remote(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
// Wait (acquire, cluster scope): the arrivals may come from other CTAs.
RNSW_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t"
      "}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
// 16-byte store into another CTA's shared memory through the async proxy,
// counted as 16 transaction bytes on that CTA's mbarrier (remote_bar): the
// consumer waits on its own barrier, no cluster-scope fences.
RNSW_DEV void st_async_v4(uint32_t remote_addr, uint4 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   remote_addr),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(remote_bar)
               : "memory");
}

// 16-byte load from another CTA's shared memory.
RNSW_DEV uint4 ld_dsmem_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

// Full cluster barrier (all threads of all CTAs), release/acquire.
RNSW_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

RNSW_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
RNSW_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <uint32_t kCols>
RNSW_DEV void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

template <uint32_t kCols>
RNSW_DEV void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}

// ---- CTA pairs (cta_group::2): one MMA spans the TMEM of both CTAs of a
// 2-CTA cluster (M = 256, each CTA's TMEM holds its 128 rows; B is split
// along N, each CTA's shared memory holding its N/2 columns at the same
// offset).  Only the even CTA issues; loads of both CTAs complete on its
// mbarrier; commits multicast to both.
template <uint32_t kCols>
RNSW_DEV void tmem_alloc_2sm(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <uint32_t kCols>
RNSW_DEV void tmem_dealloc_2sm(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
// 4-D tensor load into this CTA's shared memory whose transaction bytes
// complete on the pair leader's mbarrier (leader_bar: shared::cluster address)
RNSW_DEV void tma_load_4d_2sm(void* dst, const void* desc, uint32_t leader_bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// A from tensor memory, B from shared memory, across the CTA pair (warp-collective issue)
RNSW_DEV void mma_i8_ts_warp_2sm(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// 3-D tensor load into this CTA's shared memory, bytes completing on the
// pair leader's mbarrier
RNSW_DEV void tma_load_3d_2sm(void* dst, const void* desc, uint32_t leader_bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// both operands from shared memory, across the CTA pair, one issuing thread
RNSW_DEV void mma_i8_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// ... warp-collective (one elected lane; operands stay in uniform registers)
RNSW_DEV void mma_i8_warp_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                              uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// one issuing thread: commit the pair's prior MMAs to the mbarrier at this offset in both CTAs
RNSW_DEV void mma_commit_2sm(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
// commit the pair's prior MMAs to the mbarrier at this offset in both CTAs
RNSW_DEV void mma_commit_warp_2sm(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

// D[tmem] (+)= A[smem] * B[smem], s8 x s8 -> s32, one elected thread.
RNSW_DEV void mma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Warp-collective variants: every lane of the (converged) warp executes them
// with the same operands, one elected lane issues.  The operands then stay in
// uniform registers (no per-lane uniformisation loop around each MMA).
RNSW_DEV void mma_i8_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// A from tensor memory (K-major, 4 int8 per 32-bit column), B from shared memory.
RNSW_DEV void mma_i8_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// Issue f(0) .. f(n-1), n <= 8, as a fully unrolled, branch-free sequence.
// A runtime bound tested between consecutive tcgen05.mma instructions
// (`#pragma unroll` + `if (ks < n)`) measured 50 instead of 32 cycles per
// M=128 N=64 K=32 MMA on B200 (tools/k1_mma_probe.cu, K1 issue timing).
template <int kN, typename F>
RNSW_DEV void unrolled_steps(F& f) {
#pragma unroll
  for (int i = 0; i < kN; ++i) f(i);
}
template <typename F>
RNSW_DEV void for_ksteps(int n, F&& f) {
  switch (n) {
    case 8: unrolled_steps<8>(f); break;
    case 7: unrolled_steps<7>(f); break;
    case 6: unrolled_steps<6>(f); break;
    case 5: unrolled_steps<5>(f); break;
    case 4: unrolled_steps<4>(f); break;
    case 3: unrolled_steps<3>(f); break;
    case 2: unrolled_steps<2>(f); break;
    case 1: unrolled_steps<1>(f); break;
    default:
      for (int i = 0; i < n; ++i) f(i);
  }
}

RNSW_DEV void mma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05.mma complete.
// Arrive on the mbarrier at this offset in every CTA of ctaMask once all
// previously issued MMAs of this thread have completed.
RNSW_DEV void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

RNSW_DEV void mma_commit_warp_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

RNSW_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread.
RNSW_DEV void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// 32 lanes x 32 bit, 8 consecutive columns per thread.
RNSW_DEV void tmem_ld8(uint32_t taddr, int32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

RNSW_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 bit: the same value into 16 consecutive columns of this
// thread's lane (accumulator bias initialisation).
RNSW_DEV void tmem_st16_fill(uint32_t taddr, uint32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
      "r"(v)
      : "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns from 16 registers.
RNSW_DEV void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
// 32 lanes x 32 bit, 8 consecutive columns from 8 registers.
RNSW_DEV void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
RNSW_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor for a K-major operand tile whose rows are
// `row_bytes` (32/64/128) wide and swizzled by the matching TMA mode.  Rows
// are grouped in 8-row core matrices (SBO = 8 * row_bytes apart).
RNSW_DEV uint64_t umma_desc_kmajor(uint32_t smem_addr, uint32_t row_bytes) {
  uint64_t layout = row_bytes == 128 ? 2ull : (row_bytes == 64 ? 4ull : 6ull);
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                                  // LBO (unused for swizzled K-major)
  d |= (uint64_t)(((8 * row_bytes) >> 4) & 0x3FFF) << 32;  // SBO
  d |= (uint64_t)1 << 46;                                  // descriptor version (sm_100)
  d |= layout << 61;
  return d;
}

// UMMA descriptor for an MN-major operand in the 128B-swizzled canonical
// layout: each K index is one 128-byte row of 128 consecutive M (or N)
// int8 elements, 8-row groups 1024 bytes apart (SBO); M = 128 is a single
// atom wide, so LBO is unused.
RNSW_DEV uint64_t umma_desc_mn_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                   // LBO (unused: one MN atom)
  d |= (uint64_t)(1024 >> 4) << 32;         // SBO: next 8 K rows
  d |= (uint64_t)1 << 46;                   // descriptor version (sm_100)
  d |= 2ull << 61;                          // SWIZZLE_128B
  return d;
}

// ... in the 32B-swizzled canonical layout: each K index is one 32-byte row
// of 32 consecutive M elements, 8-row K groups 256 bytes apart (SBO), the
// next 32 M elements (MN atom) `atom_stride` bytes further (LBO).
RNSW_DEV uint64_t umma_desc_mn_sw32(uint32_t smem_addr, uint32_t atom_stride) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((atom_stride >> 4) & 0x3FFF) << 16;  // LBO: next MN atom
  d |= (uint64_t)(256 >> 4) << 32;                      // SBO: next 8 K rows
  d |= (uint64_t)1 << 46;
  d |= 6ull << 61;                                      // SWIZZLE_32B
  return d;
}

// ... in the 64B-swizzled canonical layout: each K index is one 64-byte row
// of 64 consecutive M (or N) elements, 8-row K groups 512 bytes apart (SBO),
// the next 64 M elements (MN atom) `atom_stride` bytes further (LBO).
RNSW_DEV uint64_t umma_desc_mn_sw64(uint32_t smem_addr, uint32_t atom_stride) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((atom_stride >> 4) & 0x3FFF) << 16;  // LBO: next MN atom
  d |= (uint64_t)(512 >> 4) << 32;                      // SBO: next 8 K rows
  d |= (uint64_t)1 << 46;
  d |= 4ull << 61;                                      // SWIZZLE_64B
  return d;
}

// Byte offset of element (row, col) of a dense array of 32-byte rows under
// the 32B swizzle (16-byte chunk bit 4 ^= address bit 7).
__host__ __device__ constexpr uint32_t swz32(uint32_t off) { return off ^ (((off >> 7) & 1u) << 4); }
// ... of 128-byte rows under the 128B swizzle (chunk ^= row & 7).
__host__ __device__ constexpr uint32_t swz128(uint32_t off) { return off ^ (((off >> 7) & 7u) << 4); }

// Instruction descriptor for kind::i8 with explicit operand signedness and
// majorness (a_mn / b_mn: MN-major operand).
__host__ __device__ constexpr uint32_t idesc_i8x(uint32_t m, uint32_t n, bool a_signed, bool b_signed, bool a_mn,
                                                 bool b_mn) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

// Instruction descriptor: s8 x s8 -> s32, both K-major, M x N tile.
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t m, uint32_t n) {
  return (2u << 4)             // D format: S32
         | (1u << 7)           // A: signed 8-bit
         | (1u << 10)          // B: signed 8-bit
         | ((n >> 3) << 17)    // N / 8
         | ((m >> 4) << 24);   // M / 16
}

// ---------------------------------------------------------------------------
// Warp-level int8 tensor-core MMA (mma.sync m16n8k16) for the small,
// register-resident Winograd transforms.  Fragment ownership (g = lane/4,
// t = lane%4): A rows g / g+8, k = 4t..4t+3; B k = 4t..4t+3, column g;
// C rows g (c0,c1) / g+8 (c2,c3), columns 2t, 2t+1.

RNSW_DEV void imma_ss(int32_t (&c)[4], uint32_t a0, uint32_t a1, uint32_t b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(b));
}

RNSW_DEV void imma_us(int32_t (&c)[4], uint32_t a0, uint32_t a1, uint32_t b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(b));
}

RNSW_DEV void imma_su(int32_t (&c)[4], uint32_t a0, uint32_t a1, uint32_t b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(b));
}

// Low bytes of four int32 values packed little-endian into one register.
RNSW_DEV uint32_t pack4_lo(int32_t x0, int32_t x1, int32_t x2, int32_t x3) {
  const uint32_t a = __byte_perm((uint32_t)x0, (uint32_t)x1, 0x0040);
  const uint32_t b = __byte_perm((uint32_t)x2, (uint32_t)x3, 0x0040);
  return __byte_perm(a, b, 0x5410);
}

// Byte k (0..3) of four words packed into one (pack4_lo is k = 0).
template <int k>
RNSW_DEV uint32_t pack4_byte(int32_t x0, int32_t x1, int32_t x2, int32_t x3) {
  constexpr uint32_t sel = ((4u + k) << 4) | k;
  const uint32_t a = __byte_perm((uint32_t)x0, (uint32_t)x1, sel);
  const uint32_t b = __byte_perm((uint32_t)x2, (uint32_t)x3, sel);
  return __byte_perm(a, b, 0x5410);
}

// High limb of the balanced split v = 256*hi + lo, lo in [-128, 127].
RNSW_DEV int32_t limb_hi(int32_t v) { return (v + 128) >> 8; }

