// Probe: the K1 (input_umma.cu) MMA sequence in isolation on every SM -- bias
// MMAs + 8 K-steps x 2 limbs of TS-mode M=128 N=64 K=32 per unit, B from 8
// rotating 16 KB stages -- with features toggled, to find what makes it run
// slower than the 32-cycle microbenchmark rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/k1_mma_probe tools/k1_mma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2007_12216_b200/csrc/common.cuh"

// kV bit 0: bias MMAs, bit 1: per-unit commits, bit 2: B advances over stages/K-steps,
// bit 3: both limbs share B (else the lo limb reads the next K-step), bit 4: D double buffer by unit,
// bit 5: 11 more warps spin on an mbarrier meanwhile, bit 6: per-unit tfull/tempty handshake with warp 4
template <int kV, int kEpi = 1, bool kFence = false, int kAlu = 0>
__global__ void probe_kernel(long long* out, int units) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[8];  // 0,1 commits, 2 end, 3 spin, 4-5 tfull, 6-7 tempty
  __shared__ uint32_t slot;
  __shared__ int done_flag;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) done_flag = 0;
  for (int i = threadIdx.x; i < (8 * 16384 + 4096) / 4; i += blockDim.x) {
    uint32_t r = (uint32_t)i * 2654435761u + 12345u;
    r ^= r >> 13; r *= 0x5bd1e995u; r ^= r >> 15;
    reinterpret_cast<uint32_t*>(smem)[i] = r;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 6; ++i) mbar_init(&bar[i], 1);
    mbar_init(&bar[6], kEpi);
    mbar_init(&bar[7], kEpi);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  if (warp == 0) {
    constexpr uint32_t idesc = idesc_i8x(128, 64, true, true, false, true);
    uint8_t* sB = smem;
    uint8_t* sBias = smem + 8 * 16384;
    const uint64_t db0 = umma_desc_mn_sw64(smem_u32(sB), 16);
    const uint64_t dbh = umma_desc_mn_sw64(smem_u32(sBias), 16);
    const uint64_t dbl = umma_desc_mn_sw64(smem_u32(sBias + 2048), 16);
    const uint32_t ta = tbase + 256;
    long long t0 = clock64();
    int stage = 0;
    for (int it = 0; it < units; ++it) {
      const int as = (kV & 16) ? (it & 1) : 0;
      if (kV & 64) mbar_wait(&bar[6 + (it & 1)], ((it >> 1) & 1) ^ 1);
      const uint32_t d0 = tbase + as * 128;
      const uint64_t db_stage = (kV & 4) ? db0 + (uint64_t)(stage * 1024) : db0;
      if (kV & 1) {
        mma_i8_ts_warp(d0, tbase + 384, dbh, idesc, 0u);
        mma_i8_ts_warp(d0 + 64, tbase + 384, dbl, idesc, 0u);
      }
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint64_t db = (kV & 4) ? db_stage + (uint64_t)(ks * 128) : db_stage;
        const uint32_t acc = ((kV & 1) || ks > 0) ? 1u : 0u;
        mma_i8_ts_warp(d0, ta + ks * 8, db, idesc, acc);
        mma_i8_ts_warp(d0 + 64, ta + 64 + ks * 8, (kV & 8) ? db : db + 128, idesc, acc);
      }
      if (kV & 2) {
        mma_commit_warp(&bar[0]);
        mma_commit_warp((kV & 64) ? &bar[4 + (it & 1)] : &bar[1]);
      }
      if (++stage == 8) stage = 0;
    }
    mma_commit_warp(&bar[2]);
    mbar_wait(&bar[2], 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (threadIdx.x == 0) mbar_arrive(&bar[3]);  // release the spinning warps
    if (threadIdx.x == 0) *(volatile int*)&done_flag = 1;
  } else if ((kV & 64) && warp >= 4 && warp < 4 + kEpi) {
    for (int it = 0; it < units; ++it) {  // "epilogue": wait for the unit's accumulator, hand it back
      mbar_wait(&bar[4 + (it & 1)], (it >> 1) & 1);
      tc_fence_after();
      tc_fence_before();
      if (kFence) fence_proxy_async();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&bar[6 + (it & 1)]);
    }
  } else if (kV & 32) {
    mbar_wait(&bar[3], 0);
  } else if (kAlu && warp >= 4) {  // 8 warps of CUDA-core work until warp 0 is done
    uint32_t a = threadIdx.x, b = threadIdx.x * 7 + 1, c = 3, e = 5;
    float fa = (float)threadIdx.x, fb = 1.0001f;
    while (*(volatile uint64_t*)&bar[3] == 0 || true) {
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        if (kAlu == 1) { a = a * 2654435761u + b; b = __umulhi(b, 0x9E3779B9u) + c; c = c * e + a; e = e * a + 7; }
        if (kAlu == 2) { fa = fa * fb + 1.0f; fb = fb * 0.9999f + 0.0001f; }
        if (kAlu == 3) { a = (a ^ b) + (c >> 3); b = __byte_perm(a, b, 0x5140) ^ c; c = (c << 1) | (a & 1); e += a ^ b; }
      }
      if (*(volatile int*)&done_flag) break;
    }
    if (a + b + c + e == 0x12345 || fa == 1.5f) out[0] = a;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int kV, int kEpi = 1, bool kFence = false, int kAlu = 0>
void run(const char* name, int units = 2000) {
  long long* d;
  const int blocks = 148;
  cudaMalloc(&d, sizeof(long long) * blocks);
  auto k = probe_kernel<kV, kEpi, kFence, kAlu>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k<<<blocks, 384, 140 * 1024>>>(d, units);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
  const int mmas = ((kV & 1) ? 18 : 16);
  printf("%-52s %7.1f cyc/unit  %5.1f cyc/MMA  (%s)\n", name, (double)mx / units, (double)mx / units / mmas,
         e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("plain: 16 MMAs, fixed B, lo reads next K-step");
  run<8>("limbs share B");
  run<4>("B advances");
  run<12>("B advances, limbs share B");
  run<13>("+ bias MMAs");
  run<15>("+ commits (= K1 sequence, single D)");
  run<31>("+ D double buffer (= K1 sequence)");
  run<31 + 32>("+ 11 warps spinning on an mbarrier");
  run<31 + 64>("+ tfull/tempty handshake with an epilogue warp");
  run<31 + 96>("+ both");
  run<31 + 64, 8>("handshake with 8 epilogue warps");
  run<31 + 64, 8, true>("handshake with 8 epilogue warps + fence.proxy.async");
  run<31 + 64, 1, true>("handshake with 1 epilogue warp + fence.proxy.async");
  run<31, 1, false, 1>("K1 sequence + 8 warps of IMAD/IMAD.HI chains");
  run<31, 1, false, 2>("K1 sequence + 8 warps of FFMA chains");
  run<31, 1, false, 3>("K1 sequence + 8 warps of ALU (LOP/PRMT/SHF) chains");
  return 0;
}
