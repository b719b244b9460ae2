// Microbenchmark: the two-pass K4's MMA shapes in isolation (M = 128, K = 32,
// N = 16 / 32 / 64 per instruction, both operands from shared memory) by A
// operand layout: MN-major under the 32B swizzle (pass 1: the Mw8 boxes as
// TMA lands them), MN-major under the 128B swizzle (pass 2: the z limbs) and
// K-major 32-byte rows, with B K-major (the 1 KB constant tiles).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/k4_mma_probe tools/k4_mma_probe.cu
// Run:   ./tools/k4_mma_probe   (cycles per MMA, one CTA per SM and two)
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2007_12216_b200/csrc/common.cuh"


// kA: 0 = MN-major SW32 (LBO 1 KB), 1 = MN-major SW128, 2 = K-major 32-byte rows
// kPairs: consecutive MMA pairs accumulate into the same columns (pass 2) instead of 8 distinct accumulators
template <int N, int kA, int kPairs>
__global__ void __launch_bounds__(128) probe(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 80 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(&slot);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  if (warp == 0) {
    constexpr uint32_t idesc = idesc_i8x(128, N, false, true, kA != 2, false);
    uint64_t da[16];
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      const uint32_t a = smem_u32(smem + v * 4096);
      da[v] = kA == 0 ? umma_desc_mn_sw32(a, 1024) : (kA == 1 ? umma_desc_mn_sw128(a) : umma_desc_kmajor(a, 32));
    }
    const uint64_t db = umma_desc_kmajor(smem_u32(smem + 64 * 1024), 32);
    mma_i8_warp(tbase, da[0], db, idesc, 0u);
    mma_commit_warp(&bar);
    mbar_wait(&bar, 0);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t dcol = kPairs ? (k >> 1) * 32 : (k & 7) * (N <= 32 ? 32 : 64) % 256;
        mma_i8_warp(tbase + dcol, da[k], db + (k & 3) * 64, idesc, kPairs ? (uint32_t)(k & 1) : 0u);
      }
    }
    mma_commit_warp(&bar);
    mbar_wait(&bar, 1);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tbase);
  }
}

template <int N, int kA, int kPairs>
void run(const char* name, int blocks) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * blocks);
  const int iters = 1000;
  auto k = probe<N, kA, kPairs>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<blocks, 128, 100 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[512];
  cudaMemcpy(h, d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  const double cyc = (double)h[0] / (iters * 16.0);
  printf("%-44s blocks=%3d  %6.1f cyc/MMA  (%s)\n", name, blocks, cyc, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int blocks : {148, 296}) {
    run<32, 0, 0>("N=32 A MN-major SW32 (pass 1)", blocks);
    run<32, 1, 0>("N=32 A MN-major SW128", blocks);
    run<32, 1, 1>("N=32 A MN-major SW128 pairs (pass 2)", blocks);
    run<32, 2, 0>("N=32 A K-major 32B rows", blocks);
    run<16, 0, 0>("N=16 A MN-major SW32", blocks);
    run<16, 1, 0>("N=16 A MN-major SW128", blocks);
    run<64, 0, 0>("N=64 A MN-major SW32", blocks);
    run<64, 1, 0>("N=64 A MN-major SW128", blocks);
    run<64, 2, 0>("N=64 A K-major 32B rows", blocks);
  }
  return 0;
}
