// Microbenchmark: tcgen05.mma kind::i8 issue/execution rate on one SM for the
// operand layouts the kernels use (SS K-major, SS with MN-major B, TS with A
// in TMEM), M = 128, N = 64 / 128 / 256, K = 32 per instruction.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o mma_rate tools/mma_rate.cu
// Run:   ./mma_rate   (prints cycles per MMA and MACs/clk for each variant)
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2007_12216_b200/csrc/common.cuh"

template <int N, int kMode, int kAcc = 2, int kRand = 0>  // kRand: random operand bytes (1) instead of small constants; kAcc: independent accumulators cycled; kMode 0: SS both K-major, 1: SS, B MN-major (SW128/SW64), 2: TS (A in TMEM), B MN-major
__global__ void mma_rate_kernel(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) {
    uint32_t r = (uint32_t)i * 2654435761u + 12345u;
    r ^= r >> 13; r *= 0x5bd1e995u; r ^= r >> 15;
    reinterpret_cast<uint32_t*>(smem)[i] = kRand ? r : 0x01010101u * (i & 7);
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  if (kRand && warp < 4) {  // random A operand bytes in TMEM columns 384..511
    for (int c = 0; c < 128; c += 8) {
      uint32_t v[8];
      for (int j = 0; j < 8; ++j) {
        uint32_t r = (uint32_t)(threadIdx.x * 977 + c * 31 + j) * 2654435761u;
        r ^= r >> 13; r *= 0x5bd1e995u; r ^= r >> 15;
        v[j] = r;
      }
      tmem_st8(tbase + ((uint32_t)(warp * 32) << 16) + 384 + c, v);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  long long t0 = 0, t1 = 0;
  if (warp == 0) {
    constexpr bool bmn = kMode >= 1;
    constexpr uint32_t idesc = idesc_i8x(128, N, true, true, false, bmn);
    const uint64_t da = umma_desc_kmajor(smem_u32(smem), 128);
    uint64_t db;
    if (kMode == 0) db = umma_desc_kmajor(smem_u32(smem + 32768), 128);
    else if (N == 64) db = umma_desc_mn_sw64(smem_u32(smem + 32768), 16);
    else db = umma_desc_mn_sw128(smem_u32(smem + 32768));
    // warm-up
    for (int i = 0; i < 4; ++i) {
      if (kMode == 2) mma_i8_ts_warp(tbase, tbase + 384, db, idesc, 1u);
      else mma_i8_warp(tbase, da, db, idesc, 1u);
    }
    mma_commit_warp(&bar);
    mbar_wait(&bar, 0);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t dcol = N <= 128 ? (k % kAcc) * N : 0;
        if (kMode == 2) mma_i8_ts_warp(tbase + dcol, tbase + 384 + k * 8, db + k * 2, idesc, 1u);
        else mma_i8_warp(tbase + dcol, da + k * 2, db + k * 2, idesc, 1u);
      }
    }
    mma_commit_warp(&bar);
    mbar_wait(&bar, 1);
    t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int N, int kMode, int kAcc = 2, int kRand = 0>
void run(const char* name, int blocks) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * blocks);
  const int iters = 2000;
  auto k = mma_rate_kernel<N, kMode, kAcc, kRand>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<blocks, 128, 100 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double cyc = (double)h[0] / (iters * 8.0);
  printf("%-34s blocks=%3d  %7.1f cyc/MMA  %7.0f MACs/clk/SM  (%s)\n", name, blocks, cyc, 128.0 * N * 32 / cyc,
         e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int blocks : {1, 148}) {
    run<64, 0>("SS K-major/K-major  N=64", blocks);
    run<128, 0>("SS K-major/K-major  N=128", blocks);
    run<256, 0>("SS K-major/K-major  N=256", blocks);
    run<64, 1>("SS K-major/MN-major N=64", blocks);
    run<128, 1>("SS K-major/MN-major N=128", blocks);
    run<256, 1>("SS K-major/MN-major N=256", blocks);
    run<64, 2>("TS A-tmem/MN-major  N=64", blocks);
    run<128, 2>("TS A-tmem/MN-major  N=128", blocks);
    run<256, 2>("TS A-tmem/MN-major  N=256", blocks);
  }
  // dependent accumulation: how many independent accumulators keep the pipe full
  run<64, 2, 1>("TS N=64  one accumulator", 148);
  run<64, 2, 2>("TS N=64  two accumulators", 148);
  run<64, 2, 4>("TS N=64  four accumulators", 148);
  run<128, 2, 1>("TS N=128 one accumulator", 148);
  run<128, 2, 2>("TS N=128 two accumulators", 148);
  run<64, 1, 1>("SS N=64  one accumulator", 148);
  run<64, 1, 4>("SS N=64  four accumulators", 148);
  run<128, 1, 1>("SS N=128 one accumulator", 148);
  run<128, 1, 2>("SS N=128 two accumulators", 148);
  // operand values: random bytes instead of small constants
  run<64, 2, 2, 1>("TS N=64  random operands", 148);
  run<128, 2, 2, 1>("TS N=128 random operands", 148);
  run<256, 2, 1, 1>("TS N=256 random operands", 148);
  run<128, 1, 2, 1>("SS N=128 random operands", 148);
  run<256, 1, 1, 1>("SS N=256 random operands", 148);
  run<256, 0, 1, 1>("SS K/K N=256 random operands", 148);
  return 0;
}
