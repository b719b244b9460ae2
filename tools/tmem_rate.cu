// Microbenchmark: TMEM read bandwidth (tcgen05.ld 32x32b) per SM, alone and
// while one warp keeps the tensor pipe busy with TS-mode kind::i8 MMAs into
// other TMEM columns.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/tmem_rate tools/tmem_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2007_12216_b200/csrc/common.cuh"

// warps 0..nld-1 read TMEM (x16 loads, 8 in flight per wait); warp 4 (if
// mma) issues MMAs (M=128, N=64) into columns 256..383, A at 448.
template <int kLdWarps, bool kMma, int kX>
__global__ void tmem_rate_kernel(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ int stop;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    stop = 0;
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  if (warp < kLdWarps) {
    const int q = warp & 3, half = warp >> 2;
    const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) + half * 128;
    int32_t acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      int32_t v[kX][16];
#pragma unroll
      for (int j = 0; j < kX; ++j) tmem_ld16(ta + j * 16, v[j]);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < kX; ++j) acc += v[j][0] ^ v[j][15];
    }
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x * 16 + warp] = t1 - t0;
    if (acc == 0x12345678) out[0] = acc;
    if (threadIdx.x == 0) atomicExch(&stop, 1);
  } else if (kMma && warp == 8) {
    constexpr uint32_t idesc = idesc_i8x(128, 64, true, true, false, true);
    const uint64_t db = umma_desc_mn_sw64(smem_u32(smem), 16);
    long long n = 0;
    long long t0 = clock64();
    while (kLdWarps > 0 ? *(volatile int*)&stop == 0 : n < 8 * iters) {
#pragma unroll
      for (int k = 0; k < 8; ++k) mma_i8_ts_warp(tbase + 256 + (k & 1) * 64, tbase + 448 + k * 8, db, idesc, 1u);
      n += 8;
      mma_commit_warp(&bar);
      mbar_wait(&bar, (uint32_t)((n / 8 - 1) & 1));
    }
    if ((threadIdx.x & 31) == 0) {
      out[blockIdx.x * 16 + 15] = n;
      out[blockIdx.x * 16 + 14] = clock64() - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int kLdWarps, bool kMma, int kX>
void run(const char* name) {
  long long* d;
  const int blocks = 148;
  cudaMalloc(&d, sizeof(long long) * blocks * 16);
  cudaMemset(d, 0, sizeof(long long) * blocks * 16);
  const int iters = 4000;
  auto k = tmem_rate_kernel<kLdWarps, kMma, kX>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<blocks, 288, 64 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[16];
  cudaMemcpy(h, d, sizeof(long long) * 16, cudaMemcpyDeviceToHost);
  long long cyc = 0;
  for (int w = 0; w < kLdWarps; ++w) cyc = h[w] > cyc ? h[w] : cyc;
  if (kLdWarps == 0) cyc = h[14];
  const double bytes = (double)kLdWarps * 32 * 16 * 4 * kX * iters;
  const double mma_cyc = kMma && h[15] ? (double)cyc / h[15] : 0;
  if (kLdWarps == 0) { printf("%-40s %6.1f cyc/MMA\n", name, (double)h[14] / h[15]); cudaFree(d); return; }
  printf("%-40s %8.1f B/clk TMEM read   %s%6.1f cyc/MMA  (%s)\n", name, bytes / cyc, kMma ? "MMA: " : "",
         mma_cyc, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<4, false, 2>("4 warps, x16 x2 per wait");
  run<4, false, 4>("4 warps, x16 x4 per wait");
  run<4, false, 8>("4 warps, x16 x8 per wait");
  run<8, false, 4>("8 warps, x16 x4 per wait");
  run<8, false, 8>("8 warps, x16 x8 per wait");
  run<4, true, 4>("4 warps + MMA warp (N=64 TS)");
  run<4, true, 8>("4 warps x8 + MMA warp (N=64 TS)");
  run<0, true, 4>("MMA warp alone (N=64 TS)");
  return 0;
}
