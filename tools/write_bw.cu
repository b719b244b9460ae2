// HBM bandwidth of write-only and read+write streams on this GPU, with
// non-constant data (constant or zero data may be compressed by the memory
// system and overstate the rate): the roofline for write-dominated kernels
// (K1 writes five bytes of V per byte it reads).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/write_bw tools/write_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void write_kernel(uint4* dst, size_t n16, uint32_t salt) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t h = (uint32_t)i * 2654435761u ^ salt;
    dst[i] = make_uint4(h, h * 0x9E3779B9u, h ^ 0x85EBCA6Bu, h * 0xC2B2AE35u);
  }
}
__global__ void copy_kernel(const uint4* __restrict__ src, uint4* dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) dst[i] = src[i];
}
__global__ void read_kernel(const uint4* __restrict__ src, size_t n16, uint32_t* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = src[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  const size_t bytes = 4ull << 30, n16 = bytes / 16;
  uint4 *a, *b;
  uint32_t* o;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&o, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 148 * 8, block = 512;
  write_kernel<<<grid, block>>>(a, n16, 1);
  write_kernel<<<grid, block>>>(b, n16, 2);
  cudaDeviceSynchronize();
  float best_w = 1e9, best_c = 1e9, best_r = 1e9;
  for (int r = 0; r < 10; ++r) {
    float ms;
    cudaEventRecord(e0);
    write_kernel<<<grid, block>>>(a, n16, 3 + r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best_w = ms < best_w ? ms : best_w;
    cudaEventRecord(e0);
    copy_kernel<<<grid, block>>>(b, a, n16);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best_c = ms < best_c ? ms : best_c;
    cudaEventRecord(e0);
    read_kernel<<<grid, block>>>(b, n16, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best_r = ms < best_r ? ms : best_r;
  }
  printf("{\"write_only_GBs\": %.1f, \"read_only_GBs\": %.1f, \"copy_read_plus_write_GBs\": %.1f}\n",
         bytes / (best_w * 1e-3) / 1e9, bytes / (best_r * 1e-3) / 1e9, 2.0 * bytes / (best_c * 1e-3) / 1e9);
  return 0;
}
