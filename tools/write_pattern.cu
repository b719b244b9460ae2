// HBM write bandwidth by access pattern, with non-constant data: does the
// way K1 scatters V (128-byte pieces into 1024 streams 4 MB apart) cost DRAM
// efficiency against larger contiguous pieces or a blocked layout?
// 148 CTAs in 4 groups; group g owns 256 of the 1024 streams; a CTA walks the
// pieces pr = cta / 4, + 37, ... and writes `piece` bytes to each of its 256
// streams per step (one thread per stream, 16-byte stores; L2 merges them).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/write_pattern tools/write_pattern.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// blocked = 0: stream s at s * stream_bytes (K1's V: [stream][tile pieces])
// blocked = 1: [block of 64 pieces][stream][64 pieces]: a stream's pieces of one block are contiguous (8 KB at 128 B)
__global__ void __launch_bounds__(256) pattern_kernel(uint8_t* dst, size_t stream_bytes, int piece, int blocked, uint32_t salt) {
  const int group = blockIdx.x & 3, row = threadIdx.x;
  const size_t stream = (size_t)group * 256 + row;
  const size_t npieces = stream_bytes / piece;
  for (size_t pr = blockIdx.x >> 2; pr < npieces; pr += gridDim.x >> 2) {
    size_t off;
    if (blocked)
      off = ((pr >> 6) * 1024 + stream) * (size_t)(64 * piece) + (pr & 63) * (size_t)piece;
    else
      off = stream * stream_bytes + pr * (size_t)piece;
    uint4* p = reinterpret_cast<uint4*>(dst + off);
    const uint32_t h = (uint32_t)(off >> 4) * 2654435761u ^ salt;
    for (int i = 0; i < piece / 16; ++i) p[i] = make_uint4(h + i, h * 0x9E3779B9u, h ^ 0x85EBCA6Bu, (h + i) * 0xC2B2AE35u);
  }
}

int main() {
  const size_t stream_bytes = 4ull << 20, bytes = 1024 * stream_bytes;
  uint8_t* a;
  cudaMalloc(&a, bytes);
  cudaMemset(a, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int blocked = 0; blocked < 2; ++blocked)
    for (int piece : {64, 128, 256, 512, 1024, 4096}) {
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        float ms;
        cudaEventRecord(e0);
        pattern_kernel<<<148, 256>>>(a, stream_bytes, piece, blocked, 7 + r);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      printf("%s piece %5d B: %7.1f GB/s (%s)\n", blocked ? "blocked  " : "streams  ", piece, bytes / (best * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
