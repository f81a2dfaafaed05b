// L2 visit ceiling: random 1-byte probes over a map-sized footprint,
// the access pattern of the DDA's class probe, at full occupancy. Prints probes/s for
// footprints of 0.25, 1 and 4 MB (class bytes of 500^2, 1000^2, 2000^2 maps) and 8 MB
// of doubles (the upper-bound layer of 1000^2). Compare with V/t of k_rays_pass1.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/l2_ceiling.cu -o l2_ceiling
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <typename T>
__global__ void probe(const T* __restrict__ buf, uint32_t mask, int iters, unsigned long long* sink) {
  uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  T acc = 0;
#pragma unroll 8
  for (int k = 0; k < iters; ++k) {
    h = mix(h + k);
    acc += __ldg(buf + (h & mask));
  }
  if (acc == T(123)) atomicAdd(sink, 1ull);
}

int main() {
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int which = 0; which < 4; ++which) {
    const size_t bytes = which == 0 ? (1u << 18) : which == 1 ? (1u << 20) : which == 2 ? (1u << 22) : (1u << 23);
    void* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (which < 3) probe<uint8_t><<<blocks, threads>>>((const uint8_t*)buf, bytes - 1, iters, sink);
      else probe<double><<<blocks, threads>>>((const double*)buf, bytes / 8 - 1, iters, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    const double n = double(blocks) * threads * iters;
    printf("%s footprint %6.2f MB: %.1f G probes/s\n", which < 3 ? "u8 " : "f64", bytes / 1048576.0, n / (ms * 1e-3) / 1e9);
    cudaFree(buf);
  }
  return 0;
}
