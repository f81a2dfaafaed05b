// Host->device transfer options for the e2e leg: cudaMemcpyAsync from pinned
// memory (1, 2, 4 streams) vs a kernel reading mapped pinned memory directly.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/h2d_bench.cu -o /tmp/h2d
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

__global__ void k_read(const double* __restrict__ src, double* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void k_read2(const double2* __restrict__ src, double2* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main() {
  const size_t bytes = 24001536;
  const size_t n = bytes / 8;
  double *h, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  cudaMalloc(&d, bytes);
  for (size_t i = 0; i < n; ++i) h[i] = i;
  cudaStream_t s[4];
  for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int ns : {1, 2, 4}) {
    float best = 1e9;
    for (int it = 0; it < 20; ++it) {
      cudaEventRecord(a, s[0]);
      for (int k = 1; k < ns; ++k) cudaStreamWaitEvent(s[k], a);
      cudaEvent_t e[4];
      for (int k = 0; k < ns; ++k) {
        size_t lo = bytes * k / ns, hi = bytes * (k + 1) / ns;
        cudaMemcpyAsync((char*)d + lo, (char*)h + lo, hi - lo, cudaMemcpyHostToDevice, s[k]);
        cudaEventCreateWithFlags(&e[k], cudaEventDisableTiming);
        cudaEventRecord(e[k], s[k]);
      }
      for (int k = 1; k < ns; ++k) cudaStreamWaitEvent(s[0], e[k]);
      cudaEventRecord(b, s[0]);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("memcpy %d stream(s): %.1f us  %.1f GB/s\n", ns, best * 1e3, bytes / (best * 1e-3) / 1e9);
  }
  for (int blocks : {148, 296, 592, 1184, 2368}) {
    for (int v = 0; v < 2; ++v) {
      float best = 1e9;
      for (int it = 0; it < 20; ++it) {
        cudaEventRecord(a, s[0]);
        if (v == 0) k_read<<<blocks, 256, 0, s[0]>>>(h, d, n);
        else k_read2<<<blocks, 256, 0, s[0]>>>((const double2*)h, (double2*)d, n / 2);
        cudaEventRecord(b, s[0]);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("zero-copy kernel %s blocks=%d: %.1f us  %.1f GB/s\n", v ? "f64x2" : "f64", blocks, best * 1e3,
             bytes / (best * 1e-3) / 1e9);
    }
  }
  // 8 distinct pinned frames copied in turn (what bench.py's e2e leg does)
  {
    double* hs[8];
    for (auto& b : hs) {
      cudaHostAlloc(&b, bytes, cudaHostAllocDefault);
      memset(b, 1, bytes);
    }
    float tot = 0;
    for (int it = 0; it < 16; ++it) {
      cudaEventRecord(a, s[0]);
      cudaMemcpyAsync(d, hs[it % 8], bytes, cudaMemcpyHostToDevice, s[0]);
      cudaEventRecord(b, s[0]);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it >= 8) tot += ms;
    }
    printf("memcpy cycling 8 pinned buffers: %.1f us  %.1f GB/s\n", tot / 8 * 1e3, bytes / (tot / 8 * 1e-3) / 1e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
