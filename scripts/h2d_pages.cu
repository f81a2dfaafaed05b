// H2D bandwidth of a 24 MB frame (C4) by how its pinned host buffer was made:
// cudaHostAlloc (4 KiB pages), malloc + cudaHostRegister, and mmap +
// madvise(MADV_HUGEPAGE) (transparent 2 MiB pages) + cudaHostRegister; several
// fresh buffers each, min / median of 30 copies per buffer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/h2d_pages.cu -o /tmp/h2d_pages
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sys/mman.h>
#include <vector>

#include <cuda_runtime.h>

static void measure(const char* label, void* h, void* d, size_t bytes, cudaStream_t s) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> t;
  for (int it = 0; it < 30; ++it) {
    cudaEventRecord(a, s);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    t.push_back(ms);
  }
  std::sort(t.begin(), t.end());
  printf("%-28s min %.3f ms  median %.3f ms  (%.1f GB/s median)\n", label, t[0], t[t.size() / 2],
         bytes / (t[t.size() / 2] * 1e6));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
}

int main() {
  const size_t bytes = 24001536;
  void* d = nullptr;
  cudaMalloc(&d, bytes);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int rep = 0; rep < 3; ++rep) {
    void* h = nullptr;
    cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
    memset(h, 1, bytes);
    measure("cudaHostAlloc", h, d, bytes, s);
    cudaFreeHost(h);

    void* m = malloc(bytes);
    memset(m, 1, bytes);
    cudaHostRegister(m, bytes, cudaHostRegisterDefault);
    measure("malloc + register", m, d, bytes, s);
    cudaHostUnregister(m);
    free(m);

    const size_t big = (bytes + (2u << 20) - 1) & ~static_cast<size_t>((2u << 20) - 1);
    void* p = mmap(nullptr, big + (2u << 20), PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    char* q = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + (2u << 20) - 1) & ~static_cast<uintptr_t>((2u << 20) - 1));
    const int adv = madvise(q, big, MADV_HUGEPAGE);
    memset(q, 1, bytes);
    cudaHostRegister(q, big, cudaHostRegisterDefault);
    measure(adv == 0 ? "mmap 2MiB-aligned + THP" : "mmap (no THP)", q, d, bytes, s);
    cudaHostUnregister(q);
    munmap(p, big + (2u << 20));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
