// Latency of the gated fold (foldCell in csrc/pipeline.cu) on one long cell,
// one thread: cycles per point for all-fused, all-ignored (wall rule) and a
// mixed sequence like the box face of the headline frame.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 \
//   -I include -I paper_2204_12876_b200/csrc scripts/fold_bench.cu -o fold_bench
#include "../paper_2204_12876_b200/csrc/pipeline.cu"

#include <cstdio>
#include <vector>

namespace rb200 {
namespace {
__global__ void k_bench(Layers L, const uint32_t* start, const double* spz, const double* spv, int cnt,
                        FuseArgs a, DevStats* st, long long* cycles) {
  FoldCounts k;
  const long long t0 = clock64();
  foldCell(L, 0, cnt, start, spz, spv, a, st, k);
  const long long t1 = clock64();
  cycles[0] = t1 - t0;
  cycles[1] = static_cast<long long>(k.nf);
  cycles[2] = static_cast<long long>(k.ni);
  cycles[3] = static_cast<long long>(k.no);
}
__global__ void k_bench_smem(Layers L, const double* spz, const double* spv, int cnt, FuseArgs a,
                             long long* cycles) {
  __shared__ double sz[2048], sv[2048];
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
    sz[j] = spz[j];
    sv[j] = spv[j];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  FoldCounts k;
  FoldState s = foldBegin(L, 0);
  const bool wall = cnt > a.wall;
  const long long t0 = clock64();
  for (int j = 0; j < cnt; ++j)
    if (!foldPoint(s, sz[j], sv[j], wall, a, k)) break;
  const long long t1 = clock64();
  cycles[0] = t1 - t0 + (s.h > 1e300 ? 1 : 0);
  cycles[1] = static_cast<long long>(k.nf);
  cycles[2] = static_cast<long long>(k.ni);
  cycles[3] = static_cast<long long>(k.no);
}
}  // namespace
}  // namespace rb200

using namespace rb200;

int main() {
  const int n = 1233;
  DeviceMap* m = createDeviceMap(0, Grid{0.04, 16, 16, 0, 0});
  std::vector<double> z(n), v(n);
  double* dz; double* dv; uint32_t* dstart; long long* dc;
  cudaMalloc(&dz, n * 8); cudaMalloc(&dv, n * 8); cudaMalloc(&dstart, 8); cudaMalloc(&dc, 32);
  cudaMemset(dstart, 0, 8);
  FuseArgs a{1.0, 100.0, 0.01, 100.0, 2.5, 6.25, 5};
  unsigned long long s = 1;
  auto rnd = [&]() { s = s * 6364136223846793005ULL + 1442695040888963407ULL; return ((s >> 11) * 0x1.0p-53) - 0.5; };
  for (int mode = 0; mode < 3; ++mode) {
    for (int i = 0; i < n; ++i) {
      v[i] = 2e-4;
      if (mode == 0) z[i] = 0.5 + 1e-4 * rnd() + 1e-3;          // mostly above -> fused
      else if (mode == 1) z[i] = (i == 0 ? 0.6 : 0.5 + 1e-3 * rnd());   // below the first -> ignored
      else z[i] = 0.5 + 0.02 * rnd();                              // mixed
    }
    cudaMemcpy(dz, z.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, v.data(), n * 8, cudaMemcpyHostToDevice);
    fillFresh(*m);
    cudaDeviceSynchronize();
    long long c[4];
    for (int rep = 0; rep < 3; ++rep) {
      fillFresh(*m);
      k_bench<<<1, 1>>>(m->cur, dstart, dz, dv, n, a, m->stats, dc);
      cudaMemcpy(c, dc, 32, cudaMemcpyDeviceToHost);
    }
    printf("mode %d: %lld cycles, %.1f cycles/point (fused %lld ignored %lld outlier %lld)\n", mode, c[0],
           double(c[0]) / n, c[1], c[2], c[3]);
    fillFresh(*m);
    k_bench_smem<<<1, 256>>>(m->cur, dz, dv, n, a, dc);
    cudaMemcpy(c, dc, 32, cudaMemcpyDeviceToHost);
    printf("  smem single-thread: %.1f cycles/point (fused %lld ignored %lld outlier %lld)\n",
           double(c[0]) / n, c[1], c[2], c[3]);
  }
  return 0;
}
