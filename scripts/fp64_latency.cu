// Microbenchmark: dependent-chain latency (cycles) of fp64 ops on this GPU,
// and of one gated-Kalman fold step as k_fuse executes it. Development aid.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b;
  long long t0, t1;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + b;
  t1 = clock64(); cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) y = y * a;
  t1 = clock64(); cyc[1] = t1 - t0;
  // DIV chain
  double z = a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) z = b / (z + 1.0);
  t1 = clock64(); cyc[2] = t1 - t0;
  // SQRT chain
  double w = a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) w = sqrt(w + 1.0);
  t1 = clock64(); cyc[3] = t1 - t0;
  // fold step: h,v <- fuse(h,v,z,sp)
  double h = 0.1, v = 1.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const double zz = 0.1 + 1e-3 * (i & 7), sp = 0.0004;
    const double d = fabs(zz - h);
    if (d * d > 6.25 * v * 1.000000000001) { v = v + 0.01; continue; }
    const double den = v + sp;
    h = (sp * h + v * zz) / den;
    v = v * sp / den;
  }
  t1 = clock64(); cyc[4] = t1 - t0;
  out[0] = x + y + z + w + h + v;
}

int main() {
  double* d; long long* c; cudaMalloc(&d, 8); cudaMalloc(&c, 5 * 8);
  const int n = 4096;
  chain<<<1, 1>>>(d, c, 1.0000001, 0.9999999, n);
  cudaDeviceSynchronize();
  long long h[5]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  const char* names[] = {"dadd", "dmul", "ddiv(+add)", "dsqrt(+add)", "fold step"};
  for (int i = 0; i < 5; ++i) printf("%-12s %.1f cycles/op\n", names[i], (double)h[i] / n);
  return 0;
}
