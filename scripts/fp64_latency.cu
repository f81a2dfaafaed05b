// Microbenchmark: dependent-chain latency (cycles) of fp64 ops on this GPU,
// and of one gated-Kalman fold step as k_fuse executes it. Development aid.
#include <cstdio>
#include <cuda_runtime.h>
// Division certified against IEEE round-to-nearest: q is accepted iff the
// residual n - d*q (one FMA) is strictly below half the smaller spacing of
// doubles around q, times |d| -- then q is the unique nearest double to n/d,
// i.e. exactly what n / d returns. Anything not certified (magnitudes near
// under/overflow, NaN/inf, residuals near a midpoint) uses n / d itself.
__device__ __forceinline__ bool certifiedQuotient(double n, double d, double q) {
  const double rem = __fma_rn(-d, q, n);
  const long long qb = __double_as_longlong(q);
  const int qe = static_cast<int>((qb >> 52) & 0x7ff);
  const int de = static_cast<int>((__double_as_longlong(d) >> 52) & 0x7ff);
  if (qe < 200 || qe > 1800 || de < 200 || de > 1800) return false;
  const bool pow2 = (qb & 0x000fffffffffffffLL) == 0;  // spacing below q is halved
  const double half = __longlong_as_double(static_cast<long long>(qe - 53 - (pow2 ? 1 : 0)) << 52);
  return fabs(rem) < fabs(d) * half;
}

// n1/d and n2/d sharing one reciprocal (hardware approximation + 3 Newton
// steps) so the two quotients of a Kalman update take one division latency.
__device__ __forceinline__ void divPair(double n1, double n2, double d, double& q1, double& q2) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = __fma_rn(-d, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-d, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-d, r, 1.0);
  r = __fma_rn(r, e, r);
  double a = n1 * r;
  a = __fma_rn(__fma_rn(-d, a, n1), r, a);
  double b = n2 * r;
  b = __fma_rn(__fma_rn(-d, b, n2), r, b);
  q1 = certifiedQuotient(n1, d, a) ? a : n1 / d;
  q2 = certifiedQuotient(n2, d, b) ? b : n2 / d;
}


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
  double h2 = 0.1, v2 = 1.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const double zz = 0.1 + 1e-3 * (i & 7), sp = 0.0004;
    const double d = fabs(zz - h2);
    if (d * d > 6.25 * v2 * 1.000000000001) { v2 = v2 + 0.01; continue; }
    const double den = v2 + sp;
    divPair(sp * h2 + v2 * zz, v2 * sp, den, h2, v2);
  }
  t1 = clock64(); cyc[5] = t1 - t0;
  out[0] = x + y + z + w + h + v + h2 + v2;
}

int main() {
  double* d; long long* c; cudaMalloc(&d, 8); cudaMalloc(&c, 6 * 8);
  const int n = 4096;
  chain<<<1, 1>>>(d, c, 1.0000001, 0.9999999, n);
  cudaDeviceSynchronize();
  long long h[6]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  const char* names[] = {"dadd", "dmul", "ddiv(+add)", "dsqrt(+add)", "fold step", "fold divPair"};
  for (int i = 0; i < 6; ++i) printf("%-12s %.1f cycles/op\n", names[i], (double)h[i] / n);
  return 0;
}
