// Device check that div2_rn (csrc/fp_exact.cuh) returns exactly a1/b and a2/b.
// Usage: div2_check <n> <seed>; prints the number of mismatching quotients.
#include <cstdio>
#include <cstdlib>

#include "fp_exact.cuh"

__device__ unsigned long long mix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Random doubles: full exponent range, map-like magnitudes, and special values.
__device__ double pick(unsigned long long h) {
  const unsigned kind = h & 7;
  const unsigned long long m = mix(h);
  if (kind == 0) return __longlong_as_double(static_cast<long long>(m));  // any bit pattern
  if (kind == 1) {
    const double specials[8] = {0.0, -0.0, 1.0, -1.0, 1e-310, 1e308, __longlong_as_double(0x7ff0000000000000LL),
                                __longlong_as_double(0x7ff8000000000000LL)};
    return specials[m & 7];
  }
  // sign, exponent in [-60, 60] around 1 (the fold's values), random mantissa
  const long long e = static_cast<long long>((m >> 52) % 121) - 60 + 1023;
  const long long bits = ((m & 1) << 63) | (e << 52) | (m & 0xfffffffffffffULL);
  return __longlong_as_double(bits);
}

__global__ void check(unsigned long long n, unsigned long long seed, unsigned long long* bad) {
  unsigned long long local = 0;
  for (unsigned long long i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const unsigned long long h = mix(seed ^ (i * 3));
    const double a1 = pick(h), a2 = pick(mix(h + 1)), b = pick(mix(h + 2));
    double q1, q2;
    rb200::div2_rn(a1, a2, b, q1, q2);
    const double w1 = a1 / b, w2 = a2 / b;
    const bool ok1 = __double_as_longlong(q1) == __double_as_longlong(w1) || (q1 != q1 && w1 != w1);
    const bool ok2 = __double_as_longlong(q2) == __double_as_longlong(w2) || (q2 != q2 && w2 != w2);
    local += !ok1 + !ok2;
  }
  if (local) atomicAdd(bad, local);
}

int main(int argc, char** argv) {
  const unsigned long long n = argc > 1 ? strtoull(argv[1], nullptr, 10) : 1000000ULL;
  const unsigned long long seed = argc > 2 ? strtoull(argv[2], nullptr, 10) : 1ULL;
  unsigned long long* bad;
  cudaMalloc(&bad, sizeof(*bad));
  cudaMemset(bad, 0, sizeof(*bad));
  check<<<148 * 16, 256>>>(n, seed, bad);
  unsigned long long h = 0;
  if (cudaMemcpy(&h, bad, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return 2;
  printf("%llu\n", h);
  return 0;
}
