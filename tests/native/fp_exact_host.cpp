// Host build of csrc/fp_exact.cuh for tests/test_fp_exact.py (test helper, not product).
#include <cmath>
#include <cstdint>

#include "fp_exact.cuh"

extern "C" {
double rb_hypot(double x, double y) { return rb200::libm_hypot(x, y); }
int rb_to_int(double v) { return rb200::x86_to_int(v); }

// Counts disagreements between rb200::libm_hypot and the host libm hypot over n
// splitmix64-generated pairs spanning sensor-scale, tiny, huge and mixed scales.
long long rb_hypot_mismatches(long long n, unsigned long long seed) {
  unsigned long long s = seed;
  auto next = [&]() {
    unsigned long long z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  };
  auto u = [&]() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); };
  long long bad = 0;
  for (long long i = 0; i < n; ++i) {
    double x = u() * 20 - 10, y = u() * 20 - 10;
    switch (i % 7) {
      case 1: x *= 1e-3; break;
      case 2: y *= 1e-9; break;
      case 3: x *= 1e-160; y *= 1e-160; break;
      case 4: x *= 1e300; break;
      case 5: x = std::ldexp(x, static_cast<int>(u() * 2000) - 1000);
              y = std::ldexp(y, static_cast<int>(u() * 2000) - 1000); break;
      default: break;
    }
    const double a = std::hypot(x, y), b = rb200::libm_hypot(x, y);
    if (!(a == b) && !(std::isnan(a) && std::isnan(b))) ++bad;
  }
  return bad;
}
}
