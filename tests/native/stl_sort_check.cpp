// Host check of the device's libstdc++ std::sort replica (csrc/stl_sort.cuh)
// against std::sort itself: random windows of 1..121 doubles drawn from small
// value sets with +0 / -0 ties, repeated values and NaNs (which push the
// introsort into its heap-sort fallback), compared bit for bit.
// Build + run: tests/test_stl_sort.py.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "stl_sort.cuh"

// McIlroy's adversary ("A killer adversary for quicksort", 1999) run against
// std::sort itself: values are fixed lazily as the comparisons need them, so
// the returned input drives the introsort to its depth limit and into the
// heap-sort fallback.
static std::vector<double> adversary(int n) {
  std::vector<int> val(n, n), idx(n);
  const int gas = n;
  int solid = 0, candidate = 0;
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int x, int y) {
    if (val[x] == gas && val[y] == gas) {
      if (x == candidate) val[x] = solid++;
      else val[y] = solid++;
    }
    if (val[x] == gas) candidate = x;
    else if (val[y] == gas) candidate = y;
    return val[x] < val[y];
  });
  std::vector<double> a(n);
  for (int i = 0; i < n; ++i) a[i] = static_cast<double>(val[i]);
  return a;
}

static bool same(std::vector<double> a) {
  std::vector<double> want = a, got = a;
  std::sort(want.begin(), want.end());
  rb200::stl::sort(got.data(), static_cast<int>(a.size()));
  return std::memcmp(want.data(), got.data(), a.size() * sizeof(double)) == 0;
}

int main(int argc, char** argv) {
  for (int n = 2; n <= 121; ++n) {
    std::vector<double> a = adversary(n);
    if (!same(a)) {
      std::printf("MISMATCH adversary n %d\n", n);
      return 1;
    }
    for (double& x : a) x = (x == 0.0) ? -0.0 : (static_cast<int>(x) % 5 == 0 ? 0.0 : x);  // + signed zeros
    if (!same(a)) {
      std::printf("MISMATCH adversary+zeros n %d\n", n);
      return 1;
    }
  }
  const int trials = argc > 1 ? std::atoi(argv[1]) : 200000;
  std::mt19937_64 rng(12345);
  long long heapish = 0;
  for (int t = 0; t < trials; ++t) {
    const int n = 1 + static_cast<int>(rng() % 121);
    const int mode = static_cast<int>(rng() % 6);
    std::vector<double> a(n);
    for (int k = 0; k < n; ++k) {
      const uint64_t r = rng();
      switch (mode) {
        case 0: a[k] = static_cast<double>(r % 1000) * 1e-3 - 0.5; break;          // mostly distinct
        case 1: a[k] = static_cast<double>(static_cast<int>(r % 5) - 2) * 0.25; break;  // many ties
        case 2: a[k] = (r % 3 == 0) ? -0.0 : ((r % 3 == 1) ? 0.0 : 1.0); break;        // signed zeros
        case 3: a[k] = (r % 7 == 0) ? NAN : static_cast<double>(r % 9) - 4.0; break;    // a few NaNs
        case 4: a[k] = (r % 2 == 0) ? NAN : ((r % 4 == 1) ? -0.0 : 0.0); break;         // NaN-heavy
        default: a[k] = static_cast<double>(k % 7) * ((r & 1) ? 1.0 : -1.0); break;     // patterned
      }
    }
    std::vector<double> want = a, got = a;
    std::sort(want.begin(), want.end());
    rb200::stl::sort(got.data(), n);
    if (std::memcmp(want.data(), got.data(), n * sizeof(double)) != 0) {
      std::printf("MISMATCH trial %d n %d mode %d\n", t, n, mode);
      for (int k = 0; k < n; ++k) std::printf("%a %a\n", want[k], got[k]);
      return 1;
    }
    heapish += mode == 4;
  }
  std::printf("ok %d trials\n", trials);
  return 0;
}
