// Post-processing chain on the device (reference postprocess.cpp:29-197):
// min-inpaint, gaussian / box smoothing normalised over valid cells, and the
// valid-window median. Each step is one stencil launch over a masked layer;
// min-inpaint is a connected-component labelling (lock-free union-find over
// 4-neighbours) followed by a per-component atomic min over the 8-neighbour
// valid border. Sums run in the reference's row-major window order, the median
// sorts the same window values, and the inpaint minimum is order independent,
// so every step is bit-exact.
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "device_map.hpp"
#include "fp_exact.cuh"
#include "runners.hpp"

namespace rb200 {

namespace {

constexpr int kT = 256;
constexpr int kMaxMedianWindow = 121;  // radius <= 5

__global__ void __launch_bounds__(kT) k_linear(const double* __restrict__ v,
                                               const uint8_t* __restrict__ ok, int W, int H,
                                               int R, const double* __restrict__ w,
                                               double* __restrict__ out) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= W * H) return;
  if (!ok[i]) {
    out[i] = v[i];
    return;
  }
  const int r = i / W, c = i - (i / W) * W, k = 2 * R + 1;
  double acc = 0.0, ws = 0.0;
  for (int dr = -R; dr <= R; ++dr) {
    const int rr = r + dr;
    if (rr < 0 || rr >= H) continue;
    for (int dc = -R; dc <= R; ++dc) {
      const int cc = c + dc;
      if (cc < 0 || cc >= W) continue;
      const int j = rr * W + cc;
      if (!ok[j]) continue;
      const double wt = w[(dr + R) * k + (dc + R)];
      acc += wt * v[j];
      ws += wt;
    }
  }
  out[i] = acc / ws;
}

__global__ void __launch_bounds__(kT) k_median(const double* __restrict__ v,
                                               const uint8_t* __restrict__ ok, int W, int H,
                                               int R, double* __restrict__ out) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= W * H) return;
  if (!ok[i]) {
    out[i] = v[i];
    return;
  }
  const int r = i / W, c = i - (i / W) * W;
  double win[kMaxMedianWindow];
  int n = 0;
  for (int dr = -R; dr <= R; ++dr) {
    const int rr = r + dr;
    if (rr < 0 || rr >= H) continue;
    for (int dc = -R; dc <= R; ++dc) {
      const int cc = c + dc;
      if (cc < 0 || cc >= W) continue;
      const int j = rr * W + cc;
      if (!ok[j]) continue;
      // insertion keeps the window sorted ascending
      const double x = v[j];
      int p = n++;
      while (p > 0 && x < win[p - 1]) {
        win[p] = win[p - 1];
        --p;
      }
      win[p] = x;
    }
  }
  out[i] = (n % 2 == 1) ? win[n / 2] : 0.5 * (win[n / 2 - 1] + win[n / 2]);
}

// ---- min inpaint
__device__ __forceinline__ int findRoot(const int* p, int x) {
  int y = p[x];
  while (y != x) {
    x = y;
    y = p[x];
  }
  return x;
}

__device__ void unite(int* p, int a, int b) {
  while (true) {
    a = findRoot(p, a);
    b = findRoot(p, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicCAS(p + b, b, a);
    if (old == b) return;
    b = old;
  }
}

__device__ __forceinline__ unsigned long long orderKey(double v) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double fromKey(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

__global__ void __launch_bounds__(kT) k_cc_init(const uint8_t* ok, int n, int* parent,
                                                unsigned long long* key, uint8_t* border,
                                                int* any_valid) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= n) return;
  parent[i] = i;
  key[i] = 0xfff0000000000000ULL;  // orderKey(+inf)
  border[i] = 0;
  if (ok[i]) *any_valid = 1;
}

__global__ void __launch_bounds__(kT) k_cc_union(const uint8_t* ok, int W, int H, int* parent) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= W * H || ok[i]) return;
  const int r = i / W, c = i - (i / W) * W;
  if (c + 1 < W && !ok[i + 1]) unite(parent, i, i + 1);
  if (r + 1 < H && !ok[i + W]) unite(parent, i, i + W);
}

__global__ void __launch_bounds__(kT) k_cc_border(const double* v, const uint8_t* ok, int W, int H,
                                                  int* parent, unsigned long long* key,
                                                  uint8_t* border) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= W * H || ok[i]) return;
  const int root = findRoot(parent, i);
  parent[i] = root;
  const int r = i / W, c = i - (i / W) * W;
  bool any = false;
  unsigned long long best = 0xfff0000000000000ULL;
  for (int dr = -1; dr <= 1; ++dr) {
    for (int dc = -1; dc <= 1; ++dc) {
      if (dr == 0 && dc == 0) continue;
      const int rr = r + dr, cc = c + dc;
      if (rr < 0 || rr >= H || cc < 0 || cc >= W) continue;
      const int j = rr * W + cc;
      if (!ok[j]) continue;
      any = true;
      const double x = v[j];
      if (x == x) {
        const unsigned long long kx = orderKey(x);
        if (kx < best) best = kx;
      }
    }
  }
  if (any) {
    border[root] = 1;
    if (best < 0xfff0000000000000ULL) atomicMin(key + root, best);
  }
}

__global__ void __launch_bounds__(kT) k_cc_fill(const double* v, const uint8_t* ok, int n,
                                                const int* parent, const unsigned long long* key,
                                                const uint8_t* border, double* out,
                                                uint8_t* ok_out) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= n) return;
  if (ok[i]) {
    out[i] = v[i];
    ok_out[i] = 1;
    return;
  }
  const int root = findRoot(parent, i);
  if (border[root]) {
    out[i] = fromKey(key[root]);
    ok_out[i] = 1;
  } else {
    out[i] = v[i];
    ok_out[i] = 0;
  }
}

}  // namespace

void smoothChainDevice(int device, cudaStream_t s, const double* d_values, const uint8_t* d_valid,
                       int W, int H, const ChainStep* steps, int n_steps, double* d_values_out,
                       uint8_t* d_valid_out) {
  checkCuda(cudaSetDevice(device), "cudaSetDevice");
  if (W <= 0 || H <= 0) fail(Err::kUsage, "malformed masked layer");
  const int n = W * H;
  const unsigned grid = static_cast<unsigned>((n + kT - 1) / kT);
  double *va = nullptr, *vb = nullptr, *w = nullptr;
  uint8_t *oa = nullptr, *ob = nullptr, *border = nullptr;
  int *parent = nullptr, *flag = nullptr;
  unsigned long long* key = nullptr;
  struct Free {
    std::vector<void*> ptrs;
    ~Free() {
      for (void* p : ptrs) cudaFree(p);
    }
  } guard;
  const auto alloc = [&](auto** p, std::size_t bytes) {
    checkCuda(cudaMalloc(reinterpret_cast<void**>(p), bytes), "chain scratch");
    guard.ptrs.push_back(*p);
  };
  alloc(&va, n * sizeof(double));
  alloc(&vb, n * sizeof(double));
  alloc(&oa, n);
  alloc(&ob, n);
  checkCuda(cudaMemcpyAsync(va, d_values, n * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy");
  checkCuda(cudaMemcpyAsync(oa, d_valid, n, cudaMemcpyDeviceToDevice, s), "copy");
  for (int k = 0; k < n_steps; ++k) {
    const ChainStep& st = steps[k];
    if (st.kind != 3 && st.radius < 1) fail(Err::kUsage, "filter radius must be >= 1");
    if (st.kind == 0 && !(st.sigma > 0.0)) fail(Err::kUsage, "gaussian sigma must be > 0");
    if (st.kind == 0 || st.kind == 1) {
      const int kk = 2 * st.radius + 1;
      std::vector<double> hw(static_cast<std::size_t>(kk) * kk, 1.0);
      if (st.kind == 0)
        for (int dr = -st.radius; dr <= st.radius; ++dr)
          for (int dc = -st.radius; dc <= st.radius; ++dc)
            hw[static_cast<std::size_t>(dr + st.radius) * kk + (dc + st.radius)] =
                std::exp(-(dr * dr + dc * dc) / (2.0 * st.sigma * st.sigma));  // host libm
      cudaFree(w);
      w = nullptr;
      checkCuda(cudaMalloc(&w, hw.size() * sizeof(double)), "weights");
      checkCuda(cudaMemcpyAsync(w, hw.data(), hw.size() * sizeof(double), cudaMemcpyHostToDevice, s),
                "weights");
      k_linear<<<grid, kT, 0, s>>>(va, oa, W, H, st.radius, w, vb);
      checkCuda(cudaMemcpyAsync(ob, oa, n, cudaMemcpyDeviceToDevice, s), "copy");
      checkCuda(cudaStreamSynchronize(s), "linear step");
    } else if (st.kind == 2) {
      if ((2 * st.radius + 1) * (2 * st.radius + 1) > kMaxMedianWindow)
        fail(Err::kUsage, "median radius above 5 is not supported");
      k_median<<<grid, kT, 0, s>>>(va, oa, W, H, st.radius, vb);
      checkCuda(cudaMemcpyAsync(ob, oa, n, cudaMemcpyDeviceToDevice, s), "copy");
    } else {
      if (parent == nullptr) {
        alloc(&parent, n * sizeof(int));
        alloc(&key, n * sizeof(unsigned long long));
        alloc(&border, n);
        alloc(&flag, sizeof(int));
      }
      checkCuda(cudaMemsetAsync(flag, 0, sizeof(int), s), "memset");
      k_cc_init<<<grid, kT, 0, s>>>(oa, n, parent, key, border, flag);
      int any = 0;
      checkCuda(cudaMemcpyAsync(&any, flag, sizeof(int), cudaMemcpyDeviceToHost, s), "flag");
      checkCuda(cudaStreamSynchronize(s), "inpaint");
      if (!any) fail(Err::kNothingToInpaint, "layer has no valid cells");
      k_cc_union<<<grid, kT, 0, s>>>(oa, W, H, parent);
      k_cc_border<<<grid, kT, 0, s>>>(va, oa, W, H, parent, key, border);
      k_cc_fill<<<grid, kT, 0, s>>>(va, oa, n, parent, key, border, vb, ob);
    }
    checkCuda(cudaGetLastError(), "chain step");
    std::swap(va, vb);
    std::swap(oa, ob);
  }
  checkCuda(cudaMemcpyAsync(d_values_out, va, n * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy");
  checkCuda(cudaMemcpyAsync(d_valid_out, oa, n, cudaMemcpyDeviceToDevice, s), "copy");
  checkCuda(cudaStreamSynchronize(s), "chain");
  cudaFree(w);
}

namespace {
std::vector<ChainStep> makeSteps(const int* kinds, const int* radii, const double* sigmas, int n) {
  std::vector<ChainStep> steps(n > 0 ? n : 0);
  for (int k = 0; k < n; ++k) {
    if (kinds[k] < 0 || kinds[k] > 3) fail(Err::kUsage, "unknown filter kind");
    steps[k] = {kinds[k], radii[k], sigmas[k]};
  }
  return steps;
}
}  // namespace

void runHostChain(int device, const double* values, const uint8_t* valid, int W, int H,
                  const int* kinds, const int* radii, const double* sigmas, int n_steps,
                  double* values_out, uint8_t* valid_out) {
  if (W <= 0 || H <= 0) fail(Err::kUsage, "malformed masked layer");
  const std::vector<ChainStep> steps = makeSteps(kinds, radii, sigmas, n_steps);
  checkCuda(cudaSetDevice(device), "cudaSetDevice");
  const std::size_t n = static_cast<std::size_t>(W) * H;
  double* dv = nullptr;
  uint8_t* dm = nullptr;
  checkCuda(cudaMalloc(&dv, n * sizeof(double)), "chain input");
  if (cudaMalloc(&dm, n) != cudaSuccess) {
    cudaFree(dv);
    fail(Err::kDevice, "chain input allocation failed");
  }
  try {
    checkCuda(cudaMemcpy(dv, values, n * sizeof(double), cudaMemcpyHostToDevice), "upload");
    checkCuda(cudaMemcpy(dm, valid, n, cudaMemcpyHostToDevice), "upload");
    smoothChainDevice(device, nullptr, dv, dm, W, H, steps.data(), n_steps, dv, dm);
    checkCuda(cudaMemcpy(values_out, dv, n * sizeof(double), cudaMemcpyDeviceToHost), "download");
    checkCuda(cudaMemcpy(valid_out, dm, n, cudaMemcpyDeviceToHost), "download");
  } catch (...) {
    cudaFree(dv);
    cudaFree(dm);
    throw;
  }
  cudaFree(dv);
  cudaFree(dm);
}

void runMapChain(DeviceMap& m, const std::string& layer, const int* kinds, const int* radii,
                 const double* sigmas, int n_steps, double* values_out, uint8_t* valid_out) {
  const std::vector<ChainStep> steps = makeSteps(kinds, radii, sigmas, n_steps);
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  const std::size_t n = m.grid.cells();
  double* dv = nullptr;
  uint8_t* dm = nullptr;
  checkCuda(cudaMalloc(&dv, n * sizeof(double)), "chain input");
  if (cudaMalloc(&dm, n) != cudaSuccess) {
    cudaFree(dv);
    fail(Err::kDevice, "chain input allocation failed");
  }
  try {
    if (!exportLayerDevice(m, layer.c_str(), dv)) fail(Err::kUsage, "unknown layer '" + layer + "'");
    const uint8_t* mask = layer == "upper_bound" ? m.cur.ubv : m.cur.valid;
    checkCuda(cudaMemcpyAsync(dm, mask, n, cudaMemcpyDeviceToDevice, m.stream), "mask");
    smoothChainDevice(m.device, m.stream, dv, dm, m.grid.width, m.grid.height, steps.data(),
                      n_steps, dv, dm);
    checkCuda(cudaMemcpy(values_out, dv, n * sizeof(double), cudaMemcpyDeviceToHost), "download");
    checkCuda(cudaMemcpy(valid_out, dm, n, cudaMemcpyDeviceToHost), "download");
  } catch (...) {
    cudaFree(dv);
    cudaFree(dm);
    throw;
  }
  cudaFree(dv);
  cudaFree(dm);
}

}  // namespace rb200
