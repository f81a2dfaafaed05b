// Conv-net traversability on the device (reference analysis.cpp:138-216,
// used by integration.cpp:242-244 when use_convnet_traversability):
//
//   1. fillNearestValid: invalid cells take the value of the cell that claims
//      them in a multi-source 8-neighbour BFS seeded with the valid cells in
//      index order. The BFS queue is ordered by (root index, offset chain)
//      lexicographically -- level 0 is index order, and each level is ordered
//      by (parent rank, neighbour offset) -- so the first neighbour popped is
//      the previous-level neighbour with the smallest ROOT, and by induction
//      root(j) = the smallest index among the valid cells at the minimum
//      Chebyshev distance D from j (the BFS level of j: on a full grid every
//      source at distance D lies on a shortest 8-path to j). No BFS is run:
//        * D = the smallest k whose (2k+1)^2 square around j holds a valid
//          cell -- binary search over k with O(1) square counts from a
//          summed-area table of the validity mask;
//        * the sources at distance exactly D lie on the square ring of radius
//          D, so the smallest index is the first hit among: the top row
//          (next valid column >= c-D within c+D), then the two side columns
//          (next valid row >= r-D+1 within r+D-1, left column first on a tie),
//          then the bottom row -- O(1) with per-row "next valid column" and
//          per-column "next valid row" tables.
//   2. the layer stack: k x k border-replicate convolution, acc = bias then
//      acc += w * x in (kr, kc) row-major order (fp64, no FMA: bit-exact),
//      relu / sigmoid / identity, and the final clamp to [0, 1]. Every cell is
//      written, valid or not (test_io.cpp:237-238). Sigmoid uses the device
//      exp (≤ 1 ulp from glibc's), the only inexact step.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "device_map.hpp"
#include "fp_exact.cuh"

namespace rb200 {

namespace {

constexpr int kThreads = 256;
constexpr int kConvTX = 32, kConvTY = 8;

// Per row (one warp each): inclusive prefix count of valid cells (the first
// summed-area pass) and next_col[r][c] = smallest valid column >= c (W if none).
__global__ void __launch_bounds__(kThreads)
    k_cn_rows(const uint8_t* __restrict__ valid, int W, int H, uint32_t* __restrict__ sat,
              uint32_t* __restrict__ next_col) {
  const int r = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= H) return;
  const size_t row = static_cast<size_t>(r) * W;
  uint32_t carry = 0;
  for (int c0 = 0; c0 < W; c0 += 32) {
    const int c = c0 + lane;
    uint32_t v = (c < W && valid[row + c]) ? 1u : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    if (c < W) sat[row + c] = carry + v;
    carry += __shfl_sync(0xffffffffu, v, 31);
  }
  uint32_t next = static_cast<uint32_t>(W);
  for (int c0 = ((W - 1) / 32) * 32; c0 >= 0; c0 -= 32) {
    const int c = c0 + lane;
    uint32_t v = (c < W && valid[row + c]) ? static_cast<uint32_t>(c) : next;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_down_sync(0xffffffffu, v, o);
      if (lane + o < 32) v = min(v, t);
    }
    if (c < W) next_col[row + c] = v;
    next = __shfl_sync(0xffffffffu, v, 0);
  }
}

// Per column: the second summed-area pass and next_row[r][c] = smallest valid
// row >= r in column c (H if none). A block covers 32 columns (lanes) x 32
// row strips (warps): strip totals / first valid rows are combined through
// shared memory, then each strip is rewritten with its carry.
constexpr int kStrips = 32;
__global__ void __launch_bounds__(32 * kStrips)
    k_cn_cols(const uint8_t* __restrict__ valid, int W, int H, uint32_t* __restrict__ sat,
              uint32_t* __restrict__ next_row) {
  __shared__ uint32_t s_sum[kStrips][33];
  __shared__ uint32_t s_first[kStrips][33];
  const int lane = threadIdx.x & 31, strip = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  const int len = (H + kStrips - 1) / kStrips;
  const int rb = strip * len, re = min(rb + len, H);
  uint32_t sum = 0, first = static_cast<uint32_t>(H);
  if (c < W) {
    for (int r = rb; r < re; ++r) {
      const size_t i = static_cast<size_t>(r) * W + c;
      sum += sat[i];
      if (first == static_cast<uint32_t>(H) && valid[i]) first = static_cast<uint32_t>(r);
    }
  }
  s_sum[strip][lane] = sum;
  s_first[strip][lane] = first;
  __syncthreads();
  if (c >= W) return;
  uint32_t acc = 0, next = static_cast<uint32_t>(H);
  for (int k = 0; k < strip; ++k) acc += s_sum[k][lane];
  for (int k = kStrips - 1; k > strip; --k) next = min(next, s_first[k][lane]);
  for (int r = rb; r < re; ++r) {
    const size_t i = static_cast<size_t>(r) * W + c;
    acc += sat[i];
    sat[i] = acc;
  }
  for (int r = re - 1; r >= rb; --r) {
    const size_t i = static_cast<size_t>(r) * W + c;
    if (valid[i]) next = static_cast<uint32_t>(r);
    next_row[i] = next;
  }
}

struct FillTables {
  const uint8_t* valid;
  const uint32_t* sat;
  const uint32_t* next_col;
  const uint32_t* next_row;
  int W, H;
};

// Valid cells in rows [r1, r2] x cols [c1, c2] (already clipped to the grid).
__device__ __forceinline__ uint32_t squareCount(const FillTables& t, int r1, int c1, int r2, int c2) {
  const uint32_t* S = t.sat;
  const int W = t.W;
  uint32_t v = S[static_cast<size_t>(r2) * W + c2];
  if (r1 > 0) v -= S[static_cast<size_t>(r1 - 1) * W + c2];
  if (c1 > 0) v -= S[static_cast<size_t>(r2) * W + c1 - 1];
  if (r1 > 0 && c1 > 0) v += S[static_cast<size_t>(r1 - 1) * W + c1 - 1];
  return v;
}

// fillNearestValid + the first conv layer's input: out[i] = layer[root(i)].
__global__ void __launch_bounds__(kThreads)
    k_cn_fill(FillTables t, const double* __restrict__ layer, double* __restrict__ out) {
  const size_t i = blockIdx.x * static_cast<size_t>(kThreads) + threadIdx.x;
  const int W = t.W, H = t.H;
  if (i >= static_cast<size_t>(W) * H) return;
  if (t.valid[i]) {
    out[i] = layer[i];
    return;
  }
  const uint32_t total = t.sat[static_cast<size_t>(W) * H - 1];
  if (total == 0) {
    out[i] = 0.0;  // no valid cell at all
    return;
  }
  const int r = static_cast<int>(i / W), c = static_cast<int>(i % W);
  // smallest D >= 1 with a valid cell in the square of radius D
  int lo = 1, hi = max(max(r, H - 1 - r), max(c, W - 1 - c));
  while (lo < hi) {
    const int k = (lo + hi) >> 1;
    if (squareCount(t, max(r - k, 0), max(c - k, 0), min(r + k, H - 1), min(c + k, W - 1)) > 0)
      hi = k;
    else
      lo = k + 1;
  }
  const int D = lo;
  const int cl = max(c - D, 0), cr = min(c + D, W - 1);
  size_t root;
  if (r - D >= 0 && t.next_col[static_cast<size_t>(r - D) * W + cl] <= static_cast<uint32_t>(cr)) {
    root = static_cast<size_t>(r - D) * W + t.next_col[static_cast<size_t>(r - D) * W + cl];
  } else {
    root = ~static_cast<size_t>(0);
    const int top = max(r - D + 1, 0), bottom = min(r + D - 1, H - 1);
    if (c - D >= 0) {
      const uint32_t y = t.next_row[static_cast<size_t>(top) * W + (c - D)];
      if (y <= static_cast<uint32_t>(bottom)) root = static_cast<size_t>(y) * W + (c - D);
    }
    if (c + D < W) {
      const uint32_t y = t.next_row[static_cast<size_t>(top) * W + (c + D)];
      if (y <= static_cast<uint32_t>(bottom))
        root = min(root, static_cast<size_t>(y) * W + (c + D));
    }
    if (root == ~static_cast<size_t>(0))  // bottom row (exists: D is the minimum distance)
      root = static_cast<size_t>(r + D) * W + t.next_col[static_cast<size_t>(r + D) * W + cl];
  }
  out[i] = layer[root];
}

__device__ __forceinline__ double activate(double x, int act) {
  if (act == static_cast<int>(Activation::kRelu)) return x > 0.0 ? x : 0.0;
  if (act == static_cast<int>(Activation::kSigmoid)) return 1.0 / (1.0 + exp(-x));
  return x;
}

// One layer over a 32x8 output tile; the (k-1)/2 halo is staged in shared
// memory with border replication.
__global__ void __launch_bounds__(kConvTX* kConvTY)
    k_cn_conv(const double* __restrict__ in, double* __restrict__ out, int W, int H,
              const double* __restrict__ w, int k, double bias, int act, int clamp01) {
  extern __shared__ double tile[];
  const int rad = k / 2;
  const int tw = kConvTX + 2 * rad, th = kConvTY + 2 * rad;
  const int c0 = blockIdx.x * kConvTX - rad, r0 = blockIdx.y * kConvTY - rad;
  const int tid = threadIdx.y * kConvTX + threadIdx.x;
  for (int q = tid; q < tw * th; q += kConvTX * kConvTY) {
    const int rr = min(max(r0 + q / tw, 0), H - 1);
    const int cc = min(max(c0 + q % tw, 0), W - 1);
    tile[q] = in[static_cast<size_t>(rr) * W + cc];
  }
  __syncthreads();
  const int r = blockIdx.y * kConvTY + threadIdx.y, c = blockIdx.x * kConvTX + threadIdx.x;
  if (r >= H || c >= W) return;
  double acc = bias;
  for (int kr = 0; kr < k; ++kr) {
    const double* trow = tile + (threadIdx.y + kr) * tw + threadIdx.x;
    const double* wrow = w + kr * k;
    for (int kc = 0; kc < k; ++kc) acc = acc + __ldg(wrow + kc) * trow[kc];
  }
  double v = activate(acc, act);
  if (clamp01) v = sclamp(v, 0.0, 1.0);
  out[static_cast<size_t>(r) * W + c] = v;
}

// Fixed-K layer: each thread produces 4 outputs of one tile row at columns
// tx, tx+32, tx+64, tx+96 (conflict-free shared loads), so every weight read
// from shared memory feeds 4 multiply-adds; the (kr, kc) loops are unrolled.
// Each output still sums bias + w*x in (kr, kc) row-major order.
constexpr int kWideX = 4 * kConvTX;
template <int K>
__global__ void __launch_bounds__(kConvTX* kConvTY)
    k_cn_conv_k(const double* __restrict__ in, double* __restrict__ out, int W, int H,
                const double* __restrict__ w, double bias, int act, int clamp01) {
  constexpr int R = K / 2, TW = kWideX + 2 * R, TH = kConvTY + 2 * R;
  __shared__ double tile[TW * TH];
  __shared__ double sw[K * K];
  const int c0 = blockIdx.x * kWideX - R, r0 = blockIdx.y * kConvTY - R;
  const int tid = threadIdx.y * kConvTX + threadIdx.x;
  for (int q = tid; q < K * K; q += kConvTX * kConvTY) sw[q] = w[q];
  for (int q = tid; q < TW * TH; q += kConvTX * kConvTY) {
    const int rr = min(max(r0 + q / TW, 0), H - 1);
    const int cc = min(max(c0 + q % TW, 0), W - 1);
    tile[q] = in[static_cast<size_t>(rr) * W + cc];
  }
  __syncthreads();
  double acc[4] = {bias, bias, bias, bias};
#pragma unroll
  for (int kr = 0; kr < K; ++kr) {
    const double* trow = tile + (threadIdx.y + kr) * TW + threadIdx.x;
#pragma unroll
    for (int kc = 0; kc < K; ++kc) {
      const double wv = sw[kr * K + kc];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = acc[j] + wv * trow[kc + 32 * j];
    }
  }
  const int r = blockIdx.y * kConvTY + threadIdx.y;
  if (r >= H) return;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = blockIdx.x * kWideX + threadIdx.x + 32 * j;
    if (c >= W) continue;
    double v = activate(acc[j], act);
    if (clamp01) v = sclamp(v, 0.0, 1.0);
    out[static_cast<size_t>(r) * W + c] = v;
  }
}

template <int K>
void launchConvK(cudaStream_t s, const double* in, double* out, int W, int H, const double* w,
                 double bias, int act, int clamp01) {
  const dim3 grid((W + kWideX - 1) / kWideX, (H + kConvTY - 1) / kConvTY);
  k_cn_conv_k<K><<<grid, dim3(kConvTX, kConvTY), 0, s>>>(in, out, W, H, w, bias, act, clamp01);
}

// Same layer straight from global memory, for kernels whose halo tile would
// not fit in shared memory.
__global__ void __launch_bounds__(kThreads)
    k_cn_conv_global(const double* __restrict__ in, double* __restrict__ out, int W, int H,
                     const double* __restrict__ w, int k, double bias, int act, int clamp01) {
  const size_t i = blockIdx.x * static_cast<size_t>(kThreads) + threadIdx.x;
  if (i >= static_cast<size_t>(W) * H) return;
  const int r = static_cast<int>(i / W), c = static_cast<int>(i % W);
  const int rad = k / 2;
  double acc = bias;
  for (int kr = -rad; kr <= rad; ++kr) {
    const int rr = min(max(r + kr, 0), H - 1);
    for (int kc = -rad; kc <= rad; ++kc) {
      const int cc = min(max(c + kc, 0), W - 1);
      acc = acc + __ldg(w + (kr + rad) * k + (kc + rad)) * in[static_cast<size_t>(rr) * W + cc];
    }
  }
  double v = activate(acc, act);
  if (clamp01) v = sclamp(v, 0.0, 1.0);
  out[i] = v;
}

}  // namespace

void ConvScratch::ensure(std::size_t n, std::size_t n_weights) {
  if (n > cap) {
    cudaFree(sat);
    cudaFree(next_col);
    cudaFree(next_row);
    cudaFree(va);
    cudaFree(vb);
    sat = next_col = next_row = nullptr;
    va = vb = nullptr;
    checkCuda(cudaMalloc(&sat, n * sizeof(uint32_t)), "convnet scratch");
    checkCuda(cudaMalloc(&next_col, n * sizeof(uint32_t)), "convnet scratch");
    checkCuda(cudaMalloc(&next_row, n * sizeof(uint32_t)), "convnet scratch");
    checkCuda(cudaMalloc(&va, n * sizeof(double)), "convnet scratch");
    checkCuda(cudaMalloc(&vb, n * sizeof(double)), "convnet scratch");
    cap = n;
  }
  if (n_weights > wcap) {
    cudaFree(weights);
    cudaFreeHost(h_weights);
    weights = h_weights = nullptr;
    checkCuda(cudaMalloc(&weights, n_weights * sizeof(double)), "convnet weights");
    checkCuda(cudaMallocHost(&h_weights, n_weights * sizeof(double)), "convnet weights");
    wcap = n_weights;
  }
}

void ConvScratch::release() {
  cudaFree(sat);
  cudaFree(next_col);
  cudaFree(next_row);
  cudaFree(va);
  cudaFree(vb);
  cudaFree(weights);
  if (h_weights) cudaFreeHost(h_weights);
  if (upload_done) cudaEventDestroy(upload_done);
  upload_done = nullptr;
  sat = next_col = next_row = nullptr;
  va = vb = weights = h_weights = nullptr;
  cap = wcap = 0;
}

int convnetEnqueue(cudaStream_t s, ConvScratch& cs, const double* d_layer, const uint8_t* d_valid,
                   int W, int H, const ConvNetSpec& spec, double* d_out) {
  spec.validate();
  if (W <= 0 || H <= 0) fail(Err::kUsage, "layer size does not match grid dimensions");
  const std::size_t n = static_cast<std::size_t>(W) * H;
  if (n >= 0xffffffffu) fail(Err::kUsage, "layer too large for the conv-net executor");
  std::size_t nw = 0;
  for (const ConvLayer& l : spec.layers) nw += l.kernel.size();
  // Weights are staged through pinned memory; the previous call's copy may
  // still be in flight, so wait for it before the staging buffer is touched.
  if (cs.upload_done) checkCuda(cudaEventSynchronize(cs.upload_done), "convnet weights");
  else checkCuda(cudaEventCreateWithFlags(&cs.upload_done, cudaEventDisableTiming), "event");
  cs.ensure(n, nw);
  int launches = 0;
  std::size_t off = 0;
  for (const ConvLayer& l : spec.layers) {
    std::copy(l.kernel.begin(), l.kernel.end(), cs.h_weights + off);
    off += l.kernel.size();
  }
  checkCuda(cudaMemcpyAsync(cs.weights, cs.h_weights, nw * sizeof(double), cudaMemcpyHostToDevice, s),
            "convnet weights");
  checkCuda(cudaEventRecord(cs.upload_done, s), "event");

  // 1. nearest-valid fill.
  k_cn_rows<<<(H + kThreads / 32 - 1) / (kThreads / 32), kThreads, 0, s>>>(d_valid, W, H, cs.sat,
                                                                           cs.next_col);
  k_cn_cols<<<(W + 31) / 32, 32 * kStrips, 0, s>>>(d_valid, W, H, cs.sat, cs.next_row);
  const unsigned nb = static_cast<unsigned>((n + kThreads - 1) / kThreads);
  k_cn_fill<<<nb, kThreads, 0, s>>>(FillTables{d_valid, cs.sat, cs.next_col, cs.next_row, W, H},
                                    d_layer, cs.va);
  launches += 3;

  // 2. the layer stack; the last layer clamps and writes the output.
  const double* cur = cs.va;
  off = 0;
  for (std::size_t li = 0; li < spec.layers.size(); ++li) {
    const ConvLayer& l = spec.layers[li];
    const bool last = li + 1 == spec.layers.size();
    double* dst = last ? d_out : (cur == cs.va ? cs.vb : cs.va);
    const int rad = l.kernel_size / 2;
    const std::size_t smem =
        static_cast<std::size_t>(kConvTX + 2 * rad) * (kConvTY + 2 * rad) * sizeof(double);
    const int act = static_cast<int>(l.activation);
    const double* wl = cs.weights + off;
    switch (l.kernel_size) {
      case 1: launchConvK<1>(s, cur, dst, W, H, wl, l.bias, act, last); break;
      case 3: launchConvK<3>(s, cur, dst, W, H, wl, l.bias, act, last); break;
      case 5: launchConvK<5>(s, cur, dst, W, H, wl, l.bias, act, last); break;
      case 7: launchConvK<7>(s, cur, dst, W, H, wl, l.bias, act, last); break;
      case 9: launchConvK<9>(s, cur, dst, W, H, wl, l.bias, act, last); break;
      case 11: launchConvK<11>(s, cur, dst, W, H, wl, l.bias, act, last); break;
      default: break;
    }
    if (l.kernel_size <= 11) {
      // launched above
    } else if (smem <= 200 * 1024) {
      if (smem > 48 * 1024)
        checkCuda(cudaFuncSetAttribute(k_cn_conv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)),
                  "smem attribute");
      const dim3 grid((W + kConvTX - 1) / kConvTX, (H + kConvTY - 1) / kConvTY);
      k_cn_conv<<<grid, dim3(kConvTX, kConvTY), smem, s>>>(cur, dst, W, H, cs.weights + off,
                                                           l.kernel_size, l.bias, act, last);
    } else {
      k_cn_conv_global<<<nb, kThreads, 0, s>>>(cur, dst, W, H, cs.weights + off, l.kernel_size,
                                               l.bias, act, last);
    }
    ++launches;
    off += l.kernel.size();
    cur = dst;
  }
  checkCuda(cudaGetLastError(), "convnet launch");
  return launches;
}

void runHostConvnet(int device, const ConvNetSpec& spec, const double* layer, const uint8_t* valid,
                    int W, int H, double* out) {
  spec.validate();
  if (W <= 0 || H <= 0) fail(Err::kUsage, "layer size does not match grid dimensions");
  checkCuda(cudaSetDevice(device), "cudaSetDevice");
  const std::size_t n = static_cast<std::size_t>(W) * H;
  ConvScratch cs;
  struct Guard {
    ConvScratch& cs;
    double* dl = nullptr;
    double* dout = nullptr;
    uint8_t* dv = nullptr;
    ~Guard() {
      cs.release();
      cudaFree(dl);
      cudaFree(dout);
      cudaFree(dv);
    }
  } g{cs};
  checkCuda(cudaMalloc(&g.dl, n * sizeof(double)), "convnet input");
  checkCuda(cudaMalloc(&g.dout, n * sizeof(double)), "convnet output");
  checkCuda(cudaMalloc(&g.dv, n), "convnet input");
  checkCuda(cudaMemcpy(g.dl, layer, n * sizeof(double), cudaMemcpyHostToDevice), "upload");
  checkCuda(cudaMemcpy(g.dv, valid, n, cudaMemcpyHostToDevice), "upload");
  convnetEnqueue(nullptr, cs, g.dl, g.dv, W, H, spec, g.dout);
  checkCuda(cudaMemcpy(out, g.dout, n * sizeof(double), cudaMemcpyDeviceToHost), "download");
}

}  // namespace rb200
