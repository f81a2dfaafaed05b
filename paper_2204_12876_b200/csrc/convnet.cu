// Conv-net traversability on the device (reference analysis.cpp:138-216,
// used by integration.cpp:242-244 when use_convnet_traversability):
//
//   1. fillNearestValid: invalid cells take the value of the cell that claims
//      them in a multi-source 8-neighbour BFS seeded with the valid cells in
//      index order. The BFS queue is ordered by (root index, offset chain)
//      lexicographically -- level 0 is index order, and each level is ordered
//      by (parent rank, neighbour offset) -- so the first neighbour popped is
//      the previous-level neighbour with the smallest ROOT. Hence the filled
//      value is elev[root(j)] with root(j) = min over previous-level
//      neighbours p of root(p): an order-free min that a level-synchronous
//      device BFS computes exactly with atomicMin (levels = Chebyshev distance
//      to the nearest valid cell). One cooperative persistent kernel runs all
//      levels with a grid barrier between them.
//   2. the layer stack: k x k border-replicate convolution, acc = bias then
//      acc += w * x in (kr, kc) row-major order (fp64, no FMA: bit-exact),
//      relu / sigmoid / identity, and the final clamp to [0, 1]. Every cell is
//      written, valid or not (test_io.cpp:237-238). Sigmoid uses the device
//      exp (≤ 1 ulp from glibc's), the only inexact step.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "device_map.hpp"
#include "fp_exact.cuh"

namespace cg = cooperative_groups;

namespace rb200 {

namespace {

constexpr int kThreads = 256;
constexpr uint32_t kUnknown = 0xffffffffu;
constexpr int kConvTX = 32, kConvTY = 8;

// Level 0: every valid cell, its own root. Queue order is irrelevant here:
// the min-root rule makes the result independent of it.
__global__ void __launch_bounds__(kThreads)
    k_cn_seed(const uint8_t* __restrict__ valid, uint32_t n, uint32_t* __restrict__ level,
              uint32_t* __restrict__ root, uint32_t* __restrict__ frontier, uint32_t* cnt) {
  const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  const bool v = i < n && valid[i] != 0;
  if (i < n) {
    level[i] = v ? 0u : kUnknown;
    root[i] = v ? i : kUnknown;
  }
  const unsigned mask = __ballot_sync(0xffffffffu, v);
  if (mask == 0) return;
  const int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(cnt, static_cast<uint32_t>(__popc(mask)));
  base = __shfl_sync(0xffffffffu, base, __ffs(mask) - 1);
  if (v) frontier[base + __popc(mask & ((1u << lane) - 1u))] = i;
}

// All BFS levels. cnt[d % 3] holds the size of level d; the counter of level
// d + 2 is cleared while level d is expanded (nobody reads or writes it then).
__global__ void __launch_bounds__(kThreads)
    k_cn_bfs(uint32_t* level, uint32_t* root, uint32_t* fa, uint32_t* fb, uint32_t* cnt, int W,
             int H) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t stride = gridDim.x * kThreads;
  const uint32_t tid = blockIdx.x * kThreads + threadIdx.x;
  for (uint32_t d = 1;; ++d) {
    const uint32_t n = *reinterpret_cast<volatile uint32_t*>(&cnt[(d - 1) % 3]);
    if (n == 0) break;
    const uint32_t* cur = (d & 1) ? fa : fb;
    uint32_t* nxt = (d & 1) ? fb : fa;
    uint32_t* ncnt = &cnt[d % 3];
    if (tid == 0) cnt[(d + 1) % 3] = 0;
    for (uint32_t q = tid; q < n; q += stride) {
      const uint32_t p = cur[q];
      const uint32_t rp = root[p];
      const int r = static_cast<int>(p / static_cast<uint32_t>(W));
      const int c = static_cast<int>(p - static_cast<uint32_t>(r) * W);
      for (int dr = -1; dr <= 1; ++dr) {
        const int rr = r + dr;
        if (rr < 0 || rr >= H) continue;
        for (int dc = -1; dc <= 1; ++dc) {
          const int cc = c + dc;
          if ((dr == 0 && dc == 0) || cc < 0 || cc >= W) continue;
          const uint32_t j = static_cast<uint32_t>(rr) * W + cc;
          uint32_t lv = *reinterpret_cast<volatile uint32_t*>(&level[j]);
          if (lv < d) continue;  // reached at an earlier level
          if (lv == kUnknown) {
            lv = atomicCAS(&level[j], kUnknown, d);
            if (lv == kUnknown) nxt[atomicAdd(ncnt, 1u)] = j;
            else if (lv < d) continue;
          }
          atomicMin(&root[j], rp);
        }
      }
    }
    grid.sync();
  }
}

__global__ void __launch_bounds__(kThreads)
    k_cn_gather(const double* __restrict__ elev, const uint32_t* __restrict__ root, uint32_t n,
                double* __restrict__ out) {
  const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= n) return;
  const uint32_t r = root[i];
  out[i] = r == kUnknown ? 0.0 : elev[r];  // no valid cell at all: zeros
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
    cudaFree(root);
    cudaFree(level);
    cudaFree(fa);
    cudaFree(fb);
    cudaFree(va);
    cudaFree(vb);
    root = level = fa = fb = nullptr;
    va = vb = nullptr;
    checkCuda(cudaMalloc(&root, n * sizeof(uint32_t)), "convnet scratch");
    checkCuda(cudaMalloc(&level, n * sizeof(uint32_t)), "convnet scratch");
    checkCuda(cudaMalloc(&fa, n * sizeof(uint32_t)), "convnet scratch");
    checkCuda(cudaMalloc(&fb, n * sizeof(uint32_t)), "convnet scratch");
    checkCuda(cudaMalloc(&va, n * sizeof(double)), "convnet scratch");
    checkCuda(cudaMalloc(&vb, n * sizeof(double)), "convnet scratch");
    cap = n;
  }
  if (cnt == nullptr) checkCuda(cudaMalloc(&cnt, 4 * sizeof(uint32_t)), "convnet scratch");
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
  cudaFree(root);
  cudaFree(level);
  cudaFree(fa);
  cudaFree(fb);
  cudaFree(va);
  cudaFree(vb);
  cudaFree(cnt);
  cudaFree(weights);
  if (h_weights) cudaFreeHost(h_weights);
  if (upload_done) cudaEventDestroy(upload_done);
  upload_done = nullptr;
  root = level = fa = fb = cnt = nullptr;
  va = vb = weights = h_weights = nullptr;
  cap = wcap = 0;
  bfs_blocks = 0;
}

int convnetEnqueue(cudaStream_t s, ConvScratch& cs, const double* d_layer, const uint8_t* d_valid,
                   int W, int H, const ConvNetSpec& spec, double* d_out) {
  spec.validate();
  if (W <= 0 || H <= 0) fail(Err::kUsage, "layer size does not match grid dimensions");
  const std::size_t n = static_cast<std::size_t>(W) * H;
  if (n >= kUnknown) fail(Err::kUsage, "layer too large for the conv-net executor");
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
  checkCuda(cudaMemsetAsync(cs.cnt, 0, 4 * sizeof(uint32_t), s), "memset");
  const unsigned nb = static_cast<unsigned>((n + kThreads - 1) / kThreads);
  k_cn_seed<<<nb, kThreads, 0, s>>>(d_valid, static_cast<uint32_t>(n), cs.level, cs.root, cs.fa,
                                     cs.cnt);
  ++launches;
  if (cs.bfs_blocks == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    checkCuda(cudaGetDevice(&dev), "device");
    checkCuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attribute");
    checkCuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cn_bfs, kThreads, 0),
              "occupancy");
    cs.bfs_blocks = std::max(1, sms * std::min(per_sm, 4));
  }
  {
    int Wi = W, Hi = H;
    void* args[] = {&cs.level, &cs.root, &cs.fa, &cs.fb, &cs.cnt, &Wi, &Hi};
    checkCuda(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_cn_bfs), dim3(cs.bfs_blocks),
                                          dim3(kThreads), args, 0, s),
              "convnet fill launch");
    ++launches;
  }
  k_cn_gather<<<nb, kThreads, 0, s>>>(d_layer, cs.root, static_cast<uint32_t>(n), cs.va);
  ++launches;

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
    if (smem <= 200 * 1024) {
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
