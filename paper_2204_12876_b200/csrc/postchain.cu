// Post-processing chain on the device (reference postprocess.cpp:29-197):
// min-inpaint, gaussian / box smoothing normalised over valid cells, and the
// valid-window median. Each step is one stencil launch over a masked layer;
// min-inpaint is a connected-component labelling (lock-free union-find over
// 4-neighbours) followed by a per-component atomic min over the 8-neighbour
// valid border. Sums run in the reference's row-major window order, the median
// sorts the same window values, and the inpaint minimum is order independent,
// so every step is bit-exact.
//
// Everything is enqueued on one stream with scratch owned by the caller (the
// map keeps one set), so a chain is a handful of launches and no host syncs;
// a "nothing to inpaint" condition is flagged on the device and raised after.
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "device_map.hpp"
#include "fp_exact.cuh"
#include "launch.cuh"
#include "stl_sort.cuh"
#include "runners.hpp"
#include "snapshot.hpp"

namespace rb200 {

namespace {

constexpr int kT = 256;
#ifndef RB_MEDIAN3
#define RB_MEDIAN3 1  // tiled 3x3 median with a median-of-9 network (k_median3)
#endif
constexpr int kMaxWindow = 121;  // radius <= 5

struct Weights {
  double w[kMaxWindow];
};

__global__ void __launch_bounds__(kT) k_linear(const double* __restrict__ v,
                                               const uint8_t* __restrict__ ok, int W, int H,
                                               int R, Weights wt, double* __restrict__ out,
                                               uint8_t* __restrict__ ok_out) {
  pdlEnter();
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= W * H) return;
  ok_out[i] = ok[i];
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
      const double w = wt.w[(dr + R) * k + (dc + R)];
      acc += w * v[j];
      ws += w;
    }
  }
  out[i] = acc / ws;
}

__global__ void __launch_bounds__(kT) k_median(const double* __restrict__ v,
                                               const uint8_t* __restrict__ ok, int W, int H,
                                               int R, double* __restrict__ out,
                                               uint8_t* __restrict__ ok_out) {
  pdlEnter();
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= W * H) return;
  ok_out[i] = ok[i];
  if (!ok[i]) {
    out[i] = v[i];
    return;
  }
  const int r = i / W, c = i - (i / W) * W;
  double win[kMaxWindow];
  int n = 0;
  for (int dr = -R; dr <= R; ++dr) {
    const int rr = r + dr;
    if (rr < 0 || rr >= H) continue;
    for (int dc = -R; dc <= R; ++dc) {
      const int cc = c + dc;
      if (cc < 0 || cc >= W) continue;
      const int j = rr * W + cc;
      if (!ok[j]) continue;
      win[n++] = v[j];
    }
  }
  stl::sort(win, n);  // the reference's std::sort, move for move (stl_sort.cuh)
  out[i] = (n % 2 == 1) ? win[n / 2] : 0.5 * (win[n / 2 - 1] + win[n / 2]);
}

// Tiled linear filter (32 x 8 cells per block, the window halo staged in
// shared memory with coalesced loads): the same row-major window order and
// skips (outside the grid or invalid) as k_linear. (A tiled median was not
// faster: its cost is the per-cell insertion sort, not the loads.)
constexpr int kSX = 32, kSY = 8;
// 3x3 median (radius 1), 32 x 8 cells per block with the halo staged in
// shared memory. A cell whose nine window cells are all valid, non-zero and
// not NaN takes the rank-4 value from a median-of-9 exchange network (nine
// distinct-or-identical values: the rank-4 value is the same bits whatever
// sorts them); any other cell (fewer values, or a +-0 / NaN whose final place
// the reference's std::sort decides) sorts its window with stl::sort, as
// k_median.
__device__ __forceinline__ void cmpSwap(double& a, double& b) {
  const double lo = b < a ? b : a, hi = b < a ? a : b;
  a = lo;
  b = hi;
}
__global__ void __launch_bounds__(kSX* kSY) k_median3(const double* __restrict__ v,
                                                      const uint8_t* __restrict__ ok, int W, int H,
                                                      double* __restrict__ out,
                                                      uint8_t* __restrict__ ok_out) {
  pdlEnter();
  constexpr int TW = kSX + 2, TH = kSY + 2;
  __shared__ double sv[TH * TW];
  __shared__ uint8_t so[TH * TW];
  const int c0 = blockIdx.x * kSX - 1, r0 = blockIdx.y * kSY - 1;
  const int tid = threadIdx.y * kSX + threadIdx.x;
  for (int q = tid; q < TW * TH; q += kSX * kSY) {
    const int rr = r0 + q / TW, cc = c0 + q % TW;
    uint8_t o = 0;
    double x = 0.0;
    if (rr >= 0 && rr < H && cc >= 0 && cc < W) {
      const int j = rr * W + cc;
      o = ok[j];
      if (o) x = v[j];
    }
    so[q] = o;
    sv[q] = x;
  }
  __syncthreads();
  const int r = blockIdx.y * kSY + threadIdx.y, c = blockIdx.x * kSX + threadIdx.x;
  if (r >= H || c >= W) return;
  const int i = r * W + c;
  const int base = threadIdx.y * TW + threadIdx.x;  // window's top-left in the tile
  const uint8_t oi = so[base + TW + 1];
  ok_out[i] = oi;
  if (!oi) {
    out[i] = v[i];
    return;
  }
  double p[9];
  bool plain = true;  // nine valid, non-zero, non-NaN values
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int q = base + (k / 3) * TW + (k % 3);
    p[k] = sv[q];
    plain = plain && so[q] && p[k] != 0.0 && p[k] == p[k];
  }
  if (plain) {
    cmpSwap(p[1], p[2]); cmpSwap(p[4], p[5]); cmpSwap(p[7], p[8]);
    cmpSwap(p[0], p[1]); cmpSwap(p[3], p[4]); cmpSwap(p[6], p[7]);
    cmpSwap(p[1], p[2]); cmpSwap(p[4], p[5]); cmpSwap(p[7], p[8]);
    cmpSwap(p[0], p[3]); cmpSwap(p[5], p[8]); cmpSwap(p[4], p[7]);
    cmpSwap(p[3], p[6]); cmpSwap(p[1], p[4]); cmpSwap(p[2], p[5]);
    cmpSwap(p[4], p[7]); cmpSwap(p[4], p[2]); cmpSwap(p[6], p[4]);
    cmpSwap(p[4], p[2]);
    out[i] = p[4];
    return;
  }
  double win[9];
  int n = 0;
  for (int k = 0; k < 9; ++k) {
    const int q = base + (k / 3) * TW + (k % 3);
    if (so[q]) win[n++] = sv[q];
  }
  stl::sort(win, n);  // n <= 9: the library's insertion sort
  out[i] = (n % 2 == 1) ? win[n / 2] : 0.5 * (win[n / 2 - 1] + win[n / 2]);
}

template <int R, int KIND>
__global__ void __launch_bounds__(kSX* kSY) k_stencil_tile(const double* __restrict__ v,
                                                           const uint8_t* __restrict__ ok, int W,
                                                           int H, Weights wt,
                                                           double* __restrict__ out,
                                                           uint8_t* __restrict__ ok_out) {
  pdlEnter();
  static_assert(KIND == 0, "linear filter only");
  constexpr int TW = kSX + 2 * R, TH = kSY + 2 * R, k = 2 * R + 1;
  __shared__ double sv[TH * TW];
  __shared__ uint8_t so[TH * TW];
  const int c0 = blockIdx.x * kSX - R, r0 = blockIdx.y * kSY - R;
  const int tid = threadIdx.y * kSX + threadIdx.x;
  for (int q = tid; q < TW * TH; q += kSX * kSY) {
    const int rr = r0 + q / TW, cc = c0 + q % TW;
    uint8_t o = 0;
    double x = 0.0;
    if (rr >= 0 && rr < H && cc >= 0 && cc < W) {
      const int j = rr * W + cc;
      o = ok[j];
      if (o) x = v[j];
    }
    so[q] = o;
    sv[q] = x;
  }
  __syncthreads();
  const int r = blockIdx.y * kSY + threadIdx.y, c = blockIdx.x * kSX + threadIdx.x;
  if (r >= H || c >= W) return;
  const int i = r * W + c;
  const int lc = threadIdx.x + R, lr = threadIdx.y + R;
  const uint8_t oi = so[lr * TW + lc];
  ok_out[i] = oi;
  if (!oi) {
    out[i] = v[i];
    return;
  }
  double acc = 0.0, ws = 0.0;
#pragma unroll
  for (int dr = -R; dr <= R; ++dr) {
#pragma unroll
    for (int dc = -R; dc <= R; ++dc) {
      const int q = (lr + dr) * TW + (lc + dc);
      if (!so[q]) continue;
      const double w = wt.w[(dr + R) * k + (dc + R)];
      acc += w * sv[q];
      ws += w;
    }
  }
  out[i] = acc / ws;
}

template <int KIND>
bool launchStencilTile(int R, const double* v, const uint8_t* ok, int W, int H, const Weights& wt,
                       double* out, uint8_t* ok_out, cudaStream_t s) {
  const dim3 grid((W + kSX - 1) / kSX, (H + kSY - 1) / kSY), block(kSX, kSY);
  switch (R) {
    case 1: launchPdl(k_stencil_tile<1, KIND>, grid, block, 0, s, v, ok, W, H, wt, out, ok_out); return true;
    case 2: launchPdl(k_stencil_tile<2, KIND>, grid, block, 0, s, v, ok, W, H, wt, out, ok_out); return true;
    case 3: launchPdl(k_stencil_tile<3, KIND>, grid, block, 0, s, v, ok, W, H, wt, out, ok_out); return true;
    default: return false;
  }
}

// ---- min inpaint: connected components of invalid cells (4-neighbour).
// Tile-local labels in shared memory (k_cc_tile), then a lock-free
// union-find over tile roots across tile edges (ECL-CC style hooks: every
// parent index is smaller than its child, finds use intermediate pointer
// jumping), and a flatten pass makes parent[i] the root.
__device__ __forceinline__ int representative(int* p, int x) {
  int cur = p[x];
  if (cur != x) {
    int next, prev = x;
    while (cur > (next = p[cur])) {
      p[prev] = next;
      prev = cur;
      cur = next;
    }
  }
  return cur;
}

__device__ void hook(int* p, int a, int b) {
  int ra = representative(p, a), rb = representative(p, b);
  bool repeat;
  do {
    repeat = false;
    if (ra != rb) {
      if (ra < rb) {
        const int ret = atomicCAS(p + rb, rb, ra);
        if (ret != rb) {
          rb = ret;
          repeat = true;
        }
      } else {
        const int ret = atomicCAS(p + ra, ra, rb);
        if (ret != ra) {
          ra = ret;
          repeat = true;
        }
      }
    }
  } while (repeat);
}

__device__ __forceinline__ unsigned long long orderKey(double v) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double fromKey(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}
constexpr unsigned long long kKeyInf = 0xfff0000000000000ULL;  // orderKey(+inf)


// Two-level labelling: each 32x32 tile labels its invalid cells in shared
// memory, writing the tile-local root (smallest index) as a global index;
// k_cc_merge then only unions across tile edges, so the global forest's
// chains are tile-root chains instead of whole rows.
constexpr int kTileCC = 32;

__global__ void __launch_bounds__(kTileCC* kTileCC)
    k_cc_tile(const uint8_t* ok, int W, int H, int* parent, unsigned long long* key,
              uint8_t* border, int* any_valid) {
  pdlEnter();
  __shared__ int lab[kTileCC * kTileCC];
  const int tx = threadIdx.x % kTileCC, ty = threadIdx.x / kTileCC;
  const int c = blockIdx.x * kTileCC + tx, r = blockIdx.y * kTileCC + ty;
  const bool in = c < W && r < H;
  const int i = r * W + c;
  const int t = threadIdx.x;
  bool fg = false;
  if (in) {
    key[i] = kKeyInf;
    border[i] = 0;
    if (ok[i]) *any_valid = 1;
    else fg = true;
  }
  // Tile-local labels: each warp is one tile row, so a row's runs of invalid
  // cells come from one ballot (every cell points at its run's first cell);
  // runs touching across rows are then joined by a shared-memory union-find
  // whose hooks always point the larger root at the smaller one, so a
  // component's root is its smallest index (the first cell of its first
  // run), as before.
  constexpr int kNone = 1 << 30;
  static_assert(kTileCC == 32, "one warp per tile row");
  const unsigned row = __ballot_sync(0xffffffffu, fg);
  const unsigned below = tx == 31 ? 0xffffffffu : ((2u << tx) - 1u);  // lanes <= tx
  const unsigned gaps = ~row & below;
  const int run = ty * kTileCC + (gaps ? 32 - __clz(gaps) : 0);
  lab[t] = fg ? run : kNone;
  __syncthreads();
  // one union per stretch of vertical contact between two runs
  if (fg && ty > 0 && lab[t - kTileCC] != kNone &&
      !(tx > 0 && lab[t - 1] != kNone && lab[t - kTileCC - 1] != kNone)) {
    int a = run, b = lab[t - kTileCC];
    while (true) {
      while (lab[a] != a) a = lab[a];
      while (lab[b] != b) b = lab[b];
      if (a == b) break;
      const int hi = a > b ? a : b, lo = a ^ b ^ hi;
      if (atomicCAS(&lab[hi], hi, lo) == hi) break;
      a = hi;  // hi was hooked meanwhile: retry from it
      b = lo;
    }
  }
  __syncthreads();
  if (fg) {
    int x = run;
    while (lab[x] != x) x = lab[x];
    lab[t] = x;  // (only the run starts are roots; other cells are never read above)
  }
  if (!in) return;
  if (!fg) {
    parent[i] = i;
    return;
  }
  const int root = lab[t];
  parent[i] = (blockIdx.y * kTileCC + root / kTileCC) * W + blockIdx.x * kTileCC + root % kTileCC;
}

// Unions across tile edges, one thread per edge cell, consecutive threads
// walking along one boundary (the first H * (tiles_x - 1) threads the
// vertical boundaries, the rest the horizontal ones). Neighbouring edge cells
// usually join the same pair of tile roots, so each warp hooks every distinct
// (root, root) pair once.
__global__ void __launch_bounds__(kT) k_cc_merge(const uint8_t* ok, int W, int H, int* parent) {
  pdlEnter();
  const int q = blockIdx.x * kT + threadIdx.x;
  const int vx = (W - 1) / kTileCC;  // vertical boundaries
  const int hy = (H - 1) / kTileCC;  // horizontal boundaries
  int i = -1, j = -1;
  if (q < H * vx) {
    const int r = q % H, c = (q / H + 1) * kTileCC;
    i = r * W + c;
    j = i - 1;
  } else if (q < H * vx + W * hy) {
    const int e = q - H * vx;
    const int r = (e / W + 1) * kTileCC, c = e % W;
    i = r * W + c;
    j = i - W;
  }
  const bool pair = i >= 0 && !ok[i] && !ok[j];
  const int a = pair ? parent[i] : -1, b = pair ? parent[j] : -1;
  const unsigned long long key =
      (static_cast<unsigned long long>(static_cast<unsigned>(a)) << 32) | static_cast<unsigned>(b);
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  if (pair && (threadIdx.x & 31) == __ffs(peers) - 1) hook(parent, a, b);
}

// Flatten without path writes: chains are tile-root chains (short); only each
// cell's own entry is written, so concurrent walks never see a torn path.
// Also flattens (parent[i] = root, for k_cc_fill) and, in thread 0, folds
// the step's "any valid cell" flag (see k_cc_tile) into flag[1].
__global__ void __launch_bounds__(kT) k_cc_border(const double* v, const uint8_t* ok, int W, int H,
                                                  int* parent, unsigned long long* key,
                                                  uint8_t* border, int* flag) {
  pdlEnter();
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i == 0) {
    if (flag[0] == 0) flag[1] = 1;
    flag[0] = 0;
  }
  if (i >= W * H || ok[i]) return;
  int root = parent[i];
  while (parent[root] != root) root = parent[root];
  parent[i] = root;
  const int r = i / W, c = i - (i / W) * W;
  bool any = false;
  unsigned long long best = kKeyInf;
  for (int dr = -1; dr <= 1; ++dr) {
    for (int dc = -1; dc <= 1; ++dc) {
      if (dr == 0 && dc == 0) continue;
      const int rr = r + dr, cc = c + dc;
      if (rr < 0 || rr >= H || cc < 0 || cc >= W) continue;
      const int j = rr * W + cc;
      if (!ok[j]) continue;
      any = true;  // a NaN neighbour still counts as border (reference has_border)
      const double x = v[j];
      if (x == x) {
        const unsigned long long kx = orderKey(x);
        if (kx < best) best = kx;
      }
    }
  }
  if (any) {
    if (!border[root]) border[root] = 1;
    if (best < kKeyInf && best < key[root]) atomicMin(key + root, best);
  }
}

__global__ void __launch_bounds__(kT) k_cc_fill(const double* v, const uint8_t* ok, int n,
                                                const int* parent, const unsigned long long* key,
                                                const uint8_t* border, double* out,
                                                uint8_t* ok_out) {
  pdlEnter();
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= n) return;
  if (ok[i]) {
    out[i] = v[i];
    ok_out[i] = 1;
    return;
  }
  const int root = parent[i];
  if (border[root]) {
    out[i] = fromKey(key[root]);
    ok_out[i] = 1;
  } else {
    out[i] = v[i];
    ok_out[i] = 0;
  }
}

}  // namespace

void ChainScratch::ensure(std::size_t n) {
  if (n <= cap) return;
  release();
  checkCuda(cudaMalloc(&va, n * sizeof(double)), "chain scratch");
  checkCuda(cudaMalloc(&vb, n * sizeof(double)), "chain scratch");
  checkCuda(cudaMalloc(&oa, n), "chain scratch");
  checkCuda(cudaMalloc(&ob, n), "chain scratch");
  checkCuda(cudaMalloc(&parent, n * sizeof(int)), "chain scratch");
  checkCuda(cudaMalloc(&key, n * sizeof(unsigned long long)), "chain scratch");
  checkCuda(cudaMalloc(&border, n), "chain scratch");
  checkCuda(cudaMalloc(&flag, 2 * sizeof(int)), "chain scratch");
  cap = n;
}

void ChainScratch::release() {
  cudaFree(va);
  cudaFree(vb);
  cudaFree(oa);
  cudaFree(ob);
  cudaFree(parent);
  cudaFree(key);
  cudaFree(border);
  cudaFree(flag);
  va = vb = nullptr;
  oa = ob = border = nullptr;
  parent = flag = nullptr;
  key = nullptr;
  cap = 0;
}

int smoothChainEnqueue(cudaStream_t s, ChainScratch& sc, const double* d_values,
                       const uint8_t* d_valid, int W, int H, const ChainStep* steps, int n_steps,
                       double* d_values_out, uint8_t* d_valid_out) {
  if (W <= 0 || H <= 0) fail(Err::kUsage, "malformed masked layer");
  for (int k = 0; k < n_steps; ++k) {
    const ChainStep& st = steps[k];
    if (st.kind < 0 || st.kind > 3) fail(Err::kUsage, "unknown filter kind");
    if (st.kind != 3 && st.radius < 1) fail(Err::kUsage, "filter radius must be >= 1");
    if (st.kind == 0 && !(st.sigma > 0.0)) fail(Err::kUsage, "gaussian sigma must be > 0");
    if (st.kind != 3 && (2 * st.radius + 1) * (2 * st.radius + 1) > kMaxWindow)
      fail(Err::kUsage, "filter radius above 5 is not supported");
  }
  const int n = W * H;
  sc.ensure(static_cast<std::size_t>(n));
  const unsigned grid = static_cast<unsigned>((n + kT - 1) / kT);
  int launches = 0;
  checkCuda(cudaMemsetAsync(sc.flag, 0, 2 * sizeof(int), s), "memset");
  const double* cv = d_values;
  const uint8_t* co = d_valid;
  double* bufs[2] = {sc.va, sc.vb};
  uint8_t* oks[2] = {sc.oa, sc.ob};
  int which = 0;
  for (int k = 0; k < n_steps; ++k) {
    const ChainStep& st = steps[k];
    double* nv = bufs[which];
    uint8_t* no = oks[which];
    const bool direct = k == n_steps - 1 && d_values_out != cv && d_valid_out != co;
    if (direct) {  // the last step writes the caller's buffers (no trailing copy)
      nv = d_values_out;
      no = d_valid_out;
    }
    if (st.kind == 0 || st.kind == 1) {
      Weights wt{};
      const int kk = 2 * st.radius + 1;
      for (int dr = -st.radius; dr <= st.radius; ++dr)
        for (int dc = -st.radius; dc <= st.radius; ++dc)
          wt.w[(dr + st.radius) * kk + (dc + st.radius)] =
              st.kind == 1 ? 1.0 : std::exp(-(dr * dr + dc * dc) / (2.0 * st.sigma * st.sigma));
      if (!launchStencilTile<0>(st.radius, cv, co, W, H, wt, nv, no, s))
        launchPdl(k_linear, grid, kT, 0, s, cv, co, W, H, st.radius, wt, nv, no);
      ++launches;
    } else if (st.kind == 2) {
      if (st.radius == 1 && RB_MEDIAN3)
        launchPdl(k_median3, dim3((W + kSX - 1) / kSX, (H + kSY - 1) / kSY), dim3(kSX, kSY), 0, s, cv, co,
                  W, H, nv, no);
      else
        launchPdl(k_median, grid, kT, 0, s, cv, co, W, H, st.radius, nv, no);
      ++launches;
    } else {
      const dim3 tiles((W + kTileCC - 1) / kTileCC, (H + kTileCC - 1) / kTileCC);
      launchPdl(k_cc_tile, tiles, kTileCC * kTileCC, 0, s, co, W, H, sc.parent, sc.key, sc.border, sc.flag);
      const int edges = H * ((W - 1) / kTileCC) + W * ((H - 1) / kTileCC);
      if (edges > 0) launchPdl(k_cc_merge, (edges + kT - 1) / kT, kT, 0, s, co, W, H, sc.parent);
      launchPdl(k_cc_border, grid, kT, 0, s, cv, co, W, H, sc.parent, sc.key, sc.border, sc.flag);
      launchPdl(k_cc_fill, grid, kT, 0, s, cv, co, n, sc.parent, sc.key, sc.border, nv, no);
      launches += 3 + (edges > 0 ? 1 : 0);
    }
    cv = nv;
    co = no;
    which ^= 1;
  }
  if (cv != d_values_out)
    checkCuda(cudaMemcpyAsync(d_values_out, cv, n * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy");
  if (co != d_valid_out)
    checkCuda(cudaMemcpyAsync(d_valid_out, co, n, cudaMemcpyDeviceToDevice, s), "copy");
  checkCuda(cudaGetLastError(), "chain launch");
  return launches;
}

void smoothChainCheck(cudaStream_t s, ChainScratch& sc) {
  int flags[2] = {0, 0};
  checkCuda(cudaMemcpyAsync(flags, sc.flag, sizeof flags, cudaMemcpyDeviceToHost, s), "flag");
  checkCuda(cudaStreamSynchronize(s), "chain");
  if (flags[1]) fail(Err::kNothingToInpaint, "layer has no valid cells");
}

namespace {
std::vector<ChainStep> makeSteps(const int* kinds, const int* radii, const double* sigmas, int n) {
  std::vector<ChainStep> steps(n > 0 ? n : 0);
  for (int k = 0; k < n; ++k) steps[k] = {kinds[k], radii[k], sigmas[k]};
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
  ChainScratch sc;
  struct Guard {
    ChainScratch& sc;
    double* dv = nullptr;
    uint8_t* dm = nullptr;
    ~Guard() {
      sc.release();
      cudaFree(dv);
      cudaFree(dm);
    }
  } g{sc};
  checkCuda(cudaMalloc(&g.dv, n * sizeof(double)), "chain input");
  checkCuda(cudaMalloc(&g.dm, n), "chain input");
  checkCuda(cudaMemcpy(g.dv, values, n * sizeof(double), cudaMemcpyHostToDevice), "upload");
  checkCuda(cudaMemcpy(g.dm, valid, n, cudaMemcpyHostToDevice), "upload");
  smoothChainEnqueue(nullptr, sc, g.dv, g.dm, W, H, steps.data(), n_steps, g.dv, g.dm);
  smoothChainCheck(nullptr, sc);
  checkCuda(cudaMemcpy(values_out, g.dv, n * sizeof(double), cudaMemcpyDeviceToHost), "download");
  checkCuda(cudaMemcpy(valid_out, g.dm, n, cudaMemcpyDeviceToHost), "download");
}

void runMapChainDevice(DeviceMap& m, const std::string& layer, const int* kinds, const int* radii,
                       const double* sigmas, int n_steps, double* d_values_out,
                       uint8_t* d_valid_out) {
  const std::vector<ChainStep> steps = makeSteps(kinds, radii, sigmas, n_steps);
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  const std::size_t n = m.grid.cells();
  m.chain.ensure(n);
  if (m.chain_in == nullptr) checkCuda(cudaMalloc(&m.chain_in, n * sizeof(double)), "chain input");
  if (!exportLayerDevice(m, layer.c_str(), m.chain_in))
    fail(Err::kUsage, unknownLayerMessage(layer));
  const uint8_t* mask = layer == "upper_bound" ? m.cur.ubv : m.cur.valid;
  checkCuda(cudaEventRecord(m.ev[8], m.stream), "event");
  m.last_chain_launches = smoothChainEnqueue(m.stream, m.chain, m.chain_in, mask, m.grid.width,
                                             m.grid.height, steps.data(), n_steps, d_values_out,
                                             d_valid_out);
  checkCuda(cudaEventRecord(m.ev[9], m.stream), "event");
  smoothChainCheck(m.stream, m.chain);
  float ms = 0.f;
  checkCuda(cudaEventElapsedTime(&ms, m.ev[8], m.ev[9]), "timing");
  m.last_chain_seconds = ms * 1e-3;
}

void runMapChain(DeviceMap& m, const std::string& layer, const int* kinds, const int* radii,
                 const double* sigmas, int n_steps, double* values_out, uint8_t* valid_out) {
  const std::size_t n = m.grid.cells();
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  if (m.chain_out == nullptr) {
    checkCuda(cudaMalloc(&m.chain_out, n * sizeof(double)), "chain output");
    checkCuda(cudaMalloc(&m.chain_out_ok, n), "chain output");
  }
  runMapChainDevice(m, layer, kinds, radii, sigmas, n_steps, m.chain_out, m.chain_out_ok);
  checkCuda(cudaMemcpyAsync(values_out, m.chain_out, n * sizeof(double), cudaMemcpyDeviceToHost,
                            m.stream), "download");
  checkCuda(cudaMemcpyAsync(valid_out, m.chain_out_ok, n, cudaMemcpyDeviceToHost, m.stream), "download");
  checkCuda(cudaStreamSynchronize(m.stream), "download");
}

}  // namespace rb200
