// The per-scan update path on the device: input_pointcloud / move_to /
// update_variance of the paper, reproducing the reference's deterministic
// integrateScan (reference integration.cpp:70-260) bit for bit.
//
// Launch plan per scan:
//   K4a k_shift          recenter: streaming copy of the 10 persistent layers
//   K1  k_ingest         range / exclusion / transform / sigma_p^2 / cell /
//                        drift vote / per-cell count      (one thread per point)
//                        (+ drift vote mean, fixed-order, in the last block)
//   K2  radix sort       stable LSD sort of (cell, point) -> per-cell segments
//                        in scan order; exclusive scan count -> segment start
//       (stream 2, under the sort) k_drift_finalize + k_side_prep: drift
//                        offset, fold lists, ray class + probe word per cell
//                        (cells with points "none", exact: DESIGN.md §5.1)
//   K3  gated Kalman fold: the removal candidates with points first
//                        (k_fuse_list, usually none); the short cells (stream 3,
//                        k_fuse_list) and the long ones (stream 2, k_fuse_heavy)
//                        beside the ray pass. (Frames without a ray pass:
//                        k_fuse, one thread per cell.)
//   K5  k_jump_grid      the 16x16-block bounds the rays jump over
//       k_rays_pass1     exact 2-D DDA per kept point (jumping over cleared
//                        blocks): bounds of invalid cells, k* = first removing
//                        ray per candidate cell
//   K6  k_rays_tail      retry of a failed speculation + bounds of removed cells
//                        from rays k >= k* (scratch), one cooperative launch
//   K7  k_cells          removal (k* < inf) + overlap clearance + normals +
//                        traversability + time variance, one shared-memory
//                        tile with a halo; its last block hands the stats over
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <vector>

#include "device_map.hpp"
#include "launch.cuh"
#include "fp_exact.cuh"

namespace rb200 {

namespace {

constexpr int kThreads = 256;
// Graph frames of at least kGraphMinPoints points (graph_mode 2); from
// kGraphHeadPoints on, the frame's head is launched directly and only the
// rest captured (its ingest then covers the capture and graph update).
#ifndef RB_SIDE_JUMP
#define RB_SIDE_JUMP 1  // the jump grid built on stream 2 right after the side sweep
#endif
#ifndef RB_SIDE_JUMP_CELLS
#define RB_SIDE_JUMP_CELLS 524288  // ... on maps of at least this many cells
#endif
constexpr size_t kSideJumpCells = RB_SIDE_JUMP_CELLS;
#ifndef RB_CELLS_SKIP
#define RB_CELLS_SKIP 1  // k_cells blocks whose tile has no valid cell and no points skip the staging
#endif
#ifndef RB_LIGHT_SPLIT
#define RB_LIGHT_SPLIT 32  // short-fold list: cells of <= this many points first, the rest from the far end
#endif
#ifndef RB_P1_JUMP
#define RB_P1_JUMP 1  // pass-1 rays jump over the blocks their heights clear (pass1Jump)
#endif
#ifndef RB_INGEST_TMA
#define RB_INGEST_TMA 1  // persistent ingest fed by TMA bulk copies (k_ingest_tma)
#endif
#ifndef RB_INGEST_TMA_BLOCKS
#define RB_INGEST_TMA_BLOCKS 5  // k_ingest_tma grid: blocks per SM (48 registers: 5 resident)
#endif
#ifndef RB_GRAPH_MIN_POINTS
#define RB_GRAPH_MIN_POINTS 32768
#endif
#ifndef RB_GRAPH_HEAD_POINTS
#define RB_GRAPH_HEAD_POINTS 524288
#endif
constexpr uint32_t kGraphMinPoints = RB_GRAPH_MIN_POINTS;
constexpr uint32_t kGraphHeadPoints = RB_GRAPH_HEAD_POINTS;
#ifndef RB_STATS_HANDOVER
#define RB_STATS_HANDOVER 1  // synchronous frames: stats through pinned memory (DeviceMap::h_seq)
#endif

constexpr double kInf = __builtin_huge_val();

// RB_TIMELINE (diagnostic builds): per kernel slot, the first block's start
// (sampled: every 16th block and the last) and the last block's end
// (%globaltimer, ns) of the frame, printed to stderr after each synchronous
// frame (scripts/timeline.py).
#ifdef RB_TIMELINE
constexpr int kTlSlots = 16;
__device__ unsigned long long g_tl[kTlSlots][2];
__device__ unsigned long long g_tl_end[kTlSlots][32];  // block ends spread over 32 words
__device__ __forceinline__ unsigned long long tlNow() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct TlGuard {
  int slot;
  // (every 16th block and the last one record: fewer atomics on one address)
  __device__ explicit TlGuard(int s) : slot(s) {
    if (threadIdx.x == 0 && ((blockIdx.x & 15) == 0 || blockIdx.x == gridDim.x - 1))
      atomicMin(&g_tl[s][0], tlNow());
  }
  __device__ ~TlGuard() {
    if (threadIdx.x == 0) atomicMax(&g_tl_end[slot][blockIdx.x & 31], tlNow());
  }
};
#define RB_TL(slot) TlGuard tl_guard_(slot)
__global__ void k_tl_reset() {
  if (threadIdx.x < kTlSlots) {
    g_tl[threadIdx.x][0] = ~0ull;
    g_tl[threadIdx.x][1] = 0ull;
  }
  for (int k = threadIdx.x; k < kTlSlots * 32; k += blockDim.x) g_tl_end[k / 32][k % 32] = 0ull;
}
#else
#define RB_TL(slot) \
  do {              \
  } while (0)
#endif

__device__ __forceinline__ double dnan() { return __longlong_as_double(0x7ff8000000000000LL); }
__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

template <typename T>
__device__ __forceinline__ T warpSum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Radix-sort tile geometry (K2): kTile consecutive keys per tile.
constexpr int kSortItems = 8;
constexpr int kTile = kThreads * kSortItems;
static_assert(kTile == 2048, "tshift 11");
// Small frames (RB_SMALL_TILE_N keys or fewer, single-map frames): 512-key tiles.
#ifndef RB_SMALL_TILE_N
#define RB_SMALL_TILE_N 600000
#endif
constexpr uint32_t kSmallTileN = RB_SMALL_TILE_N;
constexpr int kSmallTile = 512;
constexpr uint32_t kSmallTileShift = 9;
// Sorts of at most kFusedTiles tiles scan the tile counts inside the scatter.
#ifndef RB_FUSED_ROWSCAN
#define RB_FUSED_ROWSCAN 1
#endif
#ifndef RB_FUSED_TILES
#define RB_FUSED_TILES 48
#endif
constexpr uint32_t kFusedTiles = RB_FUSED_TILES;

// Tile digit count tc[d * pitch + tile] += 1 for every lane with ok, one
// atomic per (digit, tile) run in the warp; every lane must call.
__device__ __forceinline__ void countTileDigit(uint32_t* tc, uint32_t pitch, uint32_t d,
                                               uint32_t tile, bool ok) {
  const uint32_t slot = ok ? d * pitch + tile : 0xffffffffu;
  const unsigned peers = __match_any_sync(0xffffffffu, slot);
  if (ok && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&tc[slot], __popc(peers));
}

// Exclusive scan over a kThreads block; *total = block sum.
__device__ __forceinline__ uint32_t blockExclusiveScan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t s_warp[kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint32_t wpre = 0, tot = 0;
  for (int w = 0; w < kThreads / 32; ++w) {
    if (w < warp) wpre += s_warp[w];
    tot += s_warp[w];
  }
  __syncthreads();
  *total = tot;
  return wpre + incl - v;
}

// Invalidate one cell (reference grid.cpp:126-137).
__device__ __forceinline__ void invalidateCell(const Layers& L, size_t i) {
  L.valid[i] = 0;
  L.elev[i] = dnan();
  L.var[i] = dnan();
  L.last[i] = 0.0;
  L.trav[i] = 0.0;
  L.nx[i] = 0.0;
  L.ny[i] = 0.0;
  L.nz[i] = 0.0;
  L.ub[i] = dinf();
  L.ubv[i] = 0;
}

// ------------------------------------------------------------- K4a shift
// out[r][c] = in[r+dr][c+dc], exposed cells get the fresh fill
// (reference grid.cpp:70-111). One block row per map row (blockIdx.y), the
// columns across the block's threads: no per-element division, 32-bit
// offsets, every layer read and written along contiguous row segments.
constexpr int kShiftThreads = 256;
__global__ void __launch_bounds__(kShiftThreads) k_shift(Layers in, Layers out, int W, int H, int dc,
                                                         int dr) {
  RB_TL(0);
  const int r = blockIdx.y;
  const int sr = r + dr;
  const bool row_in = sr >= 0 && sr < H;
  const size_t ro = static_cast<size_t>(r) * W;
  const size_t so = static_cast<size_t>(row_in ? sr : 0) * W;
  for (int c = blockIdx.x * kShiftThreads + threadIdx.x; c < W; c += gridDim.x * kShiftThreads) {
    const int sc = c + dc;
    const size_t i = ro + c;
    if (row_in && sc >= 0 && sc < W) {
      const size_t j = so + sc;
      out.elev[i] = __ldcs(in.elev + j);
      out.var[i] = __ldcs(in.var + j);
      out.last[i] = __ldcs(in.last + j);
      out.ub[i] = __ldcs(in.ub + j);
      out.trav[i] = __ldcs(in.trav + j);
      out.nx[i] = __ldcs(in.nx + j);
      out.ny[i] = __ldcs(in.ny + j);
      out.nz[i] = __ldcs(in.nz + j);
      out.valid[i] = in.valid[j];
      out.ubv[i] = in.ubv[j];
    } else {
      out.elev[i] = dnan();
      out.var[i] = dnan();
      out.last[i] = 0.0;
      out.ub[i] = dinf();
      out.trav[i] = 0.0;
      out.nx[i] = 0.0;
      out.ny[i] = 0.0;
      out.nz[i] = 0.0;
      out.valid[i] = 0;
      out.ubv[i] = 0;
    }
  }
}

// The drift vote reduced by the last ingest block instead of k_drift_finalize:
// off by default -- the per-block completion atomics on one counter cost the
// ingest more than the one-block finalize kernel (C4: ingest 19 -> 29 us).
#ifndef RB_INGEST_FINALIZE
#define RB_INGEST_FINALIZE 0
#endif

// ------------------------------------------------------ drift reduction
// Mean error over the votes and the clamped offset (reference drift.cpp:24-55,
// integration.cpp:119-128) from the per-block partials. The sums run in one
// fixed tree whatever block runs it -- 1024 strided lanes, warp trees, the 32
// warp sums in order -- so the result is run-to-run deterministic and the same
// in the single-GPU frame (last block of k_ingest) and the group frame
// (k_drift_finalize over the gathered partials); it differs from the
// reference's sequential sum only in the last bits.
constexpr int kDriftLanes = 1024;
__device__ __forceinline__ void driftFinalizeBlock(const double* part, const int* npart, int nblocks,
                                                   int min_points, double max_off,
                                                   double* offset_out, DevStats* st) {
  __shared__ double s_dsum[32];
  __shared__ long long s_dcnt[32];
  __shared__ double s_lane[kDriftLanes];
  __shared__ long long s_lcnt[kDriftLanes];
  const int lane = threadIdx.x & 31;
  // lane v's strided sum part[v] + part[v + 1024] + ..., all lanes' loads in flight together
  for (int v = threadIdx.x; v < kDriftLanes; v += blockDim.x) {
    double sum = 0.0;
    long long c = 0;
    if (v < nblocks) {
      const int nb = (nblocks - 1 - v) / kDriftLanes + 1;
      double pv[4];
      int nv[4];
      for (int b0 = 0; b0 < nb; b0 += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int b = v + (b0 + u) * kDriftLanes;
          pv[u] = b0 + u < nb ? __ldcg(part + b) : 0.0;
          nv[u] = b0 + u < nb ? __ldcg(npart + b) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (b0 + u < nb) {
            sum += pv[u];
            c += nv[u];
          }
      }
    }
    s_lane[v] = sum;
    s_lcnt[v] = c;
  }
  __syncthreads();
  for (int vw = threadIdx.x >> 5; vw < 32; vw += blockDim.x >> 5) {
    double sum = s_lane[vw * 32 + lane];
    long long c = s_lcnt[vw * 32 + lane];
    sum = warpSum(sum);
    c = warpSum(c);
    if (lane == 0) {
      s_dsum[vw] = sum;
      s_dcnt[vw] = c;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double total = s_dsum[0];
    long long cnt = s_dcnt[0];
    for (int w = 1; w < 32; ++w) {
      total += s_dsum[w];
      cnt += s_dcnt[w];
    }
    const int nvote = static_cast<int>(cnt);
    double off = 0.0;
    if (nvote >= min_points) {
      const double mean = total / nvote;
      off = sclamp(mean, -max_off, max_off);
      st->drift_offset = off;
      st->drift_clamped = off != mean;
      st->drift_n = nvote;
    }
    *offset_out = off;
  }
}

// ------------------------------------------------------------- K1 ingest
struct IngestArgs {
  GridArgs g;
  double R[9];
  double t[3];
  double max_range2;
  int excl_enabled;
  double excl_b, excl_c, excl_dmax, excl_tan;
  double alpha_d, sigma_p_min2;
  int drift_enabled;
  double drift_thr;
  // drift offset computed by the last block to finish (0: not here -- a group
  // frame reduces the gathered partials in k_drift_finalize)
  uint32_t drift_blocks;  // frame-wide block count of the ingest
  int drift_min_points;
  double drift_max_off;
  double* drift_offset;
  uint32_t tshift;  // log2 of the sort tile (SortGeom::tshift)
};

// Per point (reference integration.cpp:85-113,134-140; sensing.cpp:32-41;
// drift.cpp:24-42; grid.cpp:41-47): fate, map-frame point, sigma_p^2, cell,
// drift vote against the pre-fusion map, per-cell point count.
// One 256-point tile of the ingest: the points k = k_base + tile * 256 + thread,
// read from the staged copy `sx` in shared memory (null: from xyz directly).
struct IngestCounts {  // a block's out-of-range / excluded / out-of-map points (thread 0)
  unsigned oor = 0, exc = 0, oom = 0;
};

__device__ __forceinline__ void ingestTile(const double* __restrict__ xyz, uint32_t n, const IngestArgs& a,
                                           const Layers& L, int32_t* __restrict__ count,
                                           double* __restrict__ px, double* __restrict__ py,
                                           double* __restrict__ pz, double* __restrict__ pvar,
                                           uint32_t* __restrict__ key, uint8_t* __restrict__ kept,
                                           double* __restrict__ drift_part, int* __restrict__ drift_npart,
                                           uint32_t* __restrict__ tc0, uint32_t pitch, uint32_t dmask,
                                           int count_cells, DevStats* st, uint32_t k_base,
                                           uint32_t in_base, uint32_t tile, const double* sx,
                                           IngestCounts& stat_acc) {
  const uint32_t WH = static_cast<uint32_t>(a.g.W) * static_cast<uint32_t>(a.g.H);
  const uint32_t k = k_base + tile * kThreads + threadIdx.x;
  int oor = 0, exc = 0, oom = 0, dn = 0;
  double ds = 0.0;
  uint32_t cell = WH;
  const bool staged = sx != nullptr;
  if (k < n) {
    double x, y, z;
    if (staged) {
      const double* sp = sx + 3 * threadIdx.x;
      x = sp[0];
      y = sp[1];
      z = sp[2];
    } else {
      const size_t ki = 3 * static_cast<size_t>(k - in_base);
      x = xyz[ki];
      y = xyz[ki + 1];
      z = xyz[ki + 2];
    }
    const double sq = (x * x + y * y) + z * z;
    bool keep = false;
    if (sq > a.max_range2) {
      oor = 1;
    } else if (a.excl_enabled && !(a.excl_tan >= 0.0 && z <= smin(a.excl_dmax, a.excl_b)) &&
               z > smin(a.excl_dmax,
                        a.excl_b + smax(0.0, libm_hypot(x, y) - a.excl_c) * a.excl_tan)) {
      // (the pre-test skips the hypot: with tan >= 0 the bound is >= min(d_max, b))
      exc = 1;
    } else {
      keep = true;
    }
    if (keep) {
      const double mx = ((a.R[0] * x + a.R[1] * y) + a.R[2] * z) + a.t[0];
      const double my = ((a.R[3] * x + a.R[4] * y) + a.R[5] * z) + a.t[1];
      const double mz = ((a.R[6] * x + a.R[7] * y) + a.R[8] * z) + a.t[2];
      const double d = sqrt(sq);
      px[k] = mx;
      py[k] = my;
      pz[k] = mz;
      pvar[k] = smax(a.alpha_d * d * d, a.sigma_p_min2);
      double qx, qy;  // (m - origin) / res, both quotients from one reciprocal
      div2_rn(mx - a.g.ox, my - a.g.oy, a.g.res, qx, qy);
      const int col = x86_to_int(floor(qx));
      const int row = x86_to_int(floor(qy));
      if (col >= 0 && col < a.g.W && row >= 0 && row < a.g.H) {
        cell = static_cast<uint32_t>(row) * a.g.W + col;
        if (a.drift_enabled) {
          // The three gathers are issued together (one memory round trip
          // instead of a dependent chain of three).
          const uint8_t vld = L.valid[cell];
          const double tr = L.trav[cell], el = L.elev[cell];
          if (vld && !(tr <= a.drift_thr)) {
            ds = mz - el;
            dn = 1;
          }
        }
      } else {
        oom = 1;
      }
    }
    key[k] = cell;
    kept[k] = keep ? 1 : 0;
  }
  // Per-cell point count, one atomic per run of equal cells in the warp, and
  // the first radix pass's tile digit counts (K2). A sharded frame counts the
  // gathered records instead (k_records_count).
  if (count_cells) {
    const unsigned peers = __match_any_sync(0xffffffffu, cell);
    if (cell < WH && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&count[cell], __popc(peers));
    countTileDigit(tc0, pitch, cell & dmask, k >> a.tshift, cell < WH);
  }

  // Fixed-shape block reduction: deterministic drift partial per block.
  __shared__ double s_sum[kThreads / 32];
  __shared__ int s_cnt[4][kThreads / 32];
  // (the three rejection counters packed in 10-bit fields: at most 256 per tile)
  ds = warpSum(ds);
  dn = warpSum(dn);
  const int packed = warpSum(oor | (exc << 10) | (oom << 20));
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_sum[warp] = ds;
    s_cnt[0][warp] = dn;
    s_cnt[1][warp] = packed;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bs = s_sum[0];
    int c0 = s_cnt[0][0], c1 = s_cnt[1][0];
    for (int w = 1; w < kThreads / 32; ++w) {
      bs += s_sum[w];
      c0 += s_cnt[0][w];
      c1 += s_cnt[1][w];
    }
    drift_part[k_base / kThreads + tile] = bs;
    drift_npart[k_base / kThreads + tile] = c0;
    // the block's running counters (flushed once per block: flushIngestStats)
    stat_acc.oor += c1 & 1023;
    stat_acc.exc += (c1 >> 10) & 1023;
    stat_acc.oom += (c1 >> 20) & 1023;
  }
  __syncthreads();  // (the block's reduction arrays are reused by its next tile)
}

// Thread 0: the block's rejection counters to the frame stats, once per block.
__device__ __forceinline__ void flushIngestStats(const IngestCounts& c, DevStats* st) {
  if (threadIdx.x != 0) return;
  if (c.oor) atomicAdd(&st->out_of_range, static_cast<unsigned long long>(c.oor));
  if (c.exc) atomicAdd(&st->excluded, static_cast<unsigned long long>(c.exc));
  if (c.oom) atomicAdd(&st->out_of_map, static_cast<unsigned long long>(c.oom));
}

__global__ void __launch_bounds__(kThreads)
    k_ingest(const double* __restrict__ xyz, uint32_t n, IngestArgs a, Layers L,
             int32_t* __restrict__ count, double* __restrict__ px, double* __restrict__ py,
             double* __restrict__ pz, double* __restrict__ pvar, uint32_t* __restrict__ key,
             uint8_t* __restrict__ kept, double* __restrict__ drift_part,
             int* __restrict__ drift_npart, uint32_t* __restrict__ tc0, uint32_t pitch,
             uint32_t dmask, int count_cells, DevStats* st, uint32_t k_base, uint32_t in_base) {
  RB_TL(1);
  pdlEnter();
  // k_base: first point of this launch (a chunk of a frame whose upload is
  // split); block partials are indexed by the frame-wide block k / kThreads.
  // in_base: frame index of xyz[0] (0, or a group rank's first point, whose
  // outputs land at their frame-wide indices).
  // The block's 256 points (6 KB of x y z) come in as 16-byte vector loads
  // into shared memory (every byte fetched once, full sectors), then each
  // thread reads its own triple; a misaligned caller pointer reads directly.
  __shared__ double2 s_xyz[3 * kThreads / 2];
  const uint32_t k0 = k_base + blockIdx.x * kThreads;
  const double* blk = xyz + 3 * static_cast<size_t>(k0 - in_base);
  const bool staged = (reinterpret_cast<uintptr_t>(blk) & 15u) == 0;
  if (staged) {
    const uint32_t nb = k0 < n ? min(static_cast<uint32_t>(kThreads), n - k0) : 0u;
    const double2* src = reinterpret_cast<const double2*>(blk);
    for (uint32_t q = threadIdx.x; 2 * q < 3 * nb; q += kThreads) {
      if (2 * q + 1 < 3 * nb) {
        s_xyz[q] = __ldcs(src + q);
      } else {
        s_xyz[q].x = __ldcs(blk + 2 * q);  // odd tail: the last double alone
      }
    }
    __syncthreads();
  }
  IngestCounts stat_acc;
  ingestTile(xyz, n, a, L, count, px, py, pz, pvar, key, kept, drift_part, drift_npart, tc0, pitch,
             dmask, count_cells, st, k_base, in_base, blockIdx.x,
             staged ? reinterpret_cast<const double*>(s_xyz) : nullptr, stat_acc);
  flushIngestStats(stat_acc, st);
#if RB_INGEST_FINALIZE
  if (a.drift_blocks == 0) return;
  // The last block of the frame's ingest (over all chunk launches) reduces the
  // partials: no separate finalize launch.
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&st->ingest_done, 1u) == a.drift_blocks - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  driftFinalizeBlock(drift_part, drift_npart, static_cast<int>(a.drift_blocks), a.drift_min_points,
                     a.drift_max_off, a.drift_offset, st);
#endif
}

// Persistent ingest with the input brought in by the TMA engine: each block
// takes the tiles blockIdx.x, + gridDim.x, ... of this launch (ntl tiles), and
// while it processes one tile the next tile's 6 KB of x y z lands in the other
// half of a double buffer by a bulk asynchronous copy (cp.async.bulk, mbarrier
// completion). A partial last tile (or a caller pointer not 16-B aligned) is
// read directly. Outputs, drift partials (per tile) and counts are those of
// k_ingest.
__device__ __forceinline__ uint32_t smemAddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__global__ void __launch_bounds__(kThreads)
    k_ingest_tma(const double* __restrict__ xyz, uint32_t n, IngestArgs a, Layers L,
                 int32_t* __restrict__ count, double* __restrict__ px, double* __restrict__ py,
                 double* __restrict__ pz, double* __restrict__ pvar, uint32_t* __restrict__ key,
                 uint8_t* __restrict__ kept, double* __restrict__ drift_part,
                 int* __restrict__ drift_npart, uint32_t* __restrict__ tc0, uint32_t pitch,
                 uint32_t dmask, int count_cells, DevStats* st, uint32_t k_base, uint32_t in_base,
                 uint32_t ntl) {
  RB_TL(1);
  pdlEnter();
  constexpr uint32_t kTileBytes = 3 * kThreads * sizeof(double);  // 6 KB
  __shared__ alignas(128) double s_buf[2][3 * kThreads];
  __shared__ alignas(8) unsigned long long s_bar[2];
  const double* base = xyz + 3 * static_cast<size_t>(k_base - in_base);
  const bool tma = (reinterpret_cast<uintptr_t>(base) & 15u) == 0;
  auto full = [&](uint32_t t) { return k_base + (t + 1) * kThreads <= n; };
  auto issue = [&](uint32_t t, int b) {  // thread 0: tile t into buffer b
    if (!tma || !full(t)) return;
    const uint32_t bar = smemAddr(&s_bar[b]);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the buffer's last reads first
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kTileBytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smemAddr(s_buf[b])),
        "l"(base + 3 * static_cast<size_t>(t) * kThreads), "r"(kTileBytes), "r"(bar)
        : "memory");
  };
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smemAddr(&s_bar[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smemAddr(&s_bar[1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (blockIdx.x < ntl) issue(blockIdx.x, 0);
  }
  __syncthreads();
  uint32_t it = 0;
  IngestCounts stat_acc;
  for (uint32_t t = blockIdx.x; t < ntl; t += gridDim.x, ++it) {
    const int b = static_cast<int>(it & 1u);
    // the other buffer is free: every thread finished the previous tile (the
    // barrier at the end of ingestTile)
    if (threadIdx.x == 0 && t + gridDim.x < ntl) issue(t + gridDim.x, b ^ 1);
    const double* sx = nullptr;
    if (tma && full(t)) {
      const uint32_t bar = smemAddr(&s_bar[b]), parity = (it >> 1) & 1u;
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "WAIT_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
          "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
          "r"(parity)
          : "memory");
      sx = s_buf[b];
    }
    ingestTile(xyz, n, a, L, count, px, py, pz, pvar, key, kept, drift_part, drift_npart, tc0, pitch,
               dmask, count_cells, st, k_base, in_base, t, sx, stat_acc);
  }
  flushIngestStats(stat_acc, st);
}

// ------------------------------------------------------ drift (one block)
// Mean error over the votes and the clamped offset (reference drift.cpp:24-55,
// integration.cpp:119-128). Sums run in a fixed tree, so the result is
// run-to-run deterministic; it differs from the sequential sum only in the
// last bits.
__global__ void __launch_bounds__(1024)
    k_drift_finalize(const double* part, const int* npart, int nblocks, int min_points,
                     double max_off, double* offset_out, DevStats* st) {
  RB_TL(5);
  pdlEnter();
  driftFinalizeBlock(part, npart, nblocks, min_points, max_off, offset_out, st);
}

// Reference drift.cpp:44-55 as a separate sweep (RB_FUSE_OFFSET=0 builds).
__global__ void __launch_bounds__(kThreads) k_apply_offset(Layers L, size_t n, const double* off_p) {
  RB_TL(6);
  pdlEnter();
  const double off = *off_p;
  if (off == 0.0) return;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    if (L.valid[i]) L.elev[i] += off;
    if (L.ubv[i]) L.ub[i] += off;
  }
}

// Drift offset known on the host (sharded frames: the ranks' votes summed in
// rank order).
__global__ void __launch_bounds__(kThreads) k_apply_offset_value(Layers L, size_t n, double off) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    if (L.valid[i]) L.elev[i] += off;
    if (L.ubv[i]) L.ub[i] += off;
  }
}

// Local drift vote of a sharded batch: the same fixed-shape reduction as
// k_drift_finalize, reported instead of applied.
__global__ void __launch_bounds__(1024)
    k_drift_local(const double* part, const int* npart, int nblocks, double* out) {
  __shared__ double s_sum[32];
  __shared__ long long s_cnt[32];
  double sum = 0.0;
  long long c = 0;
  for (int b = threadIdx.x; b < nblocks; b += 1024) {
    sum += part[b];
    c += npart[b];
  }
  sum = warpSum(sum);
  c = warpSum(c);
  if ((threadIdx.x & 31) == 0) {
    s_sum[threadIdx.x >> 5] = sum;
    s_cnt[threadIdx.x >> 5] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double total = s_sum[0];
    long long cnt = s_cnt[0];
    for (int w = 1; w < 32; ++w) {
      total += s_sum[w];
      cnt += s_cnt[w];
    }
    out[0] = total;
    out[1] = static_cast<double>(cnt);
  }
}

// Stable compaction of a batch's in-map kept points into fusion records
// (cell, p_z, sigma_p^2) in scan order: per-1024-point block counts, one
// block scan of the counts, then the write.
constexpr int kCompact = 1024;
__global__ void __launch_bounds__(kCompact)
    k_compact_count(const uint32_t* __restrict__ key, uint32_t n, uint32_t WH,
                    uint32_t* __restrict__ blk) {
  const uint32_t i = blockIdx.x * kCompact + threadIdx.x;
  const int c = __syncthreads_count(i < n && key[i] < WH);
  if (threadIdx.x == 0) blk[blockIdx.x] = static_cast<uint32_t>(c);
}

__global__ void __launch_bounds__(kThreads)
    k_compact_scan(uint32_t* blk, uint32_t nblk, uint32_t* total) {
  uint32_t carry = 0;
  for (uint32_t b0 = 0; b0 < nblk; b0 += kThreads) {
    const uint32_t b = b0 + threadIdx.x;
    const uint32_t v = b < nblk ? blk[b] : 0u;
    uint32_t tot;
    const uint32_t ex = blockExclusiveScan(v, &tot);
    if (b < nblk) blk[b] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kCompact)
    k_compact_write(const uint32_t* __restrict__ key, const double* __restrict__ pz,
                    const double* __restrict__ pvar, uint32_t n, uint32_t WH,
                    const uint32_t* __restrict__ blk_off, uint32_t* __restrict__ rcell,
                    double* __restrict__ rz, double* __restrict__ rvar) {
  __shared__ uint32_t s_warp[kCompact / 32];
  const uint32_t i = blockIdx.x * kCompact + threadIdx.x;
  const bool keep = i < n && key[i] < WH;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned mask = __ballot_sync(0xffffffffu, keep);
  if (lane == 0) s_warp[warp] = __popc(mask);
  __syncthreads();
  uint32_t base = blk_off[blockIdx.x];
  for (unsigned w = 0; w < warp; ++w) base += s_warp[w];
  if (keep) {
    const uint32_t pos = base + __popc(mask & ((1u << lane) - 1u));
    rcell[pos] = key[i];
    rz[pos] = pz[i];
    rvar[pos] = pvar[i];
  }
}

// Per-cell counts and the first radix pass's tile digit counts of the
// gathered records of a sharded frame (the records are the sort's input).
__global__ void __launch_bounds__(kThreads)
    k_records_count(const uint32_t* __restrict__ rcell, uint32_t m, int32_t* __restrict__ count,
                    uint32_t* __restrict__ tc0, uint32_t pitch, uint32_t dmask, uint32_t WH) {
  pdlEnter();
  const uint32_t k = blockIdx.x * kThreads + threadIdx.x;
  uint32_t cell = k < m ? rcell[k] : 0xffffffffu;
  const bool ok = cell < WH;  // keys >= WH: not in the map (group frames gather them too)
  if (!ok) cell = 0xffffffffu;
  const unsigned peers = __match_any_sync(0xffffffffu, cell);
  if (ok && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&count[cell], __popc(peers));
  countTileDigit(tc0, pitch, cell & dmask, k / kTile, ok);
}

// ------------------------------------------------ K2 stable radix sort
// LSD radix sort of the in-map kept points by cell, carrying the point index,
// reduce-then-scan style so that no tile waits on another:
//  * tile counts tc[p][d][t] = keys of tile t (kTile consecutive keys of pass
//    p's input) with digit d. Pass 0's are built by k_ingest, pass p+1's by
//    pass p's scatter (it knows where every key lands); warp-aggregated
//    atomics in both.
//  * k_sort_rowscan: one block per digit turns its row into exclusive tile
//    offsets and writes the row total (the digit's global count).
//  * k_sort_scatter: one block per tile ranks its keys stably (per-warp
//    counters + __match_any_sync), adds the digit base (block scan of the row
//    totals) and its row offset, and scatters.
// Stability keeps scan order within each cell, which the gated fold needs. The
// last pass writes the fusion payload in (cell, scan order) order and each
// cell's segment start (atomic min).
struct SortGeom {
  int passes = 0, dbits = 0;
  uint32_t ntiles = 0;  // tiles of the N input keys (bounds every pass)
  uint32_t tshift = 11; // log2 of the tile (kTile keys, or kSmallTile for small frames)
  uint32_t pitch = 0;   // row pitch of tc (ntiles rounded up to 4)
  uint32_t* tc = nullptr;      // [passes][buckets][pitch]
  uint32_t* rowsum = nullptr;  // [passes][buckets]
  __host__ __device__ uint32_t buckets() const { return 1u << dbits; }
  __host__ __device__ uint32_t* counts(int p) const {
    return tc + static_cast<size_t>(p) * buckets() * pitch;
  }
};


// Row d of tc -> exclusive offsets within the digit; rowsum[d] = row total.
__global__ void __launch_bounds__(kThreads)
    k_sort_rowscan(uint32_t* __restrict__ tc, uint32_t pitch, uint32_t* __restrict__ rowsum) {
  RB_TL(2);
  pdlEnter();
  uint4* row = reinterpret_cast<uint4*>(tc + static_cast<size_t>(blockIdx.x) * pitch);
  const uint32_t nq = pitch / 4;
  uint32_t carry = 0;
  for (uint32_t b = 0; b < nq; b += kThreads) {
    const uint32_t q = b + threadIdx.x;
    uint4 v = q < nq ? row[q] : make_uint4(0, 0, 0, 0);
    uint32_t total;
    const uint32_t run = carry + blockExclusiveScan(v.x + v.y + v.z + v.w, &total);
    if (q < nq) {
      uint4 o;
      o.x = run;
      o.y = o.x + v.x;
      o.z = o.y + v.y;
      o.w = o.z + v.z;
      row[q] = o;
    }
    carry += total;
  }
  if (threadIdx.x == 0) rowsum[blockIdx.x] = carry;
}

// kFused: the row scans are done here (frames of at most kFusedTiles tiles):
// each block sums its digits' rows itself, which saves the k_sort_rowscan
// launch of every pass.
template <int kItems, bool kFused = false>
__global__ void __launch_bounds__(kThreads)
    k_sort_scatter(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                   uint32_t n_in, int pass, SortGeom sg, uint32_t sentinel,
                   uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                   const double* __restrict__ pz, const double* __restrict__ pvar,
                   double* __restrict__ spz, double* __restrict__ spv, uint32_t* start) {
  RB_TL(3 + pass);
  pdlEnter();
  extern __shared__ unsigned char smem[];
  const int dbits = sg.dbits, shift = pass * dbits;
  const int buckets = 1 << dbits;
  const uint32_t mask = buckets - 1;
  const bool last = pass == sg.passes - 1;
  const uint32_t* __restrict__ tc = sg.counts(pass);
  const uint32_t* __restrict__ rowsum = sg.rowsum + static_cast<size_t>(pass) * buckets;
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(smem);                // [8][buckets]
  uint32_t* offs = reinterpret_cast<uint32_t*>(smem + 16 * buckets);  // [buckets]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tile = blockIdx.x;
  for (int i = threadIdx.x; i < 8 * buckets; i += kThreads) wcnt[i] = 0;
  // Digit bases: exclusive scan of the row totals; their sum is the number of
  // keys being sorted (pass 0 reads N keys and skips the sentinel ones).
  uint32_t nkeys;
  {
    const int per = (buckets + kThreads - 1) / kThreads;
    constexpr int kMaxPer = 8;  // buckets <= 2048 (11-bit digits)
    uint32_t row_total[kMaxPer], before[kMaxPer];
    uint32_t loc = 0;
    for (int j = 0; j < per; ++j) {
      const int d = threadIdx.x * per + j;
      uint32_t t = 0, b = 0;
      if (d < buckets) {
        if (kFused) {  // the digit's row: counts of all tiles, and of the tiles before this one
          const uint4* row = reinterpret_cast<const uint4*>(tc + static_cast<size_t>(d) * sg.pitch);
          for (uint32_t q = 0; q < sg.pitch / 4; ++q) {
            const uint4 v = row[q];
            const uint32_t t0 = 4 * q;
            b += (t0 < tile ? v.x : 0u) + (t0 + 1 < tile ? v.y : 0u) + (t0 + 2 < tile ? v.z : 0u) +
                 (t0 + 3 < tile ? v.w : 0u);
            t += v.x + v.y + v.z + v.w;
          }
        } else {
          t = rowsum[d];
          b = tc[static_cast<size_t>(d) * sg.pitch + tile];
        }
      }
      if (j < kMaxPer) {
        row_total[j] = t;
        before[j] = b;
      }
      loc += t;
    }
    uint32_t run = blockExclusiveScan(loc, &nkeys);
    for (int j = 0; j < per && j < kMaxPer; ++j) {
      const int d = threadIdx.x * per + j;
      if (d < buckets) {
        offs[d] = run + before[j];
        run += row_total[j];
      }
    }
  }
  const uint32_t n = pass == 0 ? n_in : nkeys;
  __syncthreads();
  uint16_t* my = wcnt + warp * buckets;
  const unsigned lt = (1u << lane) - 1u;
  constexpr uint32_t kT = kThreads * kItems;  // this instantiation's tile (1 << sg.tshift)
  const uint32_t wbase = tile * kT + warp * (kT / 8);
  uint32_t key[kItems], val[kItems];
  uint16_t rank[kItems];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const uint32_t idx = wbase + r * 32 + lane;
    key[r] = idx < n ? keys_in[idx] : sentinel;
    const bool ok = key[r] < sentinel;
    val[r] = ok ? (pass == 0 ? idx : vals_in[idx]) : 0u;
    const uint32_t d = ok ? (key[r] >> shift) & mask : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    uint16_t before = 0;
    if (ok) before = my[d];
    __syncwarp();
    rank[r] = before + __popc(peers & lt);
    if (ok && lane == __ffs(peers) - 1) my[d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // Per digit: exclusive prefix over the warps of this tile.
  for (int d = threadIdx.x; d < buckets; d += kThreads) {
    uint16_t run = 0;
    for (int w = 0; w < 8; ++w) {
      const uint16_t t = wcnt[w * buckets + d];
      wcnt[w * buckets + d] = run;
      run += t;
    }
  }
  __syncthreads();
  uint32_t* tc_next = last ? nullptr : sg.counts(pass + 1);
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const bool ok = key[r] < sentinel;
    const uint32_t d = (key[r] >> shift) & mask;
    const uint32_t pos = ok ? offs[d] + my[d] + rank[r] : 0u;
    if (!last) {
      if (ok) {
        keys_out[pos] = key[r];
        vals_out[pos] = val[r];
      }
      countTileDigit(tc_next, sg.pitch, (key[r] >> (shift + dbits)) & mask, pos >> sg.tshift, ok);
    } else {
      if (ok) {
        // Final pass: the fusion payload in (cell, scan order) order.
        spz[pos] = pz[val[r]];
        spv[pos] = pvar[val[r]];
      }
      // Segment start = smallest position of the cell (lowest lane of a run).
      const unsigned peers = __match_any_sync(0xffffffffu, ok ? key[r] : 0xffffffffu);
      if (ok && lane == __ffs(peers) - 1) atomicMin(start + key[r], pos);
    }
  }
}

// ----------------------------------------------------- ray classes
enum : uint8_t { kClsNone = 0, kClsBound = 1, kClsCandidate = 2 };

struct RayArgs {
  GridArgs g;
  double o[3];  // sensor origin = pose translation
  double now, t_free, alpha_n;
  int cleanup, bound;
  // Per-frame ray constants: the origin lies in the closed map extent, and its
  // cell (the start cell of every ray that is not clipped at its start).
  int origin_in, ocol, orow;
  // Pass-1 jump grid (k_jump_grid; null: no jumps): one probe word per
  // kJumpBlk x kJumpBlk block of cells, jw x jh blocks of side jres metres.
  const float* jgrid;
  int jw, jh;
  double jres;
};

// Post-fusion ray class per cell; also resets k* (reference raycast.cpp:
// 132-183 gates that do not depend on the ray).
//
// Speculation (heavy >= 0): cells longer than `heavy` are still being folded
// by k_fuse_heavy when this runs. A cell that fuses at least one point ends
// valid with last_update = now, i.e. class "none" whenever t_free >= 0, so
// those cells are classified "none" up front; k_fuse_heavy flags any heavy
// cell that fused nothing and the ray pass is then redone (retry = 1: this
// kernel and pass 1 run only if the flag is set).
#ifndef RB_P1_JBLK
#define RB_P1_JBLK 16
#endif
constexpr int kJumpBlk = RB_P1_JBLK;  // cells per side of a pass-1 jump block
constexpr int kJumpShift = kJumpBlk == 8 ? 3 : (kJumpBlk == 16 ? 4 : 5);
static_assert(kJumpBlk == 8 || kJumpBlk == 16 || kJumpBlk == 32, "jump block");

// Pass-1 probe word of a cell (16 bits): the ray class in the low 2 bits and,
// above it, an order-preserving key of an f16 bound F >= T of the cell's gate
// threshold T (T = upper_bound for a bound cell, elevation - sqrt(variance)
// for a removal candidate), so that a visit with ray height h >= F is rejected
// without loading the cell state: the reference's own test (h < ub, resp.
// !(h >= elev - sqrt(var))) rejects it too. F is T rounded up (double -> f32
// -> f16), its key (sign-flipped f16 bits: unsigned order == value order)
// rounded up to a multiple of 4; NaN thresholds become +inf. Class "none" is
// word 0 (below every class word) and the padded grid's border is 0xffff (its
// F decodes to NaN, which no test passes), so the unsigned max of the words
// of a run of cells is the word of the run's largest F (pass 1's run test).
typedef uint16_t ProbeT;
__device__ __forceinline__ ProbeT probeWord(uint8_t cls, double t) {
  if (cls == kClsNone) return 0u;
  // up-rounded twice (double -> f32 -> f16) stays >= t
  const __half hf = (t == t) ? __float2half_ru(__double2float_ru(t)) : __ushort_as_half(0x7c00);
  const uint32_t b = __half_as_ushort(hf);
  uint32_t key = (b & 0x8000u) ? (~b & 0xffffu) : (b | 0x8000u);
  key = (key + 3u) & ~3u;  // <= 0xfc00 (+inf) for every f16 <= +inf
  return static_cast<ProbeT>(key | cls);
}
__device__ __forceinline__ double probeBound(uint32_t w) {
  const uint32_t key = w & 0xfffcu;
  const uint32_t b = (key & 0x8000u) ? (key & 0x7fffu) : (~key & 0xffffu);
  return static_cast<double>(__half2float(__ushort_as_half(static_cast<unsigned short>(b))));
}

// Ray class + probe word of cell i from its post-fusion state, k* reset
// (the reference's ray-independent gates, raycast.cpp:132-183). A cell still
// being folded on the side stream is speculated "none" (see k_fuse_heavy).
struct ClassArgs {
  double now, t_free;
  int cleanup, bound;
  int W;  // grid width: the probe words sit on the (W+2) x (H+2) padded grid
};
__device__ __forceinline__ void classifyCell(const Layers& L, size_t i, bool speculated,
                                             const ClassArgs& a, uint8_t* cls, ProbeT* probe,
                                             int32_t* kstar) {
  uint8_t c = kClsNone;
  double t = 0.0;
  if (speculated) {
    c = kClsNone;
  } else if (!L.valid[i]) {
    c = a.bound ? kClsBound : kClsNone;
    if (c) t = L.ub[i];
  } else if (a.cleanup && !(a.now - L.last[i] <= a.t_free) &&
             (L.nx[i] != 0.0 || L.ny[i] != 0.0 || L.nz[i] != 0.0)) {
    c = kClsCandidate;
    t = L.elev[i] - sqrt(L.var[i]);
  }
  cls[i] = c;
  const size_t r = i / static_cast<unsigned>(a.W);
  probe[i + static_cast<size_t>(a.W) + 3 + 2 * r] = probeWord(c, t);  // padded (r+1, c+1)
  kstar[i] = INT_MAX;
  if (i == 0) kstar[-1] = INT_MAX;  // the frame's "any removal" flag (candidateVisit)
}

// ------------------------------------------------------------- K3 fusion
struct FuseArgs {
  double now;
  double sigma_init2, sigma_outlier2, sigma_max2, maha, maha2;
  int wall;
};

// Mahalanobis gate |z - h| / sqrt(v) > maha, decided exactly. The common case
// is settled by d^2 vs maha^2 v with a 1e-12 relative margin (the rounding of
// the reference's sqrt and division is below 3e-16 relative, so outside the
// margin both forms agree); near the boundary, or for magnitudes where d^2
// could overflow / underflow, the reference's own expression is evaluated.
__device__ __forceinline__ bool gateOutlier(double d, double cv, const FuseArgs& a) {
  if (d < 1e100 && cv > 1e-200 && cv < 1e200 && (d > 1e-100 || d == 0.0)) {
    const double lhs = d * d, rhs = a.maha2 * cv;
    if (lhs > rhs * (1.0 + 1e-12)) return true;
    if (lhs < rhs * (1.0 - 1e-12)) return false;
  }
  return d / sqrt(cv) > a.maha;
}

constexpr int kFoldBatch = 8;

// Cells with more points than this fold on the side stream (k_fuse_heavy).
#ifndef RB_HEAVY_CELL
#define RB_HEAVY_CELL 160  // = RB_VHEAVY_CELL: no lane-per-cell long fold
#endif
constexpr int kHeavyCell = RB_HEAVY_CELL;
#ifndef RB_HEAVY_BLOCKS
#define RB_HEAVY_BLOCKS 256
#endif
constexpr int kHeavyBlocks = RB_HEAVY_BLOCKS;  // one warp each

struct FoldCounts {
  unsigned long long nf = 0, no = 0, ni = 0, upd = 0;
};

// Running state of one cell's gated Kalman fold.
struct FoldState {
  bool valid, var_changed, bad, fused_any;
  double h, v;
};

__device__ __forceinline__ FoldState foldBegin(const Layers& L, size_t i) {
  return FoldState{L.valid[i] != 0, false, false, false, L.elev[i], L.var[i]};
}

// One point of the fold (reference integration.cpp:40-55, 142-203). Returns
// false when a non-positive variance stops the fold.
__device__ __forceinline__ bool foldPoint(FoldState& s, double z, double sp, bool wall,
                                          const FuseArgs& a, FoldCounts& k) {
  const double ch = s.valid ? s.h : z;
  const double cv = s.valid ? s.v : a.sigma_init2;
  if (cv <= 0.0 || sp <= 0.0) {
    s.bad = true;
    return false;
  }
  if (wall && z < ch) {
    ++k.ni;
    return true;
  }
  if (gateOutlier(fabs(z - ch), cv, a)) {
    ++k.no;
    if (s.valid) {
      s.v = smin(cv + a.sigma_outlier2, a.sigma_max2);
      s.var_changed = true;
    }
    return true;
  }
  // The two quotients share one reciprocal as straight-line code (div2_rn ==
  // IEEE a/b for all inputs), instead of two division subroutines one after
  // the other on the fold's dependent chain.
  const double denom = cv + sp;
  div2_rn(sp * ch + cv * z, cv * sp, denom, s.h, s.v);
  s.valid = true;
  s.fused_any = true;
  ++k.nf;
  return true;
}

// setEstimate (grid.cpp:139-147) for a cell that fused, else the outlier
// variance; flags a non-positive variance.
__device__ __forceinline__ bool foldEnd(const Layers& L, size_t i, const FoldState& s,
                                        const FuseArgs& a, DevStats* st, FoldCounts& k) {
  if (s.bad) atomicExch(&st->error_code, 1);
  if (s.fused_any) {
    L.elev[i] = s.h;
    L.var[i] = s.v;
    L.last[i] = a.now;
    L.valid[i] = 1;
    L.ub[i] = s.h;
    L.ubv[i] = 1;
    k.upd = k.upd + 1;
  } else if (s.var_changed) {
    L.var[i] = s.v;
  }
  return s.fused_any;
}

// Gated Kalman fold of one cell (reference integration.cpp:40-55,142-203,
// grid.cpp:139-147): the cell's points in scan order. The payload is
// contiguous per cell (written by the last radix pass), loaded in batches of 8
// with the next batch in flight while the current one is folded. Returns
// whether any point fused.
__device__ __forceinline__ bool foldCell(const Layers& L, size_t i, int cnt,
                                         const uint32_t* __restrict__ start,
                                         const double* __restrict__ spz,
                                         const double* __restrict__ spv, const FuseArgs& a,
                                         DevStats* st, FoldCounts& k) {
  FoldState s = foldBegin(L, i);
  const double* zp = spz + start[i];
  const double* vp = spv + start[i];
  const bool wall = cnt > a.wall;
  double zn[kFoldBatch], vn[kFoldBatch];
#pragma unroll
  for (int b = 0; b < kFoldBatch; ++b) {
    zn[b] = b < cnt ? zp[b] : 0.0;
    vn[b] = b < cnt ? vp[b] : 0.0;
  }
  for (int base = 0; base < cnt && !s.bad; base += kFoldBatch) {
    double zc[kFoldBatch], vc[kFoldBatch];
#pragma unroll
    for (int b = 0; b < kFoldBatch; ++b) {
      zc[b] = zn[b];
      vc[b] = vn[b];
      const int j = base + kFoldBatch + b;
      zn[b] = j < cnt ? zp[j] : 0.0;
      vn[b] = j < cnt ? vp[j] : 0.0;
    }
#pragma unroll
    for (int b = 0; b < kFoldBatch; ++b) {
      if (base + b >= cnt) break;
      if (!foldPoint(s, zc[b], vc[b], wall, a, k)) break;
    }
  }
  return foldEnd(L, i, s, a, st, k);
}

__device__ __forceinline__ void flushCounts(FoldCounts k, DevStats* st) {
  k.nf = warpSum(k.nf);
  k.no = warpSum(k.no);
  k.ni = warpSum(k.ni);
  k.upd = warpSum(k.upd);
  if ((threadIdx.x & 31) == 0 && (k.nf | k.no | k.ni | k.upd)) {
    if (k.nf) atomicAdd(&st->fused, k.nf);
    if (k.no) atomicAdd(&st->outlier, k.no);
    if (k.ni) atomicAdd(&st->ignored_low, k.ni);
    if (k.upd) atomicAdd(&st->cells_updated, k.upd);
  }
}

// Before the fold (RB_SPLIT_CLASSIFY): the drift offset (as k_apply_offset)
// and the ray class of every cell without points this scan -- its post-fusion
// state is its current one -- so the classification sweep after the fold
// shrinks to the cells k_fuse folds (which it classifies itself).
__global__ void __launch_bounds__(kThreads)
    k_prep(Layers L, size_t n, const double* off_p, const int32_t* __restrict__ count, ClassArgs ca,
           uint8_t* cls, ProbeT* probe, int32_t* kstar) {
  pdlEnter();
  const double off = off_p != nullptr ? *off_p : 0.0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    if (off != 0.0) {
      if (L.valid[i]) L.elev[i] += off;
      if (L.ubv[i]) L.ub[i] += off;
    }
    if (count[i] == 0) classifyCell(L, i, false, ca, cls, probe, kstar);
  }
}

#ifndef RB_VHEAVY_CELL
#define RB_VHEAVY_CELL 160  // (128 / 192 / 224 / 256 measured)
#endif
constexpr int kVeryHeavyCell = RB_VHEAVY_CELL;

// Queues a warp's long cells (more than `heavy` points) for k_fuse_heavy:
// more than kVeryHeavyCell points on the warp-per-cell list, the others on
// the lane-per-cell list. All 32 lanes call it.
__device__ __forceinline__ void appendHeavy(int cnt, int heavy, size_t i, uint32_t* heavy_list,
                                            uint32_t* vheavy_list, DevStats* st) {
  const bool is_heavy = cnt > heavy;
  const bool is_vheavy = is_heavy && cnt > kVeryHeavyCell;
  const int lane = threadIdx.x & 31;
  const unsigned hv = __ballot_sync(0xffffffffu, is_heavy && !is_vheavy);
  if (hv) {
    unsigned base = 0;
    if (lane == __ffs(hv) - 1)
      base = static_cast<unsigned>(atomicAdd(&st->heavy_cells, static_cast<unsigned long long>(__popc(hv))));
    base = __shfl_sync(0xffffffffu, base, __ffs(hv) - 1);
    if (is_heavy && !is_vheavy) heavy_list[base + __popc(hv & ((1u << lane) - 1u))] = static_cast<uint32_t>(i);
  }
  const unsigned vv = __ballot_sync(0xffffffffu, is_vheavy);
  if (vv) {
    unsigned base = 0;
    if (lane == __ffs(vv) - 1)
      base = static_cast<unsigned>(atomicAdd(&st->vheavy_cells, static_cast<unsigned long long>(__popc(vv))));
    base = __shfl_sync(0xffffffffu, base, __ffs(vv) - 1);
    if (is_vheavy) vheavy_list[base + __popc(vv & ((1u << lane) - 1u))] = static_cast<uint32_t>(i);
  }
}

// Appends the lanes with `pred` to `list` (warp-aggregated; order within a
// warp kept, across warps arbitrary). All 32 lanes call it.
__device__ __forceinline__ void appendCell(bool pred, size_t i, uint32_t* list, unsigned long long* n) {
  const int lane = threadIdx.x & 31;
  const unsigned b = __ballot_sync(0xffffffffu, pred);
  if (!b) return;
  unsigned base = 0;
  if (lane == __ffs(b) - 1) base = static_cast<unsigned>(atomicAdd(n, static_cast<unsigned long long>(__popc(b))));
  base = __shfl_sync(0xffffffffu, base, __ffs(b) - 1);
  if (pred) list[base + __popc(b & ((1u << lane) - 1u))] = static_cast<uint32_t>(i);
}

// appendCell filling the list downwards from `last`.
__device__ __forceinline__ void appendCellBack(bool pred, size_t i, uint32_t* last, unsigned long long* n) {
  const int lane = threadIdx.x & 31;
  const unsigned b = __ballot_sync(0xffffffffu, pred);
  if (!b) return;
  unsigned base = 0;
  if (lane == __ffs(b) - 1) base = static_cast<unsigned>(atomicAdd(n, static_cast<unsigned long long>(__popc(b))));
  base = __shfl_sync(0xffffffffu, base, __ffs(b) - 1);
  if (pred) *(last - (base + __popc(b & ((1u << lane) - 1u)))) = static_cast<uint32_t>(i);
}

// Second-stream sweep after the ingest (RB_EARLY_HEAVY): the drift offset
// (off_p null: none) and the long-cell lists from the per-cell counts, so the
// long-cell fold can start as soon as the sort is done, beside k_fuse (which
// then builds no lists).
__global__ void __launch_bounds__(kThreads)
    k_side_prep(Layers L, size_t n, const double* off_p, const int32_t* __restrict__ count, int heavy,
                uint32_t* heavy_list, uint32_t* vheavy_list, uint32_t* light_list, uint32_t* pre_list,
                DevStats* st, int classify,
                ClassArgs ca, uint8_t* __restrict__ cls, ProbeT* __restrict__ probe,
                int32_t* __restrict__ kstar) {
  RB_TL(6);
  const double off = off_p != nullptr ? *off_p : 0.0;
  const int lane = threadIdx.x & 31;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t b = blockIdx.x * static_cast<size_t>(blockDim.x) + (threadIdx.x & ~31u); b < n; b += stride) {
    const size_t i = b + lane;
    const bool in = i < n;
    if (in && off != 0.0) {
      if (L.valid[i]) L.elev[i] += off;
      if (L.ubv[i]) L.ub[i] += off;
    }
    const int cnt = in ? count[i] : 0;
    // pre_list (RB_PRESPLIT): a cell with points whose class before the fold
    // is "removal candidate" (valid, stale, with a normal) ends the fold as a
    // candidate or, if it fuses, as "none" -- it is folded and classified
    // before the ray pass. Every other cell with points ends the fold "none"
    // (it fuses, so it is fresh; or it stays valid and fresh, or without a
    // normal; only a variance error could leave it otherwise, which the folds'
    // checkSpeculation turns into a retry): classified "none" here and folded
    // beside the ray pass.
    bool pre = false;
    if (pre_list != nullptr && cnt > 0)
      pre = L.valid[i] && ca.cleanup && !(ca.now - L.last[i] <= ca.t_free) &&
            (L.nx[i] != 0.0 || L.ny[i] != 0.0 || L.nz[i] != 0.0);
    const int lc = pre ? 0 : cnt;
    if (heavy_list != nullptr) appendHeavy(lc, heavy, i, heavy_list, vheavy_list, st);
    if (light_list != nullptr) {
      // RB_LIGHT_SPLIT: cells of up to that many points from the front of the
      // list, longer ones from its far end, so a fold warp's lanes get folds of
      // similar length
      const int split = RB_LIGHT_SPLIT > 0 ? RB_LIGHT_SPLIT : heavy;
      appendCell(lc > 0 && lc <= split, i, light_list, &st->light_cells);
      if (RB_LIGHT_SPLIT > 0) appendCellBack(lc > split && lc <= heavy, i, light_list + n - 1, &st->light2_cells);
    }
    if (pre_list != nullptr) appendCell(pre, i, pre_list, &st->pre_cells);
    // (classify: the cells without points, and the long cells speculatively;
    // the short-cell fold classifies the cells it folds)
    if (pre_list != nullptr) {
      if (in && !pre) {
        classifyCell(L, i, cnt > 0, ca, cls, probe, kstar);
      } else if (pre && RB_SIDE_JUMP && n >= kSideJumpCells) {
        // provisional probe word "candidate" (the jump grid built on this
        // stream then never jumps the cell's block); the candidates' fold
        // writes the real class before the ray pass reads it
        const size_t r = i / static_cast<unsigned>(ca.W);
        probe[i + static_cast<size_t>(ca.W) + 3 + 2 * r] = probeWord(kClsCandidate, 0.0);
      }
    } else if (classify && in && (cnt == 0 || cnt > heavy)) {
      classifyCell(L, i, cnt > heavy, ca, cls, probe, kstar);
    }
  }
}

// Post-fusion ray class of a cell the concurrent ray pass treated as "none";
// flags a wrong speculation.
__device__ __forceinline__ void checkSpeculation(const Layers& L, size_t i, const FuseArgs& a,
                                                 double t_free, int cleanup, int bound, DevStats* st) {
  const bool none = L.valid[i] ? !(cleanup && !(a.now - L.last[i] <= t_free) &&
                                   (L.nx[i] != 0.0 || L.ny[i] != 0.0 || L.nz[i] != 0.0))
                               : !bound;
  if (!none) atomicExch(&st->respeculate, 1);
}

// The short cells listed by k_side_prep, one thread each (grid-stride): only
// occupied cells take threads, instead of one thread per map cell (k_fuse).
#ifndef RB_FUSE_LIST_THREADS
#define RB_FUSE_LIST_THREADS 256
#endif
#ifndef RB_FUSE_LIST_BLOCKS
#define RB_FUSE_LIST_BLOCKS 2  // k_fuse_list blocks per SM (3 x 128 threads: slower)
#endif
__global__ void __launch_bounds__(RB_FUSE_LIST_THREADS)
    k_fuse_list(Layers L, const int32_t* __restrict__ count, const uint32_t* __restrict__ list,
                const unsigned long long* n_list, const unsigned long long* n_back, size_t list_len,
                const uint32_t* __restrict__ start,
                const double* __restrict__ spz, const double* __restrict__ spv, FuseArgs a,
                DevStats* st, int classify, ClassArgs ca, uint8_t* __restrict__ cls,
                ProbeT* __restrict__ probe, int32_t* __restrict__ kstar) {
  RB_TL(7);
  pdlWait();
  pdlTrigger();
  // classify 1: classify each folded cell; 2: it was classified "none" before
  // the fold (RB_PRESPLIT) -- check that (a wrong class retries the ray pass)
  // n_back (not null): n_back entries more at the far end of the list
  const unsigned front = static_cast<unsigned>(*n_list);
  const unsigned total = front + (n_back != nullptr ? static_cast<unsigned>(*n_back) : 0u);
  FoldCounts k;
  for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < total; q += gridDim.x * blockDim.x) {
    const uint32_t i = q < front ? list[q] : list[list_len - 1 - (q - front)];
    foldCell(L, i, count[i], start, spz, spv, a, st, k);
    if (classify == 1) classifyCell(L, i, false, ca, cls, probe, kstar);
    if (classify == 2) checkSpeculation(L, i, a, ca.t_free, ca.cleanup, ca.bound, st);
  }
  flushCounts(k, st);
}

// Cells with at most `heavy` points are folded here, one thread per cell;
// longer cells are queued for k_fuse_heavy, which runs on a second stream
// concurrently with the ray pass: cells
// with more than kVeryHeavyCell points on their own list (one warp each there).
//
// Every cell also gets the frame's drift offset first (reference drift.cpp:
// 44-55, off_p: device scalar from the ingest's drift reduction; null = none)
// and, after its fold, its ray class and probe word (classify != 0), so the
// ray pass follows without a separate classification sweep.
__global__ void __launch_bounds__(kThreads)
    k_fuse(Layers L, size_t ncell, const int32_t* __restrict__ count,
           const uint32_t* __restrict__ start, const double* __restrict__ spz,
           const double* __restrict__ spv, FuseArgs a, DevStats* st, int heavy,
           uint32_t* heavy_list, uint32_t* vheavy_list, const double* __restrict__ off_p,
           int classify, ClassArgs ca, uint8_t* __restrict__ cls, ProbeT* __restrict__ probe,
           int32_t* __restrict__ kstar) {
  RB_TL(7);
  // wait first: the ray pass launched on our trigger may then read anything
  // older than this kernel before its own wait. When the ray pass follows
  // directly (classify 2), trigger only once the fold is done: resident
  // pass-1 blocks waiting for us would take the registers this low-occupancy
  // fold needs.
  pdlWait();
  if (classify != 2) pdlTrigger();
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  const int cnt = i < ncell ? count[i] : 0;
  if (off_p != nullptr && i < ncell) {
    const double off = *off_p;
    if (off != 0.0) {
      if (L.valid[i]) L.elev[i] += off;
      if (L.ubv[i]) L.ub[i] += off;
    }
  }
  const bool is_heavy = cnt > heavy;
  if (heavy_list != nullptr) appendHeavy(cnt, heavy, i, heavy_list, vheavy_list, st);
  FoldCounts k;
  if (cnt > 0 && !is_heavy) foldCell(L, i, cnt, start, spz, spv, a, st, k);
  // classify 1: every cell; 2: the cells with points (k_prep classified the rest)
  if (i < ncell && (classify == 1 || (classify == 2 && cnt > 0)))
    classifyCell(L, i, is_heavy, ca, cls, probe, kstar);
  flushCounts(k, st);
  if (classify == 2) pdlTrigger();
}

// Long cells (queued by k_fuse), concurrently with the ray pass. The very
// long ones first, one warp each: the warp stages the cell's payload into
// shared memory (coalesced, all loads in flight at once) and lane 0 folds it
// from there -- one thread folding from global memory waits an L2 round trip
// per prefetch batch (~250 cycles per point, scripts/fold_bench.cu), which made
// the longest cell (1,230 points) the critical path. Then the rest, one cell
// per lane from global memory.
constexpr int kHeavyStage = 2048;  // points staged per round (32 KB)
__global__ void __launch_bounds__(32)
    k_fuse_heavy(Layers L, const int32_t* __restrict__ count, const uint32_t* __restrict__ list,
                 const uint32_t* __restrict__ vlist, const DevStats* st_in,
                 const uint32_t* __restrict__ start, const double* __restrict__ spz,
                 const double* __restrict__ spv, FuseArgs a, DevStats* st, double t_free,
                 int cleanup, int bound) {
  RB_TL(8);
  __shared__ double sz[kHeavyStage];
  __shared__ double sv[kHeavyStage];
  const int lane = threadIdx.x;
  FoldCounts k;
  const unsigned nv = static_cast<unsigned>(st_in->vheavy_cells);
  for (unsigned q = blockIdx.x; q < nv; q += gridDim.x) {
    const uint32_t i = vlist[q];
    const int cnt = count[i];
    const uint32_t s0 = start[i];
    const bool wall = cnt > a.wall;
    FoldState s{};
    if (lane == 0) s = foldBegin(L, i);
    bool go = true;
    for (int base = 0; base < cnt && go; base += kHeavyStage) {
      const int n = min(kHeavyStage, cnt - base);
      __syncwarp();
      for (int j = lane; j < n; j += 32) {
        sz[j] = spz[s0 + base + j];
        sv[j] = spv[s0 + base + j];
      }
      __syncwarp();
      // Warp-cooperative fold: points the wall rule ignores leave (h, v)
      // unchanged, so the lanes test the next 32 points against the current
      // state at once and the whole leading run of ignored points is skipped
      // in one step (counted, in order); lane 0 then folds the first point
      // that is not ignored. Same decisions in the same order as the
      // sequential fold.
      int j = 0;
      while (j < n) {
        const bool valid = __shfl_sync(0xffffffffu, s.valid, 0);
        const double h = __shfl_sync(0xffffffffu, s.h, 0);
        const double v = __shfl_sync(0xffffffffu, s.v, 0);
        const int jj = j + lane;
        // ignored <=> no variance error (cv, sp > 0) and the wall rule fires;
        // an invalid cell compares z < z (false) -- never ignored.
        const bool ign = wall && valid && v > 0.0 && jj < n && sv[jj] > 0.0 && sz[jj] < h;
        const unsigned run_mask = ~__ballot_sync(0xffffffffu, ign);
        const int run = run_mask ? __ffs(run_mask) - 1 : 32;
        if (lane == 0) k.ni += static_cast<unsigned>(run);
        j += run;
        if (run == 32 || j >= n) continue;
        int ok = 1;
        if (lane == 0) ok = foldPoint(s, sz[j], sv[j], wall, a, k) ? 1 : 0;
        ++j;
        if (!__shfl_sync(0xffffffffu, ok, 0)) break;
      }
      go = __shfl_sync(0xffffffffu, lane == 0 ? !s.bad : 1, 0) != 0;
    }
    if (lane == 0) {
      foldEnd(L, i, s, a, st, k);
      checkSpeculation(L, i, a, t_free, cleanup, bound, st);
    }
  }
  // The other long cells, one per lane, on the blocks that had no very long
  // cell (a very long cell's fold is the kernel's critical path: its block
  // takes no further work unless every block had one).
  const unsigned total = static_cast<unsigned>(st_in->heavy_cells);
  const unsigned busy = nv < gridDim.x ? nv : 0u;
  if (blockIdx.x < busy) {
    flushCounts(k, st);
#ifdef RB_TIMELINE
    if (lane == 0) atomicMax(&g_tl_end[9][blockIdx.x & 31], tlNow());  // warp-per-cell part's end
#endif
    return;
  }
  for (unsigned q = (blockIdx.x - busy) * 32 + lane; q < total; q += (gridDim.x - busy) * 32) {
    const uint32_t i = list[q];
    foldCell(L, i, count[i], start, spz, spv, a, st, k);
    checkSpeculation(L, i, a, t_free, cleanup, bound, st);
  }
  flushCounts(k, st);
#ifdef RB_TIMELINE
  if (lane == 0) atomicMax(&g_tl_end[10][blockIdx.x & 31], tlNow());  // lane-per-cell part's end
#endif
}

// ------------------------------------------------------------- K5/K6 rays
// Classification sweep for the retry of a wrong speculation (retry = 1: runs
// only if k_fuse_heavy flagged it) and for frames whose classes k_fuse did not
// write (a shard frame without records).
__global__ void __launch_bounds__(kThreads) k_classify(Layers L, size_t n, RayArgs a, uint8_t* cls,
                                                       int32_t* kstar,
                                                       const int32_t* __restrict__ count,
                                                       int heavy, int retry, DevStats* st,
                                                       ProbeT* probe) {
  RB_TL(9 + retry);
  // wait first: the ray pass launched on our trigger may then read anything
  // older than this kernel before its own wait
  pdlWait();
  pdlTrigger();
  if (retry) {
    if (!st->respeculate) return;
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // pass 1 runs again from scratch
      st->candidate_rays = 0;
      st->visits = 0;
    }
  }
  const ClassArgs ca{a.now, a.t_free, a.cleanup, a.bound, a.g.W};
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    classifyCell(L, i, heavy >= 0 && count[i] > heavy, ca, cls, probe, kstar);
}

// Pass-1 jump grid: per kJumpBlk x kJumpBlk block of cells, the largest probe
// word over the block and a one-cell ring around it (so a cell the exact walk
// reaches while the real line runs through a neighbouring block, by rounding
// at a block edge, is covered), 0xffff (bound NaN: never jumped) when any of
// those cells is a removal candidate (its rays must be queued, exactly) or
// the border. One warp per block: lanes 0-17 take the 18 ring columns.
__global__ void __launch_bounds__(kThreads) k_jump_grid(const ProbeT* __restrict__ probe, int W, int H,
                                                        float* __restrict__ jg, int jw, int jh) {
  RB_TL(11);
  pdlWait();
  pdlTrigger();
  const int warp = static_cast<int>((blockIdx.x * static_cast<unsigned>(kThreads) + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (warp >= jw * jh) return;
  const int by = warp / jw, bx = warp - by * jw;
  uint32_t mx = 0, cand = 0;
  for (int q = lane; q < kJumpBlk + 2; q += 32) {
    const int pc = kJumpBlk * bx + q;  // padded column (the ring starts one cell left)
    if (pc > W + 1) break;
    // padded rows kJumpBlk*by .. +kJumpBlk+1 (past H + 1: the border guard rows)
    const ProbeT* p = probe + static_cast<size_t>(kJumpBlk * by) * (W + 2) + pc;
#pragma unroll 6
    for (int r = 0; r < kJumpBlk + 2; ++r) {
      const uint32_t wd = p[static_cast<size_t>(r) * (W + 2)];
      mx = max(mx, wd);
      cand |= (wd & 3u) == kClsCandidate ? 1u : 0u;
    }
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  cand = __reduce_or_sync(0xffffffffu, cand);
  // the block's bound as f32: -inf (no class cell), F of the largest word
  // (an f16 value, exact in f32), +inf for a candidate / the border / NaN
  if (lane == 0) {
    float b = -__int_as_float(0x7f800000);
    if (cand || mx == 0xffffu) b = __int_as_float(0x7f800000);
    else if (mx != 0u) b = static_cast<float>(probeBound(mx));
    jg[warp] = b == b ? b : __int_as_float(0x7f800000);
  }
}

// Liang-Barsky slab clip (reference raycast.cpp:30-42).
__device__ __forceinline__ bool clipAxis(double p, double q, double& t0, double& t1) {
  if (p == 0.0) return q >= 0.0;
  const double r = q / p;
  if (p < 0.0) {
    if (r > t1) return false;
    t0 = smax(t0, r);
  } else {
    if (r < t0) return false;
    t1 = smin(t1, r);
  }
  return t0 <= t1;
}

__device__ __forceinline__ int clampCell(int v, int n) { return v < 0 ? 0 : (v > n - 1 ? n - 1 : v); }

// Exact 2-D DDA from o to p (reference raycast.cpp:48-130). Calls
// visit(cell, t_enter, t_next, vertical) for every emitted cell; the ray
// height there is o.z + (0.5*(t_enter+t_next))*dz, or o.z + 0.5*dz for a
// vertical ray. Returns nothing; the operation sequence is the reference's.
template <typename Visit>
__device__ __forceinline__ void walkRay(const GridArgs& g, const double o[3], double px, double py,
                                        Visit&& visit) {
  const double dx = px - o[0];
  const double dy = py - o[1];
  const double res = g.res;
  if (libm_hypot(dx, dy) < 1e-12) {
    if (o[0] >= g.ox && o[0] < g.xmax && o[1] >= g.oy && o[1] < g.ymax) {
      const int row = clampCell(x86_to_int(floor((o[1] - g.oy) / res)), g.H);
      const int col = clampCell(x86_to_int(floor((o[0] - g.ox) / res)), g.W);
      visit(static_cast<uint32_t>(row) * g.W + col, 0.0, 0.0, true);
    }
    return;
  }
  double t0 = 0.0, t1 = 1.0;
  if (!clipAxis(-dx, o[0] - g.ox, t0, t1)) return;
  if (!clipAxis(dx, g.xmax - o[0], t0, t1)) return;
  if (!clipAxis(-dy, o[1] - g.oy, t0, t1)) return;
  if (!clipAxis(dy, g.ymax - o[1], t0, t1)) return;
  if (t0 >= t1) return;

  const bool end_in = px >= g.ox && px < g.xmax && py >= g.oy && py < g.ymax;
  uint32_t end_idx = 0xffffffffu;  // never equal to a cell index
  if (end_in)
    end_idx = static_cast<uint32_t>(clampCell(x86_to_int(floor((py - g.oy) / res)), g.H)) * g.W +
              clampCell(x86_to_int(floor((px - g.ox) / res)), g.W);
  const double sx = o[0] + t0 * dx;
  const double sy = o[1] + t0 * dy;
  int col = clampCell(x86_to_int(floor((sx - g.ox) / res)), g.W);
  int row = clampCell(x86_to_int(floor((sy - g.oy) / res)), g.H);
  const int step_col = dx > 0.0 ? 1 : (dx < 0.0 ? -1 : 0);
  const int step_row = dy > 0.0 ? 1 : (dy < 0.0 ? -1 : 0);
  double tmx = kInf, tmy = kInf, tdx = kInf, tdy = kInf;
  if (step_col != 0) {
    const double boundary = g.ox + (col + (step_col > 0 ? 1 : 0)) * res;
    tmx = (boundary - o[0]) / dx;
    tdx = res / fabs(dx);
  }
  if (step_row != 0) {
    const double boundary = g.oy + (row + (step_row > 0 ? 1 : 0)) * res;
    tmy = (boundary - o[1]) / dy;
    tdy = res / fabs(dy);
  }
  // Linear cell index advanced incrementally; the endpoint test compares
  // indices (row/col are in range inside the loop, so this equals the
  // reference's CellIndex comparison).
  uint32_t idx = static_cast<uint32_t>(row) * g.W + col;
  const int step_idx_row = step_row * g.W;
  double t_enter = t0;
  while (true) {
    double m = tmx;  // std::min({tmx, tmy, t1}): first smallest wins
    if (tmy < m) m = tmy;
    const double t_next = (t1 < m) ? t1 : m;
    if (idx != end_idx && t_next > t_enter) visit(idx, t_enter, t_next, false);
    if (t_next >= t1) break;
    if (tmx < tmy) {
      col += step_col;
      tmx += tdx;
      idx += step_col;
      if (static_cast<unsigned>(col) >= static_cast<unsigned>(g.W)) break;
    } else {
      row += step_row;
      tmy += tdy;
      idx += step_idx_row;
      if (static_cast<unsigned>(row) >= static_cast<unsigned>(g.H)) break;
    }
    t_enter = t_next;
  }
}

// Same traversal for rays whose xy deltas are finite (every ray of a real
// scan). Without NaNs the first-smallest min of {t_max_x, t_max_y, t1} and the
// two exit tests collapse to one comparison each: m = (tmx < tmy ? tmx : tmy)
// equals the reference's min in value (ties are equal values; +-0 only occurs
// where it is not observable), and t_next >= t1 <=> !(m < t1).
template <typename Visit>
__device__ __forceinline__ void walkRayFinite(const GridArgs& g, const double o[3], double px,
                                              double py, Visit&& visit) {
  const double dx = px - o[0];
  const double dy = py - o[1];
  const double res = g.res;
  if (libm_hypot(dx, dy) < 1e-12) {
    if (o[0] >= g.ox && o[0] < g.xmax && o[1] >= g.oy && o[1] < g.ymax) {
      const int row = clampCell(x86_to_int(floor((o[1] - g.oy) / res)), g.H);
      const int col = clampCell(x86_to_int(floor((o[0] - g.ox) / res)), g.W);
      visit(static_cast<uint32_t>(row) * g.W + col, 0.0, 0.0, true);
    }
    return;
  }
  double t0 = 0.0, t1 = 1.0;
  if (!clipAxis(-dx, o[0] - g.ox, t0, t1)) return;
  if (!clipAxis(dx, g.xmax - o[0], t0, t1)) return;
  if (!clipAxis(-dy, o[1] - g.oy, t0, t1)) return;
  if (!clipAxis(dy, g.ymax - o[1], t0, t1)) return;
  if (t0 >= t1) return;
  const bool end_in = px >= g.ox && px < g.xmax && py >= g.oy && py < g.ymax;
  uint32_t end_idx = 0xffffffffu;
  if (end_in)
    end_idx = static_cast<uint32_t>(clampCell(x86_to_int(floor((py - g.oy) / res)), g.H)) * g.W +
              clampCell(x86_to_int(floor((px - g.ox) / res)), g.W);
  int col = clampCell(x86_to_int(floor(((o[0] + t0 * dx) - g.ox) / res)), g.W);
  int row = clampCell(x86_to_int(floor(((o[1] + t0 * dy) - g.oy) / res)), g.H);
  const int step_col = dx > 0.0 ? 1 : (dx < 0.0 ? -1 : 0);
  const int step_row = dy > 0.0 ? 1 : (dy < 0.0 ? -1 : 0);
  double tmx = kInf, tmy = kInf, tdx = kInf, tdy = kInf;
  if (step_col != 0) {
    tmx = ((g.ox + (col + (step_col > 0 ? 1 : 0)) * res) - o[0]) / dx;
    tdx = res / fabs(dx);
  }
  if (step_row != 0) {
    tmy = ((g.oy + (row + (step_row > 0 ? 1 : 0)) * res) - o[1]) / dy;
    tdy = res / fabs(dy);
  }
  uint32_t idx = static_cast<uint32_t>(row) * g.W + col;
  const int step_idx_row = step_row * g.W;
  const unsigned W = static_cast<unsigned>(g.W), H = static_cast<unsigned>(g.H);
  double t_enter = t0;
  while (true) {
    const bool sx = tmx < tmy;
    const double m = sx ? tmx : tmy;
    const bool more = m < t1;
    const double t_next = more ? m : t1;
    if (idx != end_idx && t_next > t_enter) visit(idx, t_enter, t_next, false);
    if (!more) break;
    if (sx) {
      col += step_col;
      tmx += tdx;
      idx += step_col;
      if (static_cast<unsigned>(col) >= W) break;
    } else {
      row += step_row;
      tmy += tdy;
      idx += step_idx_row;
      if (static_cast<unsigned>(row) >= H) break;
    }
    t_enter = t_next;
  }
}

// Dispatch: the literal walk handles non-finite endpoints (NaN / inf points
// reach the ray phase exactly as in the reference).
template <typename Visit>
__device__ __forceinline__ void walk(const GridArgs& g, const double o[3], double px, double py,
                                     Visit&& visit) {
  if (isfinite(px - o[0]) && isfinite(py - o[1])) walkRayFinite(g, o, px, py, visit);
  else walkRay(g, o, px, py, visit);
}

__device__ __forceinline__ double rayHeight(double oz, double dz, double te, double tn, bool vertical) {
  return vertical ? oz + 0.5 * dz : oz + (0.5 * (te + tn)) * dz;
}

// Running min of the upper bound with the reference's comparison (raycast.cpp:
// 167-183): CAS while ray_h < current. `seen` is a possibly stale (L1) read of
// the bound; bounds only decrease, so a stale value is never below the true
// one and the CAS loop settles on the true minimum.
__device__ __forceinline__ void boundMinSlow(const Layers& L, uint32_t c, double h, double seen) {
  unsigned long long* addr = reinterpret_cast<unsigned long long*>(L.ub + c);
  double cur = seen;
  while (h < cur) {
    const unsigned long long want = static_cast<unsigned long long>(__double_as_longlong(cur));
    const unsigned long long got =
        atomicCAS(addr, want, static_cast<unsigned long long>(__double_as_longlong(h)));
    if (got == want) {
      L.ubv[c] = 1;
      break;
    }
    cur = __longlong_as_double(static_cast<long long>(got));
  }
}

__device__ __forceinline__ void boundMin(const Layers& L, uint32_t c, double h) {
  const double seen = L.ub[c];
  if (h < seen) boundMinSlow(L, c, h, seen);
}

// Removal gates for a candidate cell (reference raycast.cpp:138-150), literal
// comparison forms; records the ray in k*.
#ifndef RB_CAND_LAZY
#define RB_CAND_LAZY 1
#endif
__device__ __forceinline__ void candidateVisit(const Layers& L, uint32_t c, double h, double vx,
                                               double vy, double vz, double alpha_n, int32_t k,
                                               int32_t* kstar) {
  const double gate = L.elev[c] - sqrt(L.var[c]);
  if (h >= gate) return;
#if RB_CAND_LAZY
  // the direction is normalised here, on this rare path, not hoisted into
  // every ray's setup (the empty asm makes it depend on the cell)
  asm("" : "+d"(vx), "+d"(vy), "+d"(vz) : "d"(gate));
#endif
  const double n2 = (vx * vx + vy * vy) + vz * vz;
  double ux = vx, uy = vy, uz = vz;
  if (n2 > 0.0) {
    const double nrm = sqrt(n2);
    ux = vx / nrm;
    uy = vy / nrm;
    uz = vz / nrm;
  }
  const double align = fabs((ux * L.nx[c] + uy * L.ny[c]) + uz * L.nz[c]);
  if (align <= alpha_n) return;
  if (k < kstar[c]) {
    atomicMin(kstar + c, k);
    kstar[-1] = 0;  // "some cell is removed this frame" (reset with k*)
  }
}

struct Pass1Ctx {
  const uint8_t* cls;
  const ProbeT* probe;
  Layers L;
  int32_t* kstar;
  double oz, dz, vx, vy, alpha_n;
  int32_t k;
};

__device__ __forceinline__ void pass1Visit(const Pass1Ctx& c, uint8_t cl, uint32_t idx, double h,
                                           bool& touched) {
  if (cl == kClsBound) {
    boundMin(c.L, idx, h);
    return;
  }
  touched = true;
  candidateVisit(c.L, idx, h, c.vx, c.vy, c.dz, c.alpha_n, c.k, c.kstar);
}

#ifdef RB_P1_DIAG
__device__ unsigned long long g_p1diag[7];
__global__ void k_p1diag() {
  printf("P1DIAG fast_runs %llu end_runs %llu gate_runs %llu rays %llu cells %llu jumped_cells %llu jumps %llu\n",
         g_p1diag[0], g_p1diag[1], g_p1diag[2], g_p1diag[3], g_p1diag[4], g_p1diag[5], g_p1diag[6]);
  for (int i = 0; i < 7; ++i) g_p1diag[i] = 0;
}
#endif
#ifndef RB_P1_RUN
#define RB_P1_RUN 8  // cells per lookahead run in pass 1
#endif

// Pass 1 of a ray with finite xy deltas, in two parts: pass1Setup (per lane:
// the reference's clip, start / end cells and first crossing times) and
// pass1Walk (the DDA, run by every lane of the warp together).
//
// Setup shortcuts, each equal to the reference's arithmetic:
// * |dx| or |dy| >= 2e-12 implies hypot(dx, dy) >= 1e-12 (hypot is within an
//   ulp of a value >= max(|dx|, |dy|)), so the vertical test needs no hypot;
// * origin and endpoint both in the map: the four Liang-Barsky clips leave
//   t0 = 0, t1 = 1 (every q >= 0, and q >= |p| on the side the ray moves
//   towards because fl(xmax - o) >= fl(px - o) when px < xmax), so the start
//   cell is the origin's (RayArgs::ocol/orow);
// * the endpoint's cell is the point's cell from k_ingest (same expression
//   floor((p - origin) / res), in range so the clamp is the identity) when
//   that is known (pcell < W*H).
struct P1Walk {
  double tmx, tmy, tdx, tdy, t_enter, t1;
  uint32_t idx, end_idx, wd;  // padded cell index, the endpoint's, the cell's probe word
  int step_col, step_row;     // index steps (step_row = +-(W+2))
  int col, row;               // the cell (pass1Jump only; the walk keeps idx)
};

// Returns true when the ray has a walk left (the vertical and clipped-out
// cases are finished here).
__device__ __forceinline__ bool pass1Setup(const GridArgs& g, const double o[3], double px,
                                           double py, const Pass1Ctx& c, bool& touched,
                                           unsigned& visits, const RayArgs& a, uint32_t pcell,
                                           P1Walk& w) {
  const double dx = px - o[0];
  const double dy = py - o[1];
  const double res = g.res;
  if (!(fabs(dx) >= 2e-12 || fabs(dy) >= 2e-12) && libm_hypot(dx, dy) < 1e-12) {
    pdlWait();
    if (o[0] >= g.ox && o[0] < g.xmax && o[1] >= g.oy && o[1] < g.ymax) {
      const uint32_t idx =
          static_cast<uint32_t>(clampCell(x86_to_int(floor((o[1] - g.oy) / res)), g.H)) * g.W +
          clampCell(x86_to_int(floor((o[0] - g.ox) / res)), g.W);
      ++visits;
      const uint8_t cl = c.cls[idx];
      if (cl) pass1Visit(c, cl, idx, o[2] + 0.5 * c.dz, touched);
    }
    return false;
  }
  double t0 = 0.0, t1 = 1.0;
  const bool end_in = px >= g.ox && px < g.xmax && py >= g.oy && py < g.ymax;
  if (!(a.origin_in && end_in)) {
    if (!clipAxis(-dx, o[0] - g.ox, t0, t1)) return false;
    if (!clipAxis(dx, g.xmax - o[0], t0, t1)) return false;
    if (!clipAxis(-dy, o[1] - g.oy, t0, t1)) return false;
    if (!clipAxis(dy, g.ymax - o[1], t0, t1)) return false;
    if (t0 >= t1) return false;
  }
  const uint32_t W = static_cast<uint32_t>(g.W), Wp = W + 2u;  // padded grid (pass1Exact)
  uint32_t end_idx = 0xffffffffu;  // padded index of the endpoint's cell
  if (end_in) {
    uint32_t er, ec;
    if (pcell < W * static_cast<uint32_t>(g.H)) {
      er = pcell / W;
      ec = pcell - er * W;
    } else {
      er = static_cast<uint32_t>(clampCell(x86_to_int(floor((py - g.oy) / res)), g.H));
      ec = static_cast<uint32_t>(clampCell(x86_to_int(floor((px - g.ox) / res)), g.W));
    }
    end_idx = (er + 1u) * Wp + ec + 1u;
  }
  int col = a.ocol, row = a.orow;
  if (t0 != 0.0) {
    col = clampCell(x86_to_int(floor(((o[0] + t0 * dx) - g.ox) / res)), g.W);
    row = clampCell(x86_to_int(floor(((o[1] + t0 * dy) - g.oy) / res)), g.H);
  }
  const int step_col = dx > 0.0 ? 1 : (dx < 0.0 ? -1 : 0);
  const int step_row = dy > 0.0 ? 1 : (dy < 0.0 ? -1 : 0);
  double tmx = kInf, tmy = kInf, tdx = kInf, tdy = kInf;
  // t_max and t_delta share the divisor |d| (a / -b == -(a / b) exactly).
  if (step_col != 0) {
    double q;
    div2_rn(res, (g.ox + (col + (step_col > 0 ? 1 : 0)) * res) - o[0], fabs(dx), tdx, q);
    tmx = dx < 0.0 ? -q : q;
  }
  if (step_row != 0) {
    double q;
    div2_rn(res, (g.oy + (row + (step_row > 0 ? 1 : 0)) * res) - o[1], fabs(dy), tdy, q);
    tmy = dy < 0.0 ? -q : q;
  }
  w.tmx = tmx;
  w.tmy = tmy;
  w.tdx = tdx;
  w.tdy = tdy;
  w.t_enter = t0;
  w.t1 = t1;
  w.idx = (static_cast<uint32_t>(row) + 1u) * Wp + static_cast<uint32_t>(col) + 1u;
  w.end_idx = end_idx;
  w.step_col = step_col;
  w.step_row = step_row * static_cast<int>(Wp);
  w.col = col;
  w.row = row;
  return true;
}

// Exact cells of a walk, one at a time (the reference's step, raycast.cpp:
// 112-129), at most `cells` of them; returns true when the walk ended. The
// probe words live on a grid padded by one border cell on every side (word
// 0xffff, tag 3): the walk leaves the grid exactly when it steps onto the
// border (the reference's bounds test after a step), so the loop carries no
// per-axis bounds tests. Only class cells leave the common path; the endpoint
// and zero-length tests of the reference's emission (t_next > t_enter) are
// made there, on the rare branch.
__device__ __forceinline__ bool pass1Exact(P1Walk& w, const Pass1Ctx& c, uint32_t W,
                                           unsigned cells, unsigned& nv, bool& touched) {
  const uint32_t Wp = W + 2u;
#pragma unroll 1
  for (unsigned s = 0; s < cells; ++s) {
    const bool sx = w.tmx < w.tmy;
    const double m = sx ? w.tmx : w.tmy;  // = the reference's min (no NaN here)
    const bool more = m < w.t1;
    if ((w.wd & 3u) != 0) {
      if ((w.wd & 3u) == 3u) return true;  // stepped out of the grid: stop before this cell
      const double t_next = more ? m : w.t1;
      if (w.idx != w.end_idx && t_next > w.t_enter) {
        const double h = c.oz + (0.5 * (w.t_enter + t_next)) * c.dz;
        const uint8_t tag = static_cast<uint8_t>(w.wd & 3u);
        if (tag == kClsCandidate) touched = true;
        // probe filter: h >= F implies the exact gate rejects (see probeWord)
        if (!(h >= probeBound(w.wd))) {
          const uint32_t pr = w.idx / Wp;
          pass1Visit(c, tag, (pr - 1u) * W + (w.idx - pr * Wp - 1u), h, touched);
        }
      }
    }
    ++nv;
    if (!more) return true;
    if (sx) w.tmx += w.tdx;
    else w.tmy += w.tdy;
    w.idx += sx ? w.step_col : w.step_row;
    w.wd = c.probe[w.idx];
    w.t_enter = m;
  }
  return false;
}

// The walk, called by all 32 lanes of the warp (walking = false for lanes
// without one). Runs of RB_P1_RUN cells: the walk (cell sequence and
// crossing times) does not depend on the probe words, so the next RB_P1_RUN
// steps are taken with their words loaded back to back (one memory latency
// per run instead of one per cell), and the run is committed without per-cell
// work when
// (a) it is not the ray's last (its last crossing time is < t1, so every
//     cell of it continues the walk: crossing times are non-decreasing), and
// (b) no cell of it can pass its gate: every emitted height of the run lies
//     between fl(oz + t*dz) at the run's first entry and last crossing time
//     (the height's three correctly rounded operations are monotone in the
//     two times, which lie in that interval), and the smaller end is >= the
//     largest F of the run (the max of its words: 0 = no class, border =
//     NaN, see probeWord) -- so every class cell would be rejected by its
//     probe filter.
// A run failing (b) is redone exactly. A lane whose run fails (a) -- its
// last run -- waits, and all lanes finish their last cells together once
// every lane of the warp got there (the warp cannot retire before its
// longest ray anyway; a ray's last run handled when it comes up would be
// executed by a lone lane, once per lane). A run's lookahead may step past
// the border into the guard rows (DeviceMap::kProbeGuardRows), hence the
// signed index. A run holding a candidate cell marks the ray touched even if
// that cell is not emitted (the endpoint or a zero-length cell): the ray is
// then queued for pass 2 without reason, which changes nothing (pass 2 only
// acts on removed cells, all of them candidates the ray would have touched).
static_assert(RB_P1_RUN > 1 && RB_P1_RUN < DeviceMap::kProbeGuardRows, "pass-1 run length");
__device__ __forceinline__ void pass1Walk(P1Walk& w, const Pass1Ctx& c, uint32_t W, bool walking,
                                          bool& touched, unsigned& visits) {
  unsigned nv = 0;
  const bool runs = walking && isfinite(c.oz) && isfinite(c.dz);
  bool ending = !runs;  // lanes without runs do their whole walk in the final exact loop
  bool finished = !walking;
#ifdef RB_P1_DIAG
  unsigned d_fast = 0, d_end = 0, d_gate = 0;
#endif
  while (!__all_sync(0xffffffffu, ending)) {
    if (ending) continue;
    double ax = w.tmx, ay = w.tmy, mlast = 0.0;
    int j = static_cast<int>(w.idx);
    uint32_t kmax = w.wd, kor = w.wd, wl = 0;
#pragma unroll
    for (int s = 0; s < RB_P1_RUN; ++s) {
      // m = min, then the axis step (ptxas computes both sums and selects)
      int dj;
      asm("{\n\t.reg .pred p;\n\t"
          "setp.lt.f64 p, %0, %1;\n\t"
          "selp.f64 %2, %0, %1, p;\n\t"
          "selp.s32 %3, %6, %7, p;\n\t"
          "@p add.rn.f64 %0, %0, %4;\n\t"
          "@!p add.rn.f64 %1, %1, %5;\n\t}"
          : "+d"(ax), "+d"(ay), "=d"(mlast), "=r"(dj)
          : "d"(w.tdx), "d"(w.tdy), "r"(w.step_col), "r"(w.step_row));
      j += dj;
      const uint32_t wj = c.probe[j];
      if (s + 1 < RB_P1_RUN) {
        kmax = max(kmax, wj);
        kor |= wj;
      } else {
        wl = wj;
      }
    }
    if (!(mlast < w.t1)) {  // the ray's last run: wait for the warp
      ending = true;
#ifdef RB_P1_DIAG
      ++d_end;
#endif
      continue;
    }
    const double ha = c.oz + w.t_enter * c.dz, hb = c.oz + mlast * c.dz;
    if (kmax == 0u || (ha < hb ? ha : hb) >= probeBound(kmax)) {
      w.tmx = ax;
      w.tmy = ay;
      w.idx = static_cast<uint32_t>(j);
      w.wd = wl;
      w.t_enter = mlast;
      nv += RB_P1_RUN;
      if (kor & kClsCandidate) touched = true;
#ifdef RB_P1_DIAG
      ++d_fast;
#endif
    } else {
#ifdef RB_P1_DIAG
      ++d_gate;
#endif
      if (pass1Exact(w, c, W, RB_P1_RUN, nv, touched)) ending = finished = true;
    }
  }
  if (!finished) pass1Exact(w, c, W, 0xffffffffu, nv, touched);
  visits += nv;
#ifdef RB_P1_DIAG
  atomicAdd(&g_p1diag[0], d_fast);
  atomicAdd(&g_p1diag[1], d_end);
  atomicAdd(&g_p1diag[2], d_gate);
  atomicAdd(&g_p1diag[3], walking ? 1u : 0u);
  atomicAdd(&g_p1diag[4], nv);
#endif
}

// Jump ahead (RayArgs::jgrid): before its walk, a ray follows its real line
// through the jump grid (plain fp64, approximate) from the walk's entry time
// and stops at the first block whose word's bound F is not below the ray's
// height over the block's time range (less a margin far above any rounding
// of the walk's crossing times); the cells the exact walk passes before that
// time lie in the passed blocks or their one-cell rings, so none of them can
// pass its gate and no candidate is among them. The walk's state is then
// moved to the last state it enters before that time, exactly: along its
// primary axis (the smaller t_delta) the reference's running sums
// t_max += t_delta up to the last crossing before the target, along the
// other axis the sums that the reference's merge order takes first (ties
// step y, raycast.cpp:120) -- the state the reference's loop is in when it
// enters that cell. No compare / select chain per step, no probe loads.
__device__ __forceinline__ void pass1Jump(P1Walk& w, const Pass1Ctx& c, const RayArgs& a,
                                          unsigned& visits) {
  if (!isfinite(c.oz) || !isfinite(c.dz)) return;
  const int sx = w.step_col, sy = w.step_row > 0 ? 1 : (w.step_row < 0 ? -1 : 0);
  // The real line's block crossings, from the walk's own cell and crossing
  // times (blocks are whole cells): the next block face along x is crossed
  // with the column crossing (bx+1)*B-1-col (resp. col-bx*B) steps after
  // t_max_x; approximate sums are enough here (see the one-cell rings).
  int bx = w.col >> kJumpShift, by = w.row >> kJumpShift;
  double tbx = kInf, tby = kInf, dtbx = kInf, dtby = kInf;
  if (sx != 0) {
    tbx = w.tmx + (sx > 0 ? (bx + 1) * kJumpBlk - 1 - w.col : w.col - bx * kJumpBlk) * w.tdx;
    dtbx = kJumpBlk * w.tdx;
  }
  if (sy != 0) {
    tby = w.tmy + (sy > 0 ? (by + 1) * kJumpBlk - 1 - w.row : w.row - by * kJumpBlk) * w.tdy;
    dtby = kJumpBlk * w.tdy;
  }
  const double t1 = w.t1;
  const double hm = 1e-9 * (fabs(c.oz) + fabs(c.dz)) + 1e-12;
  // the block's smallest height: at its exit when the ray falls, its entry
  // when it rises (the computed height is monotone in t)
  const bool down = c.dz < 0.0;
  double ha = c.oz + w.t_enter * c.dz, t_stop = w.t_enter;
  const float* jp = a.jgrid + by * a.jw + bx;
  const int jstep = sy * a.jw;
#pragma unroll 1
  while (true) {
    const double tm = tbx < tby ? tbx : tby;
    const double tb = tm < t1 ? tm : t1;
    const double hb = c.oz + tb * c.dz;
    // the smallest height less the margin, rounded down to f32, must reach
    // the block's bound (an f32 value)
    if (!(__double2float_rd((down ? hb : ha) - hm) >= __ldg(jp))) break;
    t_stop = tb;
    if (!(tb < t1)) break;
    if (tbx < tby) {
      bx += sx;
      tbx += dtbx;
      jp += sx;
      if (static_cast<unsigned>(bx) >= static_cast<unsigned>(a.jw)) break;
    } else {
      by += sy;
      tby += dtby;
      jp += jstep;
      if (static_cast<unsigned>(by) >= static_cast<unsigned>(a.jh)) break;
    }
    ha = hb;
  }
  const double tt = t_stop - 1e-9;  // states entered before tt are skipped
  if (!(tt > w.t_enter)) return;
  // The running sums: a blind stretch two steps shorter than the real-valued
  // count (whose error is far below one step), no compares, then the exact
  // stop by comparison. Primary axis = the one with more crossings (smaller
  // t_delta); each axis' code is written out (no per-step select between them).
  const int lim_x = a.g.W + 2, lim_y = a.g.H + 2;  // the walk stays in the grid: fewer steps
  double tmx = w.tmx, tmy = w.tmy, last = w.t_enter;
  int di = 0, dj = 0;
  const double tdx = w.tdx, tdy = w.tdy;
  if (tdx <= tdy) {
    const int bx0 = static_cast<int>(fmin((tt - tmx) * (1.0 / tdx), static_cast<double>(lim_x))) - 2;
#pragma unroll 4
    for (int k = 0; k < bx0; ++k) tmx += tdx;
    di = bx0 > 0 ? bx0 : 0;
    while (tmx < tt && di < lim_x) {
      last = tmx;
      tmx += tdx;
      ++di;
    }
    if (di == 0 || di >= lim_x) return;
    // (an axis that never steps has t_max = t_delta = inf: the estimate is NaN, no blind steps)
    const double ey = (last - tmy) * (1.0 / tdy);
    const int by0 = ey == ey ? static_cast<int>(fmin(ey, static_cast<double>(lim_y))) - 2 : 0;
#pragma unroll 4
    for (int k = 0; k < by0; ++k) tmy += tdy;
    dj = by0 > 0 ? by0 : 0;
    while (tmy <= last && dj < lim_y) {  // ties step y first
      tmy += tdy;
      ++dj;
    }
  } else {
    const int by0 = static_cast<int>(fmin((tt - tmy) * (1.0 / tdy), static_cast<double>(lim_y))) - 2;
#pragma unroll 4
    for (int k = 0; k < by0; ++k) tmy += tdy;
    dj = by0 > 0 ? by0 : 0;
    while (tmy < tt && dj < lim_y) {
      last = tmy;
      tmy += tdy;
      ++dj;
    }
    if (dj == 0 || dj >= lim_y) return;
    const double ex = (last - tmx) * (1.0 / tdx);
    const int bx0 = ex == ex ? static_cast<int>(fmin(ex, static_cast<double>(lim_x))) - 2 : 0;
#pragma unroll 4
    for (int k = 0; k < bx0; ++k) tmx += tdx;
    di = bx0 > 0 ? bx0 : 0;
    while (tmx < last && di < lim_x) {  // x steps first only if strictly earlier
      tmx += tdx;
      ++di;
    }
  }
  if (di >= lim_x || dj >= lim_y) return;  // (absorbed increments: leave it to the walk)
  w.tmx = tmx;
  w.tmy = tmy;
  w.t_enter = last;
  w.idx = static_cast<uint32_t>(static_cast<int>(w.idx) + di * w.step_col + dj * w.step_row);
  visits += static_cast<unsigned>(di + dj);
#ifdef RB_P1_DIAG
  atomicAdd(&g_p1diag[5], static_cast<unsigned long long>(di + dj));
  atomicAdd(&g_p1diag[6], 1ull);
#endif
}

// 128-thread blocks, 9 per SM: 56 registers (no spills in the DDA loop) at 36
// resident warps (256 x 5 at 48 registers spilled the step increments).
#ifndef RB_PASS1_MIN_BLOCKS
#define RB_PASS1_MIN_BLOCKS 9
#endif
#ifndef RB_P1_THREADS
#define RB_P1_THREADS 128
#endif
constexpr int kP1Threads = RB_P1_THREADS;
// Pass 1 of the rays [k0, k0 + kP1Threads) of a tile, one per thread; every
// thread of the block calls it (the walk and the queueing are warp-wide).
template <typename ProbePtr, typename ClsPtr>
__device__ __forceinline__ void pass1Tile(uint32_t k0, uint32_t n, const uint8_t* __restrict__ kept,
                                          const double* __restrict__ px,
                                          const double* __restrict__ py,
                                          const double* __restrict__ pz, const RayArgs& a,
                                          const Layers& L, ClsPtr cls, int32_t* kstar,
                                          uint32_t* raylist, DevStats* st, uint32_t ray_base,
                                          ProbePtr probe, const uint32_t* __restrict__ pcell) {
  const uint32_t k = k0 + threadIdx.x;
  bool touched = false, walking = false;
  unsigned visits = 0;
  Pass1Ctx c{cls, probe, L, kstar, 0.0, 0.0, 0.0, 0.0, a.alpha_n,
             static_cast<int32_t>(ray_base + k)};  // global ray id (sharded frames)
  P1Walk w;
  if (k < n && kept[k]) {
    const double ex = px[k], ey = py[k], ez = pz[k];
    c.oz = a.o[2];
    c.dz = ez - a.o[2];
    c.vx = ex - a.o[0];
    c.vy = ey - a.o[1];
    if (isfinite(c.vx) && isfinite(c.vy)) {
      walking = pass1Setup(a.g, a.o, ex, ey, c, touched, visits, a, pcell ? pcell[k] : 0xffffffffu, w);
    } else {
      pdlWait();
      walkRay(a.g, a.o, ex, ey, [&](uint32_t cell, double te, double tn, bool vertical) {
        ++visits;
        const uint8_t cl = cls[cell];
        if (cl) pass1Visit(c, cl, cell, rayHeight(a.o[2], c.dz, te, tn, vertical), touched);
      });
    }
  }
  // Every thread is past the wait before the walk (class / probe words come
  // from the classification) and the counters.
  pdlWait();
  if (walking && a.jgrid != nullptr) pass1Jump(w, c, a, visits);
  if (walking) w.wd = probe[w.idx];
  pass1Walk(w, c, static_cast<uint32_t>(a.g.W), walking, touched, visits);
  // Queue rays that crossed a removal candidate for the k* pass (one atomic per warp).
  const unsigned lane = threadIdx.x & 31;
  const unsigned want = __ballot_sync(0xffffffffu, touched && a.bound);
  if (want) {
    unsigned base = 0;
    if (lane == __ffs(want) - 1)
      base = static_cast<unsigned>(atomicAdd(&st->candidate_rays, static_cast<unsigned long long>(__popc(want))));
    base = __shfl_sync(0xffffffffu, base, __ffs(want) - 1);
    if (touched && a.bound) raylist[base + __popc(want & ((1u << lane) - 1u))] = k;
  }
  unsigned long long v = warpSum(static_cast<unsigned long long>(visits));
  if (lane == 0 && v) atomicAdd(&st->visits, v);
}

// kStride (the retry launch of sharded frames): grid-stride over ray tiles
// with a one-wave grid, so its common no-op case costs one wave of returning
// blocks. The main launch has one block per tile (the loop runs once).
template <bool kStride>
__global__ void __launch_bounds__(kP1Threads, RB_PASS1_MIN_BLOCKS)
    k_rays_pass1(uint32_t n, const uint8_t* __restrict__ kept, const double* __restrict__ px,
                 const double* __restrict__ py, const double* __restrict__ pz, RayArgs a,
                 Layers L, const uint8_t* __restrict__ cls, int32_t* kstar, uint32_t* raylist,
                 DevStats* st, int retry, uint32_t ray_base, const ProbeT* __restrict__ probe,
                 const uint32_t* __restrict__ pcell) {
  RB_TL(12 + kStride);
  pdlTrigger();  // the per-ray setup runs before the wait (inputs from k_ingest)
  if (retry && !st->respeculate) return;
  for (uint32_t k0 = blockIdx.x * kP1Threads; k0 < n;
       k0 = kStride ? k0 + gridDim.x * kP1Threads : n)
    pass1Tile(k0, n, kept, px, py, pz, a, L, cls, kstar, raylist, st, ray_base, probe, pcell);
}

// Grid-wide barrier of a cooperative launch (all blocks co-resident):
// bar[0] arrivals, bar[1] generation (both zero at the frame's stats reset).
__device__ __forceinline__ void gridSync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g0) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

template <bool kScratch>
__device__ __forceinline__ void pass2Rays(unsigned first, unsigned stride, const uint32_t* raylist,
                                          unsigned total, const double* px, const double* py,
                                          const double* pz, const RayArgs& a, const Layers& L,
                                          const uint8_t* cls, const int32_t* kstar,
                                          uint32_t ray_base, double* ub2);

// The ray phase's tail on single-call frames, one cooperative one-wave
// launch: (retry) if k_fuse_heavy found a speculated class wrong, the
// classification and pass 1 again from scratch; then (pass2) the bounds of
// the removed cells from the queued rays (k_rays_pass2<true>). Both are
// rare; the common frame pays one launch that reads two flags.
__global__ void __launch_bounds__(kP1Threads, RB_PASS1_MIN_BLOCKS)
    k_rays_tail(int retry, int pass2, uint32_t n, const uint8_t* __restrict__ kept,
                const double* __restrict__ px, const double* __restrict__ py,
                const double* __restrict__ pz, RayArgs a, Layers L, uint8_t* cls,
                int32_t* kstar, uint32_t* raylist, DevStats* st, ProbeT* probe,
                const uint32_t* __restrict__ pcell, double* ub2) {
  RB_TL(14);
  pdlWait();
  pdlTrigger();
  if (retry && st->respeculate) {
    // (cls / probe / k* are rewritten inside this kernel: plain loads below)
    const ClassArgs ca{a.now, a.t_free, a.cleanup, a.bound, a.g.W};
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < static_cast<size_t>(a.g.W) * a.g.H;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
      classifyCell(L, i, false, ca, cls, probe, kstar);
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // pass 1 runs again from scratch
      st->candidate_rays = 0;
      st->visits = 0;
    }
    gridSync(st->grid_bar);
    for (uint32_t k0 = blockIdx.x * kP1Threads; k0 < n; k0 += gridDim.x * kP1Threads)
      pass1Tile(k0, n, kept, px, py, pz, a, L, static_cast<const uint8_t*>(cls), kstar, raylist, st,
                0u, static_cast<const ProbeT*>(probe), pcell);
    gridSync(st->grid_bar);
  }
  if (pass2 && static_cast<volatile int32_t*>(kstar)[-1] != INT_MAX)
    pass2Rays<true>(blockIdx.x * kP1Threads + threadIdx.x, gridDim.x * kP1Threads, raylist,
                    static_cast<unsigned>(static_cast<volatile unsigned long long*>(
                        &st->candidate_rays)[0]),
                    px, py, pz, a, L, cls, kstar, 0u, ub2);
}

// Invalidate every cell some ray removed (set is order independent).
__global__ void __launch_bounds__(kThreads) k_remove(Layers L, size_t n, const int32_t* kstar,
                                                     DevStats* st) {
  pdlEnter();
  unsigned long long cnt = 0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    if (kstar[i] != INT_MAX) {
      invalidateCell(L, i);
      ++cnt;
    }
  }
  cnt = warpSum(cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&st->removed, cnt);
}

// Bounds of removed cells: only rays at or after the first removing ray saw
// them invalid (reference integration.cpp:212-222 ordering).
// kScratch: the removal itself happens later in k_cells, so the bounds go to
// the scratch array ub2 (+inf when untouched) that k_cells moves into the
// removed cells; otherwise (sharded frames) k_remove has run and the bounds go
// to the map.
template <bool kScratch>
__device__ __forceinline__ void pass2Rays(unsigned first, unsigned stride, const uint32_t* raylist,
                                          unsigned total, const double* px, const double* py,
                                          const double* pz, const RayArgs& a, const Layers& L,
                                          const uint8_t* cls, const int32_t* kstar,
                                          uint32_t ray_base, double* ub2) {
  for (unsigned q = first; q < total; q += stride) {
    const uint32_t k = raylist[q];
    const double dz = pz[k] - a.o[2];
    walk(a.g, a.o, px[k], py[k], [&](uint32_t c, double te, double tn, bool vertical) {
      if (cls[c] != kClsCandidate) return;
      if (kstar[c] > static_cast<int32_t>(ray_base + k)) return;
      const double h = rayHeight(a.o[2], dz, te, tn, vertical);
      if (kScratch) {
        unsigned long long* addr = reinterpret_cast<unsigned long long*>(ub2 + c);
        double cur = ub2[c];
        while (h < cur) {
          const unsigned long long want = static_cast<unsigned long long>(__double_as_longlong(cur));
          const unsigned long long got =
              atomicCAS(addr, want, static_cast<unsigned long long>(__double_as_longlong(h)));
          if (got == want) break;
          cur = __longlong_as_double(static_cast<long long>(got));
        }
      } else {
        boundMin(L, c, h);
      }
    });
  }
}

template <bool kScratch>
__global__ void __launch_bounds__(kThreads)
    k_rays_pass2(const uint32_t* __restrict__ raylist, const DevStats* st_in,
                 const double* __restrict__ px, const double* __restrict__ py,
                 const double* __restrict__ pz, RayArgs a, Layers L,
                 const uint8_t* __restrict__ cls, const int32_t* __restrict__ kstar,
                 uint32_t ray_base, double* ub2) {
  pdlEnter();
  if (kScratch ? kstar[-1] == INT_MAX : st_in->removed == 0) return;
  pass2Rays<kScratch>(blockIdx.x * kThreads + threadIdx.x, gridDim.x * kThreads, raylist,
                      static_cast<unsigned>(st_in->candidate_rays), px, py, pz, a, L, cls, kstar,
                      ray_base, ub2);
}

// ------------------------------------------------------- K7 cell phases
struct CellArgs {
  GridArgs g;
  double rx, ry, rz;  // robot position = pose translation
  int overlap;
  double ov_r2, ov_thr;
  int radius;  // traversability window / 2
  double slope_max, step_max, rough_max, w_slope, w_step, w_rough;
  int time_var;
  double growth, sigma_max2;
  int geo_trav;  // geometric traversability (off when the conv-net writes the layer)
  // Zero the normals (and the geometric traversability) of invalid cells, as the
  // reference rebuilds both layers every scan (analysis.cpp:44-48,93). They are
  // zero already unless a snapshot was loaded or a conv-net frame wrote the
  // traversability of every cell, so this runs only after those.
  int scrub;
  // Ray-cast cleanup of this frame folded in (reference raycast.cpp:132-157,
  // grid.cpp:126-137): cells with k* < inf are removed here, their upper bound
  // taken from pass 2's scratch (ub2, reset to +inf after use).
  int fold_remove;
  const int32_t* kstar;
  double* ub2;
  // Stats hand-over of a synchronous frame (DeviceMap::h_seq; null: none):
  // the last of the nblocks blocks copies the stats to hstats, then writes seq.
  DevStats* hstats;
  unsigned long long* hseq;
  unsigned long long seq;
  unsigned nblocks;
};

// End of a k_cells block: the last block to finish copies the frame's stats
// (final: every earlier kernel of the frame has completed, and every block's
// counter atomics precede its ticket) to pinned host memory, fences, and
// publishes the frame's sequence number.
__device__ __forceinline__ void handOverStats(const CellArgs& a, DevStats* st, unsigned tid) {
  if (a.hseq == nullptr) return;
  __syncthreads();
  if (tid >= 32) return;
  unsigned ticket = 0;
  if (tid == 0) {
    __threadfence();
    ticket = atomicAdd(&st->cells_done, 1u);
  }
  if (__shfl_sync(0xffffffffu, ticket, 0) != a.nblocks - 1) return;
  // the last block's first warp: one stats word per lane, each lane fencing
  // its own store before lane 0 publishes the sequence number
  __threadfence();
  static_assert(sizeof(DevStats) % 8 == 0 && sizeof(DevStats) / 8 <= 32, "stats words");
  if (tid < sizeof(DevStats) / 8) {
    reinterpret_cast<unsigned long long*>(a.hstats)[tid] =
        reinterpret_cast<const volatile unsigned long long*>(st)[tid];
    __threadfence_system();
  }
  __syncwarp();
  if (tid == 0) *reinterpret_cast<volatile unsigned long long*>(a.hseq) = a.seq;
}

constexpr int kTileX = 32, kTileY = 8;
constexpr std::size_t kCellsMaxSmem = 200 * 1024;

// Post-overlap validity and elevation of cell (rr, cc): overlap clearance
// (analysis.cpp:296-317) evaluated by every reader, so the result does not
// depend on whether the cell's own thread has invalidated it yet.
__device__ __forceinline__ uint8_t stageCell(const Layers& L, const CellArgs& a, int rr, int cc,
                                             double& e) {
  e = 0.0;
  if (rr < 0 || rr >= a.g.H || cc < 0 || cc >= a.g.W) return 0;
  const size_t j = static_cast<size_t>(rr) * a.g.W + cc;
  uint8_t v = L.valid[j];
  if (v && a.fold_remove && a.kstar[j] != INT_MAX) v = 0;  // removed by the ray pass
  if (v) {
    e = L.elev[j];
    if (a.overlap) {
      const double cx = a.g.ox + (cc + 0.5) * a.g.res;
      const double cy = a.g.oy + (rr + 0.5) * a.g.res;
      const double ddx = cx - a.rx, ddy = cy - a.ry;
      if (!(ddx * ddx + ddy * ddy > a.ov_r2) && !(fabs(e - a.rz) <= a.ov_thr)) v = 0;
    }
  }
  return v;
}

// Window access for the cell body: a shared-memory tile with a halo, or (for
// windows whose tile exceeds shared memory) the map itself.
struct TileWin {
  const double* se;
  const uint8_t* sv;
  int tw, lr, lc;
  __device__ __forceinline__ bool ok(int dr, int dc) const { return sv[(lr + dr) * tw + lc + dc] != 0; }
  __device__ __forceinline__ double e(int dr, int dc) const { return se[(lr + dr) * tw + lc + dc]; }
};
struct GlobalWin {
  const Layers* L;
  const CellArgs* a;
  int r, c;
  __device__ __forceinline__ bool ok(int dr, int dc) const {
    double e;
    return stageCell(*L, *a, r + dr, c + dc, e) != 0;
  }
  __device__ __forceinline__ double e(int dr, int dc) const {
    double v;
    stageCell(*L, *a, r + dr, c + dc, v);
    return v;
  }
};

// One cell: overlap clearance, normals (analysis.cpp:41-86), geometric
// traversability (analysis.cpp:88-132), time variance (grid.cpp:113-124).
template <int RT, typename Win>
__device__ __forceinline__ void cellBody(const Layers& L, const CellArgs& a, int r, int c,
                                         const Win& w, int32_t* __restrict__ count,
                                         uint32_t* __restrict__ seg_start,
                                         unsigned long long& cleared,
                                         unsigned long long& removed) {
  const int W = a.g.W, H = a.g.H;
  const size_t i = static_cast<size_t>(r) * W + c;
  const int32_t cnt_i = count[i];
  if (cnt_i != 0) {  // last reader this scan: ready for the next one (the sort's
    count[i] = 0;     // atomicMin segment starts need 0xffffffff)
    seg_start[i] = 0xffffffffu;
  }
  const bool was_valid = L.valid[i] != 0;
  const bool ok = w.ok(0, 0);
  if (a.fold_remove && a.kstar[i] != INT_MAX) {  // removed by the ray pass
    invalidateCell(L, i);
    const double b = a.ub2[i];
    if (b < dinf()) {  // bounds from rays at or after the removing one
      L.ub[i] = b;
      L.ubv[i] = 1;
      a.ub2[i] = dinf();
    }
    removed = 1;
  } else if (was_valid && !ok) {
    invalidateCell(L, i);
    cleared = 1;
  } else if (ok) {
    const double res = a.g.res;
    const double center = w.e(0, 0);
    const bool hl = c > 0 && w.ok(0, -1), hr = c < W - 1 && w.ok(0, 1);
    const bool hd = r > 0 && w.ok(-1, 0), hu = r < H - 1 && w.ok(1, 0);
    double nx = 0.0, ny = 0.0, nz = 0.0;
    bool has = true;
    double dhdx = 0.0, dhdy = 0.0;
    if (hl && hr) dhdx = (w.e(0, 1) - w.e(0, -1)) / (2.0 * res);
    else if (hr) dhdx = (w.e(0, 1) - center) / res;
    else if (hl) dhdx = (center - w.e(0, -1)) / res;
    else has = false;
    if (has) {
      if (hd && hu) dhdy = (w.e(1, 0) - w.e(-1, 0)) / (2.0 * res);
      else if (hu) dhdy = (w.e(1, 0) - center) / res;
      else if (hd) dhdy = (center - w.e(-1, 0)) / res;
      else has = false;
    }
    if (has) {
      const double norm = sqrt((dhdx * dhdx + dhdy * dhdy) + 1.0);
      nx = -dhdx / norm;
      ny = -dhdy / norm;
      nz = 1.0 / norm;
    }
    L.nx[i] = nx;
    L.ny[i] = ny;
    L.nz[i] = nz;
    double trav = 0.0;
    if (a.geo_trav && (nx != 0.0 || ny != 0.0 || nz != 0.0)) {
      const double slope = acos(sclamp(nz, -1.0, 1.0));
      const double s_slope = sclamp(1.0 - slope / a.slope_max, 0.0, 1.0);
      double max_step = 0.0, sum = 0.0, sum_sq = 0.0;
      int cntw = 0;
      // Row-major window over valid cells (cells outside the grid read as
      // invalid, so they are skipped like the reference's bounds test).
      const int R = RT > 0 ? RT : a.radius;
#pragma unroll
      for (int dr = -R; dr <= R; ++dr) {
#pragma unroll
        for (int dc = -R; dc <= R; ++dc) {
          if (!w.ok(dr, dc)) continue;
          const double v = w.e(dr, dc);
          max_step = smax(max_step, fabs(v - center));
          sum += v;
          sum_sq += v * v;
          ++cntw;
        }
      }
      const double s_step = sclamp(1.0 - max_step / a.step_max, 0.0, 1.0);
      const double mean = sum / cntw;
      const double var = smax(0.0, sum_sq / cntw - mean * mean);
      const double s_rough = sclamp(1.0 - sqrt(var) / a.rough_max, 0.0, 1.0);
      trav = a.w_slope * s_slope + a.w_step * s_step + a.w_rough * s_rough;
    }
    if (a.geo_trav) L.trav[i] = trav;
    if (a.time_var && cnt_i == 0) L.var[i] = smin(L.var[i] + a.growth, a.sigma_max2);
  } else if (a.scrub) {
    L.nx[i] = 0.0;
    L.ny[i] = 0.0;
    L.nz[i] = 0.0;
    if (a.geo_trav) L.trav[i] = 0.0;
  }
}

// Overlap clearance, normals, geometric traversability and time variance in
// one pass over a shared memory tile with a (radius)-cell halo. Overlap is
// evaluated for halo cells too, so every thread sees the post-clearance
// validity of its window. RT: the traversability window radius when known at
// compile time (the 5x5 default and 3x3 are instantiated; 0 = from CellArgs).
template <int RT>
__global__ void __launch_bounds__(kTileX* kTileY)
    k_cells(Layers L, int32_t* __restrict__ count, uint32_t* __restrict__ seg_start, CellArgs a,
            DevStats* st) {
  RB_TL(15);
  pdlEnter();
  extern __shared__ unsigned char smem[];
  const int halo = a.radius > 1 ? a.radius : 1;
  const int tw = kTileX + 2 * halo, th = kTileY + 2 * halo;
  double* se = reinterpret_cast<double*>(smem);
  uint8_t* sv = reinterpret_cast<uint8_t*>(se + tw * th);
  const int W = a.g.W, H = a.g.H;
  const int c0 = blockIdx.x * kTileX - halo, r0 = blockIdx.y * kTileY - halo;
  const int tid = threadIdx.y * kTileX + threadIdx.x;
  if (RB_CELLS_SKIP && !a.scrub) {
    // A tile with no valid cell and no cell with points this scan has nothing
    // to do (no normals, no removal or clearance, no counters to reset): it
    // skips the halo staging.
    const int rr = blockIdx.y * kTileY + threadIdx.y, cc = blockIdx.x * kTileX + threadIdx.x;
    bool busy = false;
    if (rr < H && cc < W) {
      const size_t j = static_cast<size_t>(rr) * W + cc;
      busy = L.valid[j] != 0 || count[j] != 0;
    }
    if (!__syncthreads_or(busy)) {
      handOverStats(a, st, static_cast<unsigned>(tid));
      return;
    }
  }
  for (int q = tid; q < tw * th; q += kTileX * kTileY) {
    double e;
    sv[q] = stageCell(L, a, r0 + q / tw, c0 + q % tw, e);
    se[q] = e;
  }
  __syncthreads();
  const int r = blockIdx.y * kTileY + threadIdx.y, c = blockIdx.x * kTileX + threadIdx.x;
  unsigned long long cleared = 0, removed = 0;
  if (r < H && c < W)
    cellBody<RT>(L, a, r, c,
                 TileWin{se, sv, tw, static_cast<int>(threadIdx.y) + halo,
                         static_cast<int>(threadIdx.x) + halo},
                 count, seg_start, cleared, removed);
  cleared = warpSum(cleared);
  removed = warpSum(removed);
  if ((tid & 31) == 0 && cleared) atomicAdd(&st->overlap_cleared, cleared);
  if ((tid & 31) == 0 && removed) atomicAdd(&st->removed, removed);
  handOverStats(a, st, static_cast<unsigned>(tid));
}

// Same cell phases without the tile, for traversability windows too large to
// stage in shared memory (the reference accepts any odd window).
__global__ void __launch_bounds__(256)
    k_cells_global(Layers L, int32_t* __restrict__ count, uint32_t* __restrict__ seg_start,
                   CellArgs a, DevStats* st) {
  pdlEnter();
  const int r = blockIdx.y, c = blockIdx.x * 256 + threadIdx.x;
  unsigned long long cleared = 0, removed = 0;
  if (c < a.g.W) cellBody<0>(L, a, r, c, GlobalWin{&L, &a, r, c}, count, seg_start, cleared, removed);
  cleared = warpSum(cleared);
  removed = warpSum(removed);
  if ((threadIdx.x & 31) == 0 && cleared) atomicAdd(&st->overlap_cleared, cleared);
  if ((threadIdx.x & 31) == 0 && removed) atomicAdd(&st->removed, removed);
  handOverStats(a, st, threadIdx.x);
}


// Phase-boundary events (per-phase device times); an event between two
// kernels also ends their programmatic overlap, so they are recorded only
// when phase timing is requested (DeviceMap::phase_events).
// Timing events are recorded as external event nodes when the frame is
// captured into a graph (a plain record inside a capture only orders streams).
inline void recordTiming(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  checkCuda(cudaStreamIsCapturing(s, &cs), "capture status");
  checkCuda(cudaEventRecordWithFlags(e, s, cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal
                                                                               : cudaEventRecordDefault),
            "event");
}
#define RB_PHASE_EVENT(k, stream) \
  do {                           \
    if (m.phase_events) recordTiming(m.ev[k], stream); \
  } while (0)

inline unsigned gridFor(size_t n, int threads = kThreads) {
  return static_cast<unsigned>((n + threads - 1) / threads);
}
inline unsigned streamGrid(size_t n) {
  return static_cast<unsigned>(std::min<size_t>((n + kThreads - 1) / kThreads, 148 * 16));
}

int quantizedShift(double d, double res) {
  if (std::abs(d) < res) return 0;  // one-cell hysteresis (reference grid.cpp:65-68)
  return static_cast<int>(std::llround(d / res));
}

}  // namespace

// ------------------------------------------------------------------ host
namespace {

// One frame's launch context. The single-call path (integrateScanDevice) and
// the sharded path (shard*) run the same phase functions in the same order.
struct Frame {
  DeviceMap& m;
  const PipelineParams& P;
  Pose pose;
  double stamp, dt;
  cudaStream_t s;
  std::size_t ncell;
  uint32_t WH;
  GridArgs g;
  long long launches = 0;
  bool overlap = false;  // heavy cells folded on stream2 during the ray pass
  FuseArgs fa{};          // fusion parameters of the frame (for the side-stream fold)
  // Per-ray endpoint cell from k_ingest (indexed like the rays), or null when
  // the sort has overwritten it (3 passes) or the rays are a shard's.
  const uint32_t* point_cells = nullptr;
  // Index of this process's first ray in the point arrays (a group rank's
  // rays sit at their frame indices; shard and single frames start at 0).
  uint32_t ray_at = 0;
  // Device scalar holding this frame's drift offset, applied by k_fuse (null:
  // none, or applied already -- the sharded path's k_apply_offset_value).
  const double* fuse_offset = nullptr;
  bool classified = false;  // k_fuse wrote this frame's ray classes
  bool drift_join = false;  // phaseDrift(side) ran on stream2: join before the fold
  bool prepped = false;     // k_side_prep classified the cells without points
  bool presplit = false;
  bool jump_done = false;   // k_jump_grid ran on stream 2 after the side sweep (RB_SIDE_JUMP)    // RB_PRESPLIT: candidates folded before the ray pass, the rest beside it
  bool lists_built = false; // k_side_prep queued the long cells (the long fold starts after the sort)
  // Removal of k* < inf cells: in k_cells (fold_remove, set when the ray pass
  // ran with cleanup on), or by k_remove right after the ray pass
  // (explicit_remove: sharded frames, whose host exchanges the bounds after it).
  bool fold_remove = false;
  bool explicit_remove = false;
  // Stats handed over by k_cells through pinned memory (DeviceMap::h_seq)
  // instead of a D2H copy + stream synchronisation (synchronous frames whose
  // last kernel is k_cells).
  bool handover = false;
  bool small_tiles = false;  // sortGeometry's small-frame tiles (single-map frames)
  int heavy = INT_MAX;
  Frame(DeviceMap& map, const PipelineParams& params, const Pose& p, double st, double d)
      : m(map), P(params), pose(p), stamp(st), dt(d), s(map.stream), ncell(map.grid.cells()),
        WH(static_cast<uint32_t>(map.grid.cells())) {}
};

// Stats reset + move_to (reference grid.cpp:87-111).
void phaseBegin(Frame& f, bool record_start = true) {
  DeviceMap& m = f.m;
  if (record_start) recordTiming(m.ev[0], f.s);
  checkCuda(cudaMemsetAsync(m.stats, 0, sizeof(DevStats), f.s), "memset");
  const int sx = quantizedShift(f.pose.t[0] - m.grid.center_x, m.grid.resolution);
  const int sy = quantizedShift(f.pose.t[1] - m.grid.center_y, m.grid.resolution);
  if (sx != 0 || sy != 0) {
    m.grid.center_x += sx * m.grid.resolution;
    m.grid.center_y += sy * m.grid.resolution;
    const int W = m.grid.width, H = m.grid.height;
    k_shift<<<dim3(std::min((W + kShiftThreads - 1) / kShiftThreads, 4), H), kShiftThreads, 0, f.s>>>(
        m.cur, m.alt, W, H, sx, sy);
    ++f.launches;
    std::swap(m.cur, m.alt);
  }
  f.g = gridArgs(m.grid);
}

// Point + reduction scratch for n points.
void phaseScratch(Frame& f, std::size_t n) {
  DeviceMap& m = f.m;
  if (n == 0) return;
  ensurePointCapacity(m, n);
  const std::size_t nb = gridFor(n);
  if (m.rcap < nb || m.rslab == nullptr) {
    cudaFree(m.rslab);
    m.rslab = nullptr;
    m.rcap = std::max<std::size_t>(nb, 1024);
    checkCuda(cudaMalloc(&m.rslab, m.rcap * (sizeof(double) + sizeof(int) + sizeof(uint32_t)) + 1024),
              "reduce scratch");
    m.drift_sum_part = static_cast<double*>(m.rslab);
    m.drift_n_part = reinterpret_cast<int*>(m.drift_sum_part + m.rcap);
    m.blk = reinterpret_cast<uint32_t*>(m.drift_n_part + m.rcap);
    m.drift_local = reinterpret_cast<double*>(
        (reinterpret_cast<uintptr_t>(m.blk + m.rcap + 1) + 255) & ~static_cast<uintptr_t>(255));
  }
}

// Point scratch + the input stream into HBM; returns the device points.
// Chunks of an uploaded frame: multiples of the radix tile (and so of the
// block), so tile digit counts and drift block partials are those of one launch.
inline uint32_t chunkPoints(uint32_t N) {
  const uint32_t c = (N + DeviceMap::kChunks - 1) / DeviceMap::kChunks;
  return (c + kTile - 1) / kTile * kTile;
}

const double* phaseUpload(Frame& f, const double* xyz, std::size_t n, bool on_device) {
  DeviceMap& m = f.m;
  if (n == 0) return xyz;
  phaseScratch(f, n);
  if (on_device) return xyz;
  checkCuda(cudaMemcpyAsync(m.xyz_in, xyz, n * 3 * sizeof(double), cudaMemcpyHostToDevice, f.s),
            "point upload");
  return m.xyz_in;
}

// Host input of a synchronous frame: kChunks copies on copy_stream (after
// ev[0] on the frame stream), one event per chunk; phaseIngest(chunked) runs
// each chunk's k_ingest when it lands, and the per-scan resets / recenter
// run under the copy. ev[13] marks the end of the upload.
const double* phaseUploadChunked(Frame& f, const double* xyz, uint32_t N) {
  DeviceMap& m = f.m;
  phaseScratch(f, N);
  checkCuda(cudaEventRecord(m.ev_fork, f.s), "event");
  checkCuda(cudaStreamWaitEvent(m.copy_stream, m.ev_fork, 0), "stream wait");
  const uint32_t chunk = chunkPoints(N);
  for (uint32_t base = 0, c = 0; base < N; base += chunk, ++c) {
    const std::size_t len = std::min(chunk, N - base);
    checkCuda(cudaMemcpyAsync(m.xyz_in + 3 * static_cast<std::size_t>(base), xyz + 3 * static_cast<std::size_t>(base),
                              len * 3 * sizeof(double), cudaMemcpyHostToDevice, m.copy_stream),
              "point upload");
    // upload done (timing) before the last chunk's event, which the frame
    // stream waits on: the copy stream ends joined to it (graph capture)
    if (base + chunk >= N) recordTiming(m.ev[13], m.copy_stream);
    checkCuda(cudaEventRecord(m.ev_chunk[c], m.copy_stream), "event");
  }
  return m.xyz_in;
}

// K2 geometry for N keys: 1-3 LSD passes over the bits of the cell id. The
// tile digit counts are accumulated upstream, so they are zeroed here.
// small: a single-map frame of fewer than kSmallTileN keys sorts in tiles of
// kSmallTile keys (more blocks for the GPU's SMs; the per-tile ranking chain
// is 4x shorter).
SortGeom sortGeometry(DeviceMap& m, uint32_t WH, uint32_t N, bool small = false) {
  SortGeom sg;
  if (N == 0) return sg;
  const int bits = 32 - __builtin_clz(WH);
  sg.passes = bits <= 11 ? 1 : (bits <= 22 ? 2 : 3);
  sg.dbits = (bits + sg.passes - 1) / sg.passes;
  sg.tshift = (small && N < kSmallTileN) ? kSmallTileShift : 11u;
  sg.ntiles = (N + (1u << sg.tshift) - 1) >> sg.tshift;
  sg.pitch = (sg.ntiles + 3) & ~3u;
  const std::size_t tcn = static_cast<std::size_t>(sg.passes) * sg.buckets() * sg.pitch;
  const std::size_t need = tcn + static_cast<std::size_t>(sg.passes) * sg.buckets();
  if (m.hist_cap < need) {  // (reserved before a graph capture: no allocation inside one)
    cudaFree(m.hist);
    m.hist = nullptr;
    m.hist_cap = need;
    checkCuda(cudaMalloc(&m.hist, m.hist_cap * sizeof(uint32_t)), "sort scratch");
  }
  sg.tc = m.hist;
  sg.rowsum = m.hist + tcn;
  return sg;
}

SortGeom phaseSortGeometry(Frame& f, uint32_t N) {
  const SortGeom sg = sortGeometry(f.m, f.WH, N, f.small_tiles);
  if (N == 0) return sg;
  const std::size_t tcn = static_cast<std::size_t>(sg.passes) * sg.buckets() * sg.pitch;
  checkCuda(cudaMemsetAsync(sg.tc, 0, tcn * sizeof(uint32_t), f.s), "memset");
  return sg;
}

// K1 (reference integration.cpp:85-140, sensing.cpp:32-41, drift.cpp:24-42).
// lo: frame index of the first of the N points (a group rank's batch; its
// outputs land at frame indices lo .. lo+N-1).
void phaseIngest(Frame& f, const double* d_xyz, uint32_t N, const SortGeom& sg, bool count_cells,
                 bool chunked = false, uint32_t lo = 0, bool finalize_drift = false) {
  if (N == 0) return;
  DeviceMap& m = f.m;
  const UpdateParams& U = f.P.update;
  IngestArgs ia;
  ia.g = f.g;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) ia.R[3 * r + c] = f.pose.R[r][c];
    ia.t[r] = f.pose.t[r];
  }
  ia.max_range2 = U.max_range * U.max_range;
  ia.excl_enabled = U.exclusion.enabled;
  ia.excl_b = U.exclusion.b;
  ia.excl_c = U.exclusion.c;
  ia.excl_dmax = U.exclusion.d_max;
  ia.excl_tan = std::tan(U.exclusion.theta_a);  // host libm, as the reference
  ia.alpha_d = U.noise.alpha_d;
  ia.sigma_p_min2 = U.noise.sigma_p_min2;
  ia.drift_enabled = f.P.drift.enabled;
  ia.drift_thr = f.P.drift.traversability_threshold;
  ia.drift_blocks = (RB_INGEST_FINALIZE && finalize_drift && f.P.drift.enabled) ? gridFor(N) : 0u;
  ia.drift_min_points = f.P.drift.min_points;
  ia.drift_max_off = f.P.drift.max_offset_per_scan;
  ia.drift_offset = m.drift_offset;
  ia.tshift = sg.tshift;
  if (ia.drift_blocks) f.fuse_offset = m.drift_offset;  // applied by k_fuse (phaseSortFuse)
  const uint32_t chunk = chunked ? chunkPoints(N) : N;
  for (uint32_t base = 0, c = 0; base < N; base += chunk, ++c) {
    if (chunked) checkCuda(cudaStreamWaitEvent(f.s, m.ev_chunk[c], 0), "stream wait");
    const unsigned ntl = gridFor(std::min(chunk, N - base));
    if (RB_INGEST_TMA && !RB_INGEST_FINALIZE)
      launchPdl(k_ingest_tma, std::min(ntl, 148u * RB_INGEST_TMA_BLOCKS), kThreads, 0, f.s, d_xyz, lo + N,
                ia, m.cur, m.count, m.px, m.py, m.pz, m.pvar, m.key0, m.kept, m.drift_sum_part,
                m.drift_n_part, sg.tc, sg.pitch, sg.buckets() - 1, count_cells ? 1 : 0, m.stats,
                lo + base, lo, ntl);
    else
      launchPdl(k_ingest, ntl, kThreads, 0, f.s, d_xyz, lo + N, ia, m.cur, m.count, m.px, m.py, m.pz,
                m.pvar, m.key0, m.kept, m.drift_sum_part, m.drift_n_part, sg.tc, sg.pitch,
                sg.buckets() - 1, count_cells ? 1 : 0, m.stats, lo + base, lo);
    ++f.launches;
  }
}

RayArgs rayArgs(const Frame& f) {
  RayArgs ra;
  ra.g = f.g;
  for (int i = 0; i < 3; ++i) ra.o[i] = f.pose.t[i];
  ra.now = f.stamp;
  ra.t_free = f.P.cleanup.t_free;
  ra.alpha_n = f.P.cleanup.alpha_n;
  ra.cleanup = f.P.cleanup.cleanup_enabled;
  ra.bound = f.P.cleanup.upper_bound_enabled;
  const GridArgs& g = f.g;
  ra.origin_in = ra.o[0] >= g.ox && ra.o[0] <= g.xmax && ra.o[1] >= g.oy && ra.o[1] <= g.ymax;
  ra.jgrid = nullptr;
  ra.jw = ra.jh = 0;
  ra.jres = 0.0;
  auto clampc = [](int v, int n) { return v < 0 ? 0 : (v > n - 1 ? n - 1 : v); };
  ra.ocol = clampc(x86_to_int(std::floor((ra.o[0] - g.ox) / g.res)), g.W);
  ra.orow = clampc(x86_to_int(std::floor((ra.o[1] - g.oy) / g.res)), g.H);
  return ra;
}

// Drift vote mean of a single-GPU frame (unless the ingest's last block
// reduced it); the offset itself is applied before the fold (phaseSortFuse).
// side (RB_SIDE_DRIFT): the vote mean and the offset sweep run on stream2,
// forked from the frame stream after the ingest, so both overlap the radix
// sort (which touches no layer); phaseSortFuse joins before the fold.
#ifndef RB_SIDE_DRIFT
#define RB_SIDE_DRIFT 1
#endif
#ifndef RB_EARLY_HEAVY
#define RB_EARLY_HEAVY 1
#endif
#ifndef RB_FUSE_LIST
#define RB_FUSE_LIST 1  // short-cell fold over k_side_prep's list (k_fuse_list)
#endif
#ifndef RB_HEAVY_PRIO
#define RB_HEAVY_PRIO 0
#endif
#ifndef RB_MAIN_PRIO
#define RB_MAIN_PRIO 0
#endif
#ifndef RB_B_AFTER_A
#define RB_B_AFTER_A 0  // the short-cell fold beside the ray pass starts after the candidates' fold
#endif
#ifndef RB_PRE_THREADS
#define RB_PRE_THREADS 64  // block size of the fold of the removal candidates before the ray pass
#endif
#ifndef RB_SFOLD_BLOCKS
#define RB_SFOLD_BLOCKS 2  // blocks per SM of the short-cell fold beside the ray pass
#endif
#ifndef RB_PRESPLIT
#define RB_PRESPLIT 1  // fold only the removal candidates before the ray pass, the rest beside it
#endif
#ifndef RB_SIDE_CLASSIFY
#define RB_SIDE_CLASSIFY 1  // k_side_prep also classifies the cells without points and the long ones (k_fuse_list its cells)
#endif
void setOverlap(Frame& f) {
  const bool cleanup = f.P.cleanup.cleanup_enabled, bound = f.P.cleanup.upper_bound_enabled;
  f.overlap = (cleanup || bound) && (!cleanup || f.P.cleanup.t_free >= 0.0);
  f.heavy = f.overlap ? kHeavyCell : INT_MAX;
}

void phaseDrift(Frame& f, uint32_t N, bool side = false) {
  DeviceMap& m = f.m;
  const bool drift = N > 0 && f.P.drift.enabled && f.fuse_offset == nullptr;
  if (RB_SIDE_DRIFT && side) {
    setOverlap(f);
    const bool lists = RB_EARLY_HEAVY && N > 0 && f.overlap;
    if (!drift && !lists) return;
    checkCuda(cudaEventRecord(m.ev_dfork, f.s), "event");
    checkCuda(cudaStreamWaitEvent(m.stream2, m.ev_dfork, 0), "stream wait");
    if (drift) {
      k_drift_finalize<<<1, 1024, 0, m.stream2>>>(m.drift_sum_part, m.drift_n_part,
                                                   static_cast<int>(gridFor(N)), f.P.drift.min_points,
                                                   f.P.drift.max_offset_per_scan, m.drift_offset, m.stats);
      ++f.launches;
    }
    if (lists) {
      const RayArgs ra = rayArgs(f);
      const ClassArgs ca{ra.now, ra.t_free, ra.cleanup, ra.bound, ra.g.W};
      f.prepped = RB_SIDE_CLASSIFY && RB_FUSE_LIST;  // (lists imply a ray pass: cleanup or bound)
      f.presplit = f.prepped && RB_PRESPLIT;
      k_side_prep<<<streamGrid(f.ncell), kThreads, 0, m.stream2>>>(
          m.cur, f.ncell, drift ? static_cast<const double*>(m.drift_offset) : nullptr,
          static_cast<const int32_t*>(m.count), f.heavy, m.heavy, m.heavy + f.ncell,
          RB_FUSE_LIST ? m.heavy + 2 * f.ncell : nullptr, f.presplit ? m.heavy + 3 * f.ncell : nullptr,
          m.stats,
          f.prepped ? 1 : 0, ca, m.cls, m.probe, m.kstar);
    } else
      k_apply_offset<<<streamGrid(f.ncell), kThreads, 0, m.stream2>>>(m.cur, f.ncell, m.drift_offset);
    ++f.launches;
    // the jump grid under the sort as well, on large maps (on 400^2 / 500^2
    // maps the sort is too short to hide it: C2 / C3 +8 %)
    if (RB_SIDE_JUMP && RB_P1_JUMP && f.presplit && f.ncell >= kSideJumpCells) {
      const int jw = (f.g.W + kJumpBlk - 1) / kJumpBlk, jh = (f.g.H + kJumpBlk - 1) / kJumpBlk;
      k_jump_grid<<<static_cast<unsigned>((static_cast<std::size_t>(jw) * jh * 32 + kThreads - 1) / kThreads),
                    kThreads, 0, m.stream2>>>(static_cast<const ProbeT*>(m.probe), f.g.W, f.g.H, m.jgrid, jw, jh);
      ++f.launches;
      f.jump_done = true;
    }
    checkCuda(cudaEventRecord(m.ev_djoin, m.stream2), "event");
    f.drift_join = true;
    f.lists_built = lists;
    return;
  }
  if (!drift) return;
  launchPdl(k_drift_finalize, 1, 1024, 0, f.s, m.drift_sum_part, m.drift_n_part,
            static_cast<int>(gridFor(N)), f.P.drift.min_points, f.P.drift.max_offset_per_scan,
            m.drift_offset, m.stats);
  ++f.launches;
  f.fuse_offset = m.drift_offset;
}

void joinDrift(Frame& f) {
  if (!f.drift_join) return;
  checkCuda(cudaStreamWaitEvent(f.s, f.m.ev_djoin, 0), "stream wait");
  f.drift_join = false;
}

// K2 over N keys (cells; >= WH = not sorted) with payload (z, var) indexed
// by key position; then K3 gated fusion. Long cells go to stream2 when the
// ray pass can overlap them.
// The long-cell fold on the side stream, after the short-cell fold (whose
// ballots build its lists) and before the ray pass it overlaps.
void launchHeavy(Frame& f) {
  if (!f.overlap) return;
  DeviceMap& m = f.m;
  const bool cleanup = f.P.cleanup.cleanup_enabled, bound = f.P.cleanup.upper_bound_enabled;
  checkCuda(cudaEventRecord(m.ev[10], f.s), "event");
  checkCuda(cudaStreamWaitEvent(m.stream2, m.ev[10], 0), "stream wait");
  // (RB_HEAVY_PRIO: the long-cell fold, the critical path from the end of the
  // sort, at the highest scheduling priority)
  int prio_lo = 0, prio_hi = 0;
  if (RB_HEAVY_PRIO) checkCuda(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi), "stream priorities");
  launchPrio(k_fuse_heavy, kHeavyBlocks, 32, 0, m.stream2, RB_HEAVY_PRIO ? prio_hi : prio_lo, m.cur,
             static_cast<const int32_t*>(m.count), static_cast<const uint32_t*>(m.heavy),
             static_cast<const uint32_t*>(m.heavy + f.ncell), static_cast<const DevStats*>(m.stats),
             static_cast<const uint32_t*>(m.start), static_cast<const double*>(m.spz),
             static_cast<const double*>(m.spv), f.fa, m.stats, f.P.cleanup.t_free, cleanup ? 1 : 0,
             bound ? 1 : 0);
  ++f.launches;
  checkCuda(cudaEventRecord(m.ev[11], m.stream2), "event");
}

// K2 alone: spz / spv / start of the N keys' points in (cell, scan) order.
void phaseSort(Frame& f, const uint32_t* keys, uint32_t N, const double* z, const double* var,
               const SortGeom& sg) {
  DeviceMap& m = f.m;
  cudaStream_t s = f.s;
  // start[] is all 0xffffffff here: set at map creation, and k_cells resets
  // the entries of cells that had points after each scan.
  const std::size_t sc_smem = 20 * static_cast<std::size_t>(sg.buckets());
  const uint32_t* kin = keys;
  uint32_t *kout = m.key1, *vin = m.val0, *vout = m.val1;
  for (int p = 0; p < sg.passes; ++p) {
    const bool fused = RB_FUSED_ROWSCAN && sg.ntiles <= kFusedTiles;
    if (!fused) {
      launchPdl(k_sort_rowscan, sg.buckets(), kThreads, 0, s, sg.counts(p), sg.pitch,
                sg.rowsum + p * sg.buckets());
      ++f.launches;
    }
    launchPdl(fused ? (sg.tshift == kSmallTileShift ? k_sort_scatter<kSmallTile / kThreads, true>
                                                     : k_sort_scatter<kSortItems, true>)
                    : (sg.tshift == kSmallTileShift ? k_sort_scatter<kSmallTile / kThreads>
                                                     : k_sort_scatter<kSortItems>),
              sg.ntiles, kThreads, sc_smem, s, kin, vin, N, p, sg, f.WH, kout, vout, z, var, m.spz, m.spv,
              m.start);
    ++f.launches;
    // ping-pong between key1 and key0 (key0 is free once pass 0 has read it)
    const uint32_t* next_in = kout;
    kout = (kout == m.key1) ? m.key0 : m.key1;
    kin = next_in;
    std::swap(vin, vout);
  }
}

void phaseSortFuse(Frame& f, const uint32_t* keys, uint32_t N, const double* z, const double* var,
                   const SortGeom& sg) {
  DeviceMap& m = f.m;
  cudaStream_t s = f.s;
  phaseSort(f, keys, N, z, var, sg);
  RB_PHASE_EVENT(4, s);  // sort done

  const UpdateParams& U = f.P.update;
  FuseArgs fa;
  fa.now = f.stamp;
  fa.sigma_init2 = U.sigma_init2;
  fa.sigma_outlier2 = U.sigma_outlier2;
  fa.sigma_max2 = U.sigma_max2;
  fa.maha = U.mahalanobis_threshold;
  fa.maha2 = U.mahalanobis_threshold * U.mahalanobis_threshold;
  fa.wall = U.wall_count_threshold;
  setOverlap(f);
  f.fa = fa;
  if (f.lists_built) launchHeavy(f);  // lists built on stream2: start beside k_fuse
// Drift offset and ray classification as their own sweeps (default) or inside
// k_fuse: k_fuse runs at low occupancy (fold registers), so per-cell work for
// every cell there costs more than a separate streaming sweep (C4 frame +11 /
// +50 us measured).
#ifndef RB_FUSE_OFFSET
#define RB_FUSE_OFFSET 0
#endif
#ifndef RB_FUSE_CLASSIFY
#define RB_FUSE_CLASSIFY 0
#endif
#ifndef RB_SPLIT_CLASSIFY
#define RB_SPLIT_CLASSIFY 0  // measured slower
#endif
  joinDrift(f);
  const RayArgs ra = rayArgs(f);
  const ClassArgs ca{ra.now, ra.t_free, ra.cleanup, ra.bound, ra.g.W};
  int classify = 0;
  if (f.prepped) {
    classify = 2;
  } else if (RB_SPLIT_CLASSIFY && (ra.cleanup || ra.bound)) {
    launchPdl(k_prep, streamGrid(f.ncell), kThreads, 0, s, m.cur, f.ncell,
              static_cast<const double*>(f.fuse_offset), static_cast<const int32_t*>(m.count), ca,
              m.cls, m.probe, m.kstar);
    ++f.launches;
    f.fuse_offset = nullptr;
    classify = 2;
  } else {
    if (!RB_FUSE_OFFSET && f.fuse_offset != nullptr) {
      launchPdl(k_apply_offset, streamGrid(f.ncell), kThreads, 0, s, m.cur, f.ncell, f.fuse_offset);
      ++f.launches;
      f.fuse_offset = nullptr;
    }
    classify = RB_FUSE_CLASSIFY && (ra.cleanup || ra.bound) ? 1 : 0;
  }
  if (f.presplit) {
    // The removal candidates with points folded and classified first (usually
    // none: small blocks, enqueued first, so they find room beside the folds
    // below), then the short cells on stream3 beside the ray pass (checked,
    // not classified).
    checkCuda(cudaEventRecord(m.ev_sfork, s), "event");
    launchPdl(k_fuse_list, 148u, RB_PRE_THREADS, 0, s, m.cur, static_cast<const int32_t*>(m.count),
              static_cast<const uint32_t*>(m.heavy + 3 * f.ncell),
              static_cast<const unsigned long long*>(&m.stats->pre_cells),
              static_cast<const unsigned long long*>(nullptr), f.ncell, static_cast<const uint32_t*>(m.start), static_cast<const double*>(m.spz),
              static_cast<const double*>(m.spv), fa, m.stats, 1, ca, m.cls, m.probe, m.kstar);
    if (RB_B_AFTER_A) checkCuda(cudaEventRecord(m.ev_sfork, s), "event");
    checkCuda(cudaStreamWaitEvent(m.stream3, m.ev_sfork, 0), "stream wait");
    k_fuse_list<<<148u * RB_SFOLD_BLOCKS, RB_FUSE_LIST_THREADS, 0, m.stream3>>>(
        m.cur, static_cast<const int32_t*>(m.count), static_cast<const uint32_t*>(m.heavy + 2 * f.ncell),
        static_cast<const unsigned long long*>(&m.stats->light_cells),
        RB_LIGHT_SPLIT > 0 ? static_cast<const unsigned long long*>(&m.stats->light2_cells) : nullptr, f.ncell,
        static_cast<const uint32_t*>(m.start),
        static_cast<const double*>(m.spz), static_cast<const double*>(m.spv), fa, m.stats, 2, ca, m.cls,
        m.probe, m.kstar);
    checkCuda(cudaEventRecord(m.ev_sjoin, m.stream3), "event");
    ++f.launches;
  } else if (f.lists_built && RB_FUSE_LIST && (classify == 0 || f.prepped) && f.fuse_offset == nullptr)
    launchPdl(k_fuse_list, 148u * RB_FUSE_LIST_BLOCKS, RB_FUSE_LIST_THREADS, 0, s, m.cur,
              static_cast<const int32_t*>(m.count), static_cast<const uint32_t*>(m.heavy + 2 * f.ncell),
              static_cast<const unsigned long long*>(&m.stats->light_cells),
              RB_LIGHT_SPLIT > 0 ? static_cast<const unsigned long long*>(&m.stats->light2_cells) : nullptr,
              f.ncell, static_cast<const uint32_t*>(m.start), static_cast<const double*>(m.spz),
              static_cast<const double*>(m.spv), fa, m.stats, f.prepped ? 1 : 0, ca, m.cls, m.probe,
              m.kstar);
  else
    launchPdl(k_fuse, gridFor(f.ncell), kThreads, 0, s, m.cur, f.ncell, m.count, m.start, m.spz, m.spv,
              fa, m.stats, f.heavy, f.lists_built ? nullptr : m.heavy, m.heavy + f.ncell, f.fuse_offset,
              classify, ca, m.cls, m.probe, m.kstar);
  ++f.launches;
  f.fuse_offset = nullptr;
  f.classified = classify != 0;
  f.fa = fa;
  // (Launching it after k_classify instead, to keep that kernel boundary programmatic, made
  // the frame 15 % slower: the side-stream blocks then queue behind the ray pass.)
  if (!f.lists_built) launchHeavy(f);
  RB_PHASE_EVENT(5, s);  // fusion done (short cells when overlapped)
}


// K5 pass 1 over this process's rays (ids ray_base + k), joined with the
// long-cell fold (and redone if a speculated class was wrong).
void phaseRaysPass1(Frame& f, uint32_t N, uint32_t ray_base, bool tail = false) {
  DeviceMap& m = f.m;
  cudaStream_t s = f.s;
  const RayArgs ra = rayArgs(f);
  if (ra.cleanup || ra.bound) {
    if (!f.classified) {
      launchPdl(k_classify, streamGrid(f.ncell), kThreads, 0, s, m.cur, f.ncell, ra, m.cls, m.kstar,
                m.count, f.overlap ? f.heavy : -1, 0, m.stats, m.probe);
      ++f.launches;
    }
    if (N > 0) {
      RayArgs rj = ra;
      if (RB_P1_JUMP) {  // the jump grid of this frame's probe words (pass1Jump)
        const int jw = (f.g.W + kJumpBlk - 1) / kJumpBlk, jh = (f.g.H + kJumpBlk - 1) / kJumpBlk;
        if (!f.jump_done) {
          launchPdl(k_jump_grid, static_cast<unsigned>((static_cast<std::size_t>(jw) * jh * 32 + kThreads - 1) / kThreads),
                    kThreads, 0, s, static_cast<const ProbeT*>(m.probe), f.g.W, f.g.H, m.jgrid, jw, jh);
          ++f.launches;
        }
        rj.jgrid = m.jgrid;
        rj.jw = jw;
        rj.jh = jh;
        rj.jres = kJumpBlk * f.g.res;
      }
      launchPdl(k_rays_pass1<false>, gridFor(N, kP1Threads), kP1Threads, 0, s, N, m.kept + f.ray_at,
                m.px + f.ray_at, m.py + f.ray_at, m.pz + f.ray_at, rj, m.cur, m.cls, m.kstar,
                m.raylist, m.stats, 0, ray_base, m.probe, f.point_cells);
      ++f.launches;
#ifdef RB_P1_DIAG
      k_p1diag<<<1, 1, 0, s>>>();
#endif
    }
  }
  if (f.overlap && !tail) {  // (tail: phaseRaysTail joins and retries)
    // Join the long-cell fold; redo the ray pass only if a heavy cell fused
    // nothing (both kernels return immediately otherwise).
    checkCuda(cudaStreamWaitEvent(s, m.ev[11], 0), "stream wait");
    launchPdl(k_classify, 148u * 4u, kThreads, 0, s, m.cur, f.ncell, ra, m.cls, m.kstar, m.count, -1, 1,
              m.stats, m.probe);  // one wave: a no-op unless a speculation failed
    ++f.launches;
    if (N > 0) {
      launchPdl(k_rays_pass1<true>, std::min(gridFor(N, kP1Threads), 148u * RB_PASS1_MIN_BLOCKS),
                kP1Threads, 0, s, N, m.kept + f.ray_at, m.px + f.ray_at, m.py + f.ray_at,
                m.pz + f.ray_at, ra, m.cur, m.cls, m.kstar, m.raylist, m.stats, 1, ray_base,
                m.probe, f.point_cells);
      ++f.launches;
    }
  }
}

// Single-call frames: join the long-cell fold, then one cooperative launch
// for the retry of a failed speculation and pass 2 (k_rays_tail); k_cells
// removes the k* < inf cells.
void phaseRaysTail(Frame& f, uint32_t N) {
  DeviceMap& m = f.m;
  const RayArgs ra = rayArgs(f);
  const bool retry = f.overlap && N > 0;
  const bool pass2 = ra.cleanup && ra.bound;
  if (ra.cleanup) f.fold_remove = true;
  if (f.overlap) checkCuda(cudaStreamWaitEvent(f.s, m.ev[11], 0), "stream wait");
  if (f.presplit) checkCuda(cudaStreamWaitEvent(f.s, m.ev_sjoin, 0), "stream wait");
  if (!retry && !pass2) return;
  static int blocks_per_sm = 0, sms = 0;
  if (blocks_per_sm == 0) {
    checkCuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_rays_tail, kP1Threads, 0),
              "occupancy");
    checkCuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m.device), "device attribute");
  }
  launchCoopPdl(k_rays_tail, static_cast<unsigned>(blocks_per_sm * sms), kP1Threads, 0, f.s,
                retry ? 1 : 0, pass2 ? 1 : 0, N, m.kept + f.ray_at, m.px + f.ray_at, m.py + f.ray_at,
                m.pz + f.ray_at, ra, m.cur, m.cls, m.kstar, m.raylist, m.stats, m.probe,
                f.point_cells, m.ub2);
  ++f.launches;
}

// Removal of k* < inf cells, then K6 bounds of removed cells from this
// process's queued rays k >= k*.
void phaseRemovePass2(Frame& f, uint32_t ray_base) {
  DeviceMap& m = f.m;
  const RayArgs ra = rayArgs(f);
  if (!ra.cleanup) return;
  if (f.explicit_remove) {
    launchPdl(k_remove, streamGrid(f.ncell), kThreads, 0, f.s, m.cur, f.ncell, m.kstar, m.stats);
    ++f.launches;
    if (ra.bound) {
      launchPdl(k_rays_pass2<false>, 148 * 8, kThreads, 0, f.s, m.raylist, m.stats, m.px + f.ray_at,
                m.py + f.ray_at, m.pz + f.ray_at, ra, m.cur, m.cls, m.kstar, ray_base, m.ub2);
      ++f.launches;
    }
    return;
  }
  f.fold_remove = true;  // k_cells removes the k* < inf cells
  if (ra.bound) {
    launchPdl(k_rays_pass2<true>, 148 * 8, kThreads, 0, f.s, m.raylist, m.stats, m.px + f.ray_at,
              m.py + f.ray_at, m.pz + f.ray_at, ra, m.cur, m.cls, m.kstar, ray_base, m.ub2);
    ++f.launches;
  }
}

// K7 cell phases + update_variance, then the conv-net filter when selected.
void phaseCells(Frame& f) {
  joinDrift(f);
  DeviceMap& m = f.m;
  const UpdateParams& U = f.P.update;
  CellArgs ca;
  ca.g = f.g;
  ca.rx = f.pose.t[0];
  ca.ry = f.pose.t[1];
  ca.rz = f.pose.t[2];
  ca.overlap = f.P.overlap.enabled;
  ca.ov_r2 = f.P.overlap.radius * f.P.overlap.radius;
  ca.ov_thr = f.P.overlap.height_threshold;
  const TraversabilityParams& T = f.P.traversability;
  ca.geo_trav = f.P.use_convnet_traversability ? 0 : 1;
  ca.radius = ca.geo_trav ? T.window / 2 : 1;
  ca.slope_max = T.slope_max;
  ca.step_max = T.step_max;
  ca.rough_max = T.roughness_max;
  ca.w_slope = T.w_slope;
  ca.w_step = T.w_step;
  ca.w_rough = T.w_roughness;
  ca.time_var = (f.dt != 0.0 && U.sigma_t2 != 0.0) ? 1 : 0;
  ca.growth = U.sigma_t2 * (f.dt / U.nominal_update_period);
  ca.sigma_max2 = U.sigma_max2;
  ca.scrub = m.scrub_invalid ? 1 : 0;
  ca.fold_remove = f.fold_remove ? 1 : 0;
  ca.kstar = m.kstar;
  ca.ub2 = m.ub2;
  ca.hstats = nullptr;
  ca.hseq = nullptr;
  ca.seq = 0;
  ca.nblocks = 0;
  f.handover = f.handover && !f.P.use_convnet_traversability;
  if (f.handover) {
    ca.hstats = m.h_stats;
    ca.hseq = m.h_seq;
    ca.seq = ++m.frame_seq;
  }
  const int halo = std::max(1, ca.radius);
  const std::size_t sm = static_cast<std::size_t>(kTileX + 2 * halo) * (kTileY + 2 * halo) * 9 + 16;
  if (sm > kCellsMaxSmem) {  // window too large for a shared-memory tile
    ca.nblocks = static_cast<unsigned>((f.g.W + 255) / 256) * static_cast<unsigned>(f.g.H);
    launchPdl(k_cells_global, dim3((f.g.W + 255) / 256, f.g.H), 256, 0, f.s, m.cur, m.count,
              m.start, ca, m.stats);
  } else {
    const dim3 grid((f.g.W + kTileX - 1) / kTileX, (f.g.H + kTileY - 1) / kTileY);
    ca.nblocks = grid.x * grid.y;
    auto* kern = ca.radius == 2 ? k_cells<2> : (ca.radius == 1 ? k_cells<1> : k_cells<0>);
    if (sm > 48 * 1024)
      checkCuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sm)),
                "smem attribute");
    launchPdl(kern, grid, dim3(kTileX, kTileY), sm, f.s, m.cur, m.count, m.start, ca, m.stats);
  }
  ++f.launches;
  // invalid cells' normals / traversability are zero again, unless the
  // conv-net below writes the traversability of every cell
  m.scrub_invalid = f.P.use_convnet_traversability;
  RB_PHASE_EVENT(7, f.s);  // cell phases done
  // Conv-net traversability (reference integration.cpp:242-244): reads the
  // post-overlap elevation, writes the traversability of every cell.
  if (f.P.use_convnet_traversability)
    f.launches += convnetEnqueue(f.s, m.conv, m.cur.elev, m.cur.valid, f.g.W, f.g.H, f.P.convnet,
                                 m.cur.trav);
  recordTiming(m.ev[12], f.s);  // traversability done
}

// Stats to the host (one sync).
void phaseStatsEnqueue(Frame& f) {
  DeviceMap& m = f.m;
  if (!f.handover)
    checkCuda(cudaMemcpyAsync(m.h_stats, m.stats, sizeof(DevStats), cudaMemcpyDeviceToHost, f.s), "stats");
  checkCuda(cudaGetLastError(), "kernel launch");
}
const DevStats& phaseStatsWait(Frame& f) {
  DeviceMap& m = f.m;
  if (f.handover) {
    // Poll the sequence number k_cells publishes; every 1024 polls ask the
    // stream, so a failed frame (or a finished one whose write this thread
    // has not yet seen) ends the wait with the stream's status.
    const volatile unsigned long long* seq = m.h_seq;
    for (unsigned k = 1; *seq != m.frame_seq; ++k) {
      if ((k & 1023u) == 0) {
        const cudaError_t e = cudaStreamQuery(f.s);
        if (e == cudaSuccess) break;
        if (e != cudaErrorNotReady) checkCuda(e, "integrate");
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    if (*seq != m.frame_seq) fail(Err::kDevice, "frame stats were not handed over");
  } else {
    checkCuda(cudaStreamSynchronize(f.s), "integrate");
  }
  if (m.h_stats->error_code == 1) fail(Err::kInvalidVariance, "variances must be positive");
  return *m.h_stats;
}
const DevStats& phaseStats(Frame& f) {
  phaseStatsEnqueue(f);
  return phaseStatsWait(f);
}

// One CUDA graph per synchronous frame: the frame's launches
// are captured from the map's stream and the capture updates a cached
// executable graph (cudaGraphExecUpdate: new kernel arguments, copy sources,
// grid sizes); a topology not seen recently is instantiated once and kept
// (DeviceMap::kGraphs entries). Host cost per frame: the capture (~0.3 us per
// launch) + update + one launch, instead of ~3 us per direct launch
// (scripts/graph_overhead.cu). Programmatic (PDL) edges are kept in the graph.
struct FrameCapture {
  DeviceMap& m;
  cudaStream_t s;
  bool on;
  FrameCapture(DeviceMap& map, cudaStream_t st, bool enable) : m(map), s(st), on(false) {
    if (enable) begin();
  }
  void begin() {
    checkCuda(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
    on = true;
  }
  ~FrameCapture() {  // an exception mid-frame: end (and drop) the capture
    if (on) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(s, &g);
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
    }
  }
  void launch() {
    if (!on) return;
    on = false;
    cudaGraph_t g = nullptr;
    checkCuda(cudaStreamEndCapture(s, &g), "end capture");
    cudaGraphExec_t exec = nullptr;
    // most recently used first
    for (int k = 0; k < m.graph_count && exec == nullptr; ++k) {
      cudaGraphExecUpdateResultInfo info;
      if (cudaGraphExecUpdate(m.graphs[k], g, &info) == cudaSuccess) {
        exec = m.graphs[k];
        std::rotate(m.graphs, m.graphs + k, m.graphs + k + 1);
        ++m.graph_updates;
      } else {
        cudaGetLastError();
      }
    }
    if (exec == nullptr) {
      // (RB_MAIN_PRIO: the captured streams' priorities kept on the graph's nodes)
      const cudaError_t e =
          cudaGraphInstantiate(&exec, g, (RB_MAIN_PRIO || RB_HEAVY_PRIO) ? cudaGraphInstantiateFlagUseNodePriority : 0);
      if (e != cudaSuccess) {
        cudaGraphDestroy(g);
        checkCuda(e, "graph instantiate");
      }
      if (m.graph_count == DeviceMap::kGraphs) cudaGraphExecDestroy(m.graphs[--m.graph_count]);
      std::copy_backward(m.graphs, m.graphs + m.graph_count, m.graphs + m.graph_count + 1);
      m.graphs[0] = exec;
      ++m.graph_count;
      ++m.graph_instantiations;
    }
    cudaGraphDestroy(g);
    checkCuda(cudaGraphLaunch(exec, s), "graph launch");
  }
};

bool hostPinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

ScanResult resultFrom(const DevStats& d, std::size_t n) {
  ScanResult out;
  out.points_in = static_cast<std::int64_t>(n);
  out.excluded = static_cast<std::int64_t>(d.excluded);
  out.out_of_range = static_cast<std::int64_t>(d.out_of_range);
  out.out_of_map = static_cast<std::int64_t>(d.out_of_map);
  out.outlier = static_cast<std::int64_t>(d.outlier);
  out.ignored_low = static_cast<std::int64_t>(d.ignored_low);
  out.fused = static_cast<std::int64_t>(d.fused);
  out.cells_updated = static_cast<std::int64_t>(d.cells_updated);
  out.removed = static_cast<std::int64_t>(d.removed);
  out.overlap_cleared = static_cast<std::int64_t>(d.overlap_cleared);
  out.drift_offset = d.drift_offset;
  out.drift_clamped = d.drift_clamped != 0;
  out.drift_points = d.drift_n;
  return out;
}

}  // namespace

// Loads the frame kernels' code on this device now (map creation) rather than
// at their first launch: with the runtime's lazy module loading the first
// frame of a process otherwise pays ~10 ms on the device.
#ifndef RB_CARVEOUT
#define RB_CARVEOUT -1  // (-1: the driver's choice per kernel; 25 / 50 / 100 measured slower)
#endif
void preloadFrameKernels(int device) {
  static bool done[64] = {};
  if (device < 0 || device >= 64 || done[device]) return;
  done[device] = true;
  cudaFuncAttributes fa;
  const void* kernels[] = {
      reinterpret_cast<const void*>(k_shift), reinterpret_cast<const void*>(k_ingest),
      reinterpret_cast<const void*>(k_ingest_tma),
      reinterpret_cast<const void*>(k_drift_finalize), reinterpret_cast<const void*>(k_apply_offset),
      reinterpret_cast<const void*>(k_side_prep), reinterpret_cast<const void*>(k_fuse_list),
      reinterpret_cast<const void*>(k_sort_rowscan),
      reinterpret_cast<const void*>(k_sort_scatter<kSortItems>),
      reinterpret_cast<const void*>(k_sort_scatter<kSortItems, true>),
      reinterpret_cast<const void*>(k_sort_scatter<kSmallTile / kThreads>),
      reinterpret_cast<const void*>(k_sort_scatter<kSmallTile / kThreads, true>),
      reinterpret_cast<const void*>(k_fuse), reinterpret_cast<const void*>(k_fuse_heavy),
      reinterpret_cast<const void*>(k_classify), reinterpret_cast<const void*>(k_jump_grid),
      reinterpret_cast<const void*>(k_rays_pass1<false>), reinterpret_cast<const void*>(k_rays_pass1<true>),
      reinterpret_cast<const void*>(k_rays_tail), reinterpret_cast<const void*>(k_cells<0>),
      reinterpret_cast<const void*>(k_cells<1>), reinterpret_cast<const void*>(k_cells<2>),
      reinterpret_cast<const void*>(k_cells_global)};
  // One shared-memory carveout for every frame kernel (RB_CARVEOUT, percent
  // of the unified L1 / shared memory): kernels of both streams share SMs, and
  // an SM runs one carveout at a time -- with the driver's per-kernel choice,
  // blocks of the long-cell fold (34 KB) could not join an SM running the
  // short-cell fold (1 KB) until it drained.
  for (const void* k : kernels) {
    cudaFuncGetAttributes(&fa, k);
    if (RB_CARVEOUT >= 0) cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, RB_CARVEOUT);
  }
  cudaGetLastError();
}

ScanResult integrateScanDevice(DeviceMap& m, const PipelineParams& P, const double* xyz,
                               std::size_t n, bool xyz_on_device, const Pose& pose,
                               double stamp, double dt) {
  const auto t_call = std::chrono::steady_clock::now();
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  if (n >= 0xffffffffULL) fail(Err::kUsage, "too many points in one scan");
  if (m.shard.stage != 0) fail(Err::kUsage, "a sharded frame is in progress on this map");
  if (m.async_count != 0) fail(Err::kUsage, "streaming frames in flight: call relief_gpu_map_wait");
  Frame f(m, P, pose, stamp, dt);
  const uint32_t N = static_cast<uint32_t>(n);
  // Scratch first: nothing may allocate inside a graph capture.
  if (n > 0) {
    phaseScratch(f, n);
    f.small_tiles = RB_SMALL_TILE_N > 0;
    sortGeometry(m, f.WH, N, f.small_tiles);
  }
  // Pageable host input cannot be a graph's copy source: it is uploaded
  // before the capture (the frame then reads it like device input).
  const bool pageable = !xyz_on_device && n > 0 && !hostPinned(xyz);
  // Graph frames (DeviceMap::graph_mode): with direct launches the device
  // outruns the host's submission on mid-size frames; on tiny frames the
  // capture + update costs more than it saves.
  // (Phase timing: direct launches, so no phase absorbs the wait for the
  // graph launch of a head-split frame.)
  const bool graph = !P.use_convnet_traversability && !m.phase_events &&
                     (m.graph_mode == 1 || (m.graph_mode == 2 && N >= kGraphMinPoints));
  const bool graph_head = graph && N >= kGraphHeadPoints;
  // ev0 -> ev13: the input copy (host input only); everything after it is the
  // frame's device time (stats / count / tile-count resets, recenter, kernels).
  const double* d_xyz = xyz;
  if (pageable) {
    recordTiming(m.ev[0], f.s);
    d_xyz = phaseUpload(f, xyz, n, false);
    recordTiming(m.ev[13], f.s);
  }
  // Graph frames: the head of the frame (upload, resets, recenter, ingest,
  // drift) is launched directly, so the device starts at once; the rest is
  // captured and its graph updated while the ingest runs (RB_GRAPH_HEAD 0:
  // the whole frame is captured).
  FrameCapture cap(m, f.s, graph && !graph_head);
  const bool chunked = !xyz_on_device && !pageable && N >= 2 * kTile;
  if (!pageable) {
    recordTiming(m.ev[0], f.s);
    d_xyz = chunked ? phaseUploadChunked(f, xyz, N) : phaseUpload(f, xyz, n, xyz_on_device);
    if (!chunked) recordTiming(m.ev[13], f.s);  // copy done
  }
  phaseBegin(f, false);
#ifdef RB_TIMELINE
  k_tl_reset<<<1, 32, 0, f.s>>>();
#endif
  // count[] is all zero here: k_cells clears it after its last use each scan.
  const SortGeom sg = phaseSortGeometry(f, N);
  RB_PHASE_EVENT(1, f.s);  // resets done
  phaseIngest(f, d_xyz, N, sg, true, chunked, 0, true);
  RB_PHASE_EVENT(2, f.s);  // ingest done
  if (!RB_SIDE_DRIFT || n == 0) phaseDrift(f, N);
  RB_PHASE_EVENT(3, f.s);  // drift done
  if (graph_head) cap.begin();
  if (n > 0) {
    phaseDrift(f, N, true);
    phaseSortFuse(f, m.key0, N, m.pz, m.pvar, sg);
    f.point_cells = sg.passes <= 2 ? m.key0 : nullptr;  // a 3rd pass reuses key0
    phaseRaysPass1(f, N, 0, true);
    phaseRaysTail(f, N);
  } else {
    RB_PHASE_EVENT(4, f.s);
    RB_PHASE_EVENT(5, f.s);
  }
  RB_PHASE_EVENT(6, f.s);  // rays done
  f.handover = RB_STATS_HANDOVER != 0;
  phaseCells(f);
  phaseStatsEnqueue(f);
  cap.launch();
#ifdef RB_HOST_DIAG
  const auto t_sub = std::chrono::steady_clock::now();
#endif
  const DevStats& d = phaseStatsWait(f);
#ifdef RB_TIMELINE
  {
    checkCuda(cudaStreamSynchronize(f.s), "timeline");
    unsigned long long tl[kTlSlots][2];
    checkCuda(cudaMemcpyFromSymbol(tl, g_tl, sizeof(tl)), "timeline");
    unsigned long long te[kTlSlots][32];
    checkCuda(cudaMemcpyFromSymbol(te, g_tl_end, sizeof(te)), "timeline");
    for (int k = 0; k < kTlSlots; ++k)
      for (int j = 0; j < 32; ++j) tl[k][1] = std::max(tl[k][1], te[k][j]);
    fprintf(stderr, "TL");
    for (int k = 0; k < kTlSlots; ++k) fprintf(stderr, " %llu %llu", tl[k][0], tl[k][1]);
    fprintf(stderr, "\nTLC pre %llu light %llu heavy %llu vheavy %llu respec %d\n", d.pre_cells,
            d.light_cells, d.heavy_cells, d.vheavy_cells, d.respeculate);
  }
#endif
  ScanResult out = resultFrom(d, n);
#ifdef RB_HOST_DIAG
  {  // host-side split of the call: submission, wait (averages every 200 calls)
    static double s_sub = 0, s_wait = 0;
    static int s_n = 0;
    const auto t_end = std::chrono::steady_clock::now();
    s_sub += std::chrono::duration<double>(t_sub - t_call).count();
    s_wait += std::chrono::duration<double>(t_end - t_sub).count();
    if (++s_n == 200) {
      fprintf(stderr, "HOSTDIAG n=%zu submit %.2f us wait %.2f us launches %lld\n", n, s_sub / s_n * 1e6,
              s_wait / s_n * 1e6, f.launches);
      s_sub = s_wait = 0;
      s_n = 0;
    }
  }
#endif

  // Per-phase device times are read from the events only when asked for
  // (resolveTiming): nine event queries cost ~30 us of host time per call.
  m.timing_pending = true;
  m.timing_chunked = chunked;
  m.timing_phases = m.phase_events;
  out.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_call).count();
  m.last_launches = f.launches;
  m.last_visits = static_cast<long long>(d.visits);
  return out;
}

// Per-phase device times of the last synchronous frame (kernel_seconds:
// upload, ingest (+ resets / recenter), drift, sort, fusion, rays, cell
// phases, total device time after the copy; phase_seconds: the reference's
// Table I labels), from its events, on first request.
void resolveTiming(DeviceMap& m) {
  if (!m.timing_pending) return;
  m.timing_pending = false;
  // (a frame whose stats were handed over may still be recording its last event)
  checkCuda(cudaEventSynchronize(m.ev[12]), "timing");
  if (!m.timing_phases) {  // only the upload and the device total were recorded
    float ms_copy = 0.0f, ms_total = 0.0f;
    checkCuda(cudaEventElapsedTime(&ms_copy, m.ev[0], m.ev[13]), "timing");
    checkCuda(cudaEventElapsedTime(&ms_total, m.ev[13], m.ev[12]), "timing");
    for (double& v : m.kernel_seconds) v = 0.0;
    for (double& v : m.phase_seconds) v = 0.0;
    m.kernel_seconds[0] = ms_copy * 1e-3;
    m.kernel_seconds[7] = std::max(0.0f, ms_total) * 1e-3;
    m.phase_seconds[6] = m.kernel_seconds[7];
    return;
  }
  float ms[7], ms_trav = 0.0f, ms_copy = 0.0f, ms_reset = 0.0f;
  for (int k = 1; k < 7; ++k) checkCuda(cudaEventElapsedTime(&ms[k], m.ev[k], m.ev[k + 1]), "timing");
  checkCuda(cudaEventElapsedTime(&ms_trav, m.ev[7], m.ev[12]), "timing");
  checkCuda(cudaEventElapsedTime(&ms_copy, m.ev[0], m.ev[13]), "timing");
  checkCuda(cudaEventElapsedTime(&ms_reset, m.ev[13], m.ev[1]), "timing");
  // kernel_seconds: upload (input copy), ingest (+ resets / recenter), drift,
  // sort, fusion, rays, cell phases, total device time after the copy. With a
  // chunked upload the resets and all but the last chunk's ingest run under
  // the copy: "ingest" is then the part after the upload ended.
  ms[0] = ms_copy;
  if (m.timing_chunked) {
    float after = 0.0f;
    checkCuda(cudaEventElapsedTime(&after, m.ev[13], m.ev[2]), "timing");
    ms[1] = std::max(0.0f, after);
  } else {
    ms[1] += ms_reset;
  }
  for (int k = 0; k < 6; ++k) m.kernel_seconds[k] = ms[k] * 1e-3;
  m.kernel_seconds[6] = (ms[6] + ms_trav) * 1e-3;
  m.kernel_seconds[7] = (ms[1] + ms[2] + ms[3] + ms[4] + ms[5] + ms[6] + ms_trav) * 1e-3;
  m.phase_seconds[0] = ms[1] * 1e-3;                    // point transform & z error count (+ move_to)
  m.phase_seconds[1] = ms[2] * 1e-3;                    // drift compensation
  m.phase_seconds[2] = (ms[3] + ms[4] + ms[5]) * 1e-3;  // height update & ray casting
  m.phase_seconds[3] = ms[6] * 1e-3;                    // overlap + normals (+ geometric traversability, fused)
  m.phase_seconds[4] = ms_trav * 1e-3;                  // conv-net traversability
  m.phase_seconds[5] = 0.0;
  m.phase_seconds[6] = m.kernel_seconds[7];
}

// ------------------------------------------------------- streaming frames
// Same launch sequence as integrateScanDevice, but the points are copied on
// copy_stream into one of two input slots (waiting until the frame that last
// used the slot has ingested it), the stats go to that slot's pinned buffer,
// and nothing waits: frame k+1's PCIe transfer overlaps frame k's kernels.
void integrateScanAsync(DeviceMap& m, const PipelineParams& P, const double* xyz, std::size_t n,
                        const Pose& pose, double stamp, double dt) {
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  if (n >= 0xffffffffULL) fail(Err::kUsage, "too many points in one scan");
  if (m.shard.stage != 0) fail(Err::kUsage, "a sharded frame is in progress on this map");
  if (m.async_count == DeviceMap::kSlots)
    fail(Err::kUsage, "too many frames in flight: call relief_gpu_map_wait");
  const int slot = (m.async_head + m.async_count) % DeviceMap::kSlots;
  // Growing the scratch frees buffers a frame in flight may still use.
  const bool grows = n > 0 && (n > m.cap || m.pslab == nullptr || gridFor(n) > m.rcap);
  if (grows && m.async_count > 0) {
    checkCuda(cudaStreamSynchronize(m.stream), "stream sync");
    checkCuda(cudaStreamSynchronize(m.copy_stream), "stream sync");
  }
  Frame f(m, P, pose, stamp, dt);
  const uint32_t N = static_cast<uint32_t>(n);
  f.small_tiles = RB_SMALL_TILE_N > 0;
  phaseBegin(f);
  phaseScratch(f, n);
  double* d_xyz = m.xyz_slot[slot];
  if (n > 0) {
    checkCuda(cudaStreamWaitEvent(m.copy_stream, m.ev_consumed[slot], 0), "stream wait");
    checkCuda(cudaEventRecord(m.ev_copy0[slot], m.copy_stream), "event");
    checkCuda(cudaMemcpyAsync(d_xyz, xyz, n * 3 * sizeof(double), cudaMemcpyHostToDevice, m.copy_stream),
              "point upload");
    checkCuda(cudaEventRecord(m.ev_copied[slot], m.copy_stream), "event");
  }
  const SortGeom sg = phaseSortGeometry(f, N);  // count[] is zero (cleared by k_cells)
  if (n > 0) checkCuda(cudaStreamWaitEvent(f.s, m.ev_copied[slot], 0), "stream wait");
  checkCuda(cudaEventRecord(m.ev_start[slot], f.s), "event");
  RB_PHASE_EVENT(1, f.s);
  phaseIngest(f, d_xyz, N, sg, true, false, 0, true);
  checkCuda(cudaEventRecord(m.ev_consumed[slot], f.s), "event");
  RB_PHASE_EVENT(2, f.s);
  if (!RB_SIDE_DRIFT || n == 0) phaseDrift(f, N);
  RB_PHASE_EVENT(3, f.s);
  if (n > 0) {
    phaseDrift(f, N, true);
    phaseSortFuse(f, m.key0, N, m.pz, m.pvar, sg);
    f.point_cells = sg.passes <= 2 ? m.key0 : nullptr;  // a 3rd pass reuses key0
    phaseRaysPass1(f, N, 0, true);
    phaseRaysTail(f, N);
  } else {
    RB_PHASE_EVENT(4, f.s);
    RB_PHASE_EVENT(5, f.s);
  }
  RB_PHASE_EVENT(6, f.s);
  phaseCells(f);
  checkCuda(cudaMemcpyAsync(m.h_slot[slot], m.stats, sizeof(DevStats), cudaMemcpyDeviceToHost, f.s),
            "stats");
  checkCuda(cudaEventRecord(m.ev_done[slot], f.s), "event");
  checkCuda(cudaGetLastError(), "kernel launch");
  m.async_n[slot] = n;
  ++m.async_count;
  m.last_launches = f.launches;
}

ScanResult waitScan(DeviceMap& m) {
  if (m.async_count == 0) fail(Err::kUsage, "no frame in flight");
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  const int slot = m.async_head;
  checkCuda(cudaEventSynchronize(m.ev_done[slot]), "integrate");
  const DevStats d = *m.h_slot[slot];
  // Device timing of this frame: its copy, and its kernels from the moment
  // the copy had landed (kernel_seconds[0] / [7]; the other phases are not
  // separated in streaming mode).
  float ms_copy = 0.0f, ms_run = 0.0f;
  if (m.async_n[slot] > 0)
    checkCuda(cudaEventElapsedTime(&ms_copy, m.ev_copy0[slot], m.ev_copied[slot]), "timing");
  checkCuda(cudaEventElapsedTime(&ms_run, m.ev_start[slot], m.ev_done[slot]), "timing");
  m.timing_pending = false;
  for (double& v : m.kernel_seconds) v = 0.0;
  m.kernel_seconds[0] = ms_copy * 1e-3;
  m.kernel_seconds[7] = ms_run * 1e-3;
  m.async_head = (m.async_head + 1) % DeviceMap::kSlots;
  --m.async_count;
  if (d.error_code == 1) fail(Err::kInvalidVariance, "variances must be positive");
  m.last_visits = static_cast<long long>(d.visits);
  return resultFrom(d, m.async_n[slot]);
}

// ------------------------------------------------------- sharded frames
// Phase 1: recenter, this batch's K1, and its fusion records (stable
// compaction of the in-map kept points) plus the local drift vote and fate
// counters for the exchange.
void shardIngest(DeviceMap& m, const PipelineParams& P, const double* xyz, std::size_t n,
                 bool xyz_on_device, uint64_t ray_offset, uint64_t n_total, const Pose& pose,
                 double stamp, ShardIO& io) {
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  if (m.async_count != 0) fail(Err::kUsage, "streaming frames in flight: call relief_gpu_map_wait");
  if (n_total >= 0x7fffffffULL) fail(Err::kUsage, "too many points in one scan");
  if (ray_offset + n > n_total) fail(Err::kUsage, "shard batch outside the frame");
  // Point scratch sized for the whole frame now: phase 2 sorts all records
  // while this batch's points must stay resident for the ray passes.
  if (n_total > 0) ensurePointCapacity(m, static_cast<std::size_t>(n_total));
  ShardState& st = m.shard;
  st = ShardState{};
  st.params = P;
  st.pose = pose;
  st.stamp = stamp;
  st.dt = m.has_last ? std::max(0.0, stamp - m.last_stamp) : 0.0;
  st.n_local = n;
  st.ray_base = static_cast<uint32_t>(ray_offset);
  Frame f(m, st.params, pose, stamp, st.dt);
  const uint32_t N = static_cast<uint32_t>(n);
  phaseBegin(f);
  const double* d_xyz = phaseUpload(f, xyz, n, xyz_on_device);
  SortGeom none;
  phaseIngest(f, d_xyz, N, none, false);
  io = ShardIO{};
  if (n > 0) {
    if (P.drift.enabled) {
      k_drift_local<<<1, 1024, 0, f.s>>>(m.drift_sum_part, m.drift_n_part, static_cast<int>(gridFor(n)),
                                         m.drift_local);
      ++f.launches;
    }
    const uint32_t nblk = (N + kCompact - 1) / kCompact;
    k_compact_count<<<nblk, kCompact, 0, f.s>>>(m.key0, N, f.WH, m.blk);
    k_compact_scan<<<1, kThreads, 0, f.s>>>(m.blk, nblk, m.blk + m.rcap);
    k_compact_write<<<nblk, kCompact, 0, f.s>>>(m.key0, m.pz, m.pvar, N, f.WH, m.blk, m.rec_cell,
                                                m.rec_z, m.rec_var);
    f.launches += 3;
  }
  const DevStats& d = phaseStats(f);
  io.counters[0] = static_cast<int64_t>(d.out_of_range);
  io.counters[1] = static_cast<int64_t>(d.excluded);
  io.counters[2] = static_cast<int64_t>(d.out_of_map);
  if (n > 0) {
    uint32_t total = 0;
    checkCuda(cudaMemcpy(&total, m.blk + m.rcap, sizeof(total), cudaMemcpyDeviceToHost), "records");
    io.n_records = total;
    if (P.drift.enabled)
      checkCuda(cudaMemcpy(io.drift, m.drift_local, 2 * sizeof(double), cudaMemcpyDeviceToHost), "drift");
  }
  io.rec_cell = m.rec_cell;
  io.rec_z = m.rec_z;
  io.rec_var = m.rec_var;
  io.kstar = m.kstar;
  io.ub = m.cur.ub;
  io.ubv = m.cur.ubv;
  io.cells = f.ncell;
  st.launches = f.launches;
  st.stage = 1;
}

// Phase 2: drift offset from all ranks' votes (summed in rank order), sort +
// fusion of all gathered records (every rank, identical), ray pass 1 over
// this batch. Leaves k* / ub / ubv for the min / min / max all-reduce.
void shardUpdate(DeviceMap& m, const double* drift_pairs, int n_ranks, const uint32_t* d_cells,
                 const double* d_z, const double* d_var, std::size_t n_records, ShardIO& io) {
  ShardState& st = m.shard;
  if (st.stage != 1) fail(Err::kUsage, "shard phases out of order (expected update after ingest)");
  if (n_records >= 0xffffffffULL) fail(Err::kUsage, "too many points in one scan");
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  Frame f(m, st.params, st.pose, st.stamp, st.dt);
  f.g = gridArgs(m.grid);
  const PipelineParams& P = st.params;
  if (P.drift.enabled && n_ranks > 0 && drift_pairs != nullptr) {
    // Same arithmetic as k_drift_finalize (drift.cpp:44-55, integration.cpp:119-128).
    double total = 0.0;
    long long cnt = 0;
    for (int r = 0; r < n_ranks; ++r) {
      total += drift_pairs[2 * r];
      cnt += static_cast<long long>(drift_pairs[2 * r + 1]);
    }
    const int nvote = static_cast<int>(cnt);
    if (nvote >= P.drift.min_points) {
      const double mean = total / nvote;
      const double off = std::clamp(mean, -P.drift.max_offset_per_scan, P.drift.max_offset_per_scan);
      st.drift_offset = off;
      st.drift_clamped = off != mean;
      st.drift_n = nvote;
      if (off != 0.0) {
        k_apply_offset_value<<<streamGrid(f.ncell), kThreads, 0, f.s>>>(m.cur, f.ncell, off);
        ++f.launches;
      }
    }
  }
  const uint32_t M = static_cast<uint32_t>(n_records);
  if (M > 0 && M > m.cap) fail(Err::kUsage, "more fusion records than points in the frame");
  checkCuda(cudaMemsetAsync(m.count, 0, f.ncell * sizeof(int32_t), f.s), "memset");
  checkCuda(cudaMemsetAsync(m.start, 0xff, f.ncell * sizeof(uint32_t), f.s), "memset");
  if (M > 0) {
    const SortGeom sg = phaseSortGeometry(f, M);
    k_records_count<<<gridFor(M), kThreads, 0, f.s>>>(d_cells, M, m.count, sg.tc, sg.pitch,
                                                      sg.buckets() - 1, f.WH);
    ++f.launches;
    phaseSortFuse(f, d_cells, M, d_z, d_var, sg);
  } else {
    f.overlap = false;
  }
  phaseRaysPass1(f, static_cast<uint32_t>(st.n_local), st.ray_base);
  checkCuda(cudaGetLastError(), "kernel launch");
  checkCuda(cudaStreamSynchronize(f.s), "shard update");
  st.overlap = f.overlap;
  st.launches += f.launches;
  io.kstar = m.kstar;
  io.ub = m.cur.ub;
  io.ubv = m.cur.ubv;
  io.cells = f.ncell;
  st.stage = 2;
}

// Phase 3 (after k* / ub / ubv hold the all-reduced values): removal and ray
// pass 2 over this batch. Returns the cells removed (identical on every rank);
// when > 0, ub / ubv need another min / max all-reduce.
int64_t shardRemove(DeviceMap& m, ShardIO& io) {
  ShardState& st = m.shard;
  if (st.stage != 2) fail(Err::kUsage, "shard phases out of order (expected remove after update)");
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  Frame f(m, st.params, st.pose, st.stamp, st.dt);
  f.g = gridArgs(m.grid);
  f.explicit_remove = true;
  phaseRemovePass2(f, st.ray_base);
  unsigned long long removed = 0;
  checkCuda(cudaMemcpyAsync(&m.h_stats->removed, &m.stats->removed, sizeof(removed),
                            cudaMemcpyDeviceToHost, f.s),
            "stats");
  checkCuda(cudaGetLastError(), "kernel launch");
  checkCuda(cudaStreamSynchronize(f.s), "shard remove");
  removed = m.h_stats->removed;
  st.launches += f.launches;
  io.ub = m.cur.ub;
  io.ubv = m.cur.ubv;
  st.stage = 3;
  return static_cast<int64_t>(removed);
}

// Phase 4: cell phases (every rank, identical) and the frame's stats with the
// fate counters summed over the ranks.
ScanResult shardFinish(DeviceMap& m, const int64_t counters_total[3], uint64_t points_total) {
  ShardState& st = m.shard;
  if (st.stage != 3) fail(Err::kUsage, "shard phases out of order (expected finish after remove)");
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  Frame f(m, st.params, st.pose, st.stamp, st.dt);
  f.g = gridArgs(m.grid);
  phaseCells(f);
  const DevStats& d = phaseStats(f);
  ScanResult out = resultFrom(d, points_total);
  out.out_of_range = counters_total[0];
  out.excluded = counters_total[1];
  out.out_of_map = counters_total[2];
  out.drift_offset = st.drift_offset;
  out.drift_clamped = st.drift_clamped;
  out.drift_points = st.drift_n;
  m.last_launches = st.launches + f.launches;
  m.last_visits = static_cast<long long>(d.visits);
  m.last_stamp = st.stamp;
  m.has_last = true;
  st.stage = 0;
  return out;
}

// ------------------------------------------------------- group frames
// One frame split across the ranks of a group (exact variant;
// DESIGN.md §7). Rank r ingests the contiguous batch [lo, lo + n_local) of
// the frame into the frame-wide point arrays at the same indices; the batch
// size is a whole number of radix tiles, so after the in-place all-gathers of
// the cell keys, p_z, sigma_p^2 and the drift block partials every rank holds
// exactly the arrays a single-GPU frame would have built: the count, sort,
// gated fusion and drift offset that follow are the single-GPU kernels on the
// same inputs (bit-identical maps, drift included). The ray passes run over
// the rank's own rays with their frame-wide ids (the k* rule), and min / max
// all-reduces of k*, the bounds and their validity merge them.
GroupGeom groupGeom(uint64_t n_total, int ranks, int rank) {
  if (ranks <= 0 || rank < 0 || rank >= ranks) fail(Err::kUsage, "bad group rank / size");
  if (n_total >= 0x7fffffffULL) fail(Err::kUsage, "too many points in one scan");
  GroupGeom g;
  g.ranks = ranks;
  g.rank = rank;
  g.n_total = n_total;
  const uint64_t per = (n_total + ranks - 1) / ranks;
  g.chunk = static_cast<uint32_t>(std::max<uint64_t>((per + kTile - 1) / kTile, 1) * kTile);
  const uint64_t lo = std::min<uint64_t>(static_cast<uint64_t>(rank) * g.chunk, n_total);
  g.lo = static_cast<uint32_t>(lo);
  g.n_local = static_cast<uint32_t>(std::min<uint64_t>(lo + g.chunk, n_total) - lo);
  return g;
}

struct GroupFrame {
  PipelineParams P;
  GroupGeom geo;
  SortGeom sg;
  Frame f;
  bool info = false;       // information-form fusion
  uint32_t c0 = 0, wn = 0;  // info: the window of cells [c0, c0 + wn) the frame can touch
  GroupFrame(DeviceMap& m, const PipelineParams& params, const GroupGeom& g, const Pose& pose,
             double stamp, double dt)
      : P(params), geo(g), f(m, P, pose, stamp, dt) {}
};

GroupFrame* groupBegin(DeviceMap& m, const PipelineParams& P, const GroupGeom& g, const Pose& pose,
                       double stamp, double dt, bool info) {
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  if (m.shard.stage != 0) fail(Err::kUsage, "a sharded frame is in progress on this map");
  if (m.async_count != 0) fail(Err::kUsage, "streaming frames in flight: call relief_gpu_map_wait");
  if (info && !(P.update.mahalanobis_threshold >= 1e12 && P.update.wall_count_threshold >= (1 << 30)))
    fail(Err::kUsage,
         "information-form fusion needs gates that cannot fire (update.mahalanobis_threshold >= "
         "1e12, update.wall_count_threshold >= 2^30)");
  auto* gf = new GroupFrame(m, P, g, pose, stamp, dt);
  gf->info = info;
  return gf;
}

void groupEnd(GroupFrame* gf) { delete gf; }

// Recenter, this rank's batch through K1 (no counts: the gathered keys are
// counted in the update phase). Gathers: keys, p_z, sigma_p^2, drift partials.
void groupPhaseIngest(GroupFrame& gf, const double* xyz, bool on_device,
                      std::vector<XBuf>& gathers) {
  Frame& f = gf.f;
  DeviceMap& m = f.m;
  const GroupGeom& g = gf.geo;
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  checkCuda(cudaEventRecord(m.ev[0], f.s), "event");
  const double* d_xyz = xyz;
  if (g.n_total > 0) {
    phaseScratch(f, static_cast<std::size_t>(g.ranks) * g.chunk);
    if (g.n_local > 0 && !on_device) {
      checkCuda(cudaMemcpyAsync(m.xyz_in, xyz, g.n_local * 3 * sizeof(double),
                                cudaMemcpyHostToDevice, f.s),
                "point upload");
      d_xyz = m.xyz_in;
    } else if (g.n_local > 0) {
      cudaPointerAttributes pa{};
      if (cudaPointerGetAttributes(&pa, xyz) == cudaSuccess && pa.type == cudaMemoryTypeDevice &&
          pa.device != m.device) {  // a frame resident on another device of the process
        checkCuda(cudaMemcpyPeerAsync(m.xyz_in, m.device, xyz, pa.device,
                                      g.n_local * 3 * sizeof(double), f.s),
                  "point copy");
        d_xyz = m.xyz_in;
      }
      cudaGetLastError();
    }
  }
  checkCuda(cudaEventRecord(m.ev[13], f.s), "event");  // input resident
  phaseBegin(f, false);
  if (g.n_total == 0) return;
  gf.sg = phaseSortGeometry(f, static_cast<uint32_t>(g.n_total));
  RB_PHASE_EVENT(1, f.s);
  phaseIngest(f, d_xyz, g.n_local, gf.sg, false, false, g.lo);
  RB_PHASE_EVENT(2, f.s);
  if (!gf.info) {  // (information form: the points stay on their rank)
    gathers.push_back({m.key0, g.chunk, XType::kU32, XOp::kSum});
    gathers.push_back({m.pz, g.chunk, XType::kF64, XOp::kSum});
    gathers.push_back({m.pvar, g.chunk, XType::kF64, XOp::kSum});
  }
  if (gf.P.drift.enabled) {
    gathers.push_back({m.drift_sum_part, g.chunk / kThreads, XType::kF64, XOp::kSum});
    gathers.push_back({m.drift_n_part, g.chunk / kThreads, XType::kI32, XOp::kSum});
  }
}

void pushRayReduces(GroupFrame& gf, std::vector<XBuf>& reduces);

// Drift offset, counts + sort + gated fusion of the whole frame (every rank,
// identical), ray pass 1 over this rank's rays. Reduces: k*, bounds.
void groupPhaseUpdate(GroupFrame& gf, std::vector<XBuf>& reduces) {
  Frame& f = gf.f;
  DeviceMap& m = f.m;
  const GroupGeom& g = gf.geo;
  const PipelineParams& P = gf.P;
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  const uint32_t N = static_cast<uint32_t>(g.n_total);
  if (N == 0) return;
  if (P.drift.enabled) {  // the gathered partials are the single-GPU frame's
    launchPdl(k_drift_finalize, 1, 1024, 0, f.s, m.drift_sum_part, m.drift_n_part,
              static_cast<int>(gridFor(N)), P.drift.min_points, P.drift.max_offset_per_scan,
              m.drift_offset, m.stats);
    ++f.launches;
    f.fuse_offset = m.drift_offset;  // applied by k_fuse
  }
  RB_PHASE_EVENT(3, f.s);
  launchPdl(k_records_count, gridFor(N), kThreads, 0, f.s, m.key0, N, m.count, gf.sg.tc,
            gf.sg.pitch, gf.sg.buckets() - 1, f.WH);
  ++f.launches;
  phaseSortFuse(f, m.key0, N, m.pz, m.pvar, gf.sg);
  f.point_cells = gf.sg.passes <= 2 ? m.key0 + g.lo : nullptr;
  f.ray_at = g.lo;
  phaseRaysPass1(f, g.n_local, g.lo);
  pushRayReduces(gf, reduces);
}

// ------------------------------------------------ information-form frames
// Ungated fusion (update.mahalanobis_threshold >= 1e12 and
// wall_count_threshold >= 2^30: the reference's outlier and wall gates,
// integration.cpp:40-55, cannot fire) is the sequential Kalman fold
//   h_k = (v_k h_{k-1} + s_{k-1} p_k) / (s_{k-1} + v_k),  s_k = s_{k-1} v_k / (s_{k-1} + v_k)
// of each cell's points, which in exact arithmetic equals the information
// form 1/s_n = 1/s_0 + sum 1/v_k, h_n = s_n (h_0/s_0 + sum p_k/v_k), with
// (h_0, s_0) = (elevation, variance) of a valid cell and (p_first,
// sigma_init^2) of an invalid one (the first point initialises it,
// integration.cpp:148-155). So every rank sums its own batch's points per
// cell (in scan order, after a local sort), and the sums are all-reduced --
// 28 B per cell of the window the frame can reach instead of 20 B per point
// gathered and the whole frame sorted and folded on every rank. The first
// point of an invalid cell comes from the lowest rank holding points there:
// a MIN all-reduce of the rank, then that rank contributes its first point to
// a SUM. Results differ from the sequential fold by rounding only (tolerance
// 1e-9 relative in tests); the ray passes and cell phases are the exact
// mode's.
void pushRayReduces(GroupFrame& gf, std::vector<XBuf>& reduces) {
  DeviceMap& m = gf.f.m;
  if (gf.P.cleanup.cleanup_enabled)
    reduces.push_back({m.kstar - 1, gf.f.ncell + 1, XType::kI32, XOp::kMin});  // + the removal flag
  if (gf.P.cleanup.upper_bound_enabled) {
    reduces.push_back({m.cur.ub, gf.f.ncell, XType::kF64, XOp::kMin});
    reduces.push_back({m.cur.ubv, gf.f.ncell, XType::kU8, XOp::kMax});
  }
}

struct InfoBufs {
  double *a, *b, *pf, *pfl;
  int32_t *n, *first;
};

InfoBufs infoBufs(DeviceMap& m) {
  if (m.islab == nullptr) {
    const std::size_t n = m.grid.cells();
    const std::size_t a8 = (n * 8 + 255) / 256 * 256, a4 = (n * 4 + 255) / 256 * 256;
    checkCuda(cudaMalloc(&m.islab, 4 * a8 + 2 * a4), "information-form scratch");
    char* p = static_cast<char*>(m.islab);
    m.info_a = reinterpret_cast<double*>(p);
    m.info_b = reinterpret_cast<double*>(p + a8);
    m.info_pf = reinterpret_cast<double*>(p + 2 * a8);
    m.info_pfl = reinterpret_cast<double*>(p + 3 * a8);
    m.info_n = reinterpret_cast<int32_t*>(p + 4 * a8);
    m.info_first = reinterpret_cast<int32_t*>(p + 4 * a8 + a4);
  }
  return InfoBufs{m.info_a, m.info_b, m.info_pf, m.info_pfl, m.info_n, m.info_first};
}

// This rank's partials over the window: sums of p/v and 1/v of each cell's
// points in scan order, their number, the first point, this rank as the
// cell's first-rank candidate. (A non-positive sigma_p^2 is the reference's
// kInvalidVariance.)
__global__ void __launch_bounds__(kThreads)
    k_info_partials(uint32_t c0, uint32_t wn, const int32_t* __restrict__ count,
                    const uint32_t* __restrict__ start, const double* __restrict__ spz,
                    const double* __restrict__ spv, int rank, InfoBufs x, DevStats* st) {
  pdlEnter();
  const uint32_t j = blockIdx.x * kThreads + threadIdx.x;
  if (j >= wn) return;
  const uint32_t i = c0 + j;
  const int cnt = count[i];
  double sa = 0.0, sb = 0.0, pf = 0.0;
  bool bad = false;
  if (cnt > 0) {
    const double* zp = spz + start[i];
    const double* vp = spv + start[i];
    pf = zp[0];
    for (int k = 0; k < cnt; ++k) {
      const double z = zp[k], v = vp[k];
      if (v <= 0.0) bad = true;
      sa += z / v;
      sb += 1.0 / v;
    }
  }
  x.a[j] = sa;
  x.b[j] = sb;
  x.n[j] = cnt;
  x.first[j] = cnt > 0 ? rank : INT_MAX;
  x.pfl[j] = pf;
  if (bad) atomicExch(&st->error_code, 1);
}

// After the MIN of the first ranks: the first rank's first point, 0 elsewhere
// (summed next, so every rank gets it).
__global__ void __launch_bounds__(kThreads) k_info_first(uint32_t wn, int rank, InfoBufs x) {
  pdlEnter();
  const uint32_t j = blockIdx.x * kThreads + threadIdx.x;
  if (j < wn) x.pf[j] = x.first[j] == rank ? x.pfl[j] : 0.0;
}

// The merged partials folded into the map (every rank, identical): the
// information-form update and setEstimate (grid.cpp:139-147) for every cell
// with points; the scan's per-cell point count for the cell phases.
__global__ void __launch_bounds__(kThreads)
    k_info_apply(uint32_t c0, uint32_t wn, Layers L, int32_t* __restrict__ count, InfoBufs x,
                 double now, double sigma_init2, DevStats* st) {
  pdlEnter();
  const uint32_t j = blockIdx.x * kThreads + threadIdx.x;
  FoldCounts k;
  if (j < wn) {
    const uint32_t i = c0 + j;
    const int n = x.n[j];
    count[i] = n;
    if (n > 0) {
      const bool valid = L.valid[i] != 0;
      const double s0 = valid ? L.var[i] : sigma_init2;
      const double h0 = valid ? L.elev[i] : x.pf[j];
      if (s0 <= 0.0) {
        atomicExch(&st->error_code, 1);
      } else {
        const double v = 1.0 / (1.0 / s0 + x.b[j]);
        const double h = (h0 / s0 + x.a[j]) * v;
        L.elev[i] = h;
        L.var[i] = v;
        L.last[i] = now;
        L.valid[i] = 1;
        L.ub[i] = h;
        L.ubv[i] = 1;
        k.nf = static_cast<unsigned long long>(n);
        k.upd = 1;
      }
    }
  }
  flushCounts(k, st);
}

// Rows of the map the frame's in-map points can reach: within max_range of
// the sensor (|R p| <= |p| (1 + 1e-6) for a pose that passed the
// orthonormality check), with a two-row margin. The same on every rank.
void infoWindow(GroupFrame& gf) {
  const Frame& f = gf.f;
  const double reach = gf.P.update.max_range * (1.0 + 1e-6) + 2.0 * f.g.res;
  int r0 = 0, r1 = f.g.H - 1;
  if (std::isfinite(reach)) {
    const double lo = std::floor((f.pose.t[1] - reach - f.g.oy) / f.g.res) - 2.0;
    const double hi = std::floor((f.pose.t[1] + reach - f.g.oy) / f.g.res) + 2.0;
    r0 = static_cast<int>(std::max(0.0, std::min(lo, static_cast<double>(f.g.H - 1))));
    r1 = static_cast<int>(std::max(0.0, std::min(hi, static_cast<double>(f.g.H - 1))));
  }
  if (!std::isfinite(f.pose.t[1])) {
    r0 = 0;
    r1 = f.g.H - 1;
  }
  gf.c0 = static_cast<uint32_t>(r0) * static_cast<uint32_t>(f.g.W);
  gf.wn = static_cast<uint32_t>(r1 - r0 + 1) * static_cast<uint32_t>(f.g.W);
}

// Drift offset (the gathered votes, as the exact mode), this rank's batch
// counted and sorted locally, its partials. Reduces: the first ranks.
void groupPhaseInfoPartials(GroupFrame& gf, std::vector<XBuf>& reduces) {
  Frame& f = gf.f;
  DeviceMap& m = f.m;
  const GroupGeom& g = gf.geo;
  const PipelineParams& P = gf.P;
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  if (g.n_total == 0) return;
  if (P.drift.enabled) {
    launchPdl(k_drift_finalize, 1, 1024, 0, f.s, m.drift_sum_part, m.drift_n_part,
              static_cast<int>(gridFor(static_cast<uint32_t>(g.n_total))), P.drift.min_points,
              P.drift.max_offset_per_scan, m.drift_offset, m.stats);
    launchPdl(k_apply_offset, streamGrid(f.ncell), kThreads, 0, f.s, m.cur, f.ncell,
              static_cast<const double*>(m.drift_offset));
    f.launches += 2;
  }
  RB_PHASE_EVENT(3, f.s);
  const uint32_t n = g.n_local;
  if (n > 0) {
    gf.sg = phaseSortGeometry(f, n);
    launchPdl(k_records_count, gridFor(n), kThreads, 0, f.s, m.key0 + g.lo, n, m.count, gf.sg.tc,
              gf.sg.pitch, gf.sg.buckets() - 1, f.WH);
    ++f.launches;
    phaseSort(f, m.key0 + g.lo, n, m.pz + g.lo, m.pvar + g.lo, gf.sg);
  }
  RB_PHASE_EVENT(4, f.s);
  infoWindow(gf);
  const InfoBufs x = infoBufs(m);
  launchPdl(k_info_partials, (gf.wn + kThreads - 1) / kThreads, kThreads, 0, f.s, gf.c0, gf.wn,
            static_cast<const int32_t*>(m.count), static_cast<const uint32_t*>(m.start),
            static_cast<const double*>(m.spz), static_cast<const double*>(m.spv), g.rank, x,
            m.stats);
  ++f.launches;
  reduces.push_back({x.first, gf.wn, XType::kI32, XOp::kMin});
}

// Reduces: the partials and the first points.
void groupPhaseInfoFirst(GroupFrame& gf, std::vector<XBuf>& reduces) {
  Frame& f = gf.f;
  DeviceMap& m = f.m;
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  if (gf.geo.n_total == 0) return;
  const InfoBufs x = infoBufs(m);
  launchPdl(k_info_first, (gf.wn + kThreads - 1) / kThreads, kThreads, 0, f.s, gf.wn, gf.geo.rank, x);
  ++f.launches;
  reduces.push_back({x.a, gf.wn, XType::kF64, XOp::kSum});
  reduces.push_back({x.b, gf.wn, XType::kF64, XOp::kSum});
  reduces.push_back({x.pf, gf.wn, XType::kF64, XOp::kSum});
  reduces.push_back({x.n, gf.wn, XType::kI32, XOp::kSum});
}

// The merged fold, then ray pass 1 over this rank's rays. Reduces: k*,
// bounds (as groupPhaseUpdate).
void groupPhaseInfoApply(GroupFrame& gf, std::vector<XBuf>& reduces) {
  Frame& f = gf.f;
  DeviceMap& m = f.m;
  const GroupGeom& g = gf.geo;
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  if (g.n_total == 0) return;
  const InfoBufs x = infoBufs(m);
  launchPdl(k_info_apply, (gf.wn + kThreads - 1) / kThreads, kThreads, 0, f.s, gf.c0, gf.wn, m.cur,
            m.count, x, f.stamp, gf.P.update.sigma_init2, m.stats);
  ++f.launches;
  RB_PHASE_EVENT(5, f.s);
  f.overlap = false;
  f.heavy = INT_MAX;
  f.point_cells = (g.n_local > 0 && gf.sg.passes <= 2) ? m.key0 + g.lo : nullptr;
  f.ray_at = g.lo;
  phaseRaysPass1(f, g.n_local, g.lo);
  pushRayReduces(gf, reduces);
}

// Removal (identical on every rank: k* is merged) and ray pass 2 over this
// rank's queued rays. Reduces: bounds of the removed cells.
void groupPhaseRemove(GroupFrame& gf, std::vector<XBuf>& reduces) {
  Frame& f = gf.f;
  DeviceMap& m = f.m;
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  if (gf.geo.n_total == 0) return;
  phaseRemovePass2(f, gf.geo.lo);
  if (gf.P.cleanup.cleanup_enabled && gf.P.cleanup.upper_bound_enabled)
    reduces.push_back({m.ub2, f.ncell, XType::kF64, XOp::kMin});  // bounds of removed cells
  RB_PHASE_EVENT(6, f.s);
}

// Cell phases (identical on every rank). Reduces: the batch fate counters.
void groupPhaseCells(GroupFrame& gf, std::vector<XBuf>& reduces) {
  Frame& f = gf.f;
  DeviceMap& m = f.m;
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  if (gf.geo.n_total == 0)
    for (int k = 1; k <= 6; ++k) RB_PHASE_EVENT(k, f.s);
  phaseCells(f);
  // out_of_range, excluded, out_of_map: the first three DevStats counters
  static_assert(offsetof(DevStats, excluded) == 8 && offsetof(DevStats, out_of_map) == 16,
                "fate counters must be contiguous");
  reduces.push_back({&m.stats->out_of_range, 3, XType::kU64, XOp::kSum});
}

ScanResult groupFinish(GroupFrame& gf) {
  Frame& f = gf.f;
  DeviceMap& m = f.m;
  checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
  checkCuda(cudaEventRecord(m.ev[12], f.s), "event");  // device end incl. the exchanges
  const DevStats& d = phaseStats(f);
  ScanResult out = resultFrom(d, gf.geo.n_total);
  m.timing_pending = true;
  m.timing_chunked = false;
  m.timing_phases = m.phase_events;
  m.last_launches = f.launches;
  m.last_visits = static_cast<long long>(d.visits);
  return out;
}

}  // namespace rb200
