// Device map lifecycle: allocation, fresh fill, layer export, snapshot
// upload/download.
#include <cmath>
#include <cstring>
#include <string>

#include "device_map.hpp"

namespace rb200 {

void checkCuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(Err::kDevice, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

GridArgs gridArgs(const Grid& g) {
  GridArgs a;
  a.W = g.width;
  a.H = g.height;
  a.res = g.resolution;
  a.ox = g.originX();
  a.oy = g.originY();
  a.xmax = a.ox + g.width * g.resolution;
  a.ymax = a.oy + g.height * g.resolution;
  return a;
}

namespace {

constexpr std::size_t kAlign = 256;
inline std::size_t alignUp(std::size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

// Carves typed arrays out of one allocation.
struct Carver {
  char* base;
  std::size_t off = 0;
  template <typename T>
  T* take(std::size_t n) {
    T* p = reinterpret_cast<T*>(base + off);
    off = alignUp(off + n * sizeof(T));
    return p;
  }
};

std::size_t layerBytes(std::size_t n) { return 8 * alignUp(n * 8) + 2 * alignUp(n); }

void carveLayers(Carver& c, Layers& L, std::size_t n) {
  L.elev = c.take<double>(n);
  L.var = c.take<double>(n);
  L.last = c.take<double>(n);
  L.ub = c.take<double>(n);
  L.trav = c.take<double>(n);
  L.nx = c.take<double>(n);
  L.ny = c.take<double>(n);
  L.nz = c.take<double>(n);
  L.valid = c.take<uint8_t>(n);
  L.ubv = c.take<uint8_t>(n);
}

// Probe words of the padded grid and its guard rows: the border is 0xffff
// (tag 3, "outside the grid", F = NaN) for good; the interior is rewritten by
// every frame's classification.
__global__ void k_probe_border(uint16_t* probe, std::size_t n) {
  const std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x;
  if (i < n) probe[i] = 0xffffu;
}

__global__ void k_fill_fresh(Layers L, std::size_t n, int32_t* kstar, double* ub2) {
  const std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  L.elev[i] = nan;
  L.var[i] = nan;
  L.last[i] = 0.0;
  L.ub[i] = __longlong_as_double(0x7ff0000000000000LL);
  L.trav[i] = 0.0;
  L.nx[i] = 0.0;
  L.ny[i] = 0.0;
  L.nz[i] = 0.0;
  L.valid[i] = 0;
  L.ubv[i] = 0;
  kstar[i] = INT_MAX;
  if (i == 0) kstar[-1] = INT_MAX;
  ub2[i] = __longlong_as_double(0x7ff0000000000000LL);
}

// Layer ids for the masked export; order = reference snapshot.cpp:43-48.
enum LayerId { kElev, kVar, kLast, kUb, kUbv, kTrav, kNx, kNy, kNz, kValid };

__global__ void k_export(Layers L, std::size_t n, int which, double* out) {
  const std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  const bool v = L.valid[i] != 0;
  double r;
  switch (which) {
    case kElev: r = v ? L.elev[i] : nan; break;
    case kVar: r = v ? L.var[i] : nan; break;
    case kLast: r = v ? L.last[i] : nan; break;
    case kUb: r = L.ubv[i] ? L.ub[i] : nan; break;
    case kUbv: r = L.ubv[i] ? 1.0 : 0.0; break;
    case kTrav: r = v ? L.trav[i] : nan; break;
    case kNx: r = v ? L.nx[i] : nan; break;
    case kNy: r = v ? L.ny[i] : nan; break;
    case kNz: r = v ? L.nz[i] : nan; break;
    default: r = v ? 1.0 : 0.0; break;
  }
  out[i] = r;
}

int layerId(const char* name) {
  static const char* names[] = {"elevation",      "variance", "last_update", "upper_bound",
                                "upper_bound_valid", "traversability", "normal_x", "normal_y",
                                "normal_z",       "valid"};
  for (int k = 0; k < 10; ++k)
    if (std::strcmp(name, names[k]) == 0) return k;
  return -1;
}

}  // namespace

DeviceMap* createDeviceMap(int device, const Grid& grid) {
  grid.validate();
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    fail(Err::kDevice, "no CUDA device available: librelief_b200 has no CPU fallback");
  }
  if (device < 0 || device >= count) fail(Err::kUsage, "CUDA device ordinal out of range");
  checkCuda(cudaSetDevice(device), "cudaSetDevice");
  preloadFrameKernels(device);
  auto* m = new DeviceMap();
  m->device = device;
  m->grid = grid;
  try {
    // (RB_STREAM2_PRIO: the long-cell fold's stream at the highest priority, so
    // its blocks take SM slots as the ray pass's retire; RB_MAIN_PRIO: the
    // frame stream at the highest priority)
    int prio_lo = 0, prio_hi = 0;
    checkCuda(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi), "stream priorities");
#ifndef RB_MAIN_PRIO
#define RB_MAIN_PRIO 0
#endif
    checkCuda(cudaStreamCreateWithPriority(&m->stream, cudaStreamNonBlocking, RB_MAIN_PRIO ? prio_hi : prio_lo),
              "stream create");
#ifndef RB_STREAM2_PRIO
#define RB_STREAM2_PRIO 0  // measured slower
#endif
    checkCuda(cudaStreamCreateWithPriority(&m->stream2, cudaStreamNonBlocking,
                                           RB_STREAM2_PRIO ? prio_hi : prio_lo),
              "stream create");
    for (auto& e : m->ev) checkCuda(cudaEventCreate(&e), "event create");
    checkCuda(cudaEventCreateWithFlags(&m->ev_after, cudaEventDisableTiming), "event create");
    checkCuda(cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming), "event create");
    checkCuda(cudaEventCreateWithFlags(&m->ev_dfork, cudaEventDisableTiming), "event create");
    checkCuda(cudaEventCreateWithFlags(&m->ev_djoin, cudaEventDisableTiming), "event create");
    checkCuda(cudaEventCreateWithFlags(&m->ev_sfork, cudaEventDisableTiming), "event create");
    checkCuda(cudaEventCreateWithFlags(&m->ev_sjoin, cudaEventDisableTiming), "event create");
    checkCuda(cudaStreamCreateWithFlags(&m->stream3, cudaStreamNonBlocking), "stream create");
    checkCuda(cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking), "stream create");
    for (auto& e : m->ev_chunk)
      checkCuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
    for (int k = 0; k < DeviceMap::kSlots; ++k) {
      checkCuda(cudaEventCreate(&m->ev_copied[k]), "event create");
      checkCuda(cudaEventCreateWithFlags(&m->ev_consumed[k], cudaEventDisableTiming), "event create");
      checkCuda(cudaEventCreate(&m->ev_done[k]), "event create");
      checkCuda(cudaEventCreate(&m->ev_copy0[k]), "event create");
      checkCuda(cudaEventCreate(&m->ev_start[k]), "event create");
      checkCuda(cudaMallocHost(&m->h_slot[k], sizeof(DevStats)), "pinned stats");
    }
    const std::size_t n = grid.cells();
    const std::size_t guard = static_cast<std::size_t>(DeviceMap::kProbeGuardRows) * (grid.width + 2);
    const std::size_t np = static_cast<std::size_t>(grid.width + 2) * (grid.height + 2) + 2 * guard;
    const std::size_t bytes = 2 * layerBytes(n) + 6 * alignUp(n * 4) + alignUp(np * 2) +
                              alignUp((n + 1) * 4) + alignUp(n) + alignUp(n * 8) + 8 * kAlign;
    checkCuda(cudaMalloc(&m->slab, bytes), "map allocation");
    Carver c{static_cast<char*>(m->slab)};
    carveLayers(c, m->cur, n);
    carveLayers(c, m->alt, n);
    m->count = c.take<int32_t>(n);
    m->kstar = c.take<int32_t>(n + 32) + 32;  // kstar[-1]: the frame's "any removal" flag
    m->heavy = c.take<uint32_t>(4 * n);
    m->start = c.take<uint32_t>(n + 1);
    m->cls = c.take<uint8_t>(n);
    m->probe = c.take<uint16_t>(np) + guard;
    m->ub2 = c.take<double>(n);
    m->jw = (grid.width + 7) / 8;  // sized for the smallest jump block (pipeline.cu kJumpBlk)
    m->jh = (grid.height + 7) / 8;
    checkCuda(cudaMalloc(&m->jgrid, static_cast<std::size_t>(m->jw) * m->jh * sizeof(float)), "jump grid");
    checkCuda(cudaMalloc(&m->stats, sizeof(DevStats)), "stats allocation");
    checkCuda(cudaMalloc(&m->drift_offset, sizeof(double)), "offset allocation");
    checkCuda(cudaMallocHost(&m->h_stats, sizeof(DevStats)), "pinned stats");
    checkCuda(cudaMallocHost(&m->h_seq, sizeof(unsigned long long)), "pinned stats");
    *m->h_seq = 0;
    fillFresh(*m);
    k_probe_border<<<static_cast<unsigned>((np + 255) / 256), 256, 0, m->stream>>>(m->probe - guard,
                                                                                  np);
    checkCuda(cudaGetLastError(), "probe init");
    checkCuda(cudaMemsetAsync(m->count, 0, n * sizeof(int32_t), m->stream), "map init");
    checkCuda(cudaMemsetAsync(m->start, 0xff, (n + 1) * sizeof(uint32_t), m->stream), "map init");
    checkCuda(cudaStreamSynchronize(m->stream), "map init");
  } catch (...) {
    destroyDeviceMap(m);
    throw;
  }
  return m;
}

void destroyDeviceMap(DeviceMap* m) {
  if (m == nullptr) return;
  cudaSetDevice(m->device);
  if (m->stream) cudaStreamSynchronize(m->stream);
  cudaFree(m->slab);
  cudaFree(m->jgrid);
  cudaFree(m->islab);
  cudaFree(m->pslab);
  cudaFree(m->rslab);
  cudaFree(m->export_buf);
  m->chain.release();
  m->conv.release();
  cudaFree(m->chain_in);
  cudaFree(m->chain_out);
  cudaFree(m->chain_out_ok);
  cudaFree(m->hist);
  cudaFree(m->stats);
  cudaFree(m->drift_offset);
  if (m->h_stats) cudaFreeHost(m->h_stats);
  if (m->h_seq) cudaFreeHost(m->h_seq);
  for (int k = 0; k < DeviceMap::kSlots; ++k) {
    if (m->h_slot[k]) cudaFreeHost(m->h_slot[k]);
    if (m->ev_copied[k]) cudaEventDestroy(m->ev_copied[k]);
    if (m->ev_consumed[k]) cudaEventDestroy(m->ev_consumed[k]);
    if (m->ev_done[k]) cudaEventDestroy(m->ev_done[k]);
    if (m->ev_copy0[k]) cudaEventDestroy(m->ev_copy0[k]);
    if (m->ev_start[k]) cudaEventDestroy(m->ev_start[k]);
  }
  if (m->copy_stream) {
    cudaStreamSynchronize(m->copy_stream);
    cudaStreamDestroy(m->copy_stream);
  }
  for (auto& e : m->ev)
    if (e) cudaEventDestroy(e);
  if (m->ev_after) cudaEventDestroy(m->ev_after);
  if (m->ev_fork) cudaEventDestroy(m->ev_fork);
  if (m->ev_dfork) cudaEventDestroy(m->ev_dfork);
  if (m->ev_djoin) cudaEventDestroy(m->ev_djoin);
  if (m->ev_sfork) cudaEventDestroy(m->ev_sfork);
  if (m->ev_sjoin) cudaEventDestroy(m->ev_sjoin);
  if (m->stream3) cudaStreamDestroy(m->stream3);
  for (int k = 0; k < m->graph_count; ++k) cudaGraphExecDestroy(m->graphs[k]);
  for (auto& e : m->ev_chunk)
    if (e) cudaEventDestroy(e);
  if (m->stream) cudaStreamDestroy(m->stream);
  if (m->stream2) cudaStreamDestroy(m->stream2);
  delete m;
}

void fillFresh(DeviceMap& m) {
  const std::size_t n = m.grid.cells();
  k_fill_fresh<<<static_cast<unsigned>((n + 255) / 256), 256, 0, m.stream>>>(m.cur, n, m.kstar, m.ub2);
  checkCuda(cudaGetLastError(), "fill launch");
}

void ensurePointCapacity(DeviceMap& m, std::size_t n) {
  if (n <= m.cap && m.pslab != nullptr) return;
  std::size_t cap = 1 << 16;
  while (cap < n) cap <<= 1;
  cudaFree(m.pslab);
  m.pslab = nullptr;
  const std::size_t bytes = DeviceMap::kSlots * alignUp(cap * 24) + 8 * alignUp(cap * 8) +
                            6 * alignUp(cap * 4) + alignUp(cap) + 16 * kAlign;
  checkCuda(cudaMalloc(&m.pslab, bytes), "point scratch allocation");
  Carver c{static_cast<char*>(m.pslab)};
  for (int k = 0; k < DeviceMap::kSlots; ++k) m.xyz_slot[k] = c.take<double>(cap * 3);
  m.xyz_in = m.xyz_slot[0];
  m.px = c.take<double>(cap);
  m.py = c.take<double>(cap);
  m.pz = c.take<double>(cap);
  m.pvar = c.take<double>(cap);
  m.spz = c.take<double>(cap);
  m.spv = c.take<double>(cap);
  m.key0 = c.take<uint32_t>(cap);
  m.key1 = c.take<uint32_t>(cap);
  m.val0 = c.take<uint32_t>(cap);
  m.val1 = c.take<uint32_t>(cap);
  m.raylist = c.take<uint32_t>(cap);
  m.kept = c.take<uint8_t>(cap);
  m.rec_cell = c.take<uint32_t>(cap);
  m.rec_z = c.take<double>(cap);
  m.rec_var = c.take<double>(cap);
  m.cap = cap;
}

bool exportLayerDevice(DeviceMap& m, const char* name, double* d_out) {
  const int id = layerId(name);
  if (id < 0) return false;
  const std::size_t n = m.grid.cells();
  k_export<<<static_cast<unsigned>((n + 255) / 256), 256, 0, m.stream>>>(m.cur, n, id, d_out);
  checkCuda(cudaGetLastError(), "export launch");
  return true;
}

void uploadLayers(DeviceMap& m, const double* const host[8], const uint8_t* valid,
                  const uint8_t* ubv) {
  const std::size_t n = m.grid.cells();
  double* dst[8] = {m.cur.elev, m.cur.var, m.cur.last, m.cur.ub,
                    m.cur.trav, m.cur.nx,  m.cur.ny,   m.cur.nz};
  for (int k = 0; k < 8; ++k)
    checkCuda(cudaMemcpyAsync(dst[k], host[k], n * 8, cudaMemcpyHostToDevice, m.stream), "upload");
  checkCuda(cudaMemcpyAsync(m.cur.valid, valid, n, cudaMemcpyHostToDevice, m.stream), "upload");
  checkCuda(cudaMemcpyAsync(m.cur.ubv, ubv, n, cudaMemcpyHostToDevice, m.stream), "upload");
  checkCuda(cudaStreamSynchronize(m.stream), "upload sync");
  m.scrub_invalid = true;
}

void downloadLayers(const DeviceMap& m, double* const host[8], uint8_t* valid, uint8_t* ubv) {
  const std::size_t n = m.grid.cells();
  const double* src[8] = {m.cur.elev, m.cur.var, m.cur.last, m.cur.ub,
                          m.cur.trav, m.cur.nx,  m.cur.ny,   m.cur.nz};
  for (int k = 0; k < 8; ++k)
    checkCuda(cudaMemcpyAsync(host[k], src[k], n * 8, cudaMemcpyDeviceToHost, m.stream), "download");
  checkCuda(cudaMemcpyAsync(valid, m.cur.valid, n, cudaMemcpyDeviceToHost, m.stream), "download");
  checkCuda(cudaMemcpyAsync(ubv, m.cur.ubv, n, cudaMemcpyDeviceToHost, m.stream), "download");
  checkCuda(cudaStreamSynchronize(m.stream), "download sync");
}

}  // namespace rb200
