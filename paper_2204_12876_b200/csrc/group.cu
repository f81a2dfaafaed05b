// Group frames: one frame split across GPUs (exact and
// information-form variants), and the transports that run its
// exchanges.
//
// The frame's phases live in pipeline.cu (groupPhase*): each enqueues its
// kernels on the map's stream and names the buffers to exchange next. Two
// transports run those exchanges on the same stream, so every exchange is
// ordered after the kernels that produced its input and before the kernels
// that consume it -- no host synchronisation inside the frame:
//  * NcclTransport: one process per GPU; in-place ncclAllGather and
//    ncclAllReduce over NVLink / NVSwitch. NCCL is loaded with dlopen: a
//    process that already loaded it (PyTorch does) shares that copy, a plain
//    C/C++ embedder gets the system libnccl.so.2.
//  * LocalTransport: one process drives every rank (several GPUs, or several
//    replicas of the map on one GPU for tests): peer copies for the gathers,
//    a reduction kernel on rank 0 for the reduces, events for the ordering.
// Reference being split: the scan-order fusion loop (integration.cpp:142-203)
// and the per-point ray loop (integration.cpp:205-224, ray id = index, :212).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "device_map.hpp"

namespace rb200 {

std::size_t xtypeSize(XType t) {
  switch (t) {
    case XType::kU8: return 1;
    case XType::kI32:
    case XType::kU32: return 4;
    case XType::kU64:
    case XType::kF64: return 8;
  }
  return 1;
}

namespace {

// ------------------------------------------------------------------- NCCL
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  ncclResult_t (*getVersion)(int*) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::string error;
  static bool loaded = false;
  if (!loaded) {
    // RTLD_NOLOAD first: reuse a copy the process already has (PyTorch's).
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (h == nullptr) fail(Err::kDevice, std::string("cannot load NCCL: ") + dlerror());
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (p == nullptr) fail(Err::kDevice, std::string("NCCL symbol missing: ") + name);
      return p;
    };
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(sym("ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(sym("ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(sym("ncclCommDestroy"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(sym("ncclAllGather"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(sym("ncclAllReduce"));
    api.groupStart = reinterpret_cast<decltype(api.groupStart)>(sym("ncclGroupStart"));
    api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(sym("ncclGroupEnd"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(sym("ncclGetErrorString"));
    api.getVersion = reinterpret_cast<decltype(api.getVersion)>(sym("ncclGetVersion"));
    loaded = true;
  }
  return api;
}

void ncclCheck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(Err::kDevice, std::string("NCCL error in ") + what + ": " + nccl().errorString(r));
}

ncclDataType_t ncclType(XType t) {
  switch (t) {
    case XType::kU8: return ncclUint8;
    case XType::kI32: return ncclInt32;
    case XType::kU32: return ncclUint32;
    case XType::kU64: return ncclUint64;
    case XType::kF64: return ncclFloat64;
  }
  return ncclUint8;
}

ncclRedOp_t ncclOp(XOp o) {
  switch (o) {
    case XOp::kSum: return ncclSum;
    case XOp::kMin: return ncclMin;
    case XOp::kMax: return ncclMax;
  }
  return ncclSum;
}

// --------------------------------------------------------- local reduction
// dst[i] = op over the G sources (rank order), for the in-process transport.
// f64 min keeps the first of equal values; ranks never disagree on a NaN
// bound, so the NaN handling is that of any order.
constexpr int kMaxLocalRanks = 16;
struct SrcPtrs {
  const void* p[kMaxLocalRanks];
};

template <typename T, int OP>
__global__ void k_reduce_ranks(T* dst, SrcPtrs src, int ranks, std::size_t n) {
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
    T acc = static_cast<const T*>(src.p[0])[i];
    for (int r = 1; r < ranks; ++r) {
      const T v = static_cast<const T*>(src.p[r])[i];
      if (OP == 0) acc = acc + v;
      else if (OP == 1) acc = v < acc ? v : acc;
      else acc = acc < v ? v : acc;
    }
    dst[i] = acc;
  }
}

template <typename T>
void launchReduce(XOp op, void* dst, const SrcPtrs& src, int ranks, std::size_t n, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(std::min<std::size_t>((n + 255) / 256, 148 * 8));
  if (grid == 0) return;
  T* d = static_cast<T*>(dst);
  if (op == XOp::kSum) k_reduce_ranks<T, 0><<<grid, 256, 0, s>>>(d, src, ranks, n);
  else if (op == XOp::kMin) k_reduce_ranks<T, 1><<<grid, 256, 0, s>>>(d, src, ranks, n);
  else k_reduce_ranks<T, 2><<<grid, 256, 0, s>>>(d, src, ranks, n);
  checkCuda(cudaGetLastError(), "reduce launch");
}

void reduceRanks(const XBuf& b, void* dst, const SrcPtrs& src, int ranks, cudaStream_t s) {
  switch (b.type) {
    case XType::kU8: launchReduce<uint8_t>(b.op, dst, src, ranks, b.count, s); break;
    case XType::kI32: launchReduce<int32_t>(b.op, dst, src, ranks, b.count, s); break;
    case XType::kU32: launchReduce<uint32_t>(b.op, dst, src, ranks, b.count, s); break;
    case XType::kU64: launchReduce<unsigned long long>(b.op, dst, src, ranks, b.count, s); break;
    case XType::kF64: launchReduce<double>(b.op, dst, src, ranks, b.count, s); break;
  }
}

}  // namespace

// ------------------------------------------------------------ transports
struct Transport {
  virtual ~Transport() = default;
  virtual int ranks() const = 0;
};

struct NcclTransport : Transport {
  DeviceMap* map = nullptr;
  ncclComm_t comm = nullptr;
  int n = 1, me = 0;
  int ranks() const override { return n; }
  void gather(const std::vector<XBuf>& bufs) {
    if (bufs.empty()) return;
    const NcclApi& api = nccl();
    ncclCheck(api.groupStart(), "group start");
    for (const XBuf& b : bufs) {
      char* base = static_cast<char*>(b.ptr);
      ncclCheck(api.allGather(base + static_cast<std::size_t>(me) * b.count * xtypeSize(b.type),
                              base, b.count, ncclType(b.type), comm, map->stream),
                "all-gather");
    }
    ncclCheck(api.groupEnd(), "group end");
  }
  void reduce(const std::vector<XBuf>& bufs) {
    if (bufs.empty()) return;
    const NcclApi& api = nccl();
    ncclCheck(api.groupStart(), "group start");
    for (const XBuf& b : bufs)
      ncclCheck(api.allReduce(b.ptr, b.ptr, b.count, ncclType(b.type), ncclOp(b.op), comm,
                              map->stream),
                "all-reduce");
    ncclCheck(api.groupEnd(), "group end");
  }
  ~NcclTransport() override {
    if (comm) nccl().commDestroy(comm);
  }
};

// Every rank's map in this process. Each exchange: every rank's stream records
// "ready" after its phase; the copies / reduction wait for the sources' ready
// events; then every stream waits for every rank's "consumed" event before it
// continues (no rank overwrites a buffer another rank still reads).
struct LocalTransport : Transport {
  std::vector<DeviceMap*> maps;
  std::vector<cudaEvent_t> ready, done;
  void* staging = nullptr;  // rank 0's device: the other ranks' copies for a reduce
  std::size_t staging_bytes = 0;
  int ranks() const override { return static_cast<int>(maps.size()); }

  void init(std::vector<DeviceMap*> ms) {
    maps = std::move(ms);
    for (DeviceMap* m : maps) {
      checkCuda(cudaSetDevice(m->device), "cudaSetDevice");
      cudaEvent_t a, b;
      checkCuda(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "event create");
      checkCuda(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "event create");
      ready.push_back(a);
      done.push_back(b);
    }
  }
  ~LocalTransport() override {
    for (std::size_t r = 0; r < maps.size(); ++r) {
      cudaSetDevice(maps[r]->device);
      cudaStreamSynchronize(maps[r]->stream);
      cudaEventDestroy(ready[r]);
      cudaEventDestroy(done[r]);
    }
    if (staging) {
      cudaSetDevice(maps[0]->device);
      cudaFree(staging);
    }
  }
  void markReady() {
    for (std::size_t r = 0; r < maps.size(); ++r) {
      checkCuda(cudaSetDevice(maps[r]->device), "cudaSetDevice");
      checkCuda(cudaEventRecord(ready[r], maps[r]->stream), "event");
    }
  }
  void barrier() {
    for (std::size_t r = 0; r < maps.size(); ++r) {
      checkCuda(cudaSetDevice(maps[r]->device), "cudaSetDevice");
      checkCuda(cudaEventRecord(done[r], maps[r]->stream), "event");
    }
    for (std::size_t r = 0; r < maps.size(); ++r) {
      checkCuda(cudaSetDevice(maps[r]->device), "cudaSetDevice");
      for (std::size_t q = 0; q < maps.size(); ++q)
        if (q != r) checkCuda(cudaStreamWaitEvent(maps[r]->stream, done[q], 0), "stream wait");
    }
  }
  // bufs[r]: rank r's list (same shapes on every rank, own pointers).
  void gather(const std::vector<std::vector<XBuf>>& bufs) {
    if (bufs[0].empty() || maps.size() == 1) return;
    markReady();
    const int G = ranks();
    for (int r = 0; r < G; ++r) {
      DeviceMap& m = *maps[r];
      checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
      for (int q = 0; q < G; ++q)
        if (q != r) checkCuda(cudaStreamWaitEvent(m.stream, ready[q], 0), "stream wait");
      for (std::size_t k = 0; k < bufs[r].size(); ++k) {
        const std::size_t part = bufs[r][k].count * xtypeSize(bufs[r][k].type);
        for (int q = 0; q < G; ++q) {
          if (q == r || part == 0) continue;
          char* dst = static_cast<char*>(bufs[r][k].ptr) + static_cast<std::size_t>(q) * part;
          const char* src = static_cast<const char*>(bufs[q][k].ptr) + static_cast<std::size_t>(q) * part;
          checkCuda(cudaMemcpyPeerAsync(dst, m.device, src, maps[q]->device, part, m.stream),
                    "gather copy");
        }
      }
    }
    barrier();
  }
  void reduce(const std::vector<std::vector<XBuf>>& bufs) {
    if (bufs[0].empty() || maps.size() == 1) return;
    const int G = ranks();
    if (G > kMaxLocalRanks) fail(Err::kUsage, "too many ranks in one process");
    std::size_t need = 0;
    for (const XBuf& b : bufs[0]) need += (b.count * xtypeSize(b.type) + 255) / 256 * 256;
    need *= static_cast<std::size_t>(G - 1);
    DeviceMap& m0 = *maps[0];
    checkCuda(cudaSetDevice(m0.device), "cudaSetDevice");
    if (need > staging_bytes) {
      checkCuda(cudaStreamSynchronize(m0.stream), "stream sync");
      cudaFree(staging);
      staging = nullptr;
      checkCuda(cudaMalloc(&staging, need), "exchange staging");
      staging_bytes = need;
    }
    markReady();
    checkCuda(cudaSetDevice(m0.device), "cudaSetDevice");
    for (int q = 1; q < G; ++q) checkCuda(cudaStreamWaitEvent(m0.stream, ready[q], 0), "stream wait");
    char* st = static_cast<char*>(staging);
    for (std::size_t k = 0; k < bufs[0].size(); ++k) {
      const XBuf& b = bufs[0][k];
      const std::size_t bytes = b.count * xtypeSize(b.type);
      SrcPtrs src{};
      src.p[0] = b.ptr;
      for (int q = 1; q < G; ++q) {
        checkCuda(cudaMemcpyPeerAsync(st, m0.device, bufs[q][k].ptr, maps[q]->device, bytes, m0.stream),
                  "reduce copy");
        src.p[q] = st;
        st += (bytes + 255) / 256 * 256;
      }
      reduceRanks(b, b.ptr, src, G, m0.stream);
    }
    checkCuda(cudaEventRecord(ready[0], m0.stream), "event");
    for (int r = 1; r < G; ++r) {
      DeviceMap& m = *maps[r];
      checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
      checkCuda(cudaStreamWaitEvent(m.stream, ready[0], 0), "stream wait");
      for (std::size_t k = 0; k < bufs[r].size(); ++k)
        checkCuda(cudaMemcpyPeerAsync(bufs[r][k].ptr, m.device, bufs[0][k].ptr, m0.device,
                                      bufs[0][k].count * xtypeSize(bufs[0][k].type), m.stream),
                  "reduce copy");
    }
    barrier();
  }
};

struct Group {
  bool local = false;
  int fusion = 0;  // 0 exact, 1 information form
  std::vector<DeviceMap*> maps;  // NCCL: this rank's map; local: every rank's, in rank order
  std::unique_ptr<NcclTransport> nccl;
  std::unique_ptr<LocalTransport> loc;
  int rank = 0, ranks = 1;
};

void groupUniqueId(unsigned char out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  ncclUniqueId id;
  ncclCheck(nccl().getUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

int groupNcclVersion() {
  int v = 0;
  ncclCheck(nccl().getVersion(&v), "ncclGetVersion");
  return v;
}

Group* groupCreateNccl(DeviceMap* m, const unsigned char id[128], int ranks, int rank) {
  if (ranks <= 0 || rank < 0 || rank >= ranks) fail(Err::kUsage, "bad group rank / size");
  auto g = std::make_unique<Group>();
  g->maps = {m};
  g->rank = rank;
  g->ranks = ranks;
  g->nccl = std::make_unique<NcclTransport>();
  g->nccl->map = m;
  g->nccl->n = ranks;
  g->nccl->me = rank;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  checkCuda(cudaSetDevice(m->device), "cudaSetDevice");
  ncclCheck(nccl().commInitRank(&g->nccl->comm, ranks, uid, rank), "ncclCommInitRank");
  return g.release();
}

Group* groupCreateLocal(const std::vector<DeviceMap*>& maps) {
  if (maps.empty() || maps.size() > static_cast<std::size_t>(kMaxLocalRanks))
    fail(Err::kUsage, "a local group takes 1..16 maps");
  const Grid& g0 = maps[0]->grid;
  for (DeviceMap* m : maps)
    if (m->grid.width != g0.width || m->grid.height != g0.height ||
        m->grid.resolution != g0.resolution || m->grid.center_x != g0.center_x ||
        m->grid.center_y != g0.center_y)
      fail(Err::kUsage, "the maps of a group must have the same geometry");
  auto g = std::make_unique<Group>();
  g->local = true;
  g->maps = maps;
  g->ranks = static_cast<int>(maps.size());
  g->loc = std::make_unique<LocalTransport>();
  g->loc->init(maps);
  return g.release();
}

void groupDestroy(Group* g) { delete g; }
int groupRanks(const Group& g) { return g.ranks; }
int groupRank(const Group& g) { return g.rank; }
bool groupIsLocal(const Group& g) { return g.local; }
void groupSetFusion(Group& g, int mode) {
  if (mode != 0 && mode != 1) fail(Err::kUsage, "group fusion mode must be 0 (exact) or 1 (information form)");
  g.fusion = mode;
}
int groupFusion(const Group& g) { return g.fusion; }
const std::vector<DeviceMap*>& groupMaps(const Group& g) { return g.maps; }

// One frame through a group (both transports). xyz: NCCL -- this rank's batch;
// local -- the whole frame (each rank reads its batch out of it). dts: the
// per-map dt since its last scan.
ScanResult groupIntegrate(Group& g, const PipelineParams& P, const double* xyz, std::size_t n,
                          bool on_device, uint64_t n_total, const Pose& pose, double stamp,
                          const std::vector<double>& dts) {
  const int G = g.local ? static_cast<int>(g.maps.size()) : 1;
  std::vector<GroupFrame*> frames(G, nullptr);
  struct Cleanup {
    std::vector<GroupFrame*>& f;
    ~Cleanup() {
      for (GroupFrame* p : f) groupEnd(p);
    }
  } cleanup{frames};
  std::vector<GroupGeom> geo(G);
  for (int r = 0; r < G; ++r) geo[r] = groupGeom(n_total, g.ranks, g.local ? r : g.rank);
  if (!g.local && n != geo[0].n_local)
    fail(Err::kUsage, "batch size differs from relief_gpu_group_bounds for this rank");
  if (g.local && n != n_total) fail(Err::kUsage, "a local group takes the whole frame");
  const bool info = g.fusion == 1;
  for (int r = 0; r < G; ++r)
    frames[r] = groupBegin(*g.maps[r], P, geo[r], pose, stamp, dts[r], info);
  std::vector<std::vector<XBuf>> x(G);
  auto exchange = [&](bool is_gather) {
    if (g.local) {
      if (is_gather) g.loc->gather(x);
      else g.loc->reduce(x);
    } else {
      if (is_gather) g.nccl->gather(x[0]);
      else g.nccl->reduce(x[0]);
    }
    for (auto& v : x) v.clear();
  };
  for (int r = 0; r < G; ++r) {
    const double* mine = xyz;
    if (g.local && xyz != nullptr) mine = xyz + 3 * static_cast<std::size_t>(geo[r].lo);
    groupPhaseIngest(*frames[r], mine, on_device, x[r]);
  }
  exchange(true);
  if (info) {
    for (int r = 0; r < G; ++r) groupPhaseInfoPartials(*frames[r], x[r]);
    exchange(false);
    for (int r = 0; r < G; ++r) groupPhaseInfoFirst(*frames[r], x[r]);
    exchange(false);
    for (int r = 0; r < G; ++r) groupPhaseInfoApply(*frames[r], x[r]);
  } else {
    for (int r = 0; r < G; ++r) groupPhaseUpdate(*frames[r], x[r]);
  }
  exchange(false);
  for (int r = 0; r < G; ++r) groupPhaseRemove(*frames[r], x[r]);
  exchange(false);
  for (int r = 0; r < G; ++r) groupPhaseCells(*frames[r], x[r]);
  exchange(false);
  ScanResult out;
  for (int r = 0; r < G; ++r) {
    ScanResult s = groupFinish(*frames[r]);
    if (r == 0) out = s;
  }
  return out;
}

}  // namespace rb200
