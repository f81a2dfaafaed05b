// Device-resident elevation map and the per-scan launch plan.
//
// HBM layout: structure of arrays, one contiguous
// 256-byte aligned array per layer, row-major r*W + c, exactly the layer set
// of the reference map (reference grid.hpp:90-101):
//   f64  elevation, variance, last_update, upper_bound, traversability,
//        normal_x, normal_y, normal_z
//   u8   valid, upper_bound_valid
// = 66 B/cell persistent. The persistent layers are double buffered so a
// robot-centric recenter is one streaming copy (cur -> alt, then swap).
// Per-scan scratch: i32 point count + segment start, u8 ray class, i32 k*.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

#include "relief_internal.hpp"

namespace rb200 {

struct Layers {
  double* elev = nullptr;
  double* var = nullptr;
  double* last = nullptr;
  double* ub = nullptr;
  double* trav = nullptr;
  double* nx = nullptr;
  double* ny = nullptr;
  double* nz = nullptr;
  uint8_t* valid = nullptr;
  uint8_t* ubv = nullptr;
};

// Counters written by the kernels; copied to the host once per scan.
struct DevStats {
  unsigned long long out_of_range;
  unsigned long long excluded;
  unsigned long long out_of_map;
  unsigned long long outlier;
  unsigned long long ignored_low;
  unsigned long long fused;
  unsigned long long cells_updated;
  unsigned long long removed;
  unsigned long long overlap_cleared;
  unsigned long long candidate_rays;  // rays queued for the k* pass
  unsigned long long visits;          // DDA cells emitted by pass 1
  unsigned long long heavy_cells;     // cells folded by k_fuse_heavy, one per lane
  unsigned long long vheavy_cells;    // cells folded by k_fuse_heavy, one per warp
  unsigned long long light_cells;     // cells folded by k_fuse_list (lists built by k_side_prep)
  unsigned long long light2_cells;    // ... of them, from the far end of the list (RB_LIGHT_SPLIT)
  unsigned long long pre_cells;       // cells folded before the ray pass (RB_PRESPLIT)
  double drift_offset;                // applied offset (0 when not applied)
  int drift_n;
  int drift_clamped;
  int error_code;                     // 0 ok, 1 non-positive variance
  int respeculate;                    // a heavy cell fused nothing: redo the ray pass
  unsigned int ingest_done;           // ingest blocks finished (the last one reduces the drift vote)
  unsigned int grid_bar[2];           // k_rays_tail's grid barrier (arrivals, generation)
  unsigned int cells_done;            // k_cells blocks finished (the last one hands the stats over)
};

// Geometry + parameters passed by value to kernels.
struct GridArgs {
  int W, H;
  double res;
  double ox, oy;      // origin = center - extent/2
  double xmax, ymax;  // ox + W*res, oy + H*res
};

// Device scratch of the post-processing chain (postchain.cu), sized W*H.
struct ChainScratch {
  double* va = nullptr;
  double* vb = nullptr;
  uint8_t* oa = nullptr;
  uint8_t* ob = nullptr;
  int* parent = nullptr;
  unsigned long long* key = nullptr;
  uint8_t* border = nullptr;
  int* flag = nullptr;
  std::size_t cap = 0;
  void ensure(std::size_t n);
  void release();
};

// Device scratch of the conv-net traversability executor (convnet.cu).
struct ConvScratch {
  uint32_t* sat = nullptr;       // summed-area table of the validity mask
  uint32_t* next_col = nullptr;  // per row: next valid column >= c
  uint32_t* next_row = nullptr;  // per column: next valid row >= r
  double* va = nullptr;       // layer activations ping-pong
  double* vb = nullptr;
  double* weights = nullptr;    // all layers' kernels, concatenated
  double* h_weights = nullptr;  // pinned staging copy
  std::size_t cap = 0, wcap = 0;
  cudaEvent_t upload_done = nullptr;
  void ensure(std::size_t n, std::size_t n_weights);
  void release();
};

// Cross-call state of a sharded frame (pipeline.cu, relief_gpu_shard_*).
struct ShardState {
  int stage = 0;  // 0 idle, 1 ingested, 2 updated, 3 removed
  PipelineParams params;
  Pose pose;
  double stamp = 0.0, dt = 0.0;
  std::size_t n_local = 0;
  uint32_t ray_base = 0;
  bool overlap = false;
  long long launches = 0;
  double drift_offset = 0.0;
  int drift_n = 0;
  bool drift_clamped = false;
};

struct DeviceMap {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // long-cell fold, overlapped with the ray pass
  cudaStream_t stream3 = nullptr;  // short-cell fold, overlapped with the ray pass (RB_PRESPLIT)
  Grid grid;
  Layers cur, alt;
  void* slab = nullptr;  // backing allocation of both layer sets + cell scratch
  // per-cell scratch
  int32_t* count = nullptr;
  uint32_t* start = nullptr;
  uint8_t* cls = nullptr;
  // pass-1 probe words (class + conservative gate bound), (W+2)x(H+2), with
  // kProbeGuardRows padded rows of border words before and after the grid
  // (pass 1's run lookahead may step that far past the border)
  uint16_t* probe = nullptr;
  static constexpr int kProbeGuardRows = 40;  // (also the jump grid's rings below the last rows)
  int32_t* kstar = nullptr;
  double* ub2 = nullptr;      // upper bounds of cells removed this frame (+inf between frames)
  // pass-1 jump grid (pipeline.cu k_jump_grid): one word per 16 x 16 cells
  float* jgrid = nullptr;
  int jw = 0, jh = 0;
  uint32_t* heavy = nullptr;  // ids of cells queued for the side-stream fold (2 lists of W*H),
                              // the short-cell list of k_fuse_list (W*H), the cells folded
                              // before the ray pass (W*H)
  // information-form group frames (allocated on first use, W*H each): the
  // exchanged per-cell partials (sum p/v, sum 1/v, first point, points, first
  // rank) and this rank's first point per cell
  void* islab = nullptr;
  double *info_a = nullptr, *info_b = nullptr, *info_pf = nullptr, *info_pfl = nullptr;
  int32_t *info_n = nullptr, *info_first = nullptr;
  // per-point scratch (grown on demand)
  std::size_t cap = 0;
  void* pslab = nullptr;
  double* xyz_in = nullptr;  // device copy of the caller's points
  double* px = nullptr;
  double* py = nullptr;
  double* pz = nullptr;
  double* pvar = nullptr;
  double* spz = nullptr;  // p_z sorted by (cell, scan order)
  double* spv = nullptr;  // sigma_p^2 sorted likewise
  uint32_t* key0 = nullptr;
  uint32_t* key1 = nullptr;
  uint32_t* val0 = nullptr;
  uint32_t* val1 = nullptr;
  uint32_t* raylist = nullptr;
  uint8_t* kept = nullptr;
  uint32_t* rec_cell = nullptr;  // sharded frames: this batch's fusion records
  double* rec_z = nullptr;
  double* rec_var = nullptr;
  // reduction scratch
  void* rslab = nullptr;
  std::size_t rcap = 0;
  double* drift_sum_part = nullptr;
  int* drift_n_part = nullptr;
  uint32_t* blk = nullptr;        // compaction block counts / offsets (+1: total)
  double* drift_local = nullptr;  // [2] local drift vote of a sharded batch
  uint32_t* hist = nullptr;
  uint32_t* scan_part = nullptr;
  std::size_t hist_cap = 0;
  DevStats* stats = nullptr;     // device
  DevStats* h_stats = nullptr;   // pinned host mirror
  // Synchronous frames hand their stats over through pinned host memory: the
  // last block of the frame's last kernel copies them into h_stats and then
  // writes the frame's sequence number into *h_seq, which the host polls
  // (no D2H copy, no stream synchronisation on the common path).
  unsigned long long* h_seq = nullptr;
  unsigned long long frame_seq = 0;
  double* drift_offset = nullptr;  // device scalar
  // host-side bookkeeping
  double last_stamp = 0.0;
  bool has_last = false;
  // Invalid cells may hold non-zero normals / traversability (snapshot load,
  // conv-net frame): the next cell pass zeroes them (CellArgs::scrub).
  bool scrub_invalid = false;
  double* export_buf = nullptr;  // masked-layer staging for get_layer
  ChainScratch chain;            // post-processing chain scratch
  ConvScratch conv;              // conv-net traversability scratch
  ShardState shard;              // sharded-frame bookkeeping
  // Streaming frames (relief_gpu_map_integrate_async / _wait): the input of
  // frame k+1 is copied on copy_stream while frame k computes; two slots.
  static constexpr int kSlots = 3;  // frames in flight
  cudaStream_t copy_stream = nullptr;
  DevStats* h_slot[kSlots] = {};    // pinned stats of the frames in flight
  double* xyz_slot[kSlots] = {};    // device input of each slot
  cudaEvent_t ev_copied[kSlots] = {}, ev_consumed[kSlots] = {}, ev_done[kSlots] = {};
  cudaEvent_t ev_copy0[kSlots] = {}, ev_start[kSlots] = {};  // timing: copy start, compute start
  int async_head = 0, async_count = 0;
  std::size_t async_n[kSlots] = {};
  double* chain_in = nullptr;    // masked input layer of the chain
  double* chain_out = nullptr;   // chain output staging for host callers
  uint8_t* chain_out_ok = nullptr;
  double last_chain_seconds = 0.0;
  int last_chain_launches = 0;
  cudaEvent_t ev[14] = {};
  cudaEvent_t ev_after = nullptr;  // relief_gpu_map_after_stream
  cudaEvent_t ev_fork = nullptr;   // frame stream -> copy stream (chunked upload)
  cudaEvent_t ev_dfork = nullptr, ev_djoin = nullptr;  // drift on stream2 (phaseDrift side)
  cudaEvent_t ev_sfork = nullptr, ev_sjoin = nullptr;  // short-cell fold on stream3
  // Executable graphs of recent synchronous-frame topologies, most recent
  // first (pipeline.cu FrameCapture); off: direct launches.
  static constexpr int kGraphs = 4;
  cudaGraphExec_t graphs[kGraphs] = {};
  int graph_count = 0;
  long long graph_instantiations = 0, graph_updates = 0;
  // Off by default: measured no device-time gain over PDL-chained direct
  // launches and more host time per call (profiles/r2_host_overhead.txt).
  int graph_mode = 2;  // 0 direct launches, 1 graphs, 2 graphs for frames >= kGraphMinPoints
  // Synchronous host-input frames: the upload is split into kChunks copies on
  // copy_stream and each chunk is ingested as soon as it lands.
  static constexpr int kChunks = 2;  // 2 and 4 measured alike; 8 slower
  cudaEvent_t ev_chunk[kChunks] = {};
  double phase_seconds[7] = {0, 0, 0, 0, 0, 0, 0};
  double kernel_seconds[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // upload ingest drift sort fuse rays cells total
  bool timing_pending = false;  // the arrays above still to be read from the events (resolveTiming)
#ifndef RB_PHASE_EVENTS_DEFAULT
#define RB_PHASE_EVENTS_DEFAULT false
#endif
  bool phase_events = RB_PHASE_EVENTS_DEFAULT;  // record per-phase events (relief_gpu_map_set_phase_timing)
  bool timing_phases = false;   // the pending frame recorded them
  bool timing_chunked = false;
  long long last_launches = 0;
  long long last_visits = 0;
};

GridArgs gridArgs(const Grid& g);

// Lifecycle (device_map.cu).
DeviceMap* createDeviceMap(int device, const Grid& grid);
void preloadFrameKernels(int device);  // (pipeline.cu) module loading at map creation
void destroyDeviceMap(DeviceMap* m);
void ensurePointCapacity(DeviceMap& m, std::size_t n);
void fillFresh(DeviceMap& m);  // reference grid.cpp:24-39 fill values
void checkCuda(cudaError_t e, const char* what);

// Masked export of one named layer into device memory (reference
// snapshot.cpp:50-77). Returns false for an unknown layer name.
bool exportLayerDevice(DeviceMap& m, const char* name, double* d_out);
// Raw (unmasked) upload / download of the ten persistent layers, used by
// snapshot load / save. host arrays are W*H each in the order of kLayerNames.
void uploadLayers(DeviceMap& m, const double* const host[8], const uint8_t* valid,
                  const uint8_t* ubv);
void downloadLayers(const DeviceMap& m, double* const host[8], uint8_t* valid, uint8_t* ubv);

// Whole per-scan pipeline (pipeline.cu).
struct ScanResult {
  std::int64_t points_in = 0, excluded = 0, out_of_range = 0, out_of_map = 0, outlier = 0,
               ignored_low = 0, fused = 0, cells_updated = 0, removed = 0, overlap_cleared = 0;
  double drift_offset = 0.0;
  bool drift_clamped = false;
  int drift_points = 0;
  double seconds = 0.0;
};
// Fills DeviceMap::kernel_seconds / phase_seconds of the last synchronous frame.
void resolveTiming(DeviceMap& m);
ScanResult integrateScanDevice(DeviceMap& m, const PipelineParams& params, const double* xyz,
                               std::size_t n, bool xyz_on_device, const Pose& pose,
                               double stamp, double dt);
// Streaming variant: enqueue the frame (host points, ideally pinned) and
// return; at most two frames in flight, completed in order by waitScan.
void integrateScanAsync(DeviceMap& m, const PipelineParams& params, const double* xyz,
                        std::size_t n, const Pose& pose, double stamp, double dt);
ScanResult waitScan(DeviceMap& m);

// Exact point-batch sharding of one frame: every rank holds a
// full replica and runs its contiguous batch of the frame's points; the host
// exchanges the buffers named in ShardIO between the phases (pipeline.cu).
struct ShardIO {
  int64_t n_records = 0;      // this batch's in-map kept points
  double drift[2] = {0, 0};   // local drift vote (sum, count)
  int64_t counters[3] = {0, 0, 0};  // local out_of_range, excluded, out_of_map
  uint32_t* rec_cell = nullptr;     // device, n_records (scan order)
  double* rec_z = nullptr;
  double* rec_var = nullptr;
  int32_t* kstar = nullptr;    // device, cells: first removing ray per cell
  double* ub = nullptr;       // device, cells: upper-bound layer
  uint8_t* ubv = nullptr;     // device, cells: upper-bound validity
  std::size_t cells = 0;
};
void shardIngest(DeviceMap& m, const PipelineParams& params, const double* xyz, std::size_t n,
                 bool xyz_on_device, uint64_t ray_offset, uint64_t n_total, const Pose& pose,
                 double stamp, ShardIO& io);
void shardUpdate(DeviceMap& m, const double* drift_pairs, int n_ranks, const uint32_t* d_cells,
                 const double* d_z, const double* d_var, std::size_t n_records, ShardIO& io);
int64_t shardRemove(DeviceMap& m, ShardIO& io);
ScanResult shardFinish(DeviceMap& m, const int64_t counters_total[3], uint64_t points_total);

// Group frames (pipeline.cu, SURVEY.md §8e exact variant): one frame split
// over the ranks of a group, every rank keeping a full replica. The phases
// enqueue on the map's stream and list the buffers to exchange after them;
// the group's transport (group.cpp: NCCL across processes, or peer copies +
// reduction kernels inside one process) runs the exchanges on the same stream.
enum class XType { kU8, kI32, kU32, kU64, kF64 };
enum class XOp { kSum, kMin, kMax };
// All-gather: `count` elements per rank, in place (rank r's part at r*count).
// All-reduce: `count` elements, op applied elementwise.
struct XBuf {
  void* ptr;
  std::size_t count;
  XType type;
  XOp op;
};
std::size_t xtypeSize(XType t);
struct GroupGeom {
  int ranks = 1, rank = 0;
  uint64_t n_total = 0;
  uint32_t chunk = 0;    // points per rank: ceil(n_total / ranks) rounded up to a radix tile
  uint32_t lo = 0;       // this rank's batch [lo, lo + n_local) of the frame
  uint32_t n_local = 0;
};
GroupGeom groupGeom(uint64_t n_total, int ranks, int rank);
struct GroupFrame;
GroupFrame* groupBegin(DeviceMap& m, const PipelineParams& P, const GroupGeom& g, const Pose& pose,
                       double stamp, double dt, bool info = false);
void groupEnd(GroupFrame* gf);
void groupPhaseIngest(GroupFrame& gf, const double* xyz, bool on_device,
                      std::vector<XBuf>& gathers);
void groupPhaseUpdate(GroupFrame& gf, std::vector<XBuf>& reduces);
// Information-form variant of the update (ungated fusion only):
// local per-cell partials (reduces: first rank), then the first points
// (reduces: the partials), then the fold of the merged partials + ray pass 1
// (reduces: k*, bounds, as groupPhaseUpdate).
void groupPhaseInfoPartials(GroupFrame& gf, std::vector<XBuf>& reduces);
void groupPhaseInfoFirst(GroupFrame& gf, std::vector<XBuf>& reduces);
void groupPhaseInfoApply(GroupFrame& gf, std::vector<XBuf>& reduces);
void groupPhaseRemove(GroupFrame& gf, std::vector<XBuf>& reduces);
void groupPhaseCells(GroupFrame& gf, std::vector<XBuf>& reduces);
ScanResult groupFinish(GroupFrame& gf);
// group.cu: the group object and its transports.
struct Group;
void groupUniqueId(unsigned char out[128]);
int groupNcclVersion();
Group* groupCreateNccl(DeviceMap* m, const unsigned char id[128], int ranks, int rank);
Group* groupCreateLocal(const std::vector<DeviceMap*>& maps);
void groupDestroy(Group* g);
int groupRanks(const Group& g);
int groupRank(const Group& g);
bool groupIsLocal(const Group& g);
// Fusion of group frames: 0 exact (gated, bit-identical to one GPU), 1
// information form (ungated partial sums + all-reduce; needs gates that
// cannot fire: mahalanobis_threshold >= 1e12, wall_count_threshold >= 2^30).
void groupSetFusion(Group& g, int mode);
int groupFusion(const Group& g);
const std::vector<DeviceMap*>& groupMaps(const Group& g);
ScanResult groupIntegrate(Group& g, const PipelineParams& P, const double* xyz, std::size_t n,
                          bool on_device, uint64_t n_total, const Pose& pose, double stamp,
                          const std::vector<double>& dts);

// Post-processing chain on a masked layer held in device memory (postchain.cu).
struct ChainStep {
  int kind;  // 0 gaussian, 1 box, 2 median, 3 min_inpaint
  int radius;
  double sigma;
};
// Enqueues the chain on `s` (no host sync); returns the number of launches.
int smoothChainEnqueue(cudaStream_t s, ChainScratch& sc, const double* d_values,
                       const uint8_t* d_valid, int W, int H, const ChainStep* steps, int n_steps,
                       double* d_values_out, uint8_t* d_valid_out);
// Conv-net traversability (convnet.cu): nearest-valid fill of d_layer by
// d_valid, then the spec's layer stack; writes all W*H cells of d_out.
// Enqueued on `s`; returns the number of launches.
int convnetEnqueue(cudaStream_t s, ConvScratch& cs, const double* d_layer, const uint8_t* d_valid,
                   int W, int H, const ConvNetSpec& spec, double* d_out);

// Same on caller-supplied host arrays, on `device` (synchronous).
void runHostConvnet(int device, const ConvNetSpec& spec, const double* layer, const uint8_t* valid,
                    int W, int H, double* out);

// Syncs `s` and raises NothingToInpaint if an inpaint step saw no valid cell.
void smoothChainCheck(cudaStream_t s, ChainScratch& sc);

}  // namespace rb200
