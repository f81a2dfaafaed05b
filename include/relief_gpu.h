/*
 * relief_gpu.h -- additive B200 entry points of librelief_b200.so.
 *
 * Nothing here exists in the reference; relief.h alone is the drop-in ABI.
 * These calls expose what the GPU build adds on top of it:
 *   - device selection and device-resident input (no host round trip),
 *   - per-phase device timings under the reference's Table-I labels
 *     (reference integration.hpp:119-126),
 *   - the post-processing chain of the reference (postprocess.cpp:40-197)
 *     run on the device map,
 *   - the synthetic scan generator used by tests and bench.py (an independent
 *     implementation of the reference simulator, sim.cpp:29-262).
 * All calls follow relief.h's conventions: relief_status return values and a
 * thread-local message behind relief_last_error().
 */
#ifndef RELIEF_GPU_H
#define RELIEF_GPU_H

#include "relief.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Number of CUDA devices visible to this process (0 when none). */
RELIEF_API int relief_gpu_device_count(void);

/* relief_map_create on an explicit CUDA device ordinal. */
RELIEF_API relief_map* relief_gpu_map_create_on(int device, double resolution, int width,
                                                int height, double center_x, double center_y);
RELIEF_API int relief_gpu_map_device(const relief_map* map);

/* relief_map_integrate with the point stream already in device memory of the
 * map's device (d_xyz: 3*n doubles, x y z packed). Synchronous like the
 * reference call: stats are final on return. d_xyz must be complete when the
 * call is made: produced on another stream, order it first with
 * relief_gpu_map_after_stream. */
RELIEF_API relief_status relief_gpu_map_integrate_device(relief_map* map,
                                                         const relief_config* config,
                                                         const double* d_xyz, size_t n_points,
                                                         const double pose[12], double stamp,
                                                         relief_scan_stats* stats_out);

/* Device time (seconds) of the last integrate call per phase, in the
 * reference's Table-I order: point transform & z error count, drift
 * compensation, height update & ray casting, overlap clearance,
 * traversability, normal calculation, total. Phases fused into one kernel
 * report their combined time under the first label and 0 for the others. */
RELIEF_API relief_status relief_gpu_map_phase_seconds(const relief_map* map, double out[7]);

/* Finer device-time breakdown of the last integrate call (seconds): host->device
 * upload (+ recenter shift), ingest, drift, cell sort, gated fusion, ray
 * casting, cell phases, total excluding the upload. */
RELIEF_API relief_status relief_gpu_map_kernel_seconds(const relief_map* map, double out[8]);
/* Per-phase device timing (default off): with it on, every frame records CUDA events at the
 * phase boundaries and relief_gpu_map_phase_seconds / _kernel_seconds report each phase; off,
 * only the upload and the device total are recorded, because an event between two kernels
 * also ends their programmatic (overlapped) launch. The runners turn it on. */
RELIEF_API relief_status relief_gpu_map_set_phase_timing(relief_map* map, int on);

/* CUDA graphs for synchronous frames. on = 1: each relief_map_integrate /
 * relief_gpu_map_integrate_device call captures its launches and replays them
 * as one graph launch, updating a cached executable graph in place (frames of
 * >= 512Ki points launch their head -- upload, resets, ingest -- directly and
 * capture the rest while it runs). on = 0: the launches are issued one by one,
 * chained by programmatic dependent launch. on = 2 (default): graphs for
 * frames of >= 32Ki points, direct launches below (where the capture costs
 * more than it saves). Results are identical either way; any
 * other value: RELIEF_ERROR_USAGE. graph_stats: out[0] graphs instantiated,
 * out[1] frames that updated a cached graph. */
RELIEF_API relief_status relief_gpu_map_set_graphs(relief_map* map, int on);
RELIEF_API relief_status relief_gpu_map_graph_stats(const relief_map* map, int64_t out[2]);

/* Kernel launches issued by the last integrate call (evidence for bench.py). */
RELIEF_API int64_t relief_gpu_map_last_launches(const relief_map* map);

/* DDA cell visits emitted by the last integrate call's ray pass (roofline
 * accounting: one class probe per visit). */
RELIEF_API int64_t relief_gpu_map_last_visits(const relief_map* map);

/* Copies one masked layer (same semantics as relief_map_layer) into device
 * memory of the map's device. */
RELIEF_API relief_status relief_gpu_map_layer_device(const relief_map* map, const char* layer,
                                                     double* d_out, size_t capacity);

/* Post-processing chain (reference postprocess.hpp:28-44, postprocess.cpp:
 * 40-197) on one masked layer of the map, computed on the device. kinds[s]:
 * 0 gaussian, 1 box, 2 median, 3 min_inpaint; radii/sigmas as FilterStep.
 * The map itself is not modified. values_out/valid_out are host buffers of
 * width*height entries. */
RELIEF_API relief_status relief_gpu_map_smooth_chain(const relief_map* map, const char* layer,
                                                     const int* kinds, const int* radii,
                                                     const double* sigmas, int n_steps,
                                                     double* values_out, uint8_t* valid_out);

/* Same chain with outputs left in device memory of the map's device
 * (d_values_out: width*height doubles, d_valid_out: width*height bytes).
 * Synchronous; relief_gpu_map_chain_seconds() reports its device time. */
RELIEF_API relief_status relief_gpu_map_smooth_chain_device(const relief_map* map,
                                                            const char* layer, const int* kinds,
                                                            const int* radii,
                                                            const double* sigmas, int n_steps,
                                                            double* d_values_out,
                                                            uint8_t* d_valid_out);
RELIEF_API double relief_gpu_map_chain_seconds(const relief_map* map);

/* Same chain on caller-supplied host data (values + 0/1 validity). */
RELIEF_API relief_status relief_gpu_smooth_chain(const double* values, const uint8_t* valid,
                                                 int width, int height, const int* kinds,
                                                 const int* radii, const double* sigmas,
                                                 int n_steps, double* values_out,
                                                 uint8_t* valid_out);

/* Page-locked host buffer for point clouds (cudaHostAlloc, portable): the
 * H2D copy inside relief_map_integrate / _async then runs at full PCIe speed.
 * NULL on failure. */
RELIEF_API void* relief_gpu_host_alloc(size_t bytes);
RELIEF_API void relief_gpu_host_free(void* ptr);

/* Streaming integrate for sensor pipelines: enqueues the frame (xyz in host
 * memory -- pinned memory lets the copy run asynchronously) and returns. Frames
 * are processed in call order; the PCIe copy of frame k+1 overlaps the kernels
 * of frame k. At most three frames may be in flight: relief_gpu_map_wait blocks
 * until the oldest one completes and returns its stats (same values as
 * relief_map_integrate). The caller keeps xyz unchanged until that frame's
 * wait returns. relief_map_integrate and the shard calls refuse while frames
 * are in flight (RELIEF_ERROR_USAGE). */
RELIEF_API relief_status relief_gpu_map_integrate_async(relief_map* map,
                                                        const relief_config* config,
                                                        const double* xyz, size_t n_points,
                                                        const double pose[12], double stamp);
RELIEF_API relief_status relief_gpu_map_wait(relief_map* map, relief_scan_stats* stats_out);
RELIEF_API int relief_gpu_map_in_flight(const relief_map* map);

/* Conv-net traversability (reference analysis.cpp:138-290). Loads the weight
 * file into the config and switches the pipeline to the learned filter, so
 * relief_map_integrate runs it (the reference reaches it only through its
 * runners, runner.cpp:53-60: its relief_config_load records the path but never
 * loads the layers). Errors: RELIEF_ERROR_IO (cannot open), ..._INVALID_MODEL. */
RELIEF_API relief_status relief_gpu_config_load_convnet(relief_config* config,
                                                        const char* model_path);

/* convFilterInference on caller-supplied host data with the config's model:
 * nearest-valid fill of `layer` by `valid`, the layer stack, clamp to [0,1];
 * writes width*height values. */
RELIEF_API relief_status relief_gpu_convnet_infer(const relief_config* config, const double* layer,
                                                  const uint8_t* valid, int width, int height,
                                                  double* out);

/* ---- Exact point-batch sharding of one frame -----------------
 * Every rank (one process per GPU) keeps a full replica of the map and feeds
 * its contiguous batch [ray_offset, ray_offset + n_local) of the frame's
 * n_total points (scan order). Per frame, in order:
 *   1. relief_gpu_shard_ingest  -> io: n_records, drift[2], counters[3] (host);
 *      rec_cell / rec_z / rec_var (device, n_records, scan order).
 *      Exchange: all-gather drift pairs and records in rank order, sum counters.
 *   2. relief_gpu_shard_update(all ranks' drift pairs, all records) -> fusion of
 *      every cell (identical on all ranks) + ray pass 1 over the local rays;
 *      io.kstar / io.upper_bound / io.upper_bound_valid (device, cells).
 *      Exchange: all-reduce MIN kstar, MIN upper_bound, MAX upper_bound_valid.
 *   3. relief_gpu_shard_remove -> removal + ray pass 2 over the local rays;
 *      *removed (identical on all ranks). If > 0, exchange again:
 *      all-reduce MIN upper_bound, MAX upper_bound_valid.
 *   4. relief_gpu_shard_finish(summed counters, n_total) -> cell phases, stats.
 * The result equals relief_map_integrate of the whole frame on one GPU (bit for
 * bit; with drift enabled the offset is the ranks' partial sums added in rank
 * order, so heights agree to the drift tolerance). Device pointers stay valid
 * until the next integrate / shard call on the map.
 * Ordering: every shard call returns with its outputs complete. The exchanged
 * inputs of the next call (records, k*, bounds) are read on the map's own
 * stream: if the caller's transport wrote them on another stream (NCCL under
 * torch.distributed, cudaMemcpyAsync, ...), it must call
 * relief_gpu_map_after_stream(map, that_stream) (or synchronise it) first.
 * relief_gpu_group_* does the whole frame, exchanges included, in-library. */
typedef struct relief_gpu_shard_io {
  int64_t n_records;
  double drift[2];       /* local drift vote: sum, count */
  int64_t counters[3];   /* local points_out_of_range, points_excluded, points_out_of_map */
  uint32_t* rec_cell;
  double* rec_z;
  double* rec_var;
  int32_t* kstar;
  double* upper_bound;
  uint8_t* upper_bound_valid;
  size_t cells;
} relief_gpu_shard_io;

RELIEF_API relief_status relief_gpu_shard_ingest(relief_map* map, const relief_config* config,
                                                 const double* xyz, size_t n_local,
                                                 int xyz_on_device, uint64_t ray_offset,
                                                 uint64_t n_total, const double pose[12],
                                                 double stamp, relief_gpu_shard_io* io);
RELIEF_API relief_status relief_gpu_shard_update(relief_map* map, const double* drift_pairs,
                                                 int n_ranks, const uint32_t* rec_cell,
                                                 const double* rec_z, const double* rec_var,
                                                 size_t n_records, relief_gpu_shard_io* io);
RELIEF_API relief_status relief_gpu_shard_remove(relief_map* map, int64_t* removed,
                                                 relief_gpu_shard_io* io);
RELIEF_API relief_status relief_gpu_shard_finish(relief_map* map, const int64_t counters_total[3],
                                                 uint64_t points_total, relief_scan_stats* stats);

/* ---- Group frames: one frame split across GPUs, exchanges inside the library
 * (SURVEY.md §8e exact variant). Replaces the point loop of the
 * reference's integrateScan (integration.cpp:142-224) by a split of the
 * frame's points into contiguous batches, one per rank, in scan order:
 *   relief_gpu_group_bounds(n_total, n_ranks, rank) -> [lo, hi) of the rank
 *   (whole radix tiles, so the gathered arrays equal the single-GPU ones).
 * Every rank keeps a full replica of the map. Per frame each rank ingests its
 * batch; the library all-gathers the cell keys, p_z, sigma_p^2 and drift
 * partials, runs the (identical) count, sort, gated fusion and drift offset on
 * every rank, casts its own rays, and merges k* / bounds / validity with
 * min / min / max all-reduces -- all on the map's stream, one host sync per
 * frame (the stats). The maps and stats equal relief_map_integrate of the
 * whole frame on one GPU bit for bit, drift compensation included.
 * Transports:
 *   relief_gpu_group_create: one process per GPU over NCCL (libnccl.so.2,
 *   loaded at run time; a copy already in the process is reused). Rank 0 makes
 *   the id with relief_gpu_group_unique_id and the caller broadcasts its 128
 *   bytes (MPI, torch.distributed, a file); every rank then calls create
 *   collectively. relief_gpu_group_integrate takes this rank's batch
 *   (xyz = points [lo, hi) of the frame, n_points = hi - lo) and must be
 *   called by every rank for every frame, in the same order.
 *   relief_gpu_group_create_local: one process drives n_maps maps (on several
 *   GPUs, or replicas on one GPU); the exchanges are peer copies and a
 *   reduction kernel. relief_gpu_group_integrate then takes the whole frame.
 * The maps must have the same geometry and history. The group does not own
 * them: free the group before its maps. Ordering: the group's work runs on
 * the maps' streams; device input must be complete before the call (see
 * relief_gpu_map_after_stream). Errors: RELIEF_ERROR_USAGE (bad rank / batch
 * size / geometry), RELIEF_ERROR_DATA (CUDA / NCCL failure, message set). */
typedef struct relief_gpu_group relief_gpu_group;
#define RELIEF_GPU_GROUP_ID_BYTES 128
RELIEF_API relief_status relief_gpu_group_unique_id(uint8_t id_out[RELIEF_GPU_GROUP_ID_BYTES]);
RELIEF_API relief_gpu_group* relief_gpu_group_create(relief_map* map,
                                                     const uint8_t id[RELIEF_GPU_GROUP_ID_BYTES],
                                                     int n_ranks, int rank);
RELIEF_API relief_gpu_group* relief_gpu_group_create_local(relief_map* const* maps, int n_maps);
RELIEF_API void relief_gpu_group_free(relief_gpu_group* group);
RELIEF_API relief_status relief_gpu_group_bounds(uint64_t n_total, int n_ranks, int rank,
                                                 uint64_t* lo, uint64_t* hi);
RELIEF_API relief_status relief_gpu_group_integrate(relief_gpu_group* group,
                                                    const relief_config* config,
                                                    const double* xyz, size_t n_points,
                                                    int xyz_on_device, uint64_t n_total,
                                                    const double pose[12], double stamp,
                                                    relief_scan_stats* stats_out);
/* Fusion of the group's frames (set before a frame; every rank the same):
 *   RELIEF_GPU_GROUP_EXACT (default): the gated, order-dependent fold on every
 *   rank from the gathered records -- bit-identical to one GPU.
 *   RELIEF_GPU_GROUP_INFORMATION: ungated fusion in information form -- each
 *   rank sums p/sigma_p^2 and 1/sigma_p^2 of its own points per cell, the sums
 *   (and each invalid cell's first point) are all-reduced, and every rank folds
 *   them into its replica: no point records exchanged and no redundant sort /
 *   fold. Equal to the reference's sequential Kalman fold up to rounding when
 *   its gates cannot fire, which the mode requires of the config:
 *   update.mahalanobis_threshold >= 1e12 and update.wall_count_threshold >=
 *   2^30 (else the frame fails with RELIEF_ERROR_USAGE). The ray passes and
 *   cell phases are the exact mode's.
 * relief_gpu_group_fusion returns the mode (-1 for a null group). */
#define RELIEF_GPU_GROUP_EXACT 0
#define RELIEF_GPU_GROUP_INFORMATION 1
RELIEF_API relief_status relief_gpu_group_set_fusion(relief_gpu_group* group, int mode);
RELIEF_API int relief_gpu_group_fusion(const relief_gpu_group* group);
/* Version of the NCCL library the group transport uses (e.g. 22809), or -1. */
RELIEF_API int relief_gpu_nccl_version(void);

/* Stream ordering for device-resident input: everything enqueued so far on
 * cuda_stream (a cudaStream_t of this process, on the map's device; NULL = the
 * legacy default stream) completes before the map's next device work reads
 * anything. The library runs on its own non-blocking stream, so a caller that
 * produces d_xyz (or exchanged shard buffers) on another stream calls this
 * before relief_gpu_map_integrate_device / relief_gpu_shard_* / the group
 * calls. Host synchronisation is not needed. Outputs are complete when a
 * synchronous call returns. */
RELIEF_API relief_status relief_gpu_map_after_stream(relief_map* map, void* cuda_stream);

/* Synthetic scan: scene + sensor of a reliefmap config file, rendered from
 * pose (row-major [R|t]) at `time` with splitmix64 stream (seed, scan_index)
 * per ray. Returns the point count (only min(count, capacity) points are
 * written), or -1 on error. Host code; matches the reference simulator
 * bit for bit (tests/test_sim_parity.py). */
RELIEF_API int64_t relief_gpu_sim_render(const char* config_path, const double pose[12],
                                         double time, uint64_t seed, uint64_t scan_index,
                                         double* xyz, int64_t capacity);

#ifdef __cplusplus
}
#endif

#endif /* RELIEF_GPU_H */
