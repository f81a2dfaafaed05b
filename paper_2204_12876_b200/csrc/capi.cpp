// C ABI of librelief_b200.so: relief.h (drop-in, reference capi.cpp:106-334)
// plus the additive relief_gpu.h entry points.
//
// Exceptions never cross the boundary: every entry point runs its body under
// `guard`, which maps rb200::Err onto relief_status exactly as the reference
// maps relief::ErrorCode (reference capi.cpp:43-85) and stores the message
// in a thread-local string.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "../../include/relief_gpu.h"
#include "device_map.hpp"
#include "runners.hpp"
#include "snapshot.hpp"

struct relief_config {
  rb200::RunConfig config;
};

struct relief_map {
  rb200::DeviceMap* dev = nullptr;
};

struct relief_gpu_group {
  rb200::Group* g = nullptr;
  std::vector<relief_map*> maps;
};

namespace {

thread_local std::string t_last_error;

relief_status statusOf(rb200::Err e) {
  switch (e) {
    case rb200::Err::kOutOfMap: return RELIEF_ERROR_OUT_OF_MAP;
    case rb200::Err::kInvalidPose: return RELIEF_ERROR_INVALID_POSE;
    case rb200::Err::kInvalidVariance: return RELIEF_ERROR_INVALID_VARIANCE;
    case rb200::Err::kInvalidModel: return RELIEF_ERROR_INVALID_MODEL;
    case rb200::Err::kDegeneratePlane: return RELIEF_ERROR_DEGENERATE_PLANE;
    case rb200::Err::kNothingToInpaint: return RELIEF_ERROR_NOTHING_TO_INPAINT;
    case rb200::Err::kOutOfTrajectory: return RELIEF_ERROR_OUT_OF_TRAJECTORY;
    case rb200::Err::kParse: return RELIEF_ERROR_PARSE;
    case rb200::Err::kIo: return RELIEF_ERROR_IO;
    case rb200::Err::kUsage: return RELIEF_ERROR_USAGE;
    case rb200::Err::kDevice: return RELIEF_ERROR_DATA;
  }
  return RELIEF_ERROR_DATA;
}

template <typename Body>
relief_status guard(Body&& body) {
  try {
    body();
    return RELIEF_OK;
  } catch (const rb200::Error& e) {
    t_last_error = e.what();
    return statusOf(e.code());
  } catch (const std::exception& e) {
    t_last_error = e.what();
    return RELIEF_ERROR_DATA;
  }
}

template <typename T, typename Body>
T* guardCreate(Body&& body) {
  try {
    return body();
  } catch (const std::exception& e) {
    t_last_error = e.what();
    return nullptr;
  }
}

relief_status usage(const char* msg) {
  t_last_error = msg;
  return RELIEF_ERROR_USAGE;
}

int currentDevice() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return d;
}

// Parameter + pose checks done before any device work (reference
// integration.cpp:72-75; the traversability / overlap checks the reference
// runs after mutating the map are hoisted here).
void validateScan(const rb200::PipelineParams& p, const rb200::Pose& pose) {
  p.update.validate();
  p.drift.validate();
  p.cleanup.validate();
  if (!pose.isValid()) rb200::fail(rb200::Err::kInvalidPose, "rotation is not orthonormal");
  if (p.overlap.enabled) p.overlap.validate();
  // The reference validates whichever traversability filter runs
  // (analysis.cpp:89 / 187). A config loaded through relief_config_load names
  // the model file but carries no layers, so the conv-net path fails with
  // "model has no layers" exactly as the reference's C API does, unless the
  // model was attached with relief_gpu_config_load_convnet.
  if (p.use_convnet_traversability) p.convnet.validate();
  else p.traversability.validate();
}

void exportShardIO(const rb200::ShardIO& s, relief_gpu_shard_io* io) {
  io->n_records = s.n_records;
  io->drift[0] = s.drift[0];
  io->drift[1] = s.drift[1];
  for (int k = 0; k < 3; ++k) io->counters[k] = s.counters[k];
  io->rec_cell = s.rec_cell;
  io->rec_z = s.rec_z;
  io->rec_var = s.rec_var;
  io->kstar = s.kstar;
  io->upper_bound = s.ub;
  io->upper_bound_valid = s.ubv;
  io->cells = s.cells;
}

void fillStats(const rb200::ScanResult& r, relief_scan_stats* s) {
  if (s == nullptr) return;
  s->points_in = r.points_in;
  s->points_excluded = r.excluded;
  s->points_out_of_range = r.out_of_range;
  s->points_out_of_map = r.out_of_map;
  s->points_rejected_outlier = r.outlier;
  s->points_ignored_low = r.ignored_low;
  s->points_fused = r.fused;
  s->cells_updated = r.cells_updated;
  s->cells_removed_by_cleanup = r.removed;
  s->cells_cleared_by_overlap = r.overlap_cleared;
  s->drift_offset_applied = r.drift_offset;
  s->total_seconds = r.seconds;
}

relief_status integrateCommon(relief_map* map, const relief_config* config, const double* xyz,
                              size_t n, bool on_device, const double pose[12], double stamp,
                              relief_scan_stats* stats_out) {
  if (map == nullptr || pose == nullptr || (xyz == nullptr && n > 0))
    return usage("null argument");
  return guard([&] {
    const rb200::Pose p = rb200::Pose::fromRowMajor34(pose);
    const rb200::PipelineParams params =
        config ? config->config.pipeline : rb200::PipelineParams{};
    validateScan(params, p);
    rb200::DeviceMap& m = *map->dev;
    const double dt = m.has_last ? std::max(0.0, stamp - m.last_stamp) : 0.0;
    const rb200::ScanResult r = rb200::integrateScanDevice(m, params, xyz, n, on_device, p, stamp, dt);
    m.last_stamp = stamp;
    m.has_last = true;
    fillStats(r, stats_out);
  });
}

}  // namespace

extern "C" {

const char* relief_last_error(void) { return t_last_error.c_str(); }
const char* relief_version(void) { return "reliefmap 1.0.0"; }

relief_config* relief_config_default(void) {
  return guardCreate<relief_config>([] { return new relief_config{}; });
}

relief_config* relief_config_load(const char* path) {
  if (path == nullptr) {
    t_last_error = "config path is null";
    return nullptr;
  }
  return guardCreate<relief_config>(
      [&] { return new relief_config{rb200::loadRunConfigFile(path)}; });
}

void relief_config_free(relief_config* config) { delete config; }

relief_status relief_config_set_mode(relief_config* config, const char* mode) {
  if (config == nullptr) return usage("config handle is null");
  if (mode == nullptr) return RELIEF_OK;
  rb200::ExecMode m;
  if (!rb200::parseMode(mode, m)) return usage("mode must be det or par");
  config->config.pipeline.mode = m;
  return RELIEF_OK;
}

relief_status relief_config_set_seed(relief_config* config, uint64_t seed) {
  if (config == nullptr) return usage("config handle is null");
  config->config.seed = seed;
  return RELIEF_OK;
}

relief_map* relief_map_create(double resolution, int width, int height, double center_x,
                              double center_y) {
  return relief_gpu_map_create_on(currentDevice(), resolution, width, height, center_x, center_y);
}

relief_map* relief_map_load(const char* path) {
  if (path == nullptr) {
    t_last_error = "snapshot path is null";
    return nullptr;
  }
  return guardCreate<relief_map>([&] {
    const rb200::HostLayers h = rb200::readSnapshotFile(path);
    auto* m = new relief_map;
    m->dev = rb200::uploadHost(currentDevice(), h);
    return m;
  });
}

relief_status relief_map_save(const relief_map* map, const char* path) {
  if (map == nullptr || path == nullptr) return usage("map handle or path is null");
  return guard([&] { rb200::writeSnapshotFile(rb200::downloadHost(*map->dev), path); });
}

void relief_map_free(relief_map* map) {
  if (map == nullptr) return;
  rb200::destroyDeviceMap(map->dev);
  delete map;
}

int relief_map_width(const relief_map* map) { return map ? map->dev->grid.width : 0; }
int relief_map_height(const relief_map* map) { return map ? map->dev->grid.height : 0; }
double relief_map_resolution(const relief_map* map) {
  return map ? map->dev->grid.resolution : 0.0;
}

relief_status relief_map_center(const relief_map* map, double* x, double* y) {
  if (map == nullptr || x == nullptr || y == nullptr) return usage("null argument");
  *x = map->dev->grid.center_x;
  *y = map->dev->grid.center_y;
  return RELIEF_OK;
}

relief_status relief_map_layer(const relief_map* map, const char* layer, double* out,
                               size_t capacity) {
  if (map == nullptr || layer == nullptr || out == nullptr) return usage("null argument");
  rb200::DeviceMap& m = *map->dev;
  if (capacity < m.grid.cells()) return usage("output buffer too small");
  return guard([&] {
    rb200::checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
    if (m.export_buf == nullptr)
      rb200::checkCuda(cudaMalloc(&m.export_buf, m.grid.cells() * sizeof(double)), "export buffer");
    if (!rb200::exportLayerDevice(m, layer, m.export_buf))
      rb200::fail(rb200::Err::kUsage, rb200::unknownLayerMessage(layer));
    rb200::checkCuda(cudaMemcpyAsync(out, m.export_buf, m.grid.cells() * sizeof(double),
                                     cudaMemcpyDeviceToHost, m.stream),
                     "layer download");
    rb200::checkCuda(cudaStreamSynchronize(m.stream), "layer download");
  });
}

relief_status relief_map_integrate(relief_map* map, const relief_config* config,
                                   const double* xyz, size_t n_points, const double pose[12],
                                   double stamp, relief_scan_stats* stats_out) {
  return integrateCommon(map, config, xyz, n_points, false, pose, stamp, stats_out);
}

// ---------------------------------------------------------------- runners
relief_status relief_run_simulate(const char* config_path, const char* out_dir, uint64_t seed,
                                  int has_seed, const char* mode) {
  if (config_path == nullptr || out_dir == nullptr)
    return usage("config path and output directory are required");
  return guard([&] { rb200::runSimulate(config_path, out_dir, seed, has_seed != 0, mode); });
}

relief_status relief_run_replay(const char* config_path, const char* const* cloud_paths,
                                size_t n_clouds, const char* poses_path, const char* out_dir,
                                const char* mode) {
  if (config_path == nullptr || poses_path == nullptr || out_dir == nullptr ||
      (cloud_paths == nullptr && n_clouds > 0))
    return usage("config, poses, clouds and output directory are required");
  return guard([&] {
    rb200::runReplay(config_path, std::vector<std::string>(cloud_paths, cloud_paths + n_clouds),
                     poses_path, out_dir, mode);
  });
}

relief_status relief_run_bench(const char* config_path, const size_t* counts, size_t n_counts,
                               int repetitions, const char* out_csv, const char* mode) {
  if (config_path == nullptr || counts == nullptr || n_counts == 0 || out_csv == nullptr)
    return usage("config, point counts and output CSV are required");
  return guard([&] {
    rb200::runBench(config_path, std::vector<size_t>(counts, counts + n_counts), repetitions,
                    out_csv, mode);
  });
}

relief_status relief_run_export(const char* snapshot_path, const char* layer, const char* format,
                                const char* out_path) {
  if (snapshot_path == nullptr || layer == nullptr || format == nullptr || out_path == nullptr)
    return usage("snapshot, layer, format and output path are required");
  const std::string f = format;
  if (f != "csv" && f != "pgm") return usage("format must be csv or pgm");
  return guard([&] { rb200::runExport(snapshot_path, layer, f == "pgm", out_path); });
}

relief_status relief_run_segment(const char* snapshot_path, const char* config_path,
                                 const char* out_path, size_t* n_regions_out) {
  if (snapshot_path == nullptr || out_path == nullptr)
    return usage("snapshot and output path are required");
  return guard([&] {
    const size_t n = rb200::runSegment(snapshot_path, config_path, out_path);
    if (n_regions_out != nullptr) *n_regions_out = n;
  });
}

// ------------------------------------------------------- relief_gpu.h
int relief_gpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

relief_map* relief_gpu_map_create_on(int device, double resolution, int width, int height,
                                     double center_x, double center_y) {
  return guardCreate<relief_map>([&] {
    rb200::Grid g;
    g.resolution = resolution;
    g.width = width;
    g.height = height;
    g.center_x = center_x;
    g.center_y = center_y;
    g.validate();
    auto* m = new relief_map;
    try {
      m->dev = rb200::createDeviceMap(device, g);
    } catch (...) {
      delete m;
      throw;
    }
    return m;
  });
}

int relief_gpu_map_device(const relief_map* map) { return map ? map->dev->device : -1; }

relief_status relief_gpu_map_integrate_device(relief_map* map, const relief_config* config,
                                              const double* d_xyz, size_t n_points,
                                              const double pose[12], double stamp,
                                              relief_scan_stats* stats_out) {
  return integrateCommon(map, config, d_xyz, n_points, true, pose, stamp, stats_out);
}

relief_status relief_gpu_map_phase_seconds(const relief_map* map, double out[7]) {
  if (map == nullptr || out == nullptr) return usage("null argument");
  return guard([&] {
    rb200::resolveTiming(*map->dev);
    for (int k = 0; k < 7; ++k) out[k] = map->dev->phase_seconds[k];
  });
}

relief_status relief_gpu_map_set_phase_timing(relief_map* map, int on) {
  if (map == nullptr) return usage("null argument");
  map->dev->phase_events = on != 0;
  return RELIEF_OK;
}

relief_status relief_gpu_map_kernel_seconds(const relief_map* map, double out[8]) {
  if (map == nullptr || out == nullptr) return usage("null argument");
  return guard([&] {
    rb200::resolveTiming(*map->dev);
    for (int k = 0; k < 8; ++k) out[k] = map->dev->kernel_seconds[k];
  });
}

int64_t relief_gpu_map_last_visits(const relief_map* map) {
  return map ? map->dev->last_visits : 0;
}

int64_t relief_gpu_map_last_launches(const relief_map* map) {
  return map ? map->dev->last_launches : 0;
}

relief_status relief_gpu_map_layer_device(const relief_map* map, const char* layer, double* d_out,
                                          size_t capacity) {
  if (map == nullptr || layer == nullptr || d_out == nullptr) return usage("null argument");
  rb200::DeviceMap& m = *map->dev;
  if (capacity < m.grid.cells()) return usage("output buffer too small");
  return guard([&] {
    rb200::checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
    if (!rb200::exportLayerDevice(m, layer, d_out))
      rb200::fail(rb200::Err::kUsage, rb200::unknownLayerMessage(layer));
    rb200::checkCuda(cudaStreamSynchronize(m.stream), "layer export");
  });
}

relief_status relief_gpu_map_smooth_chain(const relief_map* map, const char* layer,
                                          const int* kinds, const int* radii,
                                          const double* sigmas, int n_steps, double* values_out,
                                          uint8_t* valid_out) {
  if (map == nullptr || layer == nullptr || values_out == nullptr || valid_out == nullptr ||
      (n_steps > 0 && (kinds == nullptr || radii == nullptr || sigmas == nullptr)))
    return usage("null argument");
  return guard([&] {
    rb200::runMapChain(*map->dev, layer, kinds, radii, sigmas, n_steps, values_out, valid_out);
  });
}

relief_status relief_gpu_map_smooth_chain_device(const relief_map* map, const char* layer,
                                                 const int* kinds, const int* radii,
                                                 const double* sigmas, int n_steps,
                                                 double* d_values_out, uint8_t* d_valid_out) {
  if (map == nullptr || layer == nullptr || d_values_out == nullptr || d_valid_out == nullptr ||
      (n_steps > 0 && (kinds == nullptr || radii == nullptr || sigmas == nullptr)))
    return usage("null argument");
  return guard([&] {
    rb200::runMapChainDevice(*map->dev, layer, kinds, radii, sigmas, n_steps, d_values_out,
                             d_valid_out);
  });
}

double relief_gpu_map_chain_seconds(const relief_map* map) {
  return map ? map->dev->last_chain_seconds : 0.0;
}

relief_status relief_gpu_smooth_chain(const double* values, const uint8_t* valid, int width,
                                      int height, const int* kinds, const int* radii,
                                      const double* sigmas, int n_steps, double* values_out,
                                      uint8_t* valid_out) {
  if (values == nullptr || valid == nullptr || values_out == nullptr || valid_out == nullptr ||
      (n_steps > 0 && (kinds == nullptr || radii == nullptr || sigmas == nullptr)))
    return usage("null argument");
  return guard([&] {
    rb200::runHostChain(currentDevice(), values, valid, width, height, kinds, radii, sigmas,
                        n_steps, values_out, valid_out);
  });
}

void* relief_gpu_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    t_last_error = "cudaHostAlloc failed";
    return nullptr;
  }
  return p;
}

void relief_gpu_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

relief_status relief_gpu_map_integrate_async(relief_map* map, const relief_config* config,
                                            const double* xyz, size_t n_points,
                                            const double pose[12], double stamp) {
  if (map == nullptr || pose == nullptr || (xyz == nullptr && n_points > 0))
    return usage("null argument");
  return guard([&] {
    const rb200::Pose p = rb200::Pose::fromRowMajor34(pose);
    const rb200::PipelineParams params =
        config ? config->config.pipeline : rb200::PipelineParams{};
    validateScan(params, p);
    rb200::DeviceMap& m = *map->dev;
    const double dt = m.has_last ? std::max(0.0, stamp - m.last_stamp) : 0.0;
    rb200::integrateScanAsync(m, params, xyz, n_points, p, stamp, dt);
    m.last_stamp = stamp;
    m.has_last = true;
  });
}

relief_status relief_gpu_map_wait(relief_map* map, relief_scan_stats* stats_out) {
  if (map == nullptr) return usage("null argument");
  return guard([&] { fillStats(rb200::waitScan(*map->dev), stats_out); });
}

int relief_gpu_map_in_flight(const relief_map* map) { return map ? map->dev->async_count : 0; }

relief_status relief_gpu_config_load_convnet(relief_config* config, const char* model_path) {
  if (config == nullptr || model_path == nullptr) return usage("null argument");
  return guard([&] {
    rb200::ConvNetSpec spec = rb200::loadConvNetSpecFile(model_path);
    config->config.convnet_path = model_path;
    config->config.pipeline.convnet = std::move(spec);
    config->config.pipeline.use_convnet_traversability = true;
  });
}

relief_status relief_gpu_convnet_infer(const relief_config* config, const double* layer,
                                       const uint8_t* valid, int width, int height,
                                       double* out) {
  if (config == nullptr || layer == nullptr || valid == nullptr || out == nullptr)
    return usage("null argument");
  return guard([&] {
    rb200::runHostConvnet(currentDevice(), config->config.pipeline.convnet, layer, valid, width,
                          height, out);
  });
}

relief_status relief_gpu_shard_ingest(relief_map* map, const relief_config* config,
                                      const double* xyz, size_t n_local, int xyz_on_device,
                                      uint64_t ray_offset, uint64_t n_total, const double pose[12],
                                      double stamp, relief_gpu_shard_io* io) {
  if (map == nullptr || pose == nullptr || io == nullptr || (xyz == nullptr && n_local > 0))
    return usage("null argument");
  return guard([&] {
    const rb200::Pose p = rb200::Pose::fromRowMajor34(pose);
    const rb200::PipelineParams params = config ? config->config.pipeline : rb200::PipelineParams{};
    validateScan(params, p);
    rb200::ShardIO sio;
    rb200::shardIngest(*map->dev, params, xyz, n_local, xyz_on_device != 0, ray_offset, n_total, p,
                       stamp, sio);
    exportShardIO(sio, io);
  });
}

relief_status relief_gpu_shard_update(relief_map* map, const double* drift_pairs, int n_ranks,
                                      const uint32_t* rec_cell, const double* rec_z,
                                      const double* rec_var, size_t n_records,
                                      relief_gpu_shard_io* io) {
  if (map == nullptr || io == nullptr ||
      (n_records > 0 && (rec_cell == nullptr || rec_z == nullptr || rec_var == nullptr)))
    return usage("null argument");
  return guard([&] {
    rb200::ShardIO sio;
    rb200::shardUpdate(*map->dev, drift_pairs, n_ranks, rec_cell, rec_z, rec_var, n_records, sio);
    exportShardIO(sio, io);
  });
}

relief_status relief_gpu_shard_remove(relief_map* map, int64_t* removed, relief_gpu_shard_io* io) {
  if (map == nullptr || io == nullptr) return usage("null argument");
  return guard([&] {
    rb200::ShardIO sio;
    const int64_t r = rb200::shardRemove(*map->dev, sio);
    if (removed) *removed = r;
    io->upper_bound = sio.ub;
    io->upper_bound_valid = sio.ubv;
  });
}

relief_status relief_gpu_shard_finish(relief_map* map, const int64_t counters_total[3],
                                      uint64_t points_total, relief_scan_stats* stats) {
  if (map == nullptr || counters_total == nullptr) return usage("null argument");
  return guard([&] {
    const rb200::ScanResult r = rb200::shardFinish(*map->dev, counters_total, points_total);
    fillStats(r, stats);
  });
}

relief_status relief_gpu_map_set_graphs(relief_map* map, int on) {
  if (map == nullptr) return usage("null argument");
  if (on < 0 || on > 2) return usage("graph mode must be 0, 1 or 2");
  map->dev->graph_mode = on;
  return RELIEF_OK;
}

relief_status relief_gpu_map_graph_stats(const relief_map* map, int64_t out[2]) {
  if (map == nullptr || out == nullptr) return usage("null argument");
  out[0] = map->dev->graph_instantiations;
  out[1] = map->dev->graph_updates;
  return RELIEF_OK;
}

relief_status relief_gpu_map_after_stream(relief_map* map, void* cuda_stream) {
  if (map == nullptr) return usage("null argument");
  return guard([&] {
    rb200::DeviceMap& m = *map->dev;
    rb200::checkCuda(cudaSetDevice(m.device), "cudaSetDevice");
    rb200::checkCuda(cudaEventRecord(m.ev_after, static_cast<cudaStream_t>(cuda_stream)),
                     "event record on the caller's stream");
    rb200::checkCuda(cudaStreamWaitEvent(m.stream, m.ev_after, 0), "stream wait");
  });
}

relief_status relief_gpu_group_unique_id(uint8_t id_out[RELIEF_GPU_GROUP_ID_BYTES]) {
  if (id_out == nullptr) return usage("null argument");
  return guard([&] { rb200::groupUniqueId(id_out); });
}

int relief_gpu_nccl_version(void) {
  int v = -1;
  guard([&] { v = rb200::groupNcclVersion(); });
  return v;
}

relief_gpu_group* relief_gpu_group_create(relief_map* map,
                                          const uint8_t id[RELIEF_GPU_GROUP_ID_BYTES],
                                          int n_ranks, int rank) {
  if (map == nullptr || id == nullptr) {
    t_last_error = "null argument";
    return nullptr;
  }
  return guardCreate<relief_gpu_group>([&] {
    auto* g = new relief_gpu_group{};
    try {
      g->g = rb200::groupCreateNccl(map->dev, id, n_ranks, rank);
    } catch (...) {
      delete g;
      throw;
    }
    g->maps = {map};
    return g;
  });
}

relief_gpu_group* relief_gpu_group_create_local(relief_map* const* maps, int n_maps) {
  if (maps == nullptr || n_maps <= 0) {
    t_last_error = "null argument";
    return nullptr;
  }
  return guardCreate<relief_gpu_group>([&] {
    std::vector<rb200::DeviceMap*> dev;
    for (int r = 0; r < n_maps; ++r) {
      if (maps[r] == nullptr) rb200::fail(rb200::Err::kUsage, "null map in the group");
      dev.push_back(maps[r]->dev);
    }
    auto* g = new relief_gpu_group{};
    try {
      g->g = rb200::groupCreateLocal(dev);
    } catch (...) {
      delete g;
      throw;
    }
    g->maps.assign(maps, maps + n_maps);
    return g;
  });
}

void relief_gpu_group_free(relief_gpu_group* group) {
  if (group == nullptr) return;
  rb200::groupDestroy(group->g);
  delete group;
}

relief_status relief_gpu_group_set_fusion(relief_gpu_group* group, int mode) {
  if (group == nullptr) return usage("null argument");
  return guard([&] { rb200::groupSetFusion(*group->g, mode); });
}

int relief_gpu_group_fusion(const relief_gpu_group* group) {
  return group ? rb200::groupFusion(*group->g) : -1;
}

relief_status relief_gpu_group_bounds(uint64_t n_total, int n_ranks, int rank, uint64_t* lo,
                                      uint64_t* hi) {
  if (lo == nullptr || hi == nullptr) return usage("null argument");
  return guard([&] {
    const rb200::GroupGeom g = rb200::groupGeom(n_total, n_ranks, rank);
    *lo = g.lo;
    *hi = static_cast<uint64_t>(g.lo) + g.n_local;
  });
}

relief_status relief_gpu_group_integrate(relief_gpu_group* group, const relief_config* config,
                                         const double* xyz, size_t n_points, int xyz_on_device,
                                         uint64_t n_total, const double pose[12], double stamp,
                                         relief_scan_stats* stats_out) {
  if (group == nullptr || pose == nullptr || (xyz == nullptr && n_points > 0))
    return usage("null argument");
  return guard([&] {
    const rb200::Pose p = rb200::Pose::fromRowMajor34(pose);
    const rb200::PipelineParams params =
        config ? config->config.pipeline : rb200::PipelineParams{};
    validateScan(params, p);
    std::vector<double> dts;
    for (relief_map* m : group->maps)
      dts.push_back(m->dev->has_last ? std::max(0.0, stamp - m->dev->last_stamp) : 0.0);
    const auto t0 = std::chrono::steady_clock::now();
    rb200::ScanResult r = rb200::groupIntegrate(*group->g, params, xyz, n_points,
                                                xyz_on_device != 0, n_total, p, stamp, dts);
    r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (relief_map* m : group->maps) {
      m->dev->last_stamp = stamp;
      m->dev->has_last = true;
    }
    fillStats(r, stats_out);
  });
}

int64_t relief_gpu_sim_render(const char* config_path, const double pose[12], double time,
                              uint64_t seed, uint64_t scan_index, double* xyz, int64_t capacity) {
  if (config_path == nullptr || pose == nullptr || (xyz == nullptr && capacity > 0)) {
    t_last_error = "null argument";
    return -1;
  }
  int64_t n = -1;
  const relief_status st = guard([&] {
    const rb200::RunConfig cfg = rb200::loadRunConfigFile(config_path);
    const std::vector<double> pts = rb200::renderScan(
        cfg.scene, rb200::Pose::fromRowMajor34(pose), cfg.sensor, time, seed, scan_index);
    n = static_cast<int64_t>(pts.size() / 3);
    const int64_t w = std::min<int64_t>(n, capacity);
    if (w > 0) std::memcpy(xyz, pts.data(), static_cast<size_t>(w) * 3 * sizeof(double));
  });
  return st == RELIEF_OK ? n : -1;
}

}  // extern "C"
