// Extra C entry points compiled INTO oracle/_ref/librelief_ref.so next to the
// unmodified reference sources, so tests can reach reference functions that
// relief.h does not export (the simulator, the DDA, the Kalman step, the
// post-processing chain).
//
// TEST INFRASTRUCTURE ONLY: never linked into the product library. Only
// tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs
// may load the library this file is part of.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "relief/core/analysis.hpp"
#include "relief/core/config.hpp"
#include "relief/core/integration.hpp"
#include "relief/core/postprocess.hpp"
#include "relief/core/raycast.hpp"
#include "relief/core/sim.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {
thread_local std::string g_err;

relief::RigidTransform poseFrom(const double* pose) {
  relief::RigidTransform rt;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) rt.rotation(r, c) = pose[4 * r + c];
    rt.translation(r) = pose[4 * r + 3];
  }
  return rt;
}
}  // namespace

REF_API const char* ref_last_error(void) { return g_err.c_str(); }

// Renders one scan of the scene + sensor described by a reliefmap config file
// (sim.cpp:241-262). Returns the number of points (may exceed capacity, in
// which case only `capacity` are written), or -1 on error.
REF_API int64_t ref_render_scan(const char* config_path, const double* pose, double time,
                                uint64_t seed, uint64_t scan_index, double* xyz,
                                int64_t capacity) {
  try {
    const relief::RunConfig cfg = relief::loadRunConfigFile(config_path);
    const relief::PointCloud cloud =
        relief::renderScan(cfg.scene, poseFrom(pose), cfg.sensor, time, seed, scan_index);
    const int64_t n = static_cast<int64_t>(cloud.points.size());
    for (int64_t k = 0; k < n && k < capacity; ++k) {
      xyz[3 * k] = cloud.points[k].x();
      xyz[3 * k + 1] = cloud.points[k].y();
      xyz[3 * k + 2] = cloud.points[k].z();
    }
    return n;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// traverseCells (raycast.cpp:48-130). Writes row, col, ray height triples.
REF_API int64_t ref_traverse_cells(const double* origin, const double* endpoint,
                                   double resolution, int width, int height, double center_x,
                                   double center_y, int32_t* rows, int32_t* cols,
                                   double* heights, int64_t capacity) {
  relief::GridSpec spec;
  spec.resolution = resolution;
  spec.width = width;
  spec.height = height;
  spec.center = {center_x, center_y};
  const auto out = relief::traverseCells({origin[0], origin[1], origin[2]},
                                         {endpoint[0], endpoint[1], endpoint[2]}, spec);
  const int64_t n = static_cast<int64_t>(out.size());
  for (int64_t k = 0; k < n && k < capacity; ++k) {
    rows[k] = out[k].index.row;
    cols[k] = out[k].index.col;
    heights[k] = out[k].ray_height;
  }
  return n;
}

// kalmanUpdateCell (integration.cpp:40-55). Returns disposition 0 fused,
// 1 outlier, 2 ignored-low, -1 error (non-positive variance).
REF_API int ref_kalman_update(double h, double sigma_m2, double p_z, double sigma_p2,
                              int cell_count, double mahalanobis_threshold,
                              double sigma_outlier2, int wall_count_threshold,
                              double sigma_max2, double* h_out, double* var_out) {
  relief::UpdateParams p;
  p.mahalanobis_threshold = mahalanobis_threshold;
  p.sigma_outlier2 = sigma_outlier2;
  p.wall_count_threshold = wall_count_threshold;
  p.sigma_max2 = sigma_max2;
  try {
    const relief::CellUpdate u = relief::kalmanUpdateCell(h, sigma_m2, p_z, sigma_p2, cell_count, p);
    *h_out = u.height;
    *var_out = u.variance;
    switch (u.disposition) {
      case relief::Disposition::kFused: return 0;
      case relief::Disposition::kOutlier: return 1;
      case relief::Disposition::kIgnoredLow: return 2;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// smoothChain (postprocess.cpp:166-197) over one masked layer. kinds:
// 0 gaussian, 1 box, 2 median, 3 min_inpaint. Returns 0, or -1 with
// ref_last_error() set (e.g. NothingToInpaint).
REF_API int ref_smooth_chain(const double* values, const uint8_t* valid, int width, int height,
                             const int* kinds, const int* radii, const double* sigmas,
                             int n_steps, double* values_out, uint8_t* valid_out) {
  try {
    relief::MaskedLayer layer;
    const std::size_t n = static_cast<std::size_t>(width) * height;
    layer.values.assign(values, values + n);
    layer.valid.assign(valid, valid + n);
    layer.width = width;
    layer.height = height;
    relief::FilterChainSpec chain;
    for (int s = 0; s < n_steps; ++s) {
      relief::FilterStep step;
      switch (kinds[s]) {
        case 0: step.kind = relief::FilterStep::Kind::kGaussian; break;
        case 1: step.kind = relief::FilterStep::Kind::kBox; break;
        case 2: step.kind = relief::FilterStep::Kind::kMedian; break;
        default: step.kind = relief::FilterStep::Kind::kMinInpaint; break;
      }
      step.radius = radii[s];
      step.sigma = sigmas[s];
      chain.steps.push_back(step);
    }
    const relief::MaskedLayer out = relief::smoothChain(layer, chain);
    std::memcpy(values_out, out.values.data(), n * sizeof(double));
    std::memcpy(valid_out, out.valid.data(), n);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// loadConvNetSpecFile + convFilterInference (analysis.cpp:138-290). Returns 0,
// or the reference ErrorCode + 1 as a negative number (-1 for anything that
// is not a relief::Error) with ref_last_error() set.
REF_API int ref_convnet_infer(const char* model_path, const double* layer, const uint8_t* valid,
                              int width, int height, double* out) {
  try {
    const relief::ConvNetSpec spec = relief::loadConvNetSpecFile(model_path);
    const std::size_t n = static_cast<std::size_t>(width) * height;
    const std::vector<double> in(layer, layer + n);
    const std::vector<std::uint8_t> ok(valid, valid + n);
    const std::vector<double> res = relief::convFilterInference(in, ok, width, height, spec);
    std::memcpy(out, res.data(), n * sizeof(double));
    return 0;
  } catch (const relief::Error& e) {
    g_err = e.what();
    return -(static_cast<int>(e.code()) + 1);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1000;
  }
}

