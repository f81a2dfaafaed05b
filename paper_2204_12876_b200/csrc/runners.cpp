// Batch runners (simulate / replay / bench / export) driving the device map,
// with the reference's file formats: stats.csv columns and Table-I phase
// labels (reference runner.cpp:57-85), snapshot cadence (runner.cpp:87-119,
// 184-219), cloud / pose CSV readers (runner.cpp:121-182), warm-started bench
// of resampled scans (runner.cpp:221-300) and CSV / PGM export
// (runner.cpp:302-347). Phase times come from CUDA events.
#include "runners.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <filesystem>
#include <fstream>
#include <limits>
#include <memory>
#include <sstream>

#include "snapshot.hpp"

namespace rb200 {

namespace {

constexpr std::array<const char*, 7> kPhaseLabels = {
    "point transform & z error count", "drift compensation", "height update & ray casting",
    "overlap clearance", "traversability", "normal calculation", "total"};

struct MapDeleter {
  void operator()(DeviceMap* m) const { destroyDeviceMap(m); }
};
using MapPtr = std::unique_ptr<DeviceMap, MapDeleter>;

int currentDevice() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) {
    cudaGetLastError();
    d = 0;
  }
  return d;
}

// Stateful wrapper tracking the inter-scan dt (reference integration.hpp:146-169).
class Pipeline {
 public:
  Pipeline(const Grid& g, const PipelineParams& p) : map_(createDeviceMap(currentDevice(), g)), params_(p) {
    map_->phase_events = true;  // the runners report the reference's per-phase timings
  }
  ScanResult integrate(const std::vector<double>& xyz, const Pose& pose, double stamp) {
    if (!pose.isValid()) fail(Err::kInvalidPose, "rotation is not orthonormal");
    const double dt = has_prev_ ? std::max(0.0, stamp - last_) : 0.0;
    ScanResult r = integrateScanDevice(*map_, params_, xyz.data(), xyz.size() / 3, false, pose, stamp, dt);
    last_ = stamp;
    has_prev_ = true;
    return r;
  }
  DeviceMap& map() { return *map_; }
  std::array<double, 7> phases() const {
    std::array<double, 7> a{};
    resolveTiming(*map_);
    for (int k = 0; k < 7; ++k) a[k] = map_->phase_seconds[k];
    return a;
  }

 private:
  MapPtr map_;
  PipelineParams params_;
  double last_ = 0.0;
  bool has_prev_ = false;
};

void ensureDir(const std::string& dir) {
  std::error_code ec;
  std::filesystem::create_directories(dir, ec);
  if (ec) fail(Err::kIo, "cannot create directory: " + dir);
}

std::string snapshotName(const std::string& dir, int index) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "snapshot_%05d.relief", index);
  return dir + "/" + buf;
}

void statsHeader(std::ostream& out) {
  out << "scan,stamp,points_in,points_excluded,points_out_of_range,points_out_of_map,"
         "points_rejected_outlier,points_ignored_low,points_fused,cells_updated,"
         "cells_removed_by_cleanup,cells_cleared_by_overlap,drift_offset_applied,"
         "drift_clamped,drift_points_used,skipped_missing_pose";
  for (const char* l : kPhaseLabels) out << ',' << l;
  out << '\n';
}

void statsRow(std::ostream& out, int scan, double stamp, const ScanResult& s, bool skipped,
              const std::array<double, 7>& phases) {
  out << scan << ',' << formatDouble(stamp) << ',' << s.points_in << ',' << s.excluded << ','
      << s.out_of_range << ',' << s.out_of_map << ',' << s.outlier << ',' << s.ignored_low << ','
      << s.fused << ',' << s.cells_updated << ',' << s.removed << ',' << s.overlap_cleared << ','
      << formatDouble(s.drift_offset) << ',' << (s.drift_clamped ? 1 : 0) << ','
      << s.drift_points << ',' << (skipped ? 1 : 0);
  for (double v : phases) out << ',' << formatDouble(v);
  out << '\n';
}

RunConfig configWithMode(const std::string& path, const char* mode) {
  RunConfig cfg = loadRunConfigFile(path);
  if (mode != nullptr) {
    ExecMode m;
    if (!parseMode(mode, m)) fail(Err::kUsage, "mode must be det or par");
    cfg.pipeline.mode = m;
  }
  return cfg;
}

void saveMap(DeviceMap& m, const std::string& path) { writeSnapshotFile(downloadHost(m), path); }

std::vector<double> loadCloudCsv(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(Err::kIo, "cannot open cloud: " + path);
  std::string line;
  int line_no = 0;
  if (!std::getline(in, line)) fail(Err::kParse, path + ": empty cloud file");
  ++line_no;
  if (!line.empty() && line.back() == '\r') line.pop_back();
  if (line != "x,y,z") fail(Err::kParse, path + " line 1: expected header 'x,y,z'");
  std::vector<double> xyz;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty() || line == "\r") continue;
    double x, y, z;
    char c1, c2;
    std::istringstream row(line);
    if (!(row >> x >> c1 >> y >> c2 >> z) || c1 != ',' || c2 != ',')
      fail(Err::kParse, path + " line " + std::to_string(line_no) + ": expected 'x,y,z' row");
    if (!std::isfinite(x) || !std::isfinite(y) || !std::isfinite(z))
      fail(Err::kParse, path + " line " + std::to_string(line_no) + ": non-finite coordinate");
    xyz.push_back(x);
    xyz.push_back(y);
    xyz.push_back(z);
  }
  return xyz;
}

struct TimedPose {
  double time;
  Pose pose;
};

std::vector<TimedPose> loadPosesCsv(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(Err::kIo, "cannot open poses: " + path);
  std::string line;
  int line_no = 0;
  if (!std::getline(in, line)) fail(Err::kParse, path + ": empty poses file");
  ++line_no;
  if (!line.empty() && line.back() == '\r') line.pop_back();
  if (line != "time,tx,ty,tz,qw,qx,qy,qz")
    fail(Err::kParse, path + " line 1: expected header 'time,tx,ty,tz,qw,qx,qy,qz'");
  std::vector<TimedPose> out;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty() || line == "\r") continue;
    std::replace(line.begin(), line.end(), ',', ' ');
    std::istringstream row(line);
    TimedPose tp{};
    double qw, qx, qy, qz;
    if (!(row >> tp.time >> tp.pose.t[0] >> tp.pose.t[1] >> tp.pose.t[2] >> qw >> qx >> qy >> qz))
      fail(Err::kParse, path + " line " + std::to_string(line_no) + ": expected 8 values");
    Quat q{qx, qy, qz, qw};
    if (std::abs(q.norm() - 1.0) > 1e-6)
      fail(Err::kParse, path + " line " + std::to_string(line_no) + ": quaternion is not normalized");
    q.normalize();
    q.toRotation(tp.pose.R);
    out.push_back(tp);
  }
  return out;
}

}  // namespace

// Loads the conv-net weights named by the config (reference runner.cpp:53-60).
static PipelineParams preparePipeline(const RunConfig& cfg) {
  PipelineParams p = cfg.pipeline;
  if (p.use_convnet_traversability && p.convnet.layers.empty()) {
    if (cfg.convnet_path.empty()) fail(Err::kUsage, "convnet traversability requested without a model");
    p.convnet = loadConvNetSpecFile(cfg.convnet_path);
  }
  return p;
}

bool parseMode(const std::string& m, ExecMode& out) {
  if (m == "det" || m == "deterministic") out = ExecMode::kDeterministic;
  else if (m == "par" || m == "parallel") out = ExecMode::kParallel;
  else return false;
  return true;
}

void runSimulate(const std::string& config_path, const std::string& out_dir, std::uint64_t seed,
                 bool has_seed, const char* mode) {
  RunConfig cfg = configWithMode(config_path, mode);
  if (has_seed) cfg.seed = seed;
  cfg.validate();
  cfg.trajectory.validate();
  ensureDir(out_dir);
  Pipeline pipe(cfg.map, preparePipeline(cfg));
  std::ofstream stats(out_dir + "/stats.csv");
  if (!stats) fail(Err::kIo, "cannot write stats.csv in " + out_dir);
  statsHeader(stats);
  const double t0 = cfg.trajectory.waypoints.front().time;
  for (int s = 0; s < cfg.scans; ++s) {
    const double time = t0 + s / cfg.sensor.rate;
    const PoseSample poses = poseAt(cfg.trajectory, time);
    const std::vector<double> cloud =
        renderScan(cfg.scene, poses.true_pose, cfg.sensor, time, cfg.seed, static_cast<std::uint64_t>(s));
    const ScanResult r = pipe.integrate(cloud, poses.estimated_pose, time);
    statsRow(stats, s, time, r, false, pipe.phases());
    if ((s + 1) % cfg.publish_every == 0) saveMap(pipe.map(), snapshotName(out_dir, s + 1));
  }
  saveMap(pipe.map(), out_dir + "/final.relief");
}

void runReplay(const std::string& config_path, const std::vector<std::string>& clouds,
               const std::string& poses_path, const std::string& out_dir, const char* mode) {
  RunConfig cfg = configWithMode(config_path, mode);
  cfg.validate();
  ensureDir(out_dir);
  const std::vector<TimedPose> poses = loadPosesCsv(poses_path);
  Pipeline pipe(cfg.map, preparePipeline(cfg));
  std::ofstream stats(out_dir + "/stats.csv");
  if (!stats) fail(Err::kIo, "cannot write stats.csv in " + out_dir);
  statsHeader(stats);
  int processed = 0;
  for (std::size_t k = 0; k < clouds.size(); ++k) {
    const int scan = static_cast<int>(k);
    if (k >= poses.size()) {
      statsRow(stats, scan, 0.0, ScanResult{}, true, std::array<double, 7>{});
      continue;
    }
    const std::vector<double> cloud = loadCloudCsv(clouds[k]);
    const ScanResult r = pipe.integrate(cloud, poses[k].pose, poses[k].time);
    statsRow(stats, scan, poses[k].time, r, false, pipe.phases());
    ++processed;
    if (processed % cfg.publish_every == 0) saveMap(pipe.map(), snapshotName(out_dir, processed));
  }
  saveMap(pipe.map(), out_dir + "/final.relief");
}

void runBench(const std::string& config_path, const std::vector<std::size_t>& counts,
              int repetitions, const std::string& out_csv, const char* mode) {
  RunConfig cfg = configWithMode(config_path, mode);
  cfg.validate();
  if (repetitions < 1) fail(Err::kUsage, "repetitions must be >= 1");
  Scene scene = cfg.scene;
  if (!scene.has_ground && scene.solids.empty()) scene.addGround(0.0);
  Pose pose;
  pose.t[2] = 1.0;
  if (!cfg.trajectory.waypoints.empty())
    pose = poseAt(cfg.trajectory, cfg.trajectory.waypoints.front().time).true_pose;
  const std::vector<double> ref = renderScan(scene, pose, cfg.sensor, 0.0, cfg.seed, 0);
  const std::size_t nref = ref.size() / 3;
  if (nref == 0) fail(Err::kUsage, "benchmark scene yields no returns");

  std::vector<std::pair<std::size_t, std::array<double, 7>>> rows;
  for (const std::size_t count : counts) {
    SplitMix rng(SplitMix::mix(cfg.seed, count));
    std::vector<double> cloud;
    cloud.reserve(count * 3);
    for (std::size_t i = 0; i < count; ++i) {
      const std::size_t pick = rng.next() % nref;
      cloud.insert(cloud.end(), ref.begin() + 3 * pick, ref.begin() + 3 * pick + 3);
    }
    Pipeline pipe(cfg.map, preparePipeline(cfg));
    {
      // Warm start: one untimed scan with a point at every cell centre.
      const Grid& g = pipe.map().grid;
      std::vector<double> fill;
      fill.reserve(g.cells() * 3);
      const double ox = g.originX(), oy = g.originY();
      for (int r = 0; r < g.height; ++r) {
        for (int c = 0; c < g.width; ++c) {
          const double v[3] = {ox + (c + 0.5) * g.resolution - pose.t[0],
                               oy + (r + 0.5) * g.resolution - pose.t[1], 0.0 - pose.t[2]};
          for (int i = 0; i < 3; ++i)
            fill.push_back((pose.R[0][i] * v[0] + pose.R[1][i] * v[1]) + pose.R[2][i] * v[2]);
        }
      }
      pipe.integrate(fill, pose, -1.0);
    }
    std::vector<std::array<double, 7>> samples;
    for (int rep = 0; rep < repetitions; ++rep) {
      pipe.integrate(cloud, pose, rep / cfg.sensor.rate);
      samples.push_back(pipe.phases());
    }
    std::array<double, 7> med{};
    for (int ph = 0; ph < 7; ++ph) {
      std::vector<double> v;
      for (const auto& s : samples) v.push_back(s[ph]);
      std::sort(v.begin(), v.end());
      med[ph] = v[v.size() / 2];
    }
    rows.emplace_back(count, med);
  }
  if (!out_csv.empty()) {
    std::ofstream out(out_csv);
    if (!out) fail(Err::kIo, "cannot write " + out_csv);
    out << "number of points";
    for (const char* l : kPhaseLabels) out << ',' << l;
    out << '\n';
    for (const auto& row : rows) {
      out << row.first;
      for (double v : row.second) out << ',' << formatDouble(v);
      out << '\n';
    }
  }
}

void runExport(const std::string& snapshot_path, const std::string& layer, bool pgm,
               const std::string& out_path) {
  const HostLayers h = readSnapshotFile(snapshot_path);
  const auto& names = layerNames();
  const auto it = std::find(names.begin(), names.end(), layer);
  if (it == names.end()) fail(Err::kUsage, unknownLayerMessage(layer));
  const std::vector<double> values = h.masked(static_cast<int>(it - names.begin()));
  std::ofstream out(out_path);
  if (!out) fail(Err::kIo, "cannot write " + out_path);
  const int W = h.grid.width, H = h.grid.height;
  if (!pgm) {
    for (int r = 0; r < H; ++r) {
      for (int c = 0; c < W; ++c) {
        const double v = values[static_cast<std::size_t>(r) * W + c];
        if (c) out << ',';
        if (std::isnan(v)) out << "nan";
        else out << formatDouble(v);
      }
      out << '\n';
    }
    return;
  }
  double lo = std::numeric_limits<double>::infinity();
  double hi = -std::numeric_limits<double>::infinity();
  for (double v : values) {
    if (std::isnan(v)) continue;
    lo = (v < lo) ? v : lo;
    hi = (hi < v) ? v : hi;
  }
  if (!std::isfinite(lo)) lo = hi = 0.0;
  out << "P2\n# scale min " << formatDouble(lo) << " max " << formatDouble(hi) << " invalid 0\n";
  out << W << " " << H << "\n65535\n";
  for (int r = 0; r < H; ++r) {
    for (int c = 0; c < W; ++c) {
      const double v = values[static_cast<std::size_t>(r) * W + c];
      int gray = 0;
      if (!std::isnan(v))
        gray = hi > lo ? static_cast<int>(std::lround((v - lo) / (hi - lo) * 65535.0)) : 65535;
      if (c) out << ' ';
      out << gray;
    }
    out << '\n';
  }
}

// Reference capi.cpp:320-332 + runner.cpp:349-362: parameters from the config
// first (if any), then the snapshot.
std::size_t runSegment(const std::string& snapshot_path, const char* config_path,
                       const std::string& out_path) {
  PlaneSegParams params;
  if (config_path != nullptr) params = loadRunConfigFile(config_path).segmentation;
  return segmentSnapshot(snapshot_path, params, out_path);
}

}  // namespace rb200
