// Run-configuration reader and parameter validation.
//
// Accepts the reference's flat `section.key = value` format with the same key
// set, defaults, degree->radian conversions, validation rules and error texts
// (reference config.cpp:25-261, types.hpp:87-140, integration.hpp:45-50,
// drift.hpp:33-35, raycast.hpp:34-37, analysis.hpp:38-47,68-72,
// postprocess.hpp:68-72, sim.hpp:124-133,150-156). The parser is table
// driven: one handler per key.
#include <fstream>
#include <functional>
#include <sstream>
#include <unordered_map>

#include "relief_internal.hpp"

namespace rb200 {

// ------------------------------------------------------------- validation
bool Pose::isValid(double tol) const {
  // (R^T R - I), each entry a left-to-right dot of two columns of R.
  double worst = 0.0;
  bool first = true;
  for (int c = 0; c < 3; ++c) {      // column-major walk, as the oracle's
    for (int r = 0; r < 3; ++r) {    // cwiseAbs().maxCoeff()
      double s = R[0][r] * R[0][c];
      s = s + R[1][r] * R[1][c];
      s = s + R[2][r] * R[2][c];
      const double e = std::abs(s - (r == c ? 1.0 : 0.0));
      if (first) {
        worst = e;
        first = false;
      } else if (e > worst) {
        worst = e;
      }
    }
  }
  const double det = R[0][0] * (R[1][1] * R[2][2] - R[1][2] * R[2][1]) -
                     R[0][1] * (R[1][0] * R[2][2] - R[1][2] * R[2][0]) +
                     R[0][2] * (R[1][0] * R[2][1] - R[1][1] * R[2][0]);
  return worst <= tol && std::abs(det - 1.0) <= tol;
}

void ExclusionParams::validate() const {
  if (theta_a < 0.0 || theta_a >= 1.5707963267948966)
    fail(Err::kUsage, "theta_a must lie in [0, pi/2)");
  if (b < 0.0 || c < 0.0) fail(Err::kUsage, "b and c must be >= 0");
  if (d_max <= b) fail(Err::kUsage, "d_max must exceed b");
}

void UpdateParams::validate() const {
  if (mahalanobis_threshold <= 0.0) fail(Err::kUsage, "mahalanobis_threshold must be > 0");
  if (wall_count_threshold < 1) fail(Err::kUsage, "wall_count_threshold must be >= 1");
}

void DriftParams::validate() const {
  if (min_points < 1) fail(Err::kUsage, "min_points must be >= 1");
}

void CleanupParams::validate() const {
  if (alpha_n < 0.0 || alpha_n > 1.0) fail(Err::kUsage, "alpha_n must lie in [0, 1]");
}

void TraversabilityParams::validate() const {
  if (window < 3 || window % 2 == 0) fail(Err::kUsage, "window must be odd and >= 3");
  if (slope_max <= 0.0 || step_max <= 0.0 || roughness_max <= 0.0)
    fail(Err::kUsage, "traversability maxima must be > 0");
  if (w_slope < 0.0 || w_step < 0.0 || w_roughness < 0.0 ||
      std::abs(w_slope + w_step + w_roughness - 1.0) > 1e-9)
    fail(Err::kUsage, "weights must be nonnegative and sum to 1");
}

void OverlapParams::validate() const {
  if (radius <= 0.0 || height_threshold <= 0.0)
    fail(Err::kUsage, "overlap radius and threshold must be > 0");
}

void PlaneSegParams::validate() const {
  if (normal_angle_max <= 0.0 || dist_max <= 0.0 || min_region_cells <= 0 ||
      polygon_simplify_tol < 0.0)
    fail(Err::kUsage, "plane segmentation params must be positive");
}

void SensorSpec::validate() const {
  if (max_range <= 0.0) fail(Err::kUsage, "max_range must be > 0");
  if (pattern == Pattern::kGrid && (cols < 1 || rows < 1))
    fail(Err::kUsage, "grid pattern needs cols, rows >= 1");
  if (pattern == Pattern::kRings && (ring_elevations.empty() || azimuth_steps < 1))
    fail(Err::kUsage, "rings pattern needs elevations and steps");
  if (rate <= 0.0) fail(Err::kUsage, "rate must be > 0");
}

void Trajectory::validate() const {
  if (waypoints.empty()) fail(Err::kUsage, "trajectory needs waypoints");
  for (std::size_t i = 1; i < waypoints.size(); ++i)
    if (waypoints[i].time <= waypoints[i - 1].time)
      fail(Err::kUsage, "waypoint times must strictly increase");
}

void RunConfig::validate() const {
  map.validate();
  pipeline.update.validate();
  pipeline.update.exclusion.validate();
  pipeline.drift.validate();
  pipeline.cleanup.validate();
  pipeline.traversability.validate();
  pipeline.overlap.validate();
  segmentation.validate();
  sensor.validate();
  if (scans < 0) fail(Err::kUsage, "run.scans must be >= 0");
  if (publish_every < 1) fail(Err::kUsage, "run.publish_every must be >= 1");
}

std::string formatDouble(double v) {
  char buf[32];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

// ---------------------------------------------------------------- parsing
namespace {

constexpr double kDeg = 0.017453292519943295;

class Values {
 public:
  Values(const std::string& text, int line) : in_(text), line_(line) {}

  [[noreturn]] void bad(const std::string& what) const {
    fail(Err::kParse, "config line " + std::to_string(line_) + ": " + what);
  }
  double num() {
    double v;
    if (!(in_ >> v)) bad("expected a number");
    return v;
  }
  int integer() { return static_cast<int>(num()); }
  bool flag() {
    std::string w;
    if (!(in_ >> w)) bad("expected true/false");
    if (w == "true" || w == "1" || w == "on") return true;
    if (w == "false" || w == "0" || w == "off") return false;
    bad("expected true/false, got '" + w + "'");
  }
  std::string word() {
    std::string w;
    if (!(in_ >> w)) bad("expected a word");
    return w;
  }
  bool more() {
    in_ >> std::ws;
    return in_.peek() != EOF;
  }
  Axis axis() {
    if (!more()) return Axis::kPosX;
    const std::string w = word();
    if (w == "+x") return Axis::kPosX;
    if (w == "-x") return Axis::kNegX;
    if (w == "+y") return Axis::kPosY;
    if (w == "-y") return Axis::kNegY;
    bad("axis must be one of +x -x +y -y");
  }
  void done() {
    if (more()) bad("trailing values");
  }

 private:
  std::istringstream in_;
  int line_;
};

struct ParseState {
  RunConfig cfg;
  bool pattern_set = false;
};

using Handler = std::function<void(ParseState&, Values&)>;

const std::unordered_map<std::string, Handler>& handlers() {
  static const std::unordered_map<std::string, Handler> table = [] {
    std::unordered_map<std::string, Handler> h;
    auto& H = h;
    // map geometry
    H["map.resolution"] = [](ParseState& s, Values& v) { s.cfg.map.resolution = v.num(); };
    H["map.width"] = [](ParseState& s, Values& v) { s.cfg.map.width = v.integer(); };
    H["map.height"] = [](ParseState& s, Values& v) { s.cfg.map.height = v.integer(); };
    H["map.center_x"] = [](ParseState& s, Values& v) { s.cfg.map.center_x = v.num(); };
    H["map.center_y"] = [](ParseState& s, Values& v) { s.cfg.map.center_y = v.num(); };
    // height update
    auto U = [](ParseState& s) -> UpdateParams& { return s.cfg.pipeline.update; };
    H["update.mahalanobis_threshold"] = [U](ParseState& s, Values& v) { U(s).mahalanobis_threshold = v.num(); };
    H["update.sigma_outlier2"] = [U](ParseState& s, Values& v) { U(s).sigma_outlier2 = v.num(); };
    H["update.wall_count_threshold"] = [U](ParseState& s, Values& v) { U(s).wall_count_threshold = v.integer(); };
    H["update.sigma_t2"] = [U](ParseState& s, Values& v) { U(s).sigma_t2 = v.num(); };
    H["update.sigma_max2"] = [U](ParseState& s, Values& v) { U(s).sigma_max2 = v.num(); };
    H["update.sigma_init2"] = [U](ParseState& s, Values& v) { U(s).sigma_init2 = v.num(); };
    H["update.nominal_period"] = [U](ParseState& s, Values& v) { U(s).nominal_update_period = v.num(); };
    H["update.max_range"] = [U](ParseState& s, Values& v) { U(s).max_range = v.num(); };
    // one noise model for the renderer and for fusion weights
    H["noise.alpha_d"] = [](ParseState& s, Values& v) {
      s.cfg.pipeline.update.noise.alpha_d = v.num();
      s.cfg.sensor.noise.alpha_d = s.cfg.pipeline.update.noise.alpha_d;
    };
    H["noise.sigma_p_min2"] = [](ParseState& s, Values& v) {
      s.cfg.pipeline.update.noise.sigma_p_min2 = v.num();
      s.cfg.sensor.noise.sigma_p_min2 = s.cfg.pipeline.update.noise.sigma_p_min2;
    };
    // exclusion ramp
    auto X = [](ParseState& s) -> ExclusionParams& { return s.cfg.pipeline.update.exclusion; };
    H["exclusion.enabled"] = [X](ParseState& s, Values& v) { X(s).enabled = v.flag(); };
    H["exclusion.theta_a_deg"] = [X](ParseState& s, Values& v) { X(s).theta_a = v.num() * kDeg; };
    H["exclusion.b"] = [X](ParseState& s, Values& v) { X(s).b = v.num(); };
    H["exclusion.c"] = [X](ParseState& s, Values& v) { X(s).c = v.num(); };
    H["exclusion.d_max"] = [X](ParseState& s, Values& v) { X(s).d_max = v.num(); };
    // drift
    auto D = [](ParseState& s) -> DriftParams& { return s.cfg.pipeline.drift; };
    H["drift.enabled"] = [D](ParseState& s, Values& v) { D(s).enabled = v.flag(); };
    H["drift.traversability_threshold"] = [D](ParseState& s, Values& v) { D(s).traversability_threshold = v.num(); };
    H["drift.min_points"] = [D](ParseState& s, Values& v) { D(s).min_points = v.integer(); };
    H["drift.max_offset"] = [D](ParseState& s, Values& v) { D(s).max_offset_per_scan = v.num(); };
    // ray-cast cleanup
    auto C = [](ParseState& s) -> CleanupParams& { return s.cfg.pipeline.cleanup; };
    H["cleanup.enabled"] = [C](ParseState& s, Values& v) { C(s).cleanup_enabled = v.flag(); };
    H["cleanup.upper_bound_enabled"] = [C](ParseState& s, Values& v) { C(s).upper_bound_enabled = v.flag(); };
    H["cleanup.alpha_n"] = [C](ParseState& s, Values& v) { C(s).alpha_n = v.num(); };
    H["cleanup.t_free"] = [C](ParseState& s, Values& v) { C(s).t_free = v.num(); };
    // traversability
    auto T = [](ParseState& s) -> TraversabilityParams& { return s.cfg.pipeline.traversability; };
    H["traversability.slope_max_deg"] = [T](ParseState& s, Values& v) { T(s).slope_max = v.num() * kDeg; };
    H["traversability.step_max"] = [T](ParseState& s, Values& v) { T(s).step_max = v.num(); };
    H["traversability.roughness_max"] = [T](ParseState& s, Values& v) { T(s).roughness_max = v.num(); };
    H["traversability.window"] = [T](ParseState& s, Values& v) { T(s).window = v.integer(); };
    H["traversability.weights"] = [T](ParseState& s, Values& v) {
      T(s).w_slope = v.num();
      T(s).w_step = v.num();
      T(s).w_roughness = v.num();
    };
    H["traversability.convnet"] = [](ParseState& s, Values& v) {
      s.cfg.convnet_path = v.word();
      s.cfg.pipeline.use_convnet_traversability = true;
    };
    // overlap clearance
    auto O = [](ParseState& s) -> OverlapParams& { return s.cfg.pipeline.overlap; };
    H["overlap.enabled"] = [O](ParseState& s, Values& v) { O(s).enabled = v.flag(); };
    H["overlap.radius"] = [O](ParseState& s, Values& v) { O(s).radius = v.num(); };
    H["overlap.height_threshold"] = [O](ParseState& s, Values& v) { O(s).height_threshold = v.num(); };
    // segmentation (host-side, on demand)
    auto P = [](ParseState& s) -> PlaneSegParams& { return s.cfg.segmentation; };
    H["segmentation.normal_angle_max_deg"] = [P](ParseState& s, Values& v) { P(s).normal_angle_max = v.num() * kDeg; };
    H["segmentation.dist_max"] = [P](ParseState& s, Values& v) { P(s).dist_max = v.num(); };
    H["segmentation.min_region_cells"] = [P](ParseState& s, Values& v) { P(s).min_region_cells = v.integer(); };
    H["segmentation.simplify_tol"] = [P](ParseState& s, Values& v) { P(s).polygon_simplify_tol = v.num(); };
    // virtual sensor
    auto S = [](ParseState& s) -> SensorSpec& { return s.cfg.sensor; };
    H["sensor.pattern"] = [S](ParseState& s, Values& v) {
      const std::string w = v.word();
      if (w == "grid") S(s).pattern = SensorSpec::Pattern::kGrid;
      else if (w == "rings") S(s).pattern = SensorSpec::Pattern::kRings;
      else v.bad("sensor.pattern must be grid or rings");
      s.pattern_set = true;
    };
    H["sensor.h_fov_deg"] = [S](ParseState& s, Values& v) { S(s).h_fov = v.num() * kDeg; };
    H["sensor.v_fov_deg"] = [S](ParseState& s, Values& v) { S(s).v_fov = v.num() * kDeg; };
    H["sensor.cols"] = [S](ParseState& s, Values& v) { S(s).cols = v.integer(); };
    H["sensor.rows"] = [S](ParseState& s, Values& v) { S(s).rows = v.integer(); };
    H["sensor.ring_elevations_deg"] = [S](ParseState& s, Values& v) {
      S(s).ring_elevations.clear();
      while (v.more()) S(s).ring_elevations.push_back(v.num() * kDeg);
      if (!s.pattern_set) S(s).pattern = SensorSpec::Pattern::kRings;
    };
    H["sensor.azimuth_steps"] = [S](ParseState& s, Values& v) { S(s).azimuth_steps = v.integer(); };
    H["sensor.max_range"] = [S](ParseState& s, Values& v) { S(s).max_range = v.num(); };
    H["sensor.rate"] = [S](ParseState& s, Values& v) { S(s).rate = v.num(); };
    // scene primitives
    H["scene.ground"] = [](ParseState& s, Values& v) { s.cfg.scene.addGround(v.num()); };
    H["scene.box"] = [](ParseState& s, Values& v) {
      double c[3], sz[3];
      for (double& x : c) x = v.num();
      for (double& x : sz) x = v.num();
      s.cfg.scene.addBox(c, sz);
    };
    H["scene.moving_box"] = [](ParseState& s, Values& v) {
      double c[3], sz[3], vel[3];
      for (double& x : c) x = v.num();
      for (double& x : sz) x = v.num();
      for (double& x : vel) x = v.num();
      const double t0 = v.num();
      const double t1 = v.num();
      s.cfg.scene.addMovingBox(c, sz, vel, t0, t1);
    };
    H["scene.stairs"] = [](ParseState& s, Values& v) {
      double o[3];
      for (double& x : o) x = v.num();
      const double sh = v.num();
      const double sd = v.num();
      const int count = v.integer();
      const double width = v.num();
      s.cfg.scene.addStairs(o, sh, sd, count, width, v.axis());
    };
    H["scene.ramp"] = [](ParseState& s, Values& v) {
      const double x0 = v.num(), y0 = v.num(), x1 = v.num(), y1 = v.num();
      const double zb = v.num(), slope = v.num();
      s.cfg.scene.addRamp(x0, y0, x1, y1, zb, slope, v.axis());
    };
    H["scene.wall"] = [](ParseState& s, Values& v) {
      const double x0 = v.num(), y0 = v.num(), x1 = v.num(), y1 = v.num();
      const double height = v.num(), thickness = v.num();
      s.cfg.scene.addWall(x0, y0, x1, y1, height, thickness);
    };
    H["scene.slab_overhang"] = [](ParseState& s, Values& v) {
      const double x0 = v.num(), y0 = v.num(), x1 = v.num(), y1 = v.num();
      const double z = v.num();
      const double th = v.more() ? v.num() : 0.1;
      s.cfg.scene.addSlabOverhang(x0, y0, x1, y1, z, th);
    };
    H["scene.floor2"] = [](ParseState& s, Values& v) {
      const double x0 = v.num(), y0 = v.num(), x1 = v.num(), y1 = v.num();
      const double z = v.num();
      const double hx0 = v.num(), hy0 = v.num(), hx1 = v.num(), hy1 = v.num();
      const double th = v.more() ? v.num() : 0.1;
      s.cfg.scene.addFloor2(x0, y0, x1, y1, z, hx0, hy0, hx1, hy1, th);
    };
    // trajectory
    H["traj.waypoint"] = [](ParseState& s, Values& v) {
      Waypoint wp;
      wp.time = v.num();
      for (double& x : wp.position) x = v.num();
      if (v.more()) {
        const double qw = v.num(), qx = v.num(), qy = v.num(), qz = v.num();
        wp.orientation = Quat{qx, qy, qz, qw};
        if (std::abs(wp.orientation.norm() - 1.0) > 1e-6)
          v.bad("waypoint quaternion is not normalized");
        wp.orientation.normalize();
      }
      s.cfg.trajectory.waypoints.push_back(wp);
    };
    H["traj.drift_rate"] = [](ParseState& s, Values& v) { s.cfg.trajectory.drift_rate = v.num(); };
    H["traj.drift_start"] = [](ParseState& s, Values& v) { s.cfg.trajectory.drift_start = v.num(); };
    // run knobs
    H["run.scans"] = [](ParseState& s, Values& v) { s.cfg.scans = v.integer(); };
    H["run.publish_every"] = [](ParseState& s, Values& v) { s.cfg.publish_every = v.integer(); };
    H["run.seed"] = [](ParseState& s, Values& v) { s.cfg.seed = static_cast<std::uint64_t>(v.num()); };
    H["run.mode"] = [](ParseState& s, Values& v) {
      const std::string w = v.word();
      if (w == "det" || w == "deterministic") s.cfg.pipeline.mode = ExecMode::kDeterministic;
      else if (w == "par" || w == "parallel") s.cfg.pipeline.mode = ExecMode::kParallel;
      else v.bad("run.mode must be det or par");
    };
    return h;
  }();
  return table;
}

}  // namespace

RunConfig parseRunConfig(const std::string& text) {
  ParseState st;
  std::istringstream in(text);
  std::string line;
  int line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    const std::size_t hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    const std::size_t first = line.find_first_not_of(" \t\r");
    if (first == std::string::npos) continue;
    const std::size_t eq = line.find('=');
    if (eq == std::string::npos)
      fail(Err::kParse, "config line " + std::to_string(line_no) + ": expected 'key = value'");
    std::string key = line.substr(first, eq - first);
    key.erase(key.find_last_not_of(" \t") + 1);
    Values values(line.substr(eq + 1), line_no);
    const auto it = handlers().find(key);
    if (it == handlers().end()) values.bad("unknown key '" + key + "'");
    it->second(st, values);
    if (key != "sensor.ring_elevations_deg") values.done();
  }
  st.cfg.validate();
  return st.cfg;
}

RunConfig loadRunConfigFile(const std::string& path) {
  std::ifstream f(path);
  if (!f) fail(Err::kIo, "cannot open config: " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return parseRunConfig(ss.str());
}

}  // namespace rb200
