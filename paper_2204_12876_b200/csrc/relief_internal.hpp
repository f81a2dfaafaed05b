// Host-side types of the B200 elevation-map engine.
//
// Parameter structs keep the reference's field names and defaults so that a
// reliefmap config file means the same thing here (reference
// integration.hpp:33-63, drift.hpp:27-36, raycast.hpp:28-38,
// analysis.hpp:29-76, types.hpp:77-140, postprocess.hpp:28-73, sim.hpp:110-160).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace rb200 {

// Error codes; map 1:1 onto relief_status through capi.cpp (reference
// types.hpp:34-45, capi.cpp:43-58).
enum class Err {
  kOutOfMap,
  kInvalidPose,
  kInvalidVariance,
  kInvalidModel,
  kDegeneratePlane,
  kNothingToInpaint,
  kOutOfTrajectory,
  kParse,
  kIo,
  kUsage,
  kDevice,
};

class Error : public std::runtime_error {
 public:
  Error(Err code, const std::string& what) : std::runtime_error(what), code_(code) {}
  Err code() const { return code_; }

 private:
  Err code_;
};

[[noreturn]] inline void fail(Err code, const std::string& what) { throw Error(code, what); }

// ---------------------------------------------------------------- geometry
// Fixed W x H robot-centric grid, row = y, col = x, linear index r*W + c,
// covering [center - extent/2, center + extent/2) (reference types.hpp:77-92).
struct Grid {
  double resolution = 0.04;
  int width = 250;
  int height = 250;
  double center_x = 0.0;
  double center_y = 0.0;

  double originX() const { return center_x - 0.5 * (width * resolution); }
  double originY() const { return center_y - 0.5 * (height * resolution); }
  std::size_t cells() const { return static_cast<std::size_t>(width) * height; }
  void validate() const {
    if (resolution <= 0.0) fail(Err::kUsage, "resolution must be > 0");
    if (width < 3 || height < 3) fail(Err::kUsage, "grid must be at least 3x3 cells");
  }
};

// Row-major 3x3 rotation + translation (reference types.hpp:107-117).
struct Pose {
  double R[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  double t[3] = {0, 0, 0};

  static Pose fromRowMajor34(const double* p) {
    Pose out;
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) out.R[r][c] = p[4 * r + c];
      out.t[r] = p[4 * r + 3];
    }
    return out;
  }
  // max|R^T R - I| <= tol and |det R - 1| <= tol; sums left to right and the
  // first-row cofactor determinant, as the oracle's pinned Eigen arithmetic.
  bool isValid(double tol = 1e-9) const;
};

// -------------------------------------------------------------- parameters
struct NoiseParams {
  double alpha_d = 0.01;
  double sigma_p_min2 = 1e-4;
};

struct ExclusionParams {
  bool enabled = true;
  double theta_a = 0.785398163397448;
  double b = 0.5;
  double c = 0.2;
  double d_max = 1.0;
  void validate() const;
};

struct UpdateParams {
  double mahalanobis_threshold = 2.5;
  double sigma_outlier2 = 0.01;
  int wall_count_threshold = 5;
  double sigma_t2 = 0.01;
  double sigma_max2 = 100.0;
  double sigma_init2 = 100.0;
  double nominal_update_period = 0.1;
  double max_range = 10.0;
  NoiseParams noise;
  ExclusionParams exclusion;
  void validate() const;
};

struct DriftParams {
  bool enabled = true;
  double traversability_threshold = 0.7;
  int min_points = 10;
  double max_offset_per_scan = 0.1;
  void validate() const;
};

struct CleanupParams {
  bool cleanup_enabled = true;
  bool upper_bound_enabled = true;
  double alpha_n = 0.2;
  double t_free = 1.0;
  void validate() const;
};

struct TraversabilityParams {
  double slope_max = 0.785398163397448;
  double step_max = 0.2;
  double roughness_max = 0.1;
  int window = 5;
  double w_slope = 0.4;
  double w_step = 0.3;
  double w_roughness = 0.3;
  void validate() const;
};

struct OverlapParams {
  bool enabled = true;
  double radius = 1.0;
  double height_threshold = 1.5;
  void validate() const;
};

enum class ExecMode { kDeterministic, kParallel };

// Learned traversability filter: a stack of k x k border-replicate
// convolutions over the nearest-valid-filled elevation (reference
// analysis.hpp:44-65, analysis.cpp:27-39,138-216).
enum class Activation { kRelu, kSigmoid, kIdentity };

struct ConvLayer {
  int kernel_size = 1;          // odd
  std::vector<double> kernel;   // kernel_size^2, row-major
  double bias = 0.0;
  Activation activation = Activation::kIdentity;
};

struct ConvNetSpec {
  std::vector<ConvLayer> layers;
  void validate() const;
};

// Weight file reader (reference analysis.cpp:218-290), same grammar and errors.
ConvNetSpec loadConvNetSpecText(const std::string& text);
ConvNetSpec loadConvNetSpecFile(const std::string& path);

struct PipelineParams {
  UpdateParams update;
  DriftParams drift;
  CleanupParams cleanup;
  TraversabilityParams traversability;
  OverlapParams overlap;
  ExecMode mode = ExecMode::kDeterministic;
  bool use_convnet_traversability = false;
  ConvNetSpec convnet;  // loaded by the runners / relief_gpu_config_load_convnet
};

struct PlaneSegParams {
  double normal_angle_max = 0.3490658503988659;
  double dist_max = 0.02;
  int min_region_cells = 50;
  double polygon_simplify_tol = 0.0;
  void validate() const;
};

// ----------------------------------------------------- synthetic scene input
enum class Axis { kPosX, kNegX, kPosY, kNegY };

// Convex solid as half-spaces n.p <= d (reference sim.hpp:29-49).
struct Solid {
  struct Face {
    double n[3];
    double d;
  };
  std::vector<Face> faces;
  bool walkable = true;
  double velocity[3] = {0, 0, 0};
  double active_from = -INFINITY;
  double active_until = INFINITY;
};

struct Scene {
  bool has_ground = false;
  double ground_z = 0.0;
  std::vector<Solid> solids;

  void addGround(double z) {
    has_ground = true;
    ground_z = z;
  }
  void addBox(const double center[3], const double size[3], bool walkable = true);
  void addMovingBox(const double center[3], const double size[3], const double vel[3],
                    double t0, double t1);
  void addStairs(const double origin[3], double step_h, double step_d, int count, double width,
                 Axis axis);
  void addRamp(double x0, double y0, double x1, double y1, double z_base, double slope, Axis axis);
  void addWall(double x0, double y0, double x1, double y1, double height, double thickness);
  void addSlabOverhang(double x0, double y0, double x1, double y1, double z, double thickness);
  void addFloor2(double x0, double y0, double x1, double y1, double z, double hx0, double hy0,
                 double hx1, double hy1, double thickness);
  // Nearest hit distance along dir (t > 0) or a negative value for a miss.
  double intersect(const double o[3], const double dir[3], double max_range, double time) const;
};

struct SensorSpec {
  enum class Pattern { kGrid, kRings };
  Pattern pattern = Pattern::kGrid;
  double h_fov = 1.5707963267948966;
  double v_fov = 1.0471975511965976;
  int cols = 80;
  int rows = 40;
  std::vector<double> ring_elevations;
  int azimuth_steps = 180;
  double max_range = 10.0;
  NoiseParams noise;
  double rate = 10.0;
  void validate() const;
  std::vector<std::array<double, 3>> rayDirections() const;
};

struct Quat {
  double x = 0, y = 0, z = 0, w = 1;  // Eigen coefficient order x y z w
  double norm() const { return std::sqrt(((x * x + y * y) + z * z) + w * w); }
  void normalize();
  void toRotation(double R[3][3]) const;
};

struct Waypoint {
  double time = 0.0;
  double position[3] = {0, 0, 0};
  Quat orientation;
};

struct Trajectory {
  std::vector<Waypoint> waypoints;
  double drift_rate = 0.0;
  double drift_start = 0.0;
  void validate() const;
};

struct PoseSample {
  Pose true_pose;
  Pose estimated_pose;
};
PoseSample poseAt(const Trajectory& traj, double time);

// Renders one scan (reference sim.cpp:241-262): per ray the nearest hit with
// range noise sqrt(alpha_d)*dist drawn from splitmix64(mix(mix(seed,scan),k)).
std::vector<double> renderScan(const Scene& scene, const Pose& pose, const SensorSpec& spec,
                               double time, std::uint64_t seed, std::uint64_t scan_index);

// --------------------------------------------------------------- run config
struct RunConfig {
  Grid map;
  PipelineParams pipeline;
  PlaneSegParams segmentation;
  Scene scene;
  SensorSpec sensor;
  Trajectory trajectory;
  int scans = 50;
  int publish_every = 5;
  std::uint64_t seed = 0;
  std::string convnet_path;
  void validate() const;
};

RunConfig loadRunConfigFile(const std::string& path);
RunConfig parseRunConfig(const std::string& text);

// splitmix64 (reference rng.hpp:28-60), used by the scene renderer.
struct SplitMix {
  std::uint64_t state;
  explicit SplitMix(std::uint64_t s) : state(s) {}
  std::uint64_t next() {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double uniform() { return (static_cast<double>(next() >> 11) + 1.0) * (1.0 / 9007199254740992.0); }
  double normal() {
    const double u1 = uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
  static std::uint64_t mix(std::uint64_t a, std::uint64_t b) {
    std::uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
};

std::string formatDouble(double v);  // "%.17g"

}  // namespace rb200
