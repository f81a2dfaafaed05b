// Synthetic scan generator: analytic scenes, ring / grid sensors, trajectory
// interpolation. This is the input generator for tests, bench.py and the
// simulate runner; it is host code and not on the GPU hot path.
//
// It reproduces the reference simulator's arithmetic so a cloud generated
// here is bit-identical to one rendered by the reference (checked by
// tests/test_sim_parity.py): primitives as half-space solids (reference
// sim.cpp:29-140), slab-clipped ray intersection (sim.cpp:142-187), ray fans
// (sim.cpp:222-239), per-ray seeded range noise (sim.cpp:241-262), pose
// interpolation (sim.cpp:284-314), quaternion -> matrix (Eigen 3.4 formula).
#include <algorithm>
#include <cmath>

#include "relief_internal.hpp"

namespace rb200 {

namespace {

// std::min / std::max / std::clamp comparison semantics, spelled out.
inline double lo2(double a, double b) { return (b < a) ? b : a; }
inline double hi2(double a, double b) { return (a < b) ? b : a; }
inline double clampd(double v, double lo, double hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }

inline double dot3(const double a[3], const double b[3]) {
  double s = a[0] * b[0];
  s = s + a[1] * b[1];
  return s + a[2] * b[2];
}

Solid boxSolid(double x0, double y0, double z0, double x1, double y1, double z1) {
  Solid s;
  s.faces = {{{1, 0, 0}, x1},  {{-1, 0, 0}, -x0}, {{0, 1, 0}, y1},
             {{0, -1, 0}, -y0}, {{0, 0, 1}, z1},  {{0, 0, -1}, -z0}};
  return s;
}

void axisDir(Axis a, double& dx, double& dy) {
  switch (a) {
    case Axis::kPosX: dx = 1; dy = 0; return;
    case Axis::kNegX: dx = -1; dy = 0; return;
    case Axis::kPosY: dx = 0; dy = 1; return;
    case Axis::kNegY: dx = 0; dy = -1; return;
  }
  dx = 1;
  dy = 0;
}

}  // namespace

void Scene::addBox(const double c[3], const double sz[3], bool walkable) {
  Solid s = boxSolid(c[0] - 0.5 * sz[0], c[1] - 0.5 * sz[1], c[2] - 0.5 * sz[2],
                     c[0] + 0.5 * sz[0], c[1] + 0.5 * sz[1], c[2] + 0.5 * sz[2]);
  s.walkable = walkable;
  solids.push_back(s);
}

void Scene::addMovingBox(const double c[3], const double sz[3], const double vel[3], double t0,
                         double t1) {
  Solid s = boxSolid(c[0] - 0.5 * sz[0], c[1] - 0.5 * sz[1], c[2] - 0.5 * sz[2],
                     c[0] + 0.5 * sz[0], c[1] + 0.5 * sz[1], c[2] + 0.5 * sz[2]);
  for (int i = 0; i < 3; ++i) s.velocity[i] = vel[i];
  s.active_from = t0;
  s.active_until = t1;
  solids.push_back(s);
}

void Scene::addStairs(const double o[3], double step_h, double step_d, int count, double width,
                      Axis axis) {
  double dx, dy;
  axisDir(axis, dx, dy);
  const double sx = -dy, sy = dx;  // tread-width direction
  for (int k = 0; k < count; ++k) {
    const double ax = o[0] + dx * k * step_d + lo2(0.0, sx * width);
    const double ay = o[1] + dy * k * step_d + lo2(0.0, sy * width);
    const double bx = o[0] + dx * (k + 1) * step_d + hi2(0.0, sx * width);
    const double by = o[1] + dy * (k + 1) * step_d + hi2(0.0, sy * width);
    solids.push_back(boxSolid(lo2(ax, bx), lo2(ay, by), o[2] - 0.5, hi2(ax, bx), hi2(ay, by),
                              o[2] + (k + 1) * step_h));
  }
}

void Scene::addRamp(double x0, double y0, double x1, double y1, double z_base, double slope,
                    Axis axis) {
  Solid s;
  s.faces = {{{1, 0, 0}, x1}, {{-1, 0, 0}, -x0}, {{0, 1, 0}, y1}, {{0, -1, 0}, -y0},
             {{0, 0, -1}, -(z_base - 0.5)}};
  double dx, dy;
  axisDir(axis, dx, dy);
  const double ex = dx > 0 ? x0 : (dx < 0 ? x1 : 0.0);
  const double ey = dy > 0 ? y0 : (dy < 0 ? y1 : 0.0);
  s.faces.push_back({{-slope * dx, -slope * dy, 1.0}, z_base - slope * (dx * ex + dy * ey)});
  solids.push_back(s);
}

void Scene::addWall(double x0, double y0, double x1, double y1, double height, double thickness) {
  const double ddx = x1 - x0, ddy = y1 - y0;
  double lx = lo2(x0, x1), ly = lo2(y0, y1), hx = hi2(x0, x1), hy = hi2(y0, y1);
  if (std::abs(ddx) >= std::abs(ddy)) {
    ly = y0 - 0.5 * thickness;
    hy = y0 + 0.5 * thickness;
    hx = lx + std::abs(ddx);
  } else {
    lx = x0 - 0.5 * thickness;
    hx = x0 + 0.5 * thickness;
    hy = ly + std::abs(ddy);
  }
  solids.push_back(boxSolid(lx, ly, -0.5, hx, hy, height));
}

void Scene::addSlabOverhang(double x0, double y0, double x1, double y1, double z,
                            double thickness) {
  Solid s = boxSolid(x0, y0, z, x1, y1, z + thickness);
  s.walkable = false;
  solids.push_back(s);
}

void Scene::addFloor2(double x0, double y0, double x1, double y1, double z, double hx0,
                      double hy0, double hx1, double hy1, double thickness) {
  const auto piece = [&](double a0, double b0, double a1, double b1) {
    if (a1 - a0 <= 1e-12 || b1 - b0 <= 1e-12) return;
    solids.push_back(boxSolid(a0, b0, z - thickness, a1, b1, z));
  };
  piece(x0, y0, x1, hy0);
  piece(x0, hy1, x1, y1);
  piece(x0, hy0, hx0, hy1);
  piece(hx1, hy0, x1, hy1);
}

double Scene::intersect(const double o[3], const double dir[3], double max_range,
                        double time) const {
  double best = max_range;
  bool hit = false;
  if (has_ground && dir[2] != 0.0) {
    const double t = (ground_z - o[2]) / dir[2];
    if (t > 1e-9 && t < best) {
      best = t;
      hit = true;
    }
  }
  for (const Solid& s : solids) {
    if (!(time >= s.active_from && time <= s.active_until)) continue;
    double shift[3] = {0, 0, 0};
    if (std::isfinite(s.active_from))
      for (int i = 0; i < 3; ++i) shift[i] = s.velocity[i] * (time - s.active_from);
    double t_in = 1e-9, t_out = best;
    bool ok = true;
    for (const Solid::Face& f : s.faces) {
      const double denom = dot3(f.n, dir);
      const double dist = f.d + dot3(f.n, shift) - dot3(f.n, o);
      if (std::abs(denom) < 1e-15) {
        if (dist < 0.0) {
          ok = false;
          break;
        }
        continue;
      }
      const double t = dist / denom;
      if (denom > 0.0) t_out = lo2(t_out, t);
      else t_in = hi2(t_in, t);
      if (t_in > t_out) {
        ok = false;
        break;
      }
    }
    if (ok && t_in < best && t_in > 1e-9) {
      best = t_in;
      hit = true;
    }
  }
  return hit ? best : -1.0;
}

std::vector<std::array<double, 3>> SensorSpec::rayDirections() const {
  validate();
  std::vector<std::array<double, 3>> out;
  const auto push = [&](double elev, double azim) {
    out.push_back({std::cos(elev) * std::cos(azim), std::cos(elev) * std::sin(azim),
                   std::sin(elev)});
  };
  if (pattern == Pattern::kGrid) {
    out.reserve(static_cast<std::size_t>(cols) * rows);
    for (int r = 0; r < rows; ++r) {
      const double elev = rows == 1 ? 0.0 : -0.5 * v_fov + v_fov * r / (rows - 1.0);
      for (int c = 0; c < cols; ++c)
        push(elev, cols == 1 ? 0.0 : -0.5 * h_fov + h_fov * c / (cols - 1.0));
    }
  } else {
    out.reserve(ring_elevations.size() * static_cast<std::size_t>(azimuth_steps));
    for (const double elev : ring_elevations)
      for (int k = 0; k < azimuth_steps; ++k) push(elev, 2.0 * M_PI * k / azimuth_steps);
  }
  return out;
}

std::vector<double> renderScan(const Scene& scene, const Pose& pose, const SensorSpec& spec,
                               double time, std::uint64_t seed, std::uint64_t scan_index) {
  if (!pose.isValid()) fail(Err::kInvalidPose, "rotation is not orthonormal");
  const auto dirs = spec.rayDirections();
  const double sigma_scale = std::sqrt(spec.noise.alpha_d);
  std::vector<double> xyz;
  xyz.reserve(dirs.size() * 3);
  const std::uint64_t scan_seed = SplitMix::mix(seed, scan_index);
  for (std::size_t k = 0; k < dirs.size(); ++k) {
    const auto& d = dirs[k];
    double w[3];
    for (int i = 0; i < 3; ++i) w[i] = (pose.R[i][0] * d[0] + pose.R[i][1] * d[1]) + pose.R[i][2] * d[2];
    const double dist = scene.intersect(pose.t, w, spec.max_range, time);
    if (dist < 0.0) continue;
    double measured = dist;
    if (sigma_scale > 0.0) {
      SplitMix rng(SplitMix::mix(scan_seed, k));
      measured += rng.normal() * sigma_scale * dist;
    }
    xyz.push_back(d[0] * measured);
    xyz.push_back(d[1] * measured);
    xyz.push_back(d[2] * measured);
  }
  return xyz;
}

void Quat::normalize() {
  const double n2 = ((x * x + y * y) + z * z) + w * w;
  if (n2 > 0.0) {
    const double n = std::sqrt(n2);
    x /= n;
    y /= n;
    z /= n;
    w /= n;
  }
}

void Quat::toRotation(double R[3][3]) const {
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  R[0][0] = 1.0 - (tyy + tzz);
  R[0][1] = txy - twz;
  R[0][2] = txz + twy;
  R[1][0] = txy + twz;
  R[1][1] = 1.0 - (txx + tzz);
  R[1][2] = tyz - twx;
  R[2][0] = txz - twy;
  R[2][1] = tyz + twx;
  R[2][2] = 1.0 - (txx + tyy);
}

PoseSample poseAt(const Trajectory& traj, double time) {
  traj.validate();
  const auto& wps = traj.waypoints;
  if (time < wps.front().time - 1e-9 || time > wps.back().time + 1e-9)
    fail(Err::kOutOfTrajectory, "time " + std::to_string(time) + " outside trajectory span");
  std::size_t hi = 1;
  while (hi < wps.size() && wps[hi].time < time) ++hi;
  PoseSample out;
  if (wps.size() == 1 || hi >= wps.size()) {
    for (int i = 0; i < 3; ++i) out.true_pose.t[i] = wps.back().position[i];
    wps.back().orientation.toRotation(out.true_pose.R);
  } else {
    const Waypoint& a = wps[hi - 1];
    const Waypoint& b = wps[hi];
    const double u = clampd((time - a.time) / (b.time - a.time), 0.0, 1.0);
    for (int i = 0; i < 3; ++i) out.true_pose.t[i] = (1.0 - u) * a.position[i] + u * b.position[i];
    Quat qb = b.orientation;
    const double d = ((a.orientation.x * qb.x + a.orientation.y * qb.y) + a.orientation.z * qb.z) +
                     a.orientation.w * qb.w;
    if (d < 0.0) qb = Quat{-qb.x, -qb.y, -qb.z, -qb.w};
    Quat q{(1.0 - u) * a.orientation.x + u * qb.x, (1.0 - u) * a.orientation.y + u * qb.y,
           (1.0 - u) * a.orientation.z + u * qb.z, (1.0 - u) * a.orientation.w + u * qb.w};
    q.normalize();
    q.toRotation(out.true_pose.R);
  }
  out.estimated_pose = out.true_pose;
  out.estimated_pose.t[2] += traj.drift_rate * hi2(0.0, time - traj.drift_start);
  return out;
}

}  // namespace rb200
