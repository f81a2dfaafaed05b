// Plane segmentation of a map snapshot, on the host.
//
// The reference runs it on demand on the CPU (runner.cpp:349-362 ->
// postprocess.cpp:199-545): a sequential greedy region growing (seeds taken
// flattest first, each region claims its cells before the next seed), so it
// stays host code here too. Same decisions, same output text:
//   * seeds: valid cells with a normal, stable-sorted by normal_z descending;
//   * growth: 4-neighbour BFS levels; a free valid cell with a normal joins if
//     n_cell . n_plane >= cos(angle_max) and |n . p - d| <= dist_max; after a
//     level that added cells (and >= 3 members) the plane is refit, a
//     degenerate refit keeping the previous plane;
//   * regions below min_region_cells are dropped (cells stay claimed); kept
//     regions get up to 8 refit + audit passes, violators returned to the pool;
//   * outline: boundary edges of the member mask traced into rings (region on
//     the left, sharpest left turn first at pinch corners), the largest
//     signed area is the outer ring, the rest holes; each ring simplified by
//     Douglas-Peucker anchored at the vertex farthest from the first.
// Plane fits use the covariance eigenvector of the smallest eigenvalue from a
// cyclic Jacobi solver with the arithmetic order of the Eigen semantics the
// oracle pins (oracle/shim/Eigen; the reference's Eigen version is unpinned,
// CMakeLists.txt:14-17), so the output matches the oracle bit for bit.
#include <algorithm>
#include <array>
#include <cmath>
#include <fstream>
#include <limits>
#include <map>
#include <string>
#include <vector>

#include "runners.hpp"
#include "snapshot.hpp"

namespace rb200 {

namespace {

struct V2 {
  double x, y;
};
struct V3 {
  double x, y, z;
};

inline double dot(const V3& a, const V3& b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline V3 sub(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline double dot2(const V2& a, const V2& b) { return a.x * b.x + a.y * b.y; }
inline V2 sub2(const V2& a, const V2& b) { return {a.x - b.x, a.y - b.y}; }
inline double norm2(const V2& a) { return std::sqrt(dot2(a, a)); }

struct PlaneEq {
  V3 n{0.0, 0.0, 1.0};
  double d = 0.0;
  double dist(const V3& p) const { return std::abs(dot(n, p) - d); }
};

// Cyclic Jacobi eigen-decomposition of a symmetric 3x3; eigenvalues
// ascending, eigenvectors as columns.
void symEigen3(const double m[3][3], double val[3], double vec[3][3]) {
  double a[3][3], v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a[i][j] = m[i][j];
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = (a[0][1] * a[0][1] + a[0][2] * a[0][2]) + a[1][2] * a[1][2];
    if (off == 0.0) break;
    for (int p = 0; p < 2; ++p) {
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0);
        const double s = t * c;
        for (int k = 0; k < 3; ++k) {  // columns p, q
          const double kp = a[k][p], kq = a[k][q];
          a[k][p] = c * kp - s * kq;
          a[k][q] = s * kp + c * kq;
        }
        for (int k = 0; k < 3; ++k) {  // rows p, q
          const double pk = a[p][k], qk = a[q][k];
          a[p][k] = c * pk - s * qk;
          a[q][k] = s * pk + c * qk;
        }
        for (int k = 0; k < 3; ++k) {
          const double kp = v[k][p], kq = v[k][q];
          v[k][p] = c * kp - s * kq;
          v[k][q] = s * kp + c * kq;
        }
      }
    }
  }
  int order[3] = {0, 1, 2};
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (a[order[j]][order[j]] < a[order[i]][order[i]]) std::swap(order[i], order[j]);
  for (int i = 0; i < 3; ++i) {
    val[i] = a[order[i]][order[i]];
    for (int k = 0; k < 3; ++k) vec[k][i] = v[k][order[i]];
  }
}

struct Fit {
  PlaneEq plane;
  double rms = 0.0;
};

// Total-least-squares plane (reference postprocess.cpp:199-236). Returns
// false where the reference throws DegeneratePlane.
bool fitPlane(const std::vector<V3>& pts, Fit& out) {
  if (pts.size() < 3) return false;
  const double n = static_cast<double>(pts.size());
  V3 c{0.0, 0.0, 0.0};
  for (const V3& p : pts) c = {c.x + p.x, c.y + p.y, c.z + p.z};
  c = {c.x / n, c.y / n, c.z / n};
  double cov[3][3] = {};
  for (const V3& p : pts) {
    const V3 d = sub(p, c);
    const double e[3] = {d.x, d.y, d.z};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) cov[i][j] = cov[i][j] + e[i] * e[j];
  }
  for (auto& row : cov)
    for (double& x : row) x = x / n;
  double val[3], vec[3][3];
  symEigen3(cov, val, vec);
  const double scale = std::max(val[2], 1e-30);
  if (val[1] <= 1e-12 * scale || val[2] <= 0.0) return false;
  V3 nrm{vec[0][0], vec[1][0], vec[2][0]};
  if (nrm.z < 0.0 || (nrm.z == 0.0 && (nrm.x < 0.0 || (nrm.x == 0.0 && nrm.y < 0.0))))
    nrm = {-nrm.x, -nrm.y, -nrm.z};
  const double n2 = dot(nrm, nrm);
  if (n2 > 0.0) {
    const double len = std::sqrt(n2);
    nrm = {nrm.x / len, nrm.y / len, nrm.z / len};
  }
  out.plane.n = nrm;
  out.plane.d = dot(nrm, c);
  double sq = 0.0;
  for (const V3& p : pts) {
    const double r = dot(nrm, p) - out.plane.d;
    sq += r * r;
  }
  out.rms = std::sqrt(sq / n);
  return true;
}

double ringArea(const std::vector<V2>& ring) {
  double twice = 0.0;
  for (std::size_t i = 0; i < ring.size(); ++i) {
    const V2& a = ring[i];
    const V2& b = ring[(i + 1) % ring.size()];
    twice += a.x * b.y - b.x * a.y;
  }
  return 0.5 * twice;
}

// Boundary rings of a cell mask in world xy (reference postprocess.cpp:240-319).
// Corners are (row, col) lattice points; every boundary edge is directed with
// the region on its left, so outer rings run counter-clockwise.
std::vector<std::vector<V2>> traceRings(const std::vector<uint8_t>& mask, const Grid& g,
                                        std::vector<double>& areas) {
  using Corner = std::pair<int, int>;  // (r, c), ordered row-major like the reference
  struct Edge {
    Corner from, to;
  };
  const int W = g.width, H = g.height;
  auto in = [&](int r, int c) {
    return r >= 0 && r < H && c >= 0 && c < W && mask[static_cast<std::size_t>(r) * W + c];
  };
  std::map<Corner, std::vector<Edge>> out_edges;
  for (int r = 0; r < H; ++r)
    for (int c = 0; c < W; ++c) {
      if (!in(r, c)) continue;
      if (!in(r - 1, c)) out_edges[{r, c}].push_back({{r, c}, {r, c + 1}});
      if (!in(r, c + 1)) out_edges[{r, c + 1}].push_back({{r, c + 1}, {r + 1, c + 1}});
      if (!in(r + 1, c)) out_edges[{r + 1, c + 1}].push_back({{r + 1, c + 1}, {r + 1, c}});
      if (!in(r, c - 1)) out_edges[{r + 1, c}].push_back({{r + 1, c}, {r, c}});
    }
  const double ox = g.originX(), oy = g.originY();
  std::vector<std::vector<V2>> rings;
  while (!out_edges.empty()) {
    auto it0 = out_edges.begin();
    Edge e = it0->second.back();
    it0->second.pop_back();
    if (it0->second.empty()) out_edges.erase(it0);
    std::vector<Corner> ring{e.from};
    const Corner start = e.from;
    while (e.to != start) {
      ring.push_back(e.to);
      auto it = out_edges.find(e.to);
      if (it == out_edges.end()) fail(Err::kUsage, "boundary tracing found an open chain");
      std::vector<Edge>& cand = it->second;
      const int dr = e.to.first - e.from.first, dc = e.to.second - e.from.second;
      const Corner left{e.to.first + dc, e.to.second - dr};
      const Corner straight{e.to.first + dr, e.to.second + dc};
      std::size_t pick = 0;
      if (cand.size() > 1) {
        for (std::size_t k = 0; k < cand.size(); ++k)
          if (cand[k].to == left) pick = k;
        if (cand[pick].to != left)
          for (std::size_t k = 0; k < cand.size(); ++k)
            if (cand[k].to == straight) pick = k;
      }
      e = cand[pick];
      cand.erase(cand.begin() + static_cast<std::ptrdiff_t>(pick));
      if (cand.empty()) out_edges.erase(it);
    }
    std::vector<V2> poly;
    poly.reserve(ring.size());
    for (const Corner& k : ring)
      poly.push_back({ox + k.second * g.resolution, oy + k.first * g.resolution});
    areas.push_back(ringArea(poly));
    rings.push_back(std::move(poly));
  }
  return rings;
}

double segDist(const V2& p, const V2& a, const V2& b) {
  const V2 ab = sub2(b, a);
  const double len2 = dot2(ab, ab);
  if (len2 == 0.0) return norm2(sub2(p, a));
  const double t = std::clamp(dot2(sub2(p, a), ab) / len2, 0.0, 1.0);
  return norm2(sub2(p, {a.x + ab.x * t, a.y + ab.y * t}));
}

void dpMark(const std::vector<V2>& pts, std::size_t lo, std::size_t hi, double tol,
            std::vector<uint8_t>& keep) {
  if (hi <= lo + 1) return;
  double worst = -1.0;
  std::size_t at = lo;
  for (std::size_t i = lo + 1; i < hi; ++i) {
    const double d = segDist(pts[i], pts[lo], pts[hi]);
    if (d > worst) {
      worst = d;
      at = i;
    }
  }
  if (worst > tol) {
    keep[at] = 1;
    dpMark(pts, lo, at, tol, keep);
    dpMark(pts, at, hi, tol, keep);
  }
}

std::vector<V2> simplify(const std::vector<V2>& ring, double tol) {
  if (tol <= 0.0 || ring.size() <= 4) return ring;
  std::size_t far = 0;
  double best = -1.0;
  for (std::size_t i = 1; i < ring.size(); ++i) {
    const V2 d = sub2(ring[i], ring[0]);
    const double d2 = dot2(d, d);
    if (d2 > best) {
      best = d2;
      far = i;
    }
  }
  std::vector<uint8_t> keep(ring.size(), 0);
  keep[0] = keep[far] = 1;
  dpMark(ring, 0, far, tol, keep);
  std::vector<V2> closed = ring;
  closed.push_back(ring[0]);
  std::vector<uint8_t> keep2(closed.size(), 0);
  keep2[far] = keep2[closed.size() - 1] = 1;
  dpMark(closed, far, closed.size() - 1, tol, keep2);
  std::vector<V2> out;
  for (std::size_t i = 0; i < ring.size(); ++i)
    if (keep[i] || keep2[i]) out.push_back(ring[i]);
  return out;
}

struct Region {
  PlaneEq plane;
  int cells = 0;
  std::vector<V2> outer;
  std::vector<std::vector<V2>> holes;
};

// computeNormals (reference analysis.cpp:41-86) for snapshots without normals.
void hostNormals(HostLayers& m) {
  const int W = m.grid.width, H = m.grid.height;
  const double res = m.grid.resolution;
  const std::size_t n = m.grid.cells();
  std::vector<double> nx(n, 0.0), ny(n, 0.0), nz(n, 0.0);
  auto at = [&](int r, int c) -> const double* {
    if (r < 0 || r >= H || c < 0 || c >= W) return nullptr;
    const std::size_t j = static_cast<std::size_t>(r) * W + c;
    return m.valid[j] ? &m.elev[j] : nullptr;
  };
  for (int r = 0; r < H; ++r)
    for (int c = 0; c < W; ++c) {
      const std::size_t i = static_cast<std::size_t>(r) * W + c;
      if (!m.valid[i]) continue;
      const double *l = at(r, c - 1), *rt = at(r, c + 1), *dn = at(r - 1, c), *up = at(r + 1, c);
      const double ctr = m.elev[i];
      double gx, gy;
      if (l && rt) gx = (*rt - *l) / (2.0 * res);
      else if (rt) gx = (*rt - ctr) / res;
      else if (l) gx = (ctr - *l) / res;
      else continue;
      if (dn && up) gy = (*up - *dn) / (2.0 * res);
      else if (up) gy = (*up - ctr) / res;
      else if (dn) gy = (ctr - *dn) / res;
      else continue;
      const double len = std::sqrt((gx * gx + gy * gy) + 1.0);
      nx[i] = -gx / len;
      ny[i] = -gy / len;
      nz[i] = 1.0 / len;
    }
  m.nx.swap(nx);
  m.ny.swap(ny);
  m.nz.swap(nz);
}

std::vector<Region> segment(const HostLayers& m, const PlaneSegParams& prm) {
  prm.validate();
  const int W = m.grid.width, H = m.grid.height;
  const std::size_t n = m.grid.cells();
  const double ox = m.grid.originX(), oy = m.grid.originY(), res = m.grid.resolution;
  auto usable = [&](std::size_t i) {
    return m.valid[i] && (m.nx[i] != 0.0 || m.ny[i] != 0.0 || m.nz[i] != 0.0);
  };
  auto point = [&](std::size_t i) -> V3 {
    const int r = static_cast<int>(i) / W, c = static_cast<int>(i) % W;
    return {ox + (c + 0.5) * res, oy + (r + 0.5) * res, m.elev[i]};
  };
  auto normal = [&](std::size_t i) -> V3 { return {m.nx[i], m.ny[i], m.nz[i]}; };
  auto points = [&](const std::vector<std::size_t>& cells) {
    std::vector<V3> pts;
    pts.reserve(cells.size());
    for (std::size_t i : cells) pts.push_back(point(i));
    return pts;
  };

  std::vector<std::size_t> seeds;
  for (std::size_t i = 0; i < n; ++i)
    if (usable(i)) seeds.push_back(i);
  std::stable_sort(seeds.begin(), seeds.end(),
                   [&](std::size_t a, std::size_t b) { return m.nz[a] > m.nz[b]; });
  const double cos_max = std::cos(prm.normal_angle_max);
  std::vector<uint8_t> taken(n, 0);
  std::vector<Region> regions;
  std::vector<std::size_t> members, frontier, grown;

  for (const std::size_t seed : seeds) {
    if (taken[seed]) continue;
    taken[seed] = 1;
    members.assign(1, seed);
    frontier.assign(1, seed);
    PlaneEq plane;
    plane.n = normal(seed);
    plane.d = dot(plane.n, point(seed));
    while (!frontier.empty()) {
      grown.clear();
      for (const std::size_t i : frontier) {
        const int r = static_cast<int>(i) / W, c = static_cast<int>(i) % W;
        const std::array<std::pair<int, int>, 4> nbs{{{r - 1, c}, {r + 1, c}, {r, c - 1}, {r, c + 1}}};
        for (const auto& [rr, cc] : nbs) {
          if (rr < 0 || rr >= H || cc < 0 || cc >= W) continue;
          const std::size_t j = static_cast<std::size_t>(rr) * W + cc;
          if (taken[j] || !usable(j)) continue;
          if (dot(normal(j), plane.n) < cos_max) continue;
          if (plane.dist(point(j)) > prm.dist_max) continue;
          taken[j] = 1;
          members.push_back(j);
          grown.push_back(j);
        }
      }
      if (!grown.empty() && members.size() >= 3) {
        Fit fit;
        if (fitPlane(points(members), fit)) plane = fit.plane;  // degenerate: keep the plane
      }
      frontier.swap(grown);
    }
    if (members.size() < static_cast<std::size_t>(prm.min_region_cells)) continue;

    Fit fit;
    for (int pass = 0; pass < 8; ++pass) {
      if (!fitPlane(points(members), fit)) {
        members.clear();
        break;
      }
      std::vector<std::size_t> kept;
      kept.reserve(members.size());
      for (const std::size_t i : members) {
        if (dot(normal(i), fit.plane.n) >= cos_max && fit.plane.dist(point(i)) <= prm.dist_max)
          kept.push_back(i);
        else
          taken[i] = 0;
      }
      const bool stable = kept.size() == members.size();
      members.swap(kept);
      if (stable) break;
    }
    if (members.size() < static_cast<std::size_t>(prm.min_region_cells)) {
      for (const std::size_t i : members) taken[i] = 0;
      continue;
    }
    Region reg;
    reg.plane = fit.plane;
    reg.cells = static_cast<int>(members.size());
    std::vector<uint8_t> mask(n, 0);
    for (const std::size_t i : members) mask[i] = 1;
    std::vector<double> areas;
    std::vector<std::vector<V2>> rings = traceRings(mask, m.grid, areas);
    std::size_t outer = 0;
    double outer_area = -std::numeric_limits<double>::infinity();
    for (std::size_t k = 0; k < rings.size(); ++k)
      if (areas[k] > outer_area) {
        outer_area = areas[k];
        outer = k;
      }
    for (std::size_t k = 0; k < rings.size(); ++k) {
      std::vector<V2> s = simplify(rings[k], prm.polygon_simplify_tol);
      if (k == outer) reg.outer = std::move(s);
      else reg.holes.push_back(std::move(s));
    }
    regions.push_back(std::move(reg));
  }
  return regions;
}

// Region list in the reference's text format (postprocess.cpp:525-545).
void writeRegionsText(const std::vector<Region>& regions, std::ostream& out) {
  out.precision(17);
  for (std::size_t k = 0; k < regions.size(); ++k) {
    const Region& r = regions[k];
    out << "region: " << k << "\n";
    out << "plane: " << r.plane.n.x << " " << r.plane.n.y << " " << r.plane.n.z << " " << r.plane.d
        << "\n";
    out << "cells: " << r.cells << "\n";
    out << "outer:\n";
    for (const V2& v : r.outer) out << v.x << " " << v.y << "\n";
    for (const auto& hole : r.holes) {
      out << "hole:\n";
      for (const V2& v : hole) out << v.x << " " << v.y << "\n";
    }
    out << "\n";
  }
}

}  // namespace

std::size_t segmentSnapshot(const std::string& snapshot_path, const PlaneSegParams& params,
                            const std::string& out_path) {
  HostLayers m = readSnapshotFile(snapshot_path);
  bool any_normal = false;
  for (std::size_t i = 0; i < m.grid.cells() && !any_normal; ++i)
    any_normal = m.valid[i] && (m.nx[i] != 0.0 || m.ny[i] != 0.0 || m.nz[i] != 0.0);
  if (!any_normal) hostNormals(m);
  const std::vector<Region> regions = segment(m, params);
  std::ofstream out(out_path);
  if (!out) fail(Err::kIo, "cannot write " + out_path);
  writeRegionsText(regions, out);
  return regions.size();
}

}  // namespace rb200
