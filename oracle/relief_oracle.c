/*
 * relief_oracle.c -- sequential C restatement of the reliefmap update path
 * (deterministic mode) for testing. TEST INFRASTRUCTURE ONLY; see
 * relief_oracle.h. Citations are into the reference, /root/reference/proj.
 *
 * Arithmetic follows the reference's source order; it is compiled with
 * -ffp-contract=off and no -march (oracle/Makefile), and calls the host libm
 * (glibc) for hypot / tan / acos exactly where the reference does.
 */
#include "relief_oracle.h"

#include <ctype.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { ST_OK = 0, ST_USAGE = 1, ST_DATA = 2, ST_POSE = 4, ST_VARIANCE = 5, ST_MODEL = 6,
       ST_PARSE = 10, ST_IO = 11 };

static __thread char g_err[512];

static int fail_with(int status, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return status;
}

/* ------------------------------------------------------------------ params */
/* Defaults: integration.hpp:33-63, types.hpp:120-140, drift.hpp:27-36,
 * raycast.hpp:28-38, analysis.hpp:29-76. */
typedef struct {
  double maha, s_out;
  int wall;
  double s_t2, s_max2, s_init2, period, max_range;
  double alpha_d, s_pmin2;
  int ex_on;
  double ex_theta, ex_b, ex_c, ex_dmax;
  int dr_on;
  double dr_thr;
  int dr_min;
  double dr_max;
  int cl_on, ub_on;
  double alpha_n, t_free;
  double tr_slope, tr_step, tr_rough;
  int tr_win;
  double w_slope, w_step, w_rough;
  int ov_on;
  double ov_r, ov_thr;
  int convnet;
  double map_res;
  int map_w, map_h;
} params_t;

struct relief_config {
  params_t p;
  uint64_t seed;
};

static params_t defaults(void) {
  params_t p;
  memset(&p, 0, sizeof p);
  p.maha = 2.5; p.s_out = 0.01; p.wall = 5; p.s_t2 = 0.01; p.s_max2 = 100.0;
  p.s_init2 = 100.0; p.period = 0.1; p.max_range = 10.0;
  p.alpha_d = 0.01; p.s_pmin2 = 1e-4;
  p.ex_on = 1; p.ex_theta = 0.785398163397448; p.ex_b = 0.5; p.ex_c = 0.2; p.ex_dmax = 1.0;
  p.dr_on = 1; p.dr_thr = 0.7; p.dr_min = 10; p.dr_max = 0.1;
  p.cl_on = 1; p.ub_on = 1; p.alpha_n = 0.2; p.t_free = 1.0;
  p.tr_slope = 0.785398163397448; p.tr_step = 0.2; p.tr_rough = 0.1; p.tr_win = 5;
  p.w_slope = 0.4; p.w_step = 0.3; p.w_rough = 0.3;
  p.ov_on = 1; p.ov_r = 1.0; p.ov_thr = 1.5;
  p.map_res = 0.04; p.map_w = 250; p.map_h = 250;
  return p;
}

/* std::min / std::max / std::clamp comparison forms */
static double mn(double a, double b) { return (b < a) ? b : a; }
static double mx(double a, double b) { return (a < b) ? b : a; }
static double clampd(double v, double lo, double hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }
/* static_cast<int>(double) as x86-64 cvttsd2si */
static int to_int(double v) { return (v > -2147483649.0 && v < 2147483648.0) ? (int)v : INT32_MIN; }

/* ------------------------------------------------------------------ config */
enum { K_D, K_I, K_B, K_DEG, K_NOISE_A, K_NOISE_P, K_W3, K_CONVNET, K_SKIP };
typedef struct {
  const char* key;
  int kind;
  size_t off;
} key_t_;

#define OFF(f) offsetof(params_t, f)
static const key_t_ kKeys[] = {
    {"map.resolution", K_D, OFF(map_res)}, {"map.width", K_I, OFF(map_w)},
    {"map.height", K_I, OFF(map_h)}, {"map.center_x", K_SKIP, 0}, {"map.center_y", K_SKIP, 0},
    {"update.mahalanobis_threshold", K_D, OFF(maha)}, {"update.sigma_outlier2", K_D, OFF(s_out)},
    {"update.wall_count_threshold", K_I, OFF(wall)}, {"update.sigma_t2", K_D, OFF(s_t2)},
    {"update.sigma_max2", K_D, OFF(s_max2)}, {"update.sigma_init2", K_D, OFF(s_init2)},
    {"update.nominal_period", K_D, OFF(period)}, {"update.max_range", K_D, OFF(max_range)},
    {"noise.alpha_d", K_D, OFF(alpha_d)}, {"noise.sigma_p_min2", K_D, OFF(s_pmin2)},
    {"exclusion.enabled", K_B, OFF(ex_on)}, {"exclusion.theta_a_deg", K_DEG, OFF(ex_theta)},
    {"exclusion.b", K_D, OFF(ex_b)}, {"exclusion.c", K_D, OFF(ex_c)},
    {"exclusion.d_max", K_D, OFF(ex_dmax)}, {"drift.enabled", K_B, OFF(dr_on)},
    {"drift.traversability_threshold", K_D, OFF(dr_thr)}, {"drift.min_points", K_I, OFF(dr_min)},
    {"drift.max_offset", K_D, OFF(dr_max)}, {"cleanup.enabled", K_B, OFF(cl_on)},
    {"cleanup.upper_bound_enabled", K_B, OFF(ub_on)}, {"cleanup.alpha_n", K_D, OFF(alpha_n)},
    {"cleanup.t_free", K_D, OFF(t_free)}, {"traversability.slope_max_deg", K_DEG, OFF(tr_slope)},
    {"traversability.step_max", K_D, OFF(tr_step)},
    {"traversability.roughness_max", K_D, OFF(tr_rough)},
    {"traversability.window", K_I, OFF(tr_win)}, {"traversability.weights", K_W3, OFF(w_slope)},
    {"traversability.convnet", K_CONVNET, OFF(convnet)}, {"overlap.enabled", K_B, OFF(ov_on)},
    {"overlap.radius", K_D, OFF(ov_r)}, {"overlap.height_threshold", K_D, OFF(ov_thr)},
};
/* Keys outside the update path (scene, sensor, trajectory, run knobs,
 * segmentation) are accepted and ignored by this restatement. */
static const char* kSkipPrefixes[] = {"scene.", "sensor.", "traj.", "run.", "segmentation."};

static char* trim(char* s) {
  while (*s == ' ' || *s == '\t' || *s == '\r') ++s;
  char* e = s + strlen(s);
  while (e > s && (e[-1] == ' ' || e[-1] == '\t' || e[-1] == '\r' || e[-1] == '\n')) *--e = 0;
  return s;
}

static int parse_flag(const char* w, int* out) {
  if (!strcmp(w, "true") || !strcmp(w, "1") || !strcmp(w, "on")) { *out = 1; return 1; }
  if (!strcmp(w, "false") || !strcmp(w, "0") || !strcmp(w, "off")) { *out = 0; return 1; }
  return 0;
}

/* Reference config.cpp:91-261 for the update-path keys. */
relief_config* relief_config_load(const char* path) {
  FILE* f = path ? fopen(path, "r") : NULL;
  if (!f) {
    snprintf(g_err, sizeof g_err, "cannot open config: %s", path ? path : "(null)");
    return NULL;
  }
  relief_config* c = calloc(1, sizeof *c);
  c->p = defaults();
  char line[65536];
  int line_no = 0;
  while (fgets(line, sizeof line, f)) {
    ++line_no;
    char* hash = strchr(line, '#');
    if (hash) *hash = 0;
    char* s = trim(line);
    if (!*s) continue;
    char* eq = strchr(s, '=');
    if (!eq) goto bad;
    *eq = 0;
    char* key = trim(s);
    char* val = trim(eq + 1);
    const key_t_* k = NULL;
    for (size_t i = 0; i < sizeof kKeys / sizeof kKeys[0]; ++i)
      if (!strcmp(kKeys[i].key, key)) k = &kKeys[i];
    if (!k) {
      int skip = 0;
      for (size_t i = 0; i < sizeof kSkipPrefixes / sizeof kSkipPrefixes[0]; ++i)
        if (!strncmp(key, kSkipPrefixes[i], strlen(kSkipPrefixes[i]))) skip = 1;
      if (skip) continue;
      goto bad;
    }
    char* end = NULL;
    char* base = (char*)&c->p;
    switch (k->kind) {
      case K_D: case K_DEG: {
        double v = strtod(val, &end);
        if (end == val) goto bad;
        if (!strcmp(key, "noise.alpha_d")) c->p.alpha_d = v;
        *(double*)(base + k->off) = k->kind == K_DEG ? v * 0.017453292519943295 : v;
        break;
      }
      case K_I: {
        double v = strtod(val, &end);
        if (end == val) goto bad;
        *(int*)(base + k->off) = (int)v;
        break;
      }
      case K_B:
        if (!parse_flag(val, (int*)(base + k->off))) goto bad;
        break;
      case K_W3: {
        double* w = (double*)(base + k->off);
        char* p = val;
        for (int i = 0; i < 3; ++i) {
          w[i] = strtod(p, &end);
          if (end == p) goto bad;
          p = end;
        }
        /* w_slope, w_step, w_rough are adjacent in params_t */
        break;
      }
      case K_CONVNET: c->p.convnet = 1; break;
      default: break;
    }
    continue;
  bad:
    snprintf(g_err, sizeof g_err, "config line %d: cannot parse", line_no);
    fclose(f);
    free(c);
    return NULL;
  }
  fclose(f);
  return c;
}

relief_config* relief_config_default(void) {
  relief_config* c = calloc(1, sizeof *c);
  c->p = defaults();
  return c;
}
void relief_config_free(relief_config* c) { free(c); }
int relief_config_set_mode(relief_config* c, const char* mode) {
  if (!c) return fail_with(ST_USAGE, "config handle is null");
  if (!mode) return ST_OK;
  if (strcmp(mode, "det") && strcmp(mode, "deterministic") && strcmp(mode, "par") &&
      strcmp(mode, "parallel"))
    return fail_with(ST_USAGE, "mode must be det or par");
  return ST_OK;
}
int relief_config_set_seed(relief_config* c, uint64_t seed) {
  if (!c) return fail_with(ST_USAGE, "config handle is null");
  c->seed = seed;
  return ST_OK;
}
const char* relief_last_error(void) { return g_err; }
const char* relief_version(void) { return "reliefmap 1.0.0 (C restatement oracle)"; }

/* --------------------------------------------------------------------- map */
/* Layers and fill values: grid.hpp:90-101, grid.cpp:24-39. */
struct relief_map {
  double res;
  int W, H;
  double cx, cy;
  double *elev, *var, *last, *ub, *trav, *nx, *ny, *nz;
  uint8_t *valid, *ubv;
  int32_t* count;
  double last_stamp;
  int has_last;
};

static void fill_cell(relief_map* m, size_t i) {
  m->elev[i] = NAN;
  m->var[i] = NAN;
  m->last[i] = 0.0;
  m->ub[i] = INFINITY;
  m->trav[i] = 0.0;
  m->nx[i] = m->ny[i] = m->nz[i] = 0.0;
  m->valid[i] = 0;
  m->ubv[i] = 0;
}

relief_map* relief_map_create(double res, int w, int h, double cx, double cy) {
  if (res <= 0.0) { fail_with(ST_USAGE, "resolution must be > 0"); return NULL; }
  if (w < 3 || h < 3) { fail_with(ST_USAGE, "grid must be at least 3x3 cells"); return NULL; }
  relief_map* m = calloc(1, sizeof *m);
  size_t n = (size_t)w * h;
  m->res = res; m->W = w; m->H = h; m->cx = cx; m->cy = cy;
  double** L[8] = {&m->elev, &m->var, &m->last, &m->ub, &m->trav, &m->nx, &m->ny, &m->nz};
  for (int k = 0; k < 8; ++k) *L[k] = malloc(n * sizeof(double));
  m->valid = malloc(n);
  m->ubv = malloc(n);
  m->count = calloc(n, sizeof(int32_t));
  for (size_t i = 0; i < n; ++i) fill_cell(m, i);
  return m;
}

void relief_map_free(relief_map* m) {
  if (!m) return;
  free(m->elev); free(m->var); free(m->last); free(m->ub); free(m->trav);
  free(m->nx); free(m->ny); free(m->nz); free(m->valid); free(m->ubv); free(m->count);
  free(m);
}
int relief_map_width(const relief_map* m) { return m ? m->W : 0; }
int relief_map_height(const relief_map* m) { return m ? m->H : 0; }
double relief_map_resolution(const relief_map* m) { return m ? m->res : 0.0; }
int relief_map_center(const relief_map* m, double* x, double* y) {
  if (!m || !x || !y) return fail_with(ST_USAGE, "null argument");
  *x = m->cx; *y = m->cy;
  return ST_OK;
}

static double origin_x(const relief_map* m) { return m->cx - 0.5 * (m->W * m->res); }
static double origin_y(const relief_map* m) { return m->cy - 0.5 * (m->H * m->res); }

/* indexAt, grid.cpp:41-47: -1 when outside. */
static long cell_at(const relief_map* m, double x, double y) {
  int col = to_int(floor((x - origin_x(m)) / m->res));
  int row = to_int(floor((y - origin_y(m)) / m->res));
  if (col < 0 || col >= m->W || row < 0 || row >= m->H) return -1;
  return (long)row * m->W + col;
}

/* invalidateCell, grid.cpp:126-137. */
static void invalidate(relief_map* m, size_t i) { fill_cell(m, i); }

/* layerValues, snapshot.cpp:50-77. */
int relief_map_layer(const relief_map* m, const char* layer, double* out, size_t cap) {
  if (!m || !layer || !out) return fail_with(ST_USAGE, "null argument");
  size_t n = (size_t)m->W * m->H;
  if (cap < n) return fail_with(ST_USAGE, "output buffer too small");
  static const char* names[] = {"elevation", "variance", "last_update", "upper_bound",
                                "upper_bound_valid", "traversability", "normal_x", "normal_y",
                                "normal_z", "valid"};
  int id = -1;
  for (int k = 0; k < 10; ++k)
    if (!strcmp(layer, names[k])) id = k;
  if (id < 0) {
    snprintf(g_err, sizeof g_err,
             "unknown layer '%s'; available: elevation, variance, last_update, upper_bound, "
             "upper_bound_valid, traversability, normal_x, normal_y, normal_z, valid", layer);
    return ST_USAGE;
  }
  for (size_t i = 0; i < n; ++i) {
    int v = m->valid[i] != 0;
    double r;
    switch (id) {
      case 0: r = v ? m->elev[i] : NAN; break;
      case 1: r = v ? m->var[i] : NAN; break;
      case 2: r = v ? m->last[i] : NAN; break;
      case 3: r = m->ubv[i] ? m->ub[i] : NAN; break;
      case 4: r = m->ubv[i] ? 1.0 : 0.0; break;
      case 5: r = v ? m->trav[i] : NAN; break;
      case 6: r = v ? m->nx[i] : NAN; break;
      case 7: r = v ? m->ny[i] : NAN; break;
      case 8: r = v ? m->nz[i] : NAN; break;
      default: r = v ? 1.0 : 0.0; break;
    }
    out[i] = r;
  }
  return ST_OK;
}

/* ------------------------------------------------------------- recenter */
/* grid.cpp:65-111: whole-cell shift with one-cell hysteresis. */
static int cell_shift(double d, double res) {
  if (fabs(d) < res) return 0;
  return (int)llround(d / res);
}

static void shift_f64(double* a, int W, int H, int dc, int dr, double fill, double* tmp) {
  for (int r = 0; r < H; ++r)
    for (int c = 0; c < W; ++c) {
      int sr = r + dr, sc = c + dc;
      tmp[(size_t)r * W + c] =
          (sr >= 0 && sr < H && sc >= 0 && sc < W) ? a[(size_t)sr * W + sc] : fill;
    }
  memcpy(a, tmp, (size_t)W * H * sizeof(double));
}

static void shift_u8(uint8_t* a, int W, int H, int dc, int dr, uint8_t* tmp) {
  for (int r = 0; r < H; ++r)
    for (int c = 0; c < W; ++c) {
      int sr = r + dr, sc = c + dc;
      tmp[(size_t)r * W + c] = (sr >= 0 && sr < H && sc >= 0 && sc < W) ? a[(size_t)sr * W + sc] : 0;
    }
  memcpy(a, tmp, (size_t)W * H);
}

static void recenter(relief_map* m, double x, double y) {
  int cx = cell_shift(x - m->cx, m->res), cy = cell_shift(y - m->cy, m->res);
  if (cx == 0 && cy == 0) return;
  m->cx += cx * m->res;
  m->cy += cy * m->res;
  size_t n = (size_t)m->W * m->H;
  double* tmp = malloc(n * sizeof(double));
  shift_f64(m->elev, m->W, m->H, cx, cy, NAN, tmp);
  shift_f64(m->var, m->W, m->H, cx, cy, NAN, tmp);
  shift_f64(m->last, m->W, m->H, cx, cy, 0.0, tmp);
  shift_f64(m->ub, m->W, m->H, cx, cy, INFINITY, tmp);
  shift_f64(m->trav, m->W, m->H, cx, cy, 0.0, tmp);
  shift_f64(m->nx, m->W, m->H, cx, cy, 0.0, tmp);
  shift_f64(m->ny, m->W, m->H, cx, cy, 0.0, tmp);
  shift_f64(m->nz, m->W, m->H, cx, cy, 0.0, tmp);
  shift_u8(m->valid, m->W, m->H, cx, cy, (uint8_t*)tmp);
  shift_u8(m->ubv, m->W, m->H, cx, cy, (uint8_t*)tmp);
  free(tmp);
}

/* -------------------------------------------------------------- ray walk */
/* clipAxis raycast.cpp:30-42. */
static int clip_axis(double p, double q, double* t0, double* t1) {
  if (p == 0.0) return q >= 0.0;
  double r = q / p;
  if (p < 0.0) {
    if (r > *t1) return 0;
    *t0 = mx(*t0, r);
  } else {
    if (r < *t0) return 0;
    *t1 = mn(*t1, r);
  }
  return *t0 <= *t1;
}

static int clamp_cell(int v, int n) { return v < 0 ? 0 : (v > n - 1 ? n - 1 : v); }

/* traverseCells raycast.cpp:48-130; writes cells + heights, returns count. */
static size_t traverse(const relief_map* m, const double o[3], const double e[3], long* cells,
                       double* hts) {
  size_t n = 0;
  const double gx = origin_x(m), gy = origin_y(m), res = m->res;
  const double dx = e[0] - o[0], dy = e[1] - o[1], dz = e[2] - o[2];
  const double xmax = gx + m->W * res, ymax = gy + m->H * res;
  if (hypot(dx, dy) < 1e-12) {
    if (o[0] >= gx && o[0] < xmax && o[1] >= gy && o[1] < ymax) {
      int row = clamp_cell(to_int(floor((o[1] - gy) / res)), m->H);
      int col = clamp_cell(to_int(floor((o[0] - gx) / res)), m->W);
      cells[n] = (long)row * m->W + col;
      hts[n++] = o[2] + 0.5 * dz;
    }
    return n;
  }
  double t0 = 0.0, t1 = 1.0;
  if (!clip_axis(-dx, o[0] - gx, &t0, &t1)) return n;
  if (!clip_axis(dx, xmax - o[0], &t0, &t1)) return n;
  if (!clip_axis(-dy, o[1] - gy, &t0, &t1)) return n;
  if (!clip_axis(dy, ymax - o[1], &t0, &t1)) return n;
  if (t0 >= t1) return n;
  int end_in = e[0] >= gx && e[0] < xmax && e[1] >= gy && e[1] < ymax;
  int erow = -1, ecol = -1;
  if (end_in) {
    erow = clamp_cell(to_int(floor((e[1] - gy) / res)), m->H);
    ecol = clamp_cell(to_int(floor((e[0] - gx) / res)), m->W);
  }
  const double sx = o[0] + t0 * dx, sy = o[1] + t0 * dy;
  int col = clamp_cell(to_int(floor((sx - gx) / res)), m->W);
  int row = clamp_cell(to_int(floor((sy - gy) / res)), m->H);
  int scol = dx > 0.0 ? 1 : (dx < 0.0 ? -1 : 0);
  int srow = dy > 0.0 ? 1 : (dy < 0.0 ? -1 : 0);
  double tmx = INFINITY, tmy = INFINITY, tdx = INFINITY, tdy = INFINITY;
  if (scol != 0) {
    double b = gx + (col + (scol > 0 ? 1 : 0)) * res;
    tmx = (b - o[0]) / dx;
    tdx = res / fabs(dx);
  }
  if (srow != 0) {
    double b = gy + (row + (srow > 0 ? 1 : 0)) * res;
    tmy = (b - o[1]) / dy;
    tdy = res / fabs(dy);
  }
  double te = t0;
  for (;;) {
    double tn = tmx;
    if (tmy < tn) tn = tmy;
    if (t1 < tn) tn = t1;
    int is_end = end_in && row == erow && col == ecol;
    if (!is_end && tn > te) {
      cells[n] = (long)row * m->W + col;
      hts[n++] = o[2] + (0.5 * (te + tn)) * dz;
    }
    if (tn >= t1) break;
    if (tmx < tmy) {
      col += scol;
      tmx += tdx;
      if (col < 0 || col >= m->W) break;
    } else {
      row += srow;
      tmy += tdy;
      if (row < 0 || row >= m->H) break;
    }
    te = tn;
  }
  return n;
}

/* ------------------------------------------------------------- integrate */
static int pose_valid(const double* P) {
  /* types.hpp:113-116 with the oracle's left-to-right sums. */
  double R[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) R[r][c] = P[4 * r + c];
  double worst = 0.0;
  int first = 1;
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) {
      double s = R[0][r] * R[0][c];
      s = s + R[1][r] * R[1][c];
      s = s + R[2][r] * R[2][c];
      double e = fabs(s - (r == c ? 1.0 : 0.0));
      if (first) { worst = e; first = 0; } else if (e > worst) worst = e;
    }
  double det = R[0][0] * (R[1][1] * R[2][2] - R[1][2] * R[2][1]) -
               R[0][1] * (R[1][0] * R[2][2] - R[1][2] * R[2][0]) +
               R[0][2] * (R[1][0] * R[2][1] - R[1][1] * R[2][0]);
  return worst <= 1e-9 && fabs(det - 1.0) <= 1e-9;
}

int relief_map_integrate(relief_map* m, const relief_config* cfg, const double* xyz, size_t n,
                         const double pose[12], double now, relief_scan_stats* st) {
  if (!m || !pose || (!xyz && n > 0)) return fail_with(ST_USAGE, "null argument");
  params_t P = cfg ? cfg->p : defaults();
  /* integration.cpp:72-75 */
  if (P.maha <= 0.0) return fail_with(ST_USAGE, "mahalanobis_threshold must be > 0");
  if (P.wall < 1) return fail_with(ST_USAGE, "wall_count_threshold must be >= 1");
  if (P.dr_min < 1) return fail_with(ST_USAGE, "min_points must be >= 1");
  if (P.alpha_n < 0.0 || P.alpha_n > 1.0) return fail_with(ST_USAGE, "alpha_n must lie in [0, 1]");
  if (!pose_valid(pose)) return fail_with(ST_POSE, "rotation is not orthonormal");
  if (P.convnet) return fail_with(ST_MODEL, "model has no layers");
  const double dt = m->has_last ? mx(0.0, now - m->last_stamp) : 0.0;
  relief_scan_stats s;
  memset(&s, 0, sizeof s);
  s.points_in = (int64_t)n;
  const size_t ncell = (size_t)m->W * m->H;
  const double t[3] = {pose[3], pose[7], pose[11]};

  recenter(m, t[0], t[1]); /* integration.cpp:83 */

  /* transform, exclusion, range: integration.cpp:85-113, sensing.cpp:32-41 */
  double* pts = malloc((n ? n : 1) * 3 * sizeof(double));
  double* pvar = malloc((n ? n : 1) * sizeof(double));
  size_t kept = 0;
  const double r2 = P.max_range * P.max_range;
  const double tan_a = tan(P.ex_theta);
  for (size_t k = 0; k < n; ++k) {
    const double x = xyz[3 * k], y = xyz[3 * k + 1], z = xyz[3 * k + 2];
    const double sq = (x * x + y * y) + z * z;
    if (sq > r2) { ++s.points_out_of_range; continue; }
    if (P.ex_on) {
      const double ramp = P.ex_b + mx(0.0, hypot(x, y) - P.ex_c) * tan_a;
      if (z > mn(P.ex_dmax, ramp)) { ++s.points_excluded; continue; }
    }
    for (int i = 0; i < 3; ++i)
      pts[3 * kept + i] = ((pose[4 * i] * x + pose[4 * i + 1] * y) + pose[4 * i + 2] * z) + t[i];
    const double d = sqrt(sq);
    pvar[kept] = mx(P.alpha_d * d * d, P.s_pmin2);
    ++kept;
  }

  /* drift.cpp:24-55, integration.cpp:115-128 */
  if (P.dr_on) {
    double sum = 0.0;
    int nv = 0;
    for (size_t k = 0; k < kept; ++k) {
      long i = cell_at(m, pts[3 * k], pts[3 * k + 1]);
      if (i < 0 || !m->valid[i] || m->trav[i] <= P.dr_thr) continue;
      sum += pts[3 * k + 2] - m->elev[i];
      ++nv;
    }
    if (nv >= P.dr_min) {
      const double mean = sum / nv;
      const double off = clampd(mean, -P.dr_max, P.dr_max);
      s.drift_offset_applied = off;
      if (off != 0.0)
        for (size_t i = 0; i < ncell; ++i) {
          if (m->valid[i]) m->elev[i] += off;
          if (m->ubv[i]) m->ub[i] += off;
        }
    }
  }

  /* precount + cell mapping: integration.cpp:57-68, 132-140 */
  memset(m->count, 0, ncell * sizeof(int32_t));
  long* pcell = malloc((kept ? kept : 1) * sizeof(long));
  for (size_t k = 0; k < kept; ++k) {
    pcell[k] = cell_at(m, pts[3 * k], pts[3 * k + 1]);
    if (pcell[k] >= 0) ++m->count[pcell[k]];
    else ++s.points_out_of_map;
  }

  /* gated Kalman fusion in scan order: integration.cpp:40-55, 142-203 */
  uint8_t* fused_cell = calloc(ncell, 1);
  int status = ST_OK;
  for (size_t k = 0; k < kept; ++k) {
    const long i = pcell[k];
    if (i < 0) continue;
    const double pz = pts[3 * k + 2], sp = pvar[k];
    const double h = m->valid[i] ? m->elev[i] : pz;
    const double sm = m->valid[i] ? m->var[i] : P.s_init2;
    if (sm <= 0.0 || sp <= 0.0) {
      status = fail_with(ST_VARIANCE, "variances must be positive");
      break;
    }
    if (m->count[i] > P.wall && pz < h) {
      ++s.points_ignored_low;
    } else if (fabs(pz - h) / sqrt(sm) > P.maha) {
      ++s.points_rejected_outlier;
      if (m->valid[i]) m->var[i] = mn(sm + P.s_out, P.s_max2);
    } else {
      const double den = sm + sp;
      const double nh = (sp * h + sm * pz) / den;
      m->elev[i] = nh;
      m->var[i] = sm * sp / den;
      m->last[i] = now;
      m->valid[i] = 1;
      m->ub[i] = nh;
      m->ubv[i] = 1;
      fused_cell[i] = 1;
      ++s.points_fused;
    }
  }
  if (status != ST_OK) goto done;
  for (size_t i = 0; i < ncell; ++i) s.cells_updated += fused_cell[i];

  /* ray casting, per kept point in order: integration.cpp:205-224,
   * raycast.cpp:132-183 */
  if (P.cl_on || P.ub_on) {
    const size_t cap = (size_t)m->W + m->H + 8;
    long* cells = malloc(cap * sizeof(long));
    double* hts = malloc(cap * sizeof(double));
    for (size_t k = 0; k < kept; ++k) {
      const size_t nv = traverse(m, t, &pts[3 * k], cells, hts);
      if (nv == 0) continue;
      if (P.cl_on) {
        const double v[3] = {pts[3 * k] - t[0], pts[3 * k + 1] - t[1], pts[3 * k + 2] - t[2]};
        const double n2 = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
        double u[3] = {v[0], v[1], v[2]};
        if (n2 > 0.0) {
          const double nn = sqrt(n2);
          for (int q = 0; q < 3; ++q) u[q] = v[q] / nn;
        }
        for (size_t j = 0; j < nv; ++j) {
          const long c = cells[j];
          if (!m->valid[c]) continue;
          if (now - m->last[c] <= P.t_free) continue;
          if (hts[j] >= m->elev[c] - sqrt(m->var[c])) continue;
          if (!(m->nx[c] != 0.0 || m->ny[c] != 0.0 || m->nz[c] != 0.0)) continue;
          if (fabs((u[0] * m->nx[c] + u[1] * m->ny[c]) + u[2] * m->nz[c]) <= P.alpha_n) continue;
          invalidate(m, (size_t)c);
          ++s.cells_removed_by_cleanup;
        }
      }
      if (P.ub_on)
        for (size_t j = 0; j < nv; ++j) {
          const long c = cells[j];
          if (m->valid[c]) continue;
          if (hts[j] < m->ub[c]) {
            m->ub[c] = hts[j];
            m->ubv[c] = 1;
          }
        }
    }
    free(cells);
    free(hts);
  }

  /* overlap clearance: analysis.cpp:296-317 */
  if (P.ov_on) {
    const double rr = P.ov_r * P.ov_r;
    for (int r = 0; r < m->H; ++r)
      for (int c = 0; c < m->W; ++c) {
        const size_t i = (size_t)r * m->W + c;
        if (!m->valid[i]) continue;
        const double ddx = (origin_x(m) + (c + 0.5) * m->res) - t[0];
        const double ddy = (origin_y(m) + (r + 0.5) * m->res) - t[1];
        if (ddx * ddx + ddy * ddy > rr) continue;
        if (fabs(m->elev[i] - t[2]) <= P.ov_thr) continue;
        invalidate(m, i);
        ++s.cells_cleared_by_overlap;
      }
  }

  /* normals from the pre-pass elevation: analysis.cpp:41-86 */
  {
    double* nx = calloc(ncell, sizeof(double));
    double* ny = calloc(ncell, sizeof(double));
    double* nz = calloc(ncell, sizeof(double));
    const double res = m->res;
    for (int r = 0; r < m->H; ++r)
      for (int c = 0; c < m->W; ++c) {
        const size_t i = (size_t)r * m->W + c;
        if (!m->valid[i]) continue;
        const int hl = c > 0 && m->valid[i - 1], hr = c < m->W - 1 && m->valid[i + 1];
        const int hd = r > 0 && m->valid[i - m->W], hu = r < m->H - 1 && m->valid[i + m->W];
        const double ctr = m->elev[i];
        double gx, gy;
        if (hl && hr) gx = (m->elev[i + 1] - m->elev[i - 1]) / (2.0 * res);
        else if (hr) gx = (m->elev[i + 1] - ctr) / res;
        else if (hl) gx = (ctr - m->elev[i - 1]) / res;
        else continue;
        if (hd && hu) gy = (m->elev[i + m->W] - m->elev[i - m->W]) / (2.0 * res);
        else if (hu) gy = (m->elev[i + m->W] - ctr) / res;
        else if (hd) gy = (ctr - m->elev[i - m->W]) / res;
        else continue;
        const double nrm = sqrt((gx * gx + gy * gy) + 1.0);
        nx[i] = -gx / nrm;
        ny[i] = -gy / nrm;
        nz[i] = 1.0 / nrm;
      }
    memcpy(m->nx, nx, ncell * sizeof(double));
    memcpy(m->ny, ny, ncell * sizeof(double));
    memcpy(m->nz, nz, ncell * sizeof(double));
    free(nx); free(ny); free(nz);
  }

  /* geometric traversability: analysis.cpp:88-132 */
  {
    double* out = calloc(ncell, sizeof(double));
    const int R = P.tr_win / 2;
    for (int r = 0; r < m->H; ++r)
      for (int c = 0; c < m->W; ++c) {
        const size_t i = (size_t)r * m->W + c;
        if (!m->valid[i]) continue;
        if (!(m->nx[i] != 0.0 || m->ny[i] != 0.0 || m->nz[i] != 0.0)) continue;
        const double slope = acos(clampd(m->nz[i], -1.0, 1.0));
        const double s_slope = clampd(1.0 - slope / P.tr_slope, 0.0, 1.0);
        const double ctr = m->elev[i];
        double mstep = 0.0, sum = 0.0, sum2 = 0.0;
        int cnt = 0;
        for (int dr = -R; dr <= R; ++dr) {
          const int rr = r + dr;
          if (rr < 0 || rr >= m->H) continue;
          for (int dc = -R; dc <= R; ++dc) {
            const int cc = c + dc;
            if (cc < 0 || cc >= m->W) continue;
            const size_t j = (size_t)rr * m->W + cc;
            if (!m->valid[j]) continue;
            const double v = m->elev[j];
            mstep = mx(mstep, fabs(v - ctr));
            sum += v;
            sum2 += v * v;
            ++cnt;
          }
        }
        const double s_step = clampd(1.0 - mstep / P.tr_step, 0.0, 1.0);
        const double mean = sum / cnt;
        const double var = mx(0.0, sum2 / cnt - mean * mean);
        const double s_rough = clampd(1.0 - sqrt(var) / P.tr_rough, 0.0, 1.0);
        out[i] = P.w_slope * s_slope + P.w_step * s_step + P.w_rough * s_rough;
      }
    memcpy(m->trav, out, ncell * sizeof(double));
    free(out);
  }

  /* time variance on cells the scan did not touch: grid.cpp:113-124,
   * integration.cpp:252-257 */
  if (dt != 0.0 && P.s_t2 != 0.0) {
    const double growth = P.s_t2 * (dt / P.period);
    for (size_t i = 0; i < ncell; ++i)
      if (m->valid[i] && m->count[i] == 0) m->var[i] = mn(m->var[i] + growth, P.s_max2);
  }

  m->last_stamp = now;
  m->has_last = 1;
  if (st) *st = s;
done:
  free(pts);
  free(pvar);
  free(pcell);
  free(fused_cell);
  return status;
}

/* -------------------------------------------------- outside the restatement */
relief_map* relief_map_load(const char* path) {
  (void)path;
  fail_with(ST_USAGE, "snapshot I/O is not part of the oracle restatement");
  return NULL;
}
int relief_map_save(const relief_map* m, const char* path) {
  (void)m; (void)path;
  return fail_with(ST_USAGE, "snapshot I/O is not part of the oracle restatement");
}
int relief_run_simulate(const char* a, const char* b, uint64_t c, int d, const char* e) {
  (void)a; (void)b; (void)c; (void)d; (void)e;
  return fail_with(ST_USAGE, "runners are not part of the oracle restatement");
}
int relief_run_replay(const char* a, const char* const* b, size_t c, const char* d, const char* e,
                      const char* f) {
  (void)a; (void)b; (void)c; (void)d; (void)e; (void)f;
  return fail_with(ST_USAGE, "runners are not part of the oracle restatement");
}
int relief_run_bench(const char* a, const size_t* b, size_t c, int d, const char* e, const char* f) {
  (void)a; (void)b; (void)c; (void)d; (void)e; (void)f;
  return fail_with(ST_USAGE, "runners are not part of the oracle restatement");
}
int relief_run_export(const char* a, const char* b, const char* c, const char* d) {
  (void)a; (void)b; (void)c; (void)d;
  return fail_with(ST_USAGE, "runners are not part of the oracle restatement");
}
int relief_run_segment(const char* a, const char* b, const char* c, size_t* d) {
  (void)a; (void)b; (void)c; (void)d;
  return fail_with(ST_USAGE, "runners are not part of the oracle restatement");
}

/* --------------------------------------------------------------- conv-net */
/* fillNearestValid (analysis.cpp:138-170): FIFO BFS from the valid cells in
 * index order over the 8-neighbourhood, (dr, dc) in row-major order; the first
 * popped neighbour claims a cell and hands it its value. */
static void fill_nearest_valid(const double* layer, const uint8_t* valid, int w, int h,
                               double* filled) {
  const size_t n = (size_t)w * h;
  uint8_t* known = calloc(n, 1);
  size_t* queue = malloc(n * sizeof *queue);
  size_t head = 0, tail = 0;
  for (size_t i = 0; i < n; ++i) {
    filled[i] = 0.0;
    if (valid[i]) {
      filled[i] = layer[i];
      known[i] = 1;
      queue[tail++] = i;
    }
  }
  while (head < tail) {
    const size_t i = queue[head++];
    const int r = (int)i / w, c = (int)i % w;
    for (int dr = -1; dr <= 1; ++dr)
      for (int dc = -1; dc <= 1; ++dc) {
        if (dr == 0 && dc == 0) continue;
        const int rr = r + dr, cc = c + dc;
        if (rr < 0 || rr >= h || cc < 0 || cc >= w) continue;
        const size_t j = (size_t)rr * w + cc;
        if (known[j]) continue;
        known[j] = 1;
        filled[j] = filled[i];
        queue[tail++] = j;
      }
  }
  free(known);
  free(queue);
}

/* applyActivation (analysis.cpp:172-179). */
static double activate(double x, int act) {
  if (act == 0) return x > 0.0 ? x : 0.0;
  if (act == 1) return 1.0 / (1.0 + exp(-x));
  return x;
}

/* convFilterInference (analysis.cpp:183-216) and ConvNetSpec::validate
 * (analysis.cpp:27-39). */
int oracle_convnet_infer(int n_layers, const int* ksize, const double* weights, const double* bias,
                         const int* act, const double* layer, const uint8_t* valid, int w, int h,
                         double* out) {
  if (n_layers < 1) return fail_with(ST_MODEL, "model has no layers");
  size_t off = 0;
  for (int li = 0; li < n_layers; ++li) {
    const int k = ksize[li];
    if (k < 1 || k % 2 == 0) return fail_with(ST_MODEL, "kernel size must be odd and positive");
    for (size_t q = 0; q < (size_t)k * k; ++q)
      if (!isfinite(weights[off + q])) return fail_with(ST_MODEL, "non-finite kernel weight");
    if (!isfinite(bias[li])) return fail_with(ST_MODEL, "non-finite bias");
    off += (size_t)k * k;
  }
  if (w <= 0 || h <= 0) return fail_with(ST_USAGE, "layer size does not match grid dimensions");
  const size_t n = (size_t)w * h;
  double* cur = malloc(n * sizeof *cur);
  double* nxt = malloc(n * sizeof *nxt);
  fill_nearest_valid(layer, valid, w, h, cur);
  off = 0;
  for (int li = 0; li < n_layers; ++li) {
    const int k = ksize[li], rad = k / 2;
    const double* kw = weights + off;
    for (int r = 0; r < h; ++r)
      for (int c = 0; c < w; ++c) {
        double acc = bias[li];
        for (int kr = -rad; kr <= rad; ++kr) {
          const int rr = r + kr < 0 ? 0 : (r + kr > h - 1 ? h - 1 : r + kr); /* border replicate */
          for (int kc = -rad; kc <= rad; ++kc) {
            const int cc = c + kc < 0 ? 0 : (c + kc > w - 1 ? w - 1 : c + kc);
            acc += kw[(size_t)(kr + rad) * k + (kc + rad)] * cur[(size_t)rr * w + cc];
          }
        }
        nxt[(size_t)r * w + c] = activate(acc, act[li]);
      }
    double* t = cur;
    cur = nxt;
    nxt = t;
    off += (size_t)k * k;
  }
  for (size_t i = 0; i < n; ++i) out[i] = clampd(cur[i], 0.0, 1.0);
  free(cur);
  free(nxt);
  return ST_OK;
}

