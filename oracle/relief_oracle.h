/*
 * relief_oracle.h -- C restatement of the reliefmap point-cloud -> elevation-map
 * update path (deterministic mode), used ONLY as a test oracle.
 *
 * TEST INFRASTRUCTURE. Not linked into, loaded by, or called from the product
 * (paper_2204_12876_b200/). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference legs may load it.
 *
 * It exports the map / config / integrate subset of relief.h with the same
 * signatures, so the same ctypes binding drives it, the reference and the
 * product. Every function cites the reference file:line it restates
 * (reference = /root/reference/proj). Pinned against the reference compiled
 * in place (oracle/_ref) by tests/test_oracle_restatement.py.
 */
#ifndef RELIEF_ORACLE_H
#define RELIEF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#define ORACLE_API __attribute__((visibility("default")))

typedef struct relief_config relief_config;
typedef struct relief_map relief_map;

typedef struct relief_scan_stats {
  int64_t points_in, points_excluded, points_out_of_range, points_out_of_map,
      points_rejected_outlier, points_ignored_low, points_fused, cells_updated,
      cells_removed_by_cleanup, cells_cleared_by_overlap;
  double drift_offset_applied, total_seconds;
} relief_scan_stats;

ORACLE_API const char* relief_last_error(void);
ORACLE_API const char* relief_version(void);
ORACLE_API relief_config* relief_config_default(void);
ORACLE_API relief_config* relief_config_load(const char* path);
ORACLE_API void relief_config_free(relief_config* c);
ORACLE_API int relief_config_set_mode(relief_config* c, const char* mode);
ORACLE_API int relief_config_set_seed(relief_config* c, uint64_t seed);
ORACLE_API relief_map* relief_map_create(double res, int w, int h, double cx, double cy);
ORACLE_API void relief_map_free(relief_map* m);
ORACLE_API int relief_map_width(const relief_map* m);
ORACLE_API int relief_map_height(const relief_map* m);
ORACLE_API double relief_map_resolution(const relief_map* m);
ORACLE_API int relief_map_center(const relief_map* m, double* x, double* y);
ORACLE_API int relief_map_layer(const relief_map* m, const char* layer, double* out, size_t cap);
ORACLE_API int relief_map_integrate(relief_map* m, const relief_config* c, const double* xyz,
                                    size_t n, const double pose[12], double stamp,
                                    relief_scan_stats* stats);
/* convFilterInference (analysis.cpp:138-216) with an explicit model: layer li
 * has kernel ksize[li] x ksize[li] at weights + sum of the previous layers'
 * k^2, bias[li], activation act[li] (0 relu, 1 sigmoid, 2 identity). The fill
 * is the reference's literal FIFO BFS. Returns 0, or ST_MODEL / ST_USAGE. */
ORACLE_API int oracle_convnet_infer(int n_layers, const int* ksize, const double* weights,
                                    const double* bias, const int* act, const double* layer,
                                    const uint8_t* valid, int w, int h, double* out);
/* Not restated (out of the path); present so the shared binding resolves. */
ORACLE_API relief_map* relief_map_load(const char* path);
ORACLE_API int relief_map_save(const relief_map* m, const char* path);
ORACLE_API int relief_run_simulate(const char*, const char*, uint64_t, int, const char*);
ORACLE_API int relief_run_replay(const char*, const char* const*, size_t, const char*, const char*,
                                 const char*);
ORACLE_API int relief_run_bench(const char*, const size_t*, size_t, int, const char*, const char*);
ORACLE_API int relief_run_export(const char*, const char*, const char*, const char*);
ORACLE_API int relief_run_segment(const char*, const char*, const char*, size_t*);

#endif
