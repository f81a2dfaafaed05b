// Host overhead of one synchronous frame through the C ABI, without Python:
// wall time of relief_gpu_map_integrate_device / relief_map_integrate per call
// vs the library's own device time (events on its stream) and the time spent
// inside the call. Graphs on and off.
//   g++ -O2 -I include scripts/host_overhead.cpp -L paper_2204_12876_b200/lib -lrelief_b200 \
//       -Wl,-rpath,$PWD/paper_2204_12876_b200/lib -lcudart -o scripts/host_overhead
//   scripts/host_overhead <config file> <res> <W> <H> [frames]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "relief_gpu.h"

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  if (argc < 5) return 2;
  const char* cfg_path = argv[1];
  const double res = atof(argv[2]);
  const int W = atoi(argv[3]), H = atoi(argv[4]);
  const int frames = argc > 5 ? atoi(argv[5]) : 200;
  relief_config* cfg = relief_config_load(cfg_path);
  double pose[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 1.0};
  std::vector<double> xyz(3u << 21);
  const int64_t n = relief_gpu_sim_render(cfg_path, pose, 0.0, 1, 0, xyz.data(), 1 << 21);
  double* d_xyz = nullptr;
  cudaMalloc(&d_xyz, n * 24);
  cudaMemcpy(d_xyz, xyz.data(), n * 24, cudaMemcpyHostToDevice);
  double* h_pin = nullptr;
  cudaMallocHost(&h_pin, n * 24);
  for (int64_t i = 0; i < 3 * n; ++i) h_pin[i] = xyz[i];
  for (int input = 0; input < 2; ++input) {
    for (int graphs = 1; graphs >= 0; --graphs) {
      relief_map* m = relief_map_create(res, W, H, 0, 0);
      relief_gpu_map_set_graphs(m, graphs);
      double wall = 0, inside = 0, dev = 0;
      relief_scan_stats st;
      for (int f = 0; f < frames + 10; ++f) {
        const double t0 = now();
        if (input == 0)
          relief_gpu_map_integrate_device(m, cfg, d_xyz, n, pose, 0.1 * f, &st);
        else
          relief_map_integrate(m, cfg, h_pin, n, pose, 0.1 * f, &st);
        const double t1 = now();
        double ks[8];
        relief_gpu_map_kernel_seconds(m, ks);
        if (f >= 10) {
          wall += t1 - t0;
          inside += st.total_seconds;
          dev += ks[7] + (input ? ks[0] : 0.0);
        }
      }
      printf("%-7s graphs=%d n=%lld  wall %8.2f us  in-call %8.2f us  device %8.2f us  overhead %7.2f us\n",
             input ? "pinned" : "device", graphs, (long long)n, wall / frames * 1e6,
             inside / frames * 1e6, dev / frames * 1e6, (wall - dev) / frames * 1e6);
      relief_map_free(m);
    }
  }
  return 0;
}
