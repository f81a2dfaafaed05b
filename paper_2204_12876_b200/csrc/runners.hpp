// Batch runners behind relief_run_* (reference runner.hpp:40-83) and the
// post-processing chain drivers behind relief_gpu_*smooth_chain.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "device_map.hpp"

namespace rb200 {

bool parseMode(const std::string& mode, ExecMode& out);

void runSimulate(const std::string& config_path, const std::string& out_dir, std::uint64_t seed,
                 bool has_seed, const char* mode);
void runReplay(const std::string& config_path, const std::vector<std::string>& clouds,
               const std::string& poses_path, const std::string& out_dir, const char* mode);
void runBench(const std::string& config_path, const std::vector<std::size_t>& counts,
              int repetitions, const std::string& out_csv, const char* mode);
void runExport(const std::string& snapshot_path, const std::string& layer, bool pgm,
               const std::string& out_path);
std::size_t runSegment(const std::string& snapshot_path, const char* config_path,
                       const std::string& out_path);
// Plane segmentation of a snapshot on the host (segment.cpp); returns the regions written.
std::size_t segmentSnapshot(const std::string& snapshot_path, const PlaneSegParams& params,
                            const std::string& out_path);

void runMapChain(DeviceMap& m, const std::string& layer, const int* kinds, const int* radii,
                 const double* sigmas, int n_steps, double* values_out, uint8_t* valid_out);
void runMapChainDevice(DeviceMap& m, const std::string& layer, const int* kinds, const int* radii,
                       const double* sigmas, int n_steps, double* d_values_out,
                       uint8_t* d_valid_out);
void runHostChain(int device, const double* values, const uint8_t* valid, int width, int height,
                  const int* kinds, const int* radii, const double* sigmas, int n_steps,
                  double* values_out, uint8_t* valid_out);

}  // namespace rb200
