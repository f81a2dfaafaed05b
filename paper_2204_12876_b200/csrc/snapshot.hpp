// Host copy of the ten persistent layers and the text snapshot format.
#pragma once

#include <iosfwd>
#include <string>
#include <vector>

#include "device_map.hpp"

namespace rb200 {

const std::vector<std::string>& layerNames();
std::string unknownLayerMessage(const std::string& layer);

struct HostLayers {
  Grid grid;
  std::vector<double> elev, var, last, ub, trav, nx, ny, nz;
  std::vector<uint8_t> valid, ubv;
  static HostLayers fresh(const Grid& g);
  // Masked values of layer `id` (index into layerNames()).
  std::vector<double> masked(int id) const;
};

void writeSnapshot(const HostLayers& h, std::ostream& out);
void writeSnapshotFile(const HostLayers& h, const std::string& path);
HostLayers readSnapshot(std::istream& in);
HostLayers readSnapshotFile(const std::string& path);

HostLayers downloadHost(const DeviceMap& m);
DeviceMap* uploadHost(int device, const HostLayers& h);

}  // namespace rb200
