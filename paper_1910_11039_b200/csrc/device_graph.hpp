// Device-side graph ingestion (device_graph.cu): same results as the host functions of the same name
// in host_graph.cpp, computed on the GPU.  `device` = CUDA ordinal, -1 = current device.
#pragma once

#include <cstdint>

#include "host_common.hpp"

namespace ebc {

HostGraph device_gen_rmat(int scale, int edge_factor, double a, double b, double c, double d, std::uint64_t seed,
                          bool take_lcc, int device);
HostGraph device_graph_from_edges(std::uint64_t n, const std::uint64_t *src, const std::uint64_t *dst,
                                  std::uint64_t count, bool take_lcc, int device);
HostGraph device_graph_lcc(const HostGraph &g, int device);

} // namespace ebc
