// Drop-in declarations of the reference quality functions (quality.hpp:19-38):
// modularity and community_stats are served by the device kernels in
// paper_2411_11468_b200/csrc/quality.cu; delta_modularity is the closed form.
#pragma once

#include <cstdint>
#include <map>
#include <span>
#include <unordered_map>

#include "labelprop/graph.hpp"

namespace labelprop {

double modularity(const CsrGraph& g, std::span<const VertexId> labels);

double delta_modularity(double m, double ki, double ki_to_c, double ki_to_d, double sigma_c,
                        double sigma_d);

struct CommunityStats {
  std::uint64_t count = 0;
  std::map<std::uint64_t, std::uint64_t> size_histogram;
  std::unordered_map<VertexId, double> sigma;
  std::unordered_map<VertexId, double> big_sigma;
};

CommunityStats community_stats(const CsrGraph& g, std::span<const VertexId> labels);

}  // namespace labelprop
