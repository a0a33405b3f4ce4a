// Drop-in declaration of the reference modularity (quality.hpp:19), served by
// the device kernel in paper_2411_11468_b200/csrc/quality.cu. delta_modularity
// and community_stats (quality.hpp:29-38) are report utilities outside the
// accelerated path and stay with the reference's quality.cpp.
#pragma once

#include <span>

#include "labelprop/graph.hpp"

namespace labelprop {

double modularity(const CsrGraph& g, std::span<const VertexId> labels);

}  // namespace labelprop
