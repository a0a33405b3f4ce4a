// Drop-in declarations of the reference membership I/O (io.hpp:12-19), host code in
// paper_2411_11468_b200/csrc/dropin.cpp with the reference's messages.
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "labelprop/graph.hpp"

namespace labelprop {

void write_membership(const std::string& path, std::span<const VertexId> labels);
std::vector<VertexId> read_membership(const std::string& path, std::uint32_t n);

}  // namespace labelprop
