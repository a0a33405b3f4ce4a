// Drop-in declaration of the reference engine API, served by the B200 build.
//
// ABI-identical to /root/reference/proj/include/labelprop/lpa.hpp:20-84
// (LpaConfig 56 B, RunStats 56 B, LpaResult 80 B on x86-64).
// The definitions in paper_2411_11468_b200/csrc/dropin.cpp forward to the
// C ABI (include/nulpa/nulpa.h), which runs sm_100a kernels. The CPU-only
// header templates of the reference (detail::scan_candidate, lpa_move) are
// not part of the accelerated path; ExecMode::Sequential is still honoured,
// by a single-CTA in-order pass on the device.
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <string_view>
#include <vector>

#include "labelprop/graph.hpp"
#include "labelprop/hashtable.hpp"

namespace labelprop {

enum class ExecMode { ParallelAsync, Sequential, Synchronous };
enum class ValuePrecision { Bits32 = 32, Bits64 = 64 };

struct LpaConfig {
  double tolerance = 0.05;
  int max_iterations = 20;
  int pl_period = 4;
  int cc_period = 0;
  ProbeStrategy strategy = ProbeStrategy::QuadraticDouble;
  std::uint32_t switch_degree = 32;
  ValuePrecision precision = ValuePrecision::Bits32;
  ExecMode exec = ExecMode::ParallelAsync;
  int workers = 0;
  std::uint64_t seed = 0;
  bool prune = true;
};

struct RunStats {
  int iterations = 0;
  std::vector<std::uint64_t> delta_n_per_iter;
  bool converged = false;
  int pl_iterations = 0;
  std::uint64_t cc_reverts = 0;
  double elapsed_seconds = 0.0;
};

struct LpaResult {
  std::vector<VertexId> labels;
  RunStats stats;
};

struct DegreePartition {
  std::vector<VertexId> low;
  std::vector<VertexId> high;
};

DegreePartition partition_by_degree(const CsrGraph& g, std::uint32_t switch_degree);

std::uint64_t cross_check(const CsrGraph& g, std::span<VertexId> labels,
                          std::span<const VertexId> prev, std::span<std::uint8_t> flags);

LpaResult lpa(const CsrGraph& g, const LpaConfig& config);

inline const char* to_string(ExecMode m) {
  switch (m) {
    case ExecMode::ParallelAsync: return "parallel";
    case ExecMode::Sequential: return "sequential";
    case ExecMode::Synchronous: return "synchronous";
  }
  return "?";
}

inline std::optional<ExecMode> parse_exec_mode(std::string_view s) {
  for (ExecMode m : {ExecMode::ParallelAsync, ExecMode::Sequential, ExecMode::Synchronous})
    if (s == to_string(m)) return m;
  return std::nullopt;
}

}  // namespace labelprop
