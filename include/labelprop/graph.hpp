// Drop-in declaration of the reference CSR input type (B200 build).
//
// ABI-identical to /root/reference/proj/include/labelprop/graph.hpp:53-84
// (same members in the same order: offsets u64[n+1], targets u32[m2],
// weights f32[m2], total weight 2m as double), so code compiled against either
// header can hand its graph to nulpa's labelprop::lpa. The constructor and
// weighted_degree are defined in paper_2411_11468_b200/csrc/dropin.cpp with the
// reference's validation message (graph.cpp:165-178). load_graph and
// write_edge_list (graph.cpp:18-161,180-184,309-325) are implemented in textio.cpp
// (chunk-parallel parsing of the mapped file, the reference's messages); build_csr
// (graph.cpp:186-307) in build_csr.cu (the CSR built on the device, bit-exact).
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace labelprop {

using VertexId = std::uint32_t;  // graph.hpp:13
using EdgeIdx = std::uint64_t;   // graph.hpp:14

// Error taxonomy, graph.hpp:17-31.
struct FormatError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ValidationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InternalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// graph.hpp:33-44
struct WeightedEdge {
  VertexId u = 0;
  VertexId v = 0;
  double w = 1.0;
};

struct EdgeList {
  std::vector<WeightedEdge> edges;
  std::optional<std::uint64_t> n_declared;
};

class CsrGraph {
 public:
  CsrGraph() = default;
  CsrGraph(std::vector<std::uint64_t> offsets, std::vector<VertexId> targets,
           std::vector<float> weights);

  std::uint32_t order() const { return static_cast<std::uint32_t>(offsets_.size() - 1); }
  std::uint64_t directed_size() const { return targets_.size(); }
  std::uint64_t degree(VertexId i) const { return offsets_[i + 1] - offsets_[i]; }
  std::uint64_t offset(VertexId i) const { return offsets_[i]; }
  double total_weight_2m() const { return total_weight_2m_; }

  std::span<const VertexId> neighbors(VertexId i) const {
    return {targets_.data() + offsets_[i], targets_.data() + offsets_[i + 1]};
  }
  std::span<const float> edge_weights(VertexId i) const {
    return {weights_.data() + offsets_[i], weights_.data() + offsets_[i + 1]};
  }

  const std::vector<std::uint64_t>& offsets() const { return offsets_; }
  const std::vector<VertexId>& targets() const { return targets_; }
  const std::vector<float>& weights() const { return weights_; }

  double weighted_degree(VertexId i) const;

 private:
  std::vector<std::uint64_t> offsets_{0};
  std::vector<VertexId> targets_;
  std::vector<float> weights_;
  double total_weight_2m_ = 0.0;
};

enum class FileFormat { MatrixMarket, EdgeListText };  // graph.hpp:86

EdgeList load_graph(const std::string& path, FileFormat format);  // graph.hpp:96
CsrGraph build_csr(const EdgeList& el, bool symmetrize);           // graph.hpp:107
void write_edge_list(const CsrGraph& g, const std::string& path);   // graph.hpp:112

}  // namespace labelprop
