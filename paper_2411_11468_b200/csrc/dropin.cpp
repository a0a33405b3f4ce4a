// C++ drop-in for the reference engine entry points, over the nulpa C ABI.
//
// Replaces (paths relative to /root/reference/proj):
//   labelprop::lpa                  include/labelprop/lpa.hpp:84, src/lpa.cpp:362-366
//   labelprop::partition_by_degree  include/labelprop/lpa.hpp:63, src/lpa.cpp:330-336
//   labelprop::cross_check          include/labelprop/lpa.hpp:72-73, src/lpa.cpp:338-360
//   labelprop::modularity           include/labelprop/quality.hpp:19, src/quality.cpp:21-49
//   CsrGraph::CsrGraph / weighted_degree   src/graph.cpp:165-178
// Error codes from the C ABI map back onto the reference exceptions:
// 1 → ValidationError, 2 → std::bad_alloc, 3 → InternalError, else runtime_error.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdlib>
#include <fstream>
#include <new>
#include <string>

#include "labelprop/graph.hpp"
#include "labelprop/io.hpp"
#include "labelprop/lpa.hpp"
#include "labelprop/quality.hpp"
#include "nulpa/nulpa.h"

namespace labelprop {

namespace {

[[noreturn]] void raise(int rc) {
  const std::string msg = nulpa_last_error();
  switch (rc) {
    case NULPA_EINVAL: throw ValidationError(msg);
    case NULPA_ENOMEM: throw std::bad_alloc();
    case NULPA_EINTERNAL: throw InternalError(msg);
    case NULPA_EFORMAT: throw FormatError(msg);
    default: throw std::runtime_error(msg);
  }
}

nulpa_csr view(const CsrGraph& g) {
  nulpa_csr c;
  c.n = g.order();
  c.reserved = 0;
  c.m2 = g.directed_size();
  c.offsets = g.offsets().data();
  c.targets = g.targets().data();
  c.weights = g.weights().empty() ? nullptr : g.weights().data();
  return c;
}

int device_from_env() {
  const char* d = std::getenv("NULPA_DEVICE");
  return d ? std::atoi(d) : 0;
}

}  // namespace

// load_graph (graph.cpp:180-184) over nulpa_load_edge_list (textio.cpp).
EdgeList load_graph(const std::string& path, FileFormat format) {
  nulpa_edge_list el{};
  const int rc = nulpa_load_edge_list(
      path.c_str(),
      format == FileFormat::MatrixMarket ? NULPA_FORMAT_MATRIX_MARKET : NULPA_FORMAT_EDGE_LIST, &el);
  if (rc != NULPA_OK) raise(rc);
  EdgeList out;
  out.edges.resize(el.ne);
  for (std::uint64_t k = 0; k < el.ne; ++k) out.edges[k] = {el.u[k], el.v[k], el.w[k]};
  if (el.n_declared >= 0) out.n_declared = static_cast<std::uint64_t>(el.n_declared);
  nulpa_edge_list_free(&el);
  return out;
}

// build_csr (graph.cpp:186-307) on the device (build_csr.cu), downloaded.
CsrGraph build_csr(const EdgeList& el, bool symmetrize) {
  const std::size_t ne = el.edges.size();
  std::vector<VertexId> u(ne), v(ne);
  std::vector<double> w(ne);
  for (std::size_t k = 0; k < ne; ++k) {
    u[k] = el.edges[k].u;
    v[k] = el.edges[k].v;
    w[k] = el.edges[k].w;
  }
  nulpa_graph* g = nullptr;
  int rc = nulpa_graph_from_edge_list(u.data(), v.data(), w.data(), ne,
                                      el.n_declared ? static_cast<std::int64_t>(*el.n_declared) : -1,
                                      symmetrize ? 1 : 0, device_from_env(), &g);
  if (rc != NULPA_OK) raise(rc);
  std::uint32_t n = 0;
  std::uint64_t m2 = 0;
  nulpa_graph_info(g, &n, &m2, nullptr, nullptr);
  std::vector<std::uint64_t> off(std::uint64_t(n) + 1);
  std::vector<VertexId> tgt(m2);
  std::vector<float> wt(m2);
  rc = nulpa_graph_download(g, off.data(), tgt.data(), wt.data());
  nulpa_graph_free(g);
  if (rc != NULPA_OK) raise(rc);
  return CsrGraph(std::move(off), std::move(tgt), std::move(wt));
}

// write_edge_list (graph.cpp:309-325) over nulpa_write_edge_list (textio.cpp).
void write_edge_list(const CsrGraph& g, const std::string& path) {
  const nulpa_csr c = view(g);
  const int rc = nulpa_write_edge_list(path.c_str(), &c);
  if (rc != NULPA_OK) raise(rc);
}

CsrGraph::CsrGraph(std::vector<std::uint64_t> offsets, std::vector<VertexId> targets,
                   std::vector<float> weights)
    : offsets_(std::move(offsets)), targets_(std::move(targets)), weights_(std::move(weights)) {
  if (offsets_.empty() || offsets_.back() != targets_.size() || targets_.size() != weights_.size())
    throw ValidationError("inconsistent CSR arrays");
  total_weight_2m_ = 0.0;
  for (float w : weights_) total_weight_2m_ += static_cast<double>(w);
}

double CsrGraph::weighted_degree(VertexId i) const {
  double k = 0.0;
  for (float w : edge_weights(i)) k += static_cast<double>(w);
  return k;
}

LpaResult lpa(const CsrGraph& g, const LpaConfig& cfg) {
  nulpa_opts o;
  nulpa_default_opts(&o);
  o.tolerance = cfg.tolerance;
  o.max_iterations = cfg.max_iterations;
  o.pl_period = cfg.pl_period;
  o.cc_period = cfg.cc_period;
  o.strategy = static_cast<int32_t>(cfg.strategy);
  o.switch_degree = cfg.switch_degree;
  o.precision = static_cast<int32_t>(cfg.precision);
  o.exec = static_cast<int32_t>(cfg.exec);
  o.workers = cfg.workers;
  o.seed = cfg.seed;
  o.prune = cfg.prune ? 1 : 0;
  o.device = device_from_env();

  LpaResult r;
  r.labels.resize(g.order());
  std::vector<std::uint64_t> dn(cfg.max_iterations > 0 ? cfg.max_iterations : 1);
  nulpa_stats st{};
  st.delta_n = dn.data();
  const nulpa_csr c = view(g);
  const int rc = nulpa_run(&c, &o, nullptr, r.labels.data(), &st);
  if (rc != NULPA_OK) raise(rc);
  r.stats.iterations = st.iterations;
  r.stats.delta_n_per_iter.assign(dn.begin(), dn.begin() + st.iterations);
  r.stats.converged = st.converged != 0;
  r.stats.pl_iterations = st.pl_iterations;
  r.stats.cc_reverts = st.cc_reverts;
  r.stats.elapsed_seconds = st.elapsed_seconds;
  return r;
}

DegreePartition partition_by_degree(const CsrGraph& g, std::uint32_t switch_degree) {
  DegreePartition p;
  p.low.resize(g.order());
  p.high.resize(g.order());
  std::uint64_t nl = 0, nh = 0;
  const nulpa_csr c = view(g);
  const int rc = nulpa_partition_by_degree(&c, switch_degree, p.low.data(), &nl, p.high.data(), &nh);
  if (rc != NULPA_OK) raise(rc);
  p.low.resize(nl);
  p.high.resize(nh);
  return p;
}

std::uint64_t cross_check(const CsrGraph& g, std::span<VertexId> labels,
                          std::span<const VertexId> prev, std::span<std::uint8_t> flags) {
  if (labels.size() != g.order() || prev.size() != g.order() || flags.size() != g.order())
    throw ValidationError("cross-check label arrays must cover every vertex");
  std::uint64_t reverted = 0;
  const nulpa_csr c = view(g);
  const int rc = nulpa_cross_check(&c, labels.data(), prev.data(), flags.data(), &reverted);
  if (rc != NULPA_OK) raise(rc);
  return reverted;
}

double modularity(const CsrGraph& g, std::span<const VertexId> labels) {
  if (labels.size() != g.order())
    throw ValidationError("labeling has " + std::to_string(labels.size()) + " entries for " +
                          std::to_string(g.order()) + " vertices");
  double q = 0.0;
  const nulpa_csr c = view(g);
  const int rc = nulpa_modularity(&c, labels.data(), &q);
  if (rc != NULPA_OK) raise(rc);
  return q;
}

// delta_modularity (quality.cpp:51-54): closed form.
double delta_modularity(double m, double ki, double ki_to_c, double ki_to_d, double sigma_c,
                        double sigma_d) {
  return (ki_to_c - ki_to_d) / m - ki * (ki + sigma_c - sigma_d) / (2.0 * m * m);
}

// community_stats (quality.cpp:56-78) over nulpa_community_stats (device).
CommunityStats community_stats(const CsrGraph& g, std::span<const VertexId> labels) {
  if (labels.size() != g.order())
    throw ValidationError("labeling has " + std::to_string(labels.size()) + " entries for " +
                          std::to_string(g.order()) + " vertices");
  const std::size_t n = std::max<std::size_t>(1, g.order());
  std::vector<std::uint32_t> comm(n);
  std::vector<double> sg(n), bg(n);
  std::vector<std::uint64_t> hs(n), hc(n);
  std::uint64_t count = 0, hl = 0;
  const nulpa_csr c = view(g);
  const int rc = nulpa_community_stats(&c, labels.data(), &count, comm.data(), sg.data(),
                                       bg.data(), hs.data(), hc.data(), &hl);
  if (rc != NULPA_OK) raise(rc);
  CommunityStats st;
  st.count = count;
  for (std::uint64_t k = 0; k < count; ++k) {
    st.sigma[comm[k]] = sg[k];
    st.big_sigma[comm[k]] = bg[k];
  }
  for (std::uint64_t k = 0; k < hl; ++k) st.size_histogram[hs[k]] = hc[k];
  return st;
}

// write_membership (io.cpp:9-14): the text is formatted on the device (textout.cu).
void write_membership(const std::string& path, std::span<const VertexId> labels) {
  const int rc = nulpa_write_membership(path.c_str(), labels.data(), labels.size(), device_from_env());
  if (rc != NULPA_OK) raise(rc);
}

// read_membership (io.cpp:16-56): chunk-parallel parse of the mapped file (textio.cpp).
std::vector<VertexId> read_membership(const std::string& path, std::uint32_t n) {
  std::vector<VertexId> labels(n);
  const int rc = nulpa_read_membership(path.c_str(), n, labels.data());
  if (rc != NULPA_OK) raise(rc);
  return labels;
}

}  // namespace labelprop
