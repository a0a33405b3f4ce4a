// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Array-only C shim over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp), compiled by oracle/Makefile into
// oracle/_ref/libnulpa_ref.so with the reference namespace renamed
// (-Dlabelprop=labelprop_ref) and every C++ symbol hidden, so it can sit in
// the same process as our drop-in `labelprop::lpa` without interposition.
//
// Only tests/, __graft_entry__.smoke() (as a checker) and bench.py's
// cpu_baseline / --impl reference leg may load this library.
//
// Each entry point forwards to the reference function named in its comment.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <atomic>
#include <new>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "labelprop/generators.hpp"
#include "labelprop/graph.hpp"
#include "labelprop/hashtable.hpp"
#include "labelprop/lpa.hpp"
#include "labelprop/io.hpp"
#include "labelprop/quality.hpp"
#include "support/oracles.hpp"  // reference test oracles (tests/support/oracles.hpp)

#define REF_API extern "C" __attribute__((visibility("default")))

using namespace labelprop;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

// Error codes mirror include/nulpa/nulpa.h.
template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ValidationError& e) {
    return fail(e, 1);
  } catch (const std::bad_alloc& e) {
    return fail(e, 2);
  } catch (const InternalError& e) {
    return fail(e, 3);
  } catch (const std::exception& e) {
    return fail(e, 5);
  }
}

struct RefStats {
  int32_t iterations;
  int32_t converged;
  int32_t pl_iterations;
  int32_t pad;
  uint64_t cc_reverts;
  double elapsed_seconds;
};

LpaConfig make_cfg(double tolerance, int max_iterations, int pl_period, int cc_period,
                   int strategy, uint32_t switch_degree, int precision_bits, int exec,
                   int workers, int prune) {
  LpaConfig c;
  c.tolerance = tolerance;
  c.max_iterations = max_iterations;
  c.pl_period = pl_period;
  c.cc_period = cc_period;
  c.strategy = static_cast<ProbeStrategy>(strategy);
  c.switch_degree = switch_degree;
  c.precision = precision_bits == 64 ? ValuePrecision::Bits64 : ValuePrecision::Bits32;
  c.exec = static_cast<ExecMode>(exec);
  c.workers = workers;
  c.prune = prune != 0;
  return c;
}
}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// ---- graph handles -------------------------------------------------------

// CsrGraph(offsets, targets, weights)  graph.cpp:165-172
REF_API void* ref_graph_from_csr(const uint64_t* offsets, const uint32_t* targets,
                                 const float* weights, uint32_t n, uint64_t m2) {
  try {
    std::vector<uint64_t> o(offsets, offsets + n + 1);
    std::vector<uint32_t> t(targets, targets + m2);
    std::vector<float> w;
    if (weights)
      w.assign(weights, weights + m2);
    else
      w.assign(m2, 1.0f);
    return new CsrGraph(std::move(o), std::move(t), std::move(w));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// build_csr(EdgeList, symmetrize)  graph.cpp:186-307
REF_API void* ref_graph_from_edges(const uint32_t* u, const uint32_t* v, const double* w,
                                   uint64_t ne, int64_t n_declared, int symmetrize) {
  try {
    EdgeList el;
    el.edges.resize(ne);
    for (uint64_t k = 0; k < ne; ++k) el.edges[k] = {u[k], v[k], w ? w[k] : 1.0};
    if (n_declared >= 0) el.n_declared = static_cast<uint64_t>(n_declared);
    return new CsrGraph(build_csr(el, symmetrize != 0));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// load_graph(path, format)  graph.cpp:68-161,180-184. Returns the number of edges (or
// -1 with the message in ref_last_error, prefixed "F:" for FormatError and "V:" for
// ValidationError); fills the arrays when cap >= that number.
REF_API int64_t ref_load_graph(const char* path, int format, uint64_t cap, uint32_t* u,
                               uint32_t* v, double* w, int64_t* n_declared) {
  try {
    EdgeList el = load_graph(path, format == 0 ? FileFormat::MatrixMarket : FileFormat::EdgeListText);
    if (cap >= el.edges.size())
      for (size_t k = 0; k < el.edges.size(); ++k) {
        u[k] = el.edges[k].u;
        v[k] = el.edges[k].v;
        w[k] = el.edges[k].w;
      }
    *n_declared = el.n_declared ? static_cast<int64_t>(*el.n_declared) : -1;
    return static_cast<int64_t>(el.edges.size());
  } catch (const FormatError& e) {
    g_err = std::string("F:") + e.what();
  } catch (const ValidationError& e) {
    g_err = std::string("V:") + e.what();
  } catch (const std::exception& e) {
    g_err = std::string("E:") + e.what();
  }
  return -1;
}

namespace {
// Run an I/O call; 0 on success, -1 with "F:"/"V:"/"E:" + message in ref_last_error.
template <typename F>
int io_guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const FormatError& e) {
    g_err = std::string("F:") + e.what();
  } catch (const ValidationError& e) {
    g_err = std::string("V:") + e.what();
  } catch (const std::exception& e) {
    g_err = std::string("E:") + e.what();
  }
  return -1;
}
}  // namespace

// write_edge_list(g, path)  graph.cpp:309-325
REF_API int ref_write_edge_list(void* h, const char* path) {
  return io_guard([&] { write_edge_list(*static_cast<CsrGraph*>(h), path); });
}

// write_membership(path, labels)  io.cpp:9-14
REF_API int ref_write_membership(const char* path, const uint32_t* labels, uint64_t n) {
  return io_guard([&] { write_membership(path, std::span<const VertexId>(labels, n)); });
}

// read_membership(path, n)  io.cpp:16-56
REF_API int ref_read_membership(const char* path, uint32_t n, uint32_t* labels) {
  return io_guard([&] {
    auto l = read_membership(path, n);
    std::copy(l.begin(), l.end(), labels);
  });
}

// planted_partition(...)  generators.cpp:45-88, then build_csr(symmetrize)
REF_API void* ref_graph_planted(uint32_t n, uint32_t communities, double p_in, double p_out,
                                uint64_t seed, uint32_t* ground_truth_out) {
  try {
    PlantedGraph pg = planted_partition(n, communities, p_in, p_out, seed);
    if (ground_truth_out)
      std::copy(pg.ground_truth.begin(), pg.ground_truth.end(), ground_truth_out);
    return new CsrGraph(build_csr(pg.edges, true));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// Raw planted-partition edge list (before build_csr), for generator parity.
REF_API int64_t ref_planted_edges(uint32_t n, uint32_t communities, double p_in, double p_out,
                                  uint64_t seed, uint32_t* u_out, uint32_t* v_out,
                                  uint64_t cap) {
  try {
    PlantedGraph pg = planted_partition(n, communities, p_in, p_out, seed);
    const uint64_t ne = pg.edges.edges.size();
    if (u_out && v_out) {
      for (uint64_t k = 0; k < std::min(ne, cap); ++k) {
        u_out[k] = pg.edges.edges[k].u;
        v_out[k] = pg.edges.edges[k].v;
      }
    }
    return static_cast<int64_t>(ne);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// star_graph  generators.cpp:113-118 ; ring_of_cliques :90-111
REF_API void* ref_graph_star(uint32_t leaves) {
  try {
    return new CsrGraph(build_csr(star_graph(leaves), true));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

REF_API void* ref_graph_ring_of_cliques(uint32_t cliques, uint32_t clique_size) {
  try {
    return new CsrGraph(build_csr(ring_of_cliques(cliques, clique_size).edges, true));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

REF_API void ref_graph_free(void* h) { delete static_cast<CsrGraph*>(h); }
REF_API uint32_t ref_graph_order(void* h) { return static_cast<CsrGraph*>(h)->order(); }
REF_API uint64_t ref_graph_m2(void* h) { return static_cast<CsrGraph*>(h)->directed_size(); }
REF_API double ref_graph_total_2m(void* h) { return static_cast<CsrGraph*>(h)->total_weight_2m(); }

REF_API void ref_graph_arrays(void* h, uint64_t* offsets, uint32_t* targets, float* weights) {
  const CsrGraph& g = *static_cast<CsrGraph*>(h);
  if (offsets) std::copy(g.offsets().begin(), g.offsets().end(), offsets);
  if (targets) std::copy(g.targets().begin(), g.targets().end(), targets);
  if (weights) std::copy(g.weights().begin(), g.weights().end(), weights);
}

// ---- engine --------------------------------------------------------------

// lpa(g, cfg)  lpa.cpp:362-366 (run_engine :246-315)
REF_API int ref_lpa(void* h, double tolerance, int max_iterations, int pl_period, int cc_period,
                    int strategy, uint32_t switch_degree, int precision_bits, int exec,
                    int workers, int prune, uint32_t* labels_out, uint64_t* dn_out,
                    RefStats* stats) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    const LpaConfig cfg = make_cfg(tolerance, max_iterations, pl_period, cc_period, strategy,
                                   switch_degree, precision_bits, exec, workers, prune);
    LpaResult r = lpa(g, cfg);
    std::copy(r.labels.begin(), r.labels.end(), labels_out);
    if (dn_out) std::copy(r.stats.delta_n_per_iter.begin(), r.stats.delta_n_per_iter.end(), dn_out);
    stats->iterations = r.stats.iterations;
    stats->converged = r.stats.converged ? 1 : 0;
    stats->pl_iterations = r.stats.pl_iterations;
    stats->pad = 0;
    stats->cc_reverts = r.stats.cc_reverts;
    stats->elapsed_seconds = r.stats.elapsed_seconds;
  });
}

// One synchronous label-choice step from arbitrary input labels: the public
// template detail::scan_candidate (lpa.hpp:92-111) with a snapshot reader,
// then the move rule of sync_move (lpa.cpp:87-88). Every vertex with degree
// >= 1 is examined (no pruning flags). Returns the changed count.
// Vertices are independent given the snapshot, and each one's table is its own
// arena region (slot_offset = 2*O_i, hashtable.hpp:41-46), so host threads take
// 4096-vertex chunks of the ids (the result does not depend on the thread count).
REF_API int ref_sync_step(void* h, const uint32_t* labels_in, int pick_less, int strategy,
                          int precision_bits, uint32_t* labels_out, uint64_t* changed) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    const uint32_t n = g.order();
    std::atomic<uint64_t> dn{0};
    std::atomic<uint32_t> next{0};
    std::atomic<bool> failed{false};
    std::string fail_msg;
    std::mutex fail_mu;
    auto run = [&](auto& arena) {
      auto work = [&] {
        uint64_t local = 0;
        try {
          for (;;) {
            const uint32_t b = next.fetch_add(4096);
            if (b >= n || failed.load()) break;
            const uint32_t e = std::min<uint64_t>(n, uint64_t(b) + 4096);
            for (VertexId i = b; i < e; ++i) {
              labels_out[i] = labels_in[i];
              if (g.degree(i) == 0) continue;
              auto cand = detail::scan_candidate(g, i, arena, static_cast<ProbeStrategy>(strategy),
                                                 false, [&](VertexId j) { return labels_in[j]; });
              if (!cand) continue;
              const bool allowed = pick_less ? (*cand < labels_in[i]) : (*cand != labels_in[i]);
              if (!allowed) continue;
              labels_out[i] = *cand;
              ++local;
            }
          }
        } catch (const std::exception& ex) {
          std::lock_guard<std::mutex> lk(fail_mu);
          if (!failed.exchange(true)) fail_msg = ex.what();
        }
        dn += local;
      };
      const unsigned t = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
      std::vector<std::thread> pool;
      for (unsigned k = 1; k < t; ++k) pool.emplace_back(work);
      work();
      for (auto& th : pool) th.join();
      if (failed) throw InternalError(fail_msg);
    };
    if (precision_bits == 64) {
      auto arena = HashArena<double>::for_graph(g);
      run(arena);
    } else {
      auto arena = HashArena<float>::for_graph(g);
      run(arena);
    }
    *changed = dn;
  });
}

// modularity(g, labels)  quality.cpp:21-49
REF_API int ref_modularity(void* h, const uint32_t* labels, double* q) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    *q = modularity(g, std::span<const VertexId>(labels, g.order()));
  });
}

// community_stats(g, labels).count  quality.cpp:56-78
REF_API int ref_community_count(void* h, const uint32_t* labels, uint64_t* count) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    *count = community_stats(g, std::span<const VertexId>(labels, g.order())).count;
  });
}

// cross_check(g, labels, prev, flags)  lpa.cpp:338-360
REF_API int ref_cross_check(void* h, uint32_t* labels, const uint32_t* prev, uint8_t* flags,
                            uint64_t* reverted) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    const uint32_t n = g.order();
    *reverted = cross_check(g, std::span<VertexId>(labels, n), std::span<const VertexId>(prev, n),
                            std::span<uint8_t>(flags, n));
  });
}

// lpa_move (Sequential single pass)  lpa.hpp:123-145
REF_API int ref_lpa_move(void* h, uint32_t* labels, uint8_t* flags, int pick_less, int strategy,
                         uint32_t switch_degree, uint64_t* dn) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    const uint32_t n = g.order();
    auto arena = HashArena<float>::for_graph(g);
    *dn = lpa_move(g, std::span<VertexId>(labels, n), std::span<uint8_t>(flags, n), arena,
                   pick_less != 0, static_cast<ProbeStrategy>(strategy), switch_degree);
  });
}

// partition_by_degree(g, switch_degree)  lpa.cpp:330-336
REF_API int ref_partition_by_degree(void* h, uint32_t switch_degree, uint32_t* low,
                                    uint64_t* n_low, uint32_t* high, uint64_t* n_high) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    DegreePartition p = partition_by_degree(g, switch_degree);
    std::copy(p.low.begin(), p.low.end(), low);
    std::copy(p.high.begin(), p.high.end(), high);
    *n_low = p.low.size();
    *n_high = p.high.size();
  });
}

// ---- hashtable -----------------------------------------------------------

// geometry_for(g, i)  hashtable.hpp:41-46
REF_API int ref_geometry(void* h, uint32_t i, uint64_t* slot_offset, uint64_t* p1,
                         uint64_t* p2) {
  return guard([&] {
    const TableGeometry geo = geometry_for(*static_cast<CsrGraph*>(h), i);
    *slot_offset = geo.slot_offset;
    *p1 = geo.capacity;
    *p2 = geo.step_mod;
  });
}

// Feed a sequence of (key, value) inserts through ht_accumulate
// (hashtable.hpp:96-149) into one region of capacity p1 / step modulus p2,
// unshared, and dump the resulting slots. Returns the failed-insert count.
REF_API uint64_t ref_ht_accumulate_seq(uint64_t p1, uint64_t p2, int strategy,
                                       const uint32_t* keys, const float* values, uint64_t count,
                                       uint32_t* slot_keys, float* slot_values) {
  const TableGeometry geo{0, p1, p2};
  HashArena<float> arena(p1);
  uint64_t failures = 0;
  for (uint64_t k = 0; k < count; ++k)
    if (ht_accumulate(arena, geo, static_cast<ProbeStrategy>(strategy), keys[k], values[k],
                      false) == AccumulateStatus::Failed)
      ++failures;
  std::copy(arena.keys.begin(), arena.keys.end(), slot_keys);
  std::copy(arena.values.begin(), arena.values.end(), slot_values);
  return failures;
}

// ---- reference test oracles (tests/support/oracles.hpp) --------------------

// reference_lpa  oracles.hpp:106-136
REF_API int ref_reference_lpa(void* h, double tolerance, int max_iterations, int pl_period,
                              uint32_t* labels_out, uint64_t* dn_out, int* iterations,
                              int* converged) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    testsupport::RefRun r = testsupport::reference_lpa(g, tolerance, max_iterations, pl_period);
    std::copy(r.labels.begin(), r.labels.end(), labels_out);
    std::copy(r.delta_n.begin(), r.delta_n.end(), dn_out);
    *iterations = static_cast<int>(r.delta_n.size());
    *converged = r.converged ? 1 : 0;
  });
}

// modularity_oracle  oracles.hpp:75-93
REF_API int ref_modularity_oracle(void* h, const uint32_t* labels, double* q) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    *q = testsupport::modularity_oracle(g, std::span<const VertexId>(labels, g.order()));
  });
}

REF_API uint32_t ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }
