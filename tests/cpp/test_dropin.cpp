// Known-answer tests for the C++ drop-in (labelprop::lpa & co. over the nulpa C ABI),
// written like the reference's own suites: each case restates one from
// /root/reference/proj/tests/test_lpa.cpp or test_quality.cpp (line cited) with
// the reference's expected values, and runs on the GPU through libnulpa.so.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <map>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "labelprop/graph.hpp"
#include "labelprop/lpa.hpp"
#include "labelprop/quality.hpp"

using namespace labelprop;

static int g_failures = 0, g_checks = 0;

#define CHECK(cond)                                                   \
  do {                                                                \
    ++g_checks;                                                       \
    if (!(cond)) {                                                    \
      ++g_failures;                                                   \
      std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
    }                                                                 \
  } while (0)

template <typename E, typename F>
static void check_throws(F&& f, const char* what) {
  ++g_checks;
  try {
    f();
  } catch (const E&) {
    return;
  } catch (...) {
  }
  ++g_failures;
  std::printf("  FAIL: expected exception (%s)\n", what);
}

// Symmetric, deduplicated, row-sorted CSR of a simple unit-weight edge list —
// what build_csr(symmetrize=true) produces for such input (graph.cpp:186-307).
static CsrGraph from_edges(const std::vector<std::pair<VertexId, VertexId>>& edges,
                           VertexId n_declared = 0) {
  VertexId n = n_declared;
  for (auto [a, b] : edges) n = std::max<VertexId>(n, std::max(a, b) + 1);
  std::vector<std::set<VertexId>> rows(n);
  for (auto [a, b] : edges) {
    rows[a].insert(b);
    rows[b].insert(a);
  }
  std::vector<std::uint64_t> off(n + 1, 0);
  std::vector<VertexId> tgt;
  for (VertexId i = 0; i < n; ++i) {
    tgt.insert(tgt.end(), rows[i].begin(), rows[i].end());
    off[i + 1] = tgt.size();
  }
  std::vector<float> w(tgt.size(), 1.0f);
  return CsrGraph(std::move(off), std::move(tgt), std::move(w));
}

static CsrGraph star(VertexId leaves) {
  std::vector<std::pair<VertexId, VertexId>> e;
  for (VertexId i = 1; i <= leaves; ++i) e.push_back({0, i});
  return from_edges(e);
}
static CsrGraph single_edge() { return from_edges({{0, 1}}); }
static CsrGraph two_triangles() {
  return from_edges({{0, 1}, {1, 2}, {0, 2}, {3, 4}, {4, 5}, {3, 5}});
}
static CsrGraph k22() { return from_edges({{0, 2}, {0, 3}, {1, 2}, {1, 3}}); }

static LpaConfig seq_config(int pl = 0, int cc = 0) {
  LpaConfig c;
  c.exec = ExecMode::Sequential;
  c.pl_period = pl;
  c.cc_period = cc;
  return c;
}

using U = std::vector<std::uint64_t>;
using L = std::vector<VertexId>;

static void run(const char* name, const std::function<void()>& body) {
  const int before = g_failures;
  try {
    body();
  } catch (const std::exception& e) {
    ++g_failures;
    std::printf("  FAIL: unexpected exception: %s\n", e.what());
  }
  std::printf("[%s] %s\n", g_failures == before ? "PASS" : "FAIL", name);
}

int main() {
  run("star: all vertices adopt the hub's smallest-neighbor label (test_lpa.cpp:57-66)", [] {
    const LpaResult r = lpa(star(3), seq_config());
    CHECK((r.labels == L{1, 1, 1, 1}));
    CHECK((r.stats.delta_n_per_iter == U{3, 0}));
    CHECK(r.stats.converged && r.stats.iterations == 2 && r.stats.pl_iterations == 0);
    CHECK(r.stats.cc_reverts == 0);
  });
  run("star under a pick-less first pass (test_lpa.cpp:68-75)", [] {
    const LpaResult r = lpa(star(3), seq_config(4));
    CHECK((r.labels == L{0, 0, 0, 0}));
    CHECK((r.stats.delta_n_per_iter == U{3, 0}) && r.stats.converged);
    CHECK(r.stats.pl_iterations == 1);
  });
  run("cross_check reverts the higher-id side of a swap (test_lpa.cpp:88-108)", [] {
    const CsrGraph g = single_edge();
    const L prev{0, 1};
    L swapped{1, 0};
    std::vector<std::uint8_t> flags{1, 1};
    CHECK(cross_check(g, swapped, prev, flags) == 1);
    CHECK((swapped == L{1, 1}));
    CHECK((flags == std::vector<std::uint8_t>{0, 0}));
    L good{1, 1};
    std::fill(flags.begin(), flags.end(), std::uint8_t(1));
    CHECK(cross_check(g, good, prev, flags) == 0);
    CHECK((flags == std::vector<std::uint8_t>{1, 1}));
    check_throws<ValidationError>([&] { cross_check(g, swapped, L{0}, flags); }, "short prev");
  });
  run("two disjoint triangles (test_lpa.cpp:110-121)", [] {
    const LpaResult plain = lpa(two_triangles(), seq_config());
    CHECK((plain.labels == L{1, 1, 1, 4, 4, 4}));
    CHECK((plain.stats.delta_n_per_iter == U{4, 0}) && plain.stats.converged);
    const LpaResult pl = lpa(two_triangles(), seq_config(4));
    CHECK((pl.labels == L{0, 0, 0, 3, 3, 3}));
  });
  run("edgeless graph keeps ids and converges (test_lpa.cpp:123-130)", [] {
    const LpaResult r = lpa(from_edges({}, 4), seq_config(4));
    CHECK((r.labels == L{0, 1, 2, 3}));
    CHECK((r.stats.delta_n_per_iter == U{0, 0}) && r.stats.converged && r.stats.iterations == 2);
  });
  run("synchronous baseline oscillates on K2,2 (test_lpa.cpp:132-140)", [] {
    LpaConfig c = seq_config();
    c.exec = ExecMode::Synchronous;
    const LpaResult r = lpa(k22(), c);
    CHECK(!r.stats.converged && r.stats.iterations == 20);
    CHECK((r.stats.delta_n_per_iter == U(20, 4)));
    CHECK((r.labels == L{0, 0, 2, 2}));
  });
  run("synchronous baseline oscillates on a single edge (test_lpa.cpp:142-149)", [] {
    LpaConfig c = seq_config();
    c.exec = ExecMode::Synchronous;
    const LpaResult r = lpa(single_edge(), c);
    CHECK(!r.stats.converged && (r.stats.delta_n_per_iter == U(20, 2)));
    CHECK((r.labels == L{0, 1}));
  });
  run("cross-check breaks the bipartite oscillation (test_lpa.cpp:151-160)", [] {
    LpaConfig c = seq_config(0, 1);
    c.exec = ExecMode::Synchronous;
    const LpaResult r = lpa(k22(), c);
    CHECK(r.stats.converged && r.stats.iterations == 3);
    CHECK((r.stats.delta_n_per_iter == U{2, 1, 0}) && r.stats.cc_reverts == 2);
    CHECK((r.labels == L{2, 2, 2, 2}));
  });
  run("cross-check breaks the single-edge oscillation (test_lpa.cpp:162-172)", [] {
    LpaConfig c = seq_config(0, 1);
    c.exec = ExecMode::Synchronous;
    const LpaResult r = lpa(single_edge(), c);
    CHECK(r.stats.converged && r.stats.iterations == 2);
    CHECK((r.stats.delta_n_per_iter == U{1, 0}) && r.stats.cc_reverts == 1);
    CHECK((r.labels == L{1, 1}));
  });
  run("pick-less every iteration (test_lpa.cpp:174-186)", [] {
    LpaConfig c = seq_config(1);
    c.exec = ExecMode::Synchronous;
    const LpaResult r = lpa(k22(), c);
    CHECK(!r.stats.converged && r.stats.iterations == 20 && r.stats.pl_iterations == 20);
    CHECK((r.labels == L{0, 0, 0, 0}));
    U want(20, 0);
    want[0] = 2;
    want[1] = 1;
    CHECK(r.stats.delta_n_per_iter == want);
  });
  run("parallel workers reach the fixed point (test_lpa.cpp:242-254)", [] {
    for (int workers : {1, 2, 4}) {
      LpaConfig c;
      c.workers = workers;
      c.pl_period = 4;
      const LpaResult r = lpa(two_triangles(), c);
      CHECK((r.labels == L{0, 0, 0, 3, 3, 3}) && r.stats.converged);
    }
  });
  run("the cooperating team path handles a high-degree hub (test_lpa.cpp:256-267)", [] {
    LpaConfig c;
    c.workers = 3;
    c.switch_degree = 8;
    c.pl_period = 0;
    const LpaResult r = lpa(star(40), c);
    CHECK((r.labels == L(41, 0)));
    CHECK((r.stats.delta_n_per_iter == U{40, 0}) && r.stats.converged);
  });
  run("degree partition (test_lpa.cpp:299-305)", [] {
    const CsrGraph g = from_edges({{0, 1}, {1, 2}, {0, 2}, {2, 3}});
    const DegreePartition p = partition_by_degree(g, 3);
    CHECK((p.low == L{0, 1, 3}) && (p.high == L{2}));
    check_throws<ValidationError>([&] { partition_by_degree(g, 1); }, "switch 1");
  });
  run("configuration and input validation (test_lpa.cpp:307-326)", [] {
    const CsrGraph g = single_edge();
    auto expect = [&](std::function<void(LpaConfig&)> m) {
      LpaConfig c;
      m(c);
      check_throws<ValidationError>([&] { lpa(g, c); }, "bad config");
    };
    expect([](LpaConfig& c) { c.tolerance = 0.0; });
    expect([](LpaConfig& c) { c.tolerance = 1.5; });
    expect([](LpaConfig& c) { c.max_iterations = 0; });
    expect([](LpaConfig& c) { c.pl_period = -1; });
    expect([](LpaConfig& c) { c.cc_period = -2; });
    expect([](LpaConfig& c) { c.switch_degree = 1; });
    expect([](LpaConfig& c) { c.workers = -1; });
    check_throws<ValidationError>([&] { lpa(CsrGraph(), LpaConfig{}); }, "empty graph");
    LpaConfig full;
    full.tolerance = 1.0;
    lpa(g, full);
  });
  run("run statistics are internally consistent (test_lpa.cpp:328-334)", [] {
    const LpaResult r = lpa(two_triangles(), seq_config(2, 2));
    CHECK(r.stats.iterations == static_cast<int>(r.stats.delta_n_per_iter.size()));
    CHECK(r.stats.elapsed_seconds >= 0.0);
    for (VertexId l : r.labels) CHECK(l < 6);
  });
  run("modularity of two bridged 5-cliques is 19/42 (test_quality.cpp:37-41)", [] {
    std::vector<std::pair<VertexId, VertexId>> e;
    for (VertexId s : {0u, 5u})
      for (VertexId a = s; a < s + 5; ++a)
        for (VertexId b = a + 1; b < s + 5; ++b) e.push_back({a, b});
    e.push_back({4, 5});
    const CsrGraph g = from_edges(e);
    CHECK(std::abs(modularity(g, L{0, 0, 0, 0, 0, 5, 5, 5, 5, 5}) - 19.0 / 42.0) < 1e-12);
    CHECK(modularity(single_edge(), L{0, 1}) == -0.5);
    check_throws<ValidationError>([&] { modularity(g, L{0, 1}); }, "short labels");
    check_throws<ValidationError>([&] { modularity(g, L(10, 99)); }, "label out of range");
  });
  run("CsrGraph rejects inconsistent arrays (graph.cpp:168-169)", [] {
    check_throws<ValidationError>(
        [] { CsrGraph({0, 2}, {1}, {1.0f}); }, "offsets/targets mismatch");
  });
  std::printf("%d checks, %d failures\n", g_checks, g_failures);
  return g_failures == 0 ? 0 : 1;
}
