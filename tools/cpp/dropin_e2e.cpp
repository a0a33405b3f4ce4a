// End-to-end timing of the C++ drop-in exactly as a reference caller uses it:
// labelprop::lpa(const CsrGraph&, const LpaConfig&) (lpa.hpp:84) on a CsrGraph whose
// offsets / targets / weights are std::vector storage (graph.hpp:53-84) — pageable host
// memory, an explicit all-ones weight array — with the reference's default LpaConfig.
// Every call uploads the graph, runs, and returns the labels (LpaResult).
//
//   dropin_e2e DIR STEPS     DIR holds offsets.u64 / targets.u32 (workloads.py export)
//
// Prints one JSON object: seconds per call (wall, steady_clock), the library's loop time
// (RunStats.elapsed_seconds), iterations.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "labelprop/graph.hpp"
#include "labelprop/lpa.hpp"

template <typename T>
static std::vector<T> read_all(const std::string& path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) throw std::runtime_error("cannot open " + path);
  const std::streamsize bytes = in.tellg();
  std::vector<T> v(static_cast<size_t>(bytes) / sizeof(T));
  in.seekg(0);
  in.read(reinterpret_cast<char*>(v.data()), bytes);
  return v;
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s DIR STEPS\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1];
  const int steps = std::atoi(argv[2]);
  auto off = read_all<std::uint64_t>(dir + "/offsets.u64");
  auto tgt = read_all<std::uint32_t>(dir + "/targets.u32");
  std::vector<float> w(tgt.size(), 1.0f);
  const labelprop::CsrGraph g(std::move(off), std::move(tgt), std::move(w));
  const labelprop::LpaConfig cfg{};
  using clk = std::chrono::steady_clock;
  labelprop::LpaResult r = labelprop::lpa(g, cfg);  // warm-up (device pool, pinned ring)
  double wall = 0.0, loop = 0.0;
  for (int k = 0; k < steps; ++k) {
    const auto t0 = clk::now();
    r = labelprop::lpa(g, cfg);
    wall += std::chrono::duration<double>(clk::now() - t0).count();
    loop += r.stats.elapsed_seconds;
  }
  std::printf("{\"steps\": %d, \"seconds_per_step\": %.6f, \"loop_seconds_per_step\": %.6f, "
              "\"iterations\": %d, \"n\": %u, \"m2\": %llu}\n",
              steps, wall / steps, loop / steps, r.stats.iterations, g.order(),
              static_cast<unsigned long long>(g.directed_size()));
  return 0;
}
