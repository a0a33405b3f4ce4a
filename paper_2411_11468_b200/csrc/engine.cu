// The ν-LPA iteration driver on the device.
//
// run_engine (lpa.cpp:246-315) re-stated for the GPU: identity labels, flags
// set for isolated vertices, Pick-Less on iterations ≡ 0 (mod pl_period),
// cross-check on iterations ≡ 0 (mod cc_period), flags reset on the first
// non-PL pass after a PL pass (or every pass without pruning), ΔN net of
// reverts, convergence iff a non-PL pass changes fewer than tolerance·n
// vertices. One stream; the ΔN/counter read-back is the only per-pass host
// synchronisation. elapsed_seconds covers the loop only (lpa.cpp:269,311),
// measured with CUDA events.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "internal.hpp"
#include "layout.hpp"
#include "lpa_kernels.cuh"
#include "plan.hpp"

namespace nulpa {

using namespace dev;

namespace {

// labels = identity (lpa.cpp:250): position p holds the vertex id stored there.
__global__ void k_init(uint32_t* lab, uint8_t* flags, const uint64_t* off, uint32_t n,
                       const uint32_t* vid) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    lab[i] = vid ? vid[i] : i;
    if (flags) flags[i] = (off[i + 1] == off[i]) ? 1 : 0;  // isolated: never examined
  }
}

// Batched runs: after pass `iter`, sum the tiers' label changes and, on a non-Pick-Less
// pass with dN / n < tolerance (lpa.cpp:306), stop the run: *stop = iter + 1, and every
// pass kernel enqueued behind it returns at once (PassCtx::stop).
__global__ void k_decide(const unsigned long long* ctr, uint32_t n, double tolerance, int pick_less,
                         int iter, unsigned* stop) {
  if (threadIdx.x != 0 || *stop) return;
  unsigned long long dn = 0;
  for (int t = 0; t < kTiers; ++t) dn += ctr[t * C_COUNT + C_DN];
  if (!pick_less && static_cast<double>(dn) / n < tolerance) *stop = static_cast<unsigned>(iter + 1);
}

inline unsigned grid_for(uint64_t work, unsigned per_block, unsigned cap) {
  const uint64_t b = (work + per_block - 1) / per_block;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(b, cap)));
}

template <typename K>
void allow_smem(K kernel, size_t bytes) {
  NULPA_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
}

// Run `setup` once per device for each `done` mask (function attributes are set per
// device: a process that runs on device 1 after device 0 must set them again). The
// bit is set only after `setup` succeeded, under a lock, so a concurrent caller never
// launches before the attributes are in place and a failed setup is retried.
template <typename F>
void once_per_device(std::atomic<uint64_t>& done, F&& setup) {
  int dev = 0;
  NULPA_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (done.load(std::memory_order_relaxed) & bit) return;
  setup();
  done.fetch_or(bit, std::memory_order_release);
}

// Grid for a grid-stride kernel: enough CTAs for `work` items at `per_block`
// items per CTA, but never more than fit on the device at once (one wave), so no
// second partial wave leaves most SMs idle at the end of the tier.
template <typename K>
unsigned resident_grid(K kernel, int threads, size_t smem, uint64_t work, unsigned per_block,
                       int sms) {
  // Occupancy is a property of (kernel, block, smem) on this architecture: query it once
  // (the query costs microseconds per launch, which small graphs feel).
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t>, int> cache;
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), threads, smem);
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) per_sm = it->second;
  }
  if (per_sm == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) !=
            cudaSuccess ||
        per_sm < 1) {
      (void)cudaGetLastError();
      per_sm = 1;
    }
    std::lock_guard<std::mutex> lock(mu);
    cache[key] = per_sm;
  }
  return grid_for(work, per_block, static_cast<unsigned>(per_sm) * sms);
}

// Shortest chunk a CHUNKED thread-tier walk gives one thread (k_thread).
#ifndef NULPA_MIN_CHUNK
#define NULPA_MIN_CHUNK 32
#endif
constexpr unsigned kMinChunk = NULPA_MIN_CHUNK;

// Optional per-tier CUDA-event timing (tuning.profile).
struct Prof {
  bool on = false;
  cudaEvent_t ev[kTiers][2];
  bool used[kTiers];
  void begin(int t, cudaStream_t s) {
    used[t] = true;
    if (on) cudaEventRecord(ev[t][0], s);
  }
  void end(int t, cudaStream_t s) {
    if (on) cudaEventRecord(ev[t][1], s);
  }
};

// Concurrent tiers (NULPA_CONCURRENT, read once). A pass is two tier groups, the
// reference's two lists (lpa.cpp:139-230): the register tiers (degree <= 32: thread,
// half warp, warp) and then the table tiers (team32 .. hub), with the group boundary
// a stream join, as the reference's low list finishes before its team list starts.
// Within a group the tiers run on their own streams, side by side: on a small graph
// every tier kernel is a fraction of the GPU and a pass stops being the SUM of its
// tiers' latency chains. Any order of the vertices inside one list is an ordering the
// reference's workers can produce. 0 = off, 1 = on, 2 = both groups for graphs of at
// most 2^22 vertices and the register group above (default), 3 = the register group
// only, 4 = the table group only, 5 = the register group plus the hub accumulation beside
// the table tiers, 6 = that hub accumulation only (R-MAT 27: 123.7 ms, web 69.2 ms: the
// resident hub accumulation holds SMs the table tiers need; off). Measured on one B200 (loop ms per run, off -> default):
// SBM-100K 0.456 -> 0.286 (with one-row small-tier batches), R-MAT 18 1.33 -> 0.72,
// R-MAT 22 5.1 -> 4.3, R-MAT 24 12.7 -> 12.3, R-MAT 27 96.9 -> 95.3, web 66.1 -> 64.6.
// The table group side by side on large graphs is slower (R-MAT 27: 108.8 ms): its
// tiers each fill the GPU and lose the read-only label path.
inline int concurrent_mode() {
  static const int m = [] {
    const char* e = std::getenv("NULPA_CONCURRENT");
    return e ? std::atoi(e) : 2;
  }();
  return m;
}

// Tier streams of one device (created once), forked from and joined into the run's
// stream. One run at a time holds them (Fork::lease); a concurrent run on the same
// device falls back to one stream.
struct Fork {
  cudaStream_t st[kTiers] = {};
  cudaEvent_t go = nullptr;
  cudaEvent_t done[kTiers] = {};
  bool used[kTiers] = {};
  unsigned groups = 3;  // bit 0: register tiers side by side, bit 1: table tiers
  std::mutex mu;
  void init() {
    if (go) return;
    for (int t = 0; t < kTiers; ++t) {
      NULPA_CUDA(cudaStreamCreateWithFlags(&st[t], cudaStreamNonBlocking));
      NULPA_CUDA(cudaEventCreateWithFlags(&done[t], cudaEventDisableTiming));
    }
    NULPA_CUDA(cudaEventCreateWithFlags(&go, cudaEventDisableTiming));
  }
  // Start a group: every tier stream waits for the work enqueued on `s` so far.
  void fork(cudaStream_t s) {
    NULPA_CUDA(cudaEventRecord(go, s));
    for (int t = 0; t < kTiers; ++t) used[t] = false;
  }
  cudaStream_t enter(int t) {
    if (!used[t]) NULPA_CUDA(cudaStreamWaitEvent(st[t], go, 0));
    used[t] = true;
    return st[t];
  }
  // End a group: `s` waits for every tier stream the group used.
  void join(cudaStream_t s) {
    for (int t = 0; t < kTiers; ++t)
      if (used[t]) {
        NULPA_CUDA(cudaEventRecord(done[t], st[t]));
        NULPA_CUDA(cudaStreamWaitEvent(s, done[t], 0));
        used[t] = false;
      }
  }
  static Fork& of_device(int dev) {
    static Fork forks[64];
    return forks[dev & 63];
  }
};

// Rows per iteration of the chunk-major walk (NULPA_CHUNK_ROWS, read once): 1 = k_thread's
// walk (a fence pair per row), 2 / 4 / 8 = k_chunk_walk (one fence pair per group), 14 / 18
// = 4 / 8 rows with the next row's targets prefetched, 24 / 28 = the same for ranges of
// degree <= 4 (4-entry row registers). 0 (default) = 24 where the range's degree is <= 4,
// else 14. 4096² grid per run: 5.67 / 4.95 / 4.47 / 4.50 / 4.23 / 4.68 / 3.66 / 3.66 ms for
// 1 / 2 / 4 / 8 / 14 / 18 / 24 / 28.
inline int chunk_rows() {
  static const int m = [] {
    const char* e = std::getenv("NULPA_CHUNK_ROWS");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

// One-row batches for team tiers of at most one row per team (NULPA_SMALL_TIER_BATCH,
// read once; 1 by default).
inline bool small_tier_batch() {
  static const bool m = [] {
    const char* e = std::getenv("NULPA_SMALL_TIER_BATCH");
    return e ? std::atoi(e) != 0 : true;
  }();
  return m;
}

// Wide-tier variant (NULPA_WIDE_MODE, read once): 0 = plain coalesced target loads,
// rounds in program order (default); 1 = label prefetch one round ahead; 2 = TMA-staged
// targets + label prefetch. Measured at R-MAT 27: 29.5 / 30.7 / 40.4 ms of
// wide tier per run, identical results, so the plain kernel is the default.
// Thread tier: two list entries per thread iteration (NULPA_THREAD_PAIR, read once; 0 by
// default) — one claim fence for both, both rows' loads in flight together. Measured at
// R-MAT 27 on one B200: thread tier 7.6 ms per run with pairs, 5.0 ms without (the
// 99-register pair kernel runs fewer warps per SM).
inline bool thread_pair() {
  static const bool m = [] {
    const char* e = std::getenv("NULPA_THREAD_PAIR");
    return e ? std::atoi(e) != 0 : false;
  }();
  return m;
}

// L2 persistence for the hot prefix of the label array (NULPA_L2_PERSIST = MB, read once;
// 0 = off). In position order the highest-degree vertices come first, so the first few
// tens of MB of labels take most of the neighbour-label gathers; a persisting access
// window keeps them resident while the adjacency streams past.
inline size_t l2_persist_bytes() {
  static const size_t m = [] {
    const char* e = std::getenv("NULPA_L2_PERSIST");
    return e ? static_cast<size_t>(std::atof(e) * (1 << 20)) : size_t(0);
  }();
  return m;
}

struct L2Window {
  cudaStream_t s = nullptr;
  bool on = false;
  L2Window(cudaStream_t st, const void* base, uint32_t n) : s(st) {
    size_t want = std::min<size_t>(l2_persist_bytes(), size_t(n) * 4);
    if (want == 0) return;
    int dev = 0, max_persist = 0, max_window = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    want = std::min<size_t>(want, std::min<size_t>(max_persist, max_window));
    if (want == 0) return;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
      (void)cudaGetLastError();
      return;
    }
    cudaStreamAttrValue a{};
    a.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    a.accessPolicyWindow.num_bytes = want;
    a.accessPolicyWindow.hitRatio = 1.0f;
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    on = cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &a) == cudaSuccess;
    if (!on) (void)cudaGetLastError();
  }
  ~L2Window() {
    if (!on) return;
    cudaStreamAttrValue a{};
    a.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &a);
    cudaCtxResetPersistingL2Cache();
    (void)cudaGetLastError();
  }
};

// Read-only label prefixes (PassCtx::ro_end; NULPA_RO=0 turns them off, read once).
inline bool ro_labels() {
  static const bool m = [] {
    const char* e = std::getenv("NULPA_RO");
    return e ? std::atoi(e) != 0 : true;
  }();
  return m;
}

// ... and the suffix of lower-degree tiers (NULPA_RO_LOW, read once; 0 by default: those
// labels are cold, and caching them in L1 cost R-MAT 27 97.3 -> 99.5 ms per run).
inline bool ro_labels_low() {
  static const bool m = [] {
    const char* e = std::getenv("NULPA_RO_LOW");
    return e ? std::atoi(e) != 0 : false;
  }();
  return m;
}

// In-warp label dedupe in the team tables after the first pass (NULPA_DEDUP_LATER, read
// once; 1 by default).
inline bool dedup_later() {
  static const bool m = [] {
    const char* e = std::getenv("NULPA_DEDUP_LATER");
    return e ? std::atoi(e) != 0 : true;
  }();
  return m;
}

// Thread tier with four claims per fence and batch-deferred wake-ups (k_thread_q;
// NULPA_THREAD_Q, read once; 0 by default). Measured on one B200: R-MAT 27 thread tier
// 5.00 -> 5.32 ms per run, web-like 5.75 -> 5.42 ms, SBM-100K 0.04 -> 0.07 ms.
inline bool thread_q() {
  static const bool m = [] {
    const char* e = std::getenv("NULPA_THREAD_Q");
    return e ? std::atoi(e) != 0 : false;
  }();
  return m;
}

// Passes enqueued per host read-back in batched runs (NULPA_BATCH_PASSES, read once).
inline int batch_passes() {
  static const int m = [] {
    const char* e = std::getenv("NULPA_BATCH_PASSES");
    return e ? std::max(1, std::atoi(e)) : 4;
  }();
  return m;
}

inline int wide_mode() {
  static const int m = [] {
    const char* e = std::getenv("NULPA_WIDE_MODE");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

// Steps of a k_group batch whose loads are issued together (NULPA_GROUP_STEPS, read once:
// 2 by default). Loading S steps' labels before any of them decides makes the half-warp /
// warp tiers read staler labels of the OTHER warps (the batch's own moves are patched in,
// k_group): measured on one B200, S = 8 took the SBM-100K run from 4 to 6 passes; S = 2
// keeps 4 passes there (0.282 -> 0.279 ms) and shortens R-MAT 22 4.30 -> 3.95 ms, R-MAT 18
// 0.730 -> 0.718, R-MAT 27 95.3 -> 95.0 ms against S = 1.
inline int group_steps() {
  static const int m = [] {
    const char* e = std::getenv("NULPA_GROUP_STEPS");
    return e ? std::atoi(e) : 2;
  }();
  return m;
}

template <int MODE, typename W, bool WEIGHTED, int G>
void launch_group(const PassCtx& c, const uint32_t* list, uint32_t count, cudaStream_t s, int sms) {
  auto go = [&](auto kernel) {
    // 32 entries per warp batch, walked in order: shorter batches on small tiers (more
    // warps busy) made the pass more Jacobi-like — SBM-100K quality dropped (Q 0.855 ->
    // 0.84) and the six-block KAT split a block — for no time gained (0.58 ms per run).
    constexpr uint32_t bsz = 32;
    kernel<<<resident_grid(kernel, 256, 0, count, 8 * bsz, sms), 256, 0, s>>>(c, list, count, bsz);
  };
  switch (group_steps()) {
    case 1: go(k_group<MODE, W, WEIGHTED, G, 1>); break;
    case 2: go(k_group<MODE, W, WEIGHTED, G, 2>); break;
    case 4: go(k_group<MODE, W, WEIGHTED, G, 4>); break;
    default: go(k_group<MODE, W, WEIGHTED, G, 8>);
  }
}

template <int MODE, typename W>
void launch_wide(const Plan& p, const PassCtx& c, cudaStream_t s, int sms) {
  const uint32_t cnt = p.count[T_CLUSTER];
  auto go = [&](auto kernel, size_t smem) {
    // (the scratch holds kWideCtasPerSm regions per SM: never launch more CTAs than that)
    const unsigned grid = std::min<unsigned>(resident_grid(kernel, kWideThreads, smem, cnt, 1, sms),
                                             unsigned(kWideCtasPerSm) * sms);
    kernel<<<grid, kWideThreads, smem, s>>>(
        c, p.list[T_CLUSTER], cnt, c.fresh, p.wide_scratch, p.wide_stride, p.m2, p.wide_hint);
  };
  switch (wide_mode()) {
    case 0: go(k_wide<MODE, W, false, false>, wide_bytes(false)); break;
    case 1: go(k_wide<MODE, W, false, true>, wide_bytes(false)); break;
    case 3: go(k_wide<MODE, W, false, true, true>, wide_bytes(false)); break;
    default: go(k_wide<MODE, W, true, true>, wide_bytes(true));
  }
}

// One pass over every tier (SURVEY §3.1 "new B200 stack"). `ctr` holds one
// C_COUNT block per tier. Returns the number of kernels launched.
template <int MODE, typename W, bool WEIGHTED>
int launch_pass(const Plan& p, PassCtx c, unsigned long long* ctr, cudaStream_t s, int sms,
                Prof& prof, unsigned tiers = ~0u, Fork* fk = nullptr) {
  using Tab = Table<kPacked<WEIGHTED>, W>;
  // Team kernels: <CTA threads, team threads, table slots, max degree> per tier.
  constexpr size_t wtab_smem = 8 * team_bytes<Tab, kWarpTabCap, kWarpTabMax>();
  constexpr size_t block_smem = 2 * team_bytes<Tab, kBlockCap, kBlockMax>();
  constexpr size_t block2_smem = 1 * team_bytes<Tab, kBlock2Cap, kBlock2Max>();
  constexpr size_t big_smem = team_bytes<Tab, kBigCap, kBigMax>();
  constexpr size_t cluster_smem = cluster_bytes<Tab>();
  constexpr size_t hub_smem = kHubCap * Tab::kSlotBytes + kHubChunk * sizeof(uint16_t);
  // First pass of a run (labels still mostly distinct): the team tables skip the
  // in-warp dedupe (see k_team).
  const bool dd = !c.fresh && dedup_later();
  constexpr int kDedupLater = 1;  // (merging only lane 0's label: 0.6 ms slower)
  auto k_wt = dd ? k_team<MODE, W, WEIGHTED, 256, 32, kWarpTabCap, kWarpTabMax, kDedupLater>
                 : k_team<MODE, W, WEIGHTED, 256, 32, kWarpTabCap, kWarpTabMax, 0>;
  auto k_b1 = dd ? k_team<MODE, W, WEIGHTED, 256, 128, kBlockCap, kBlockMax, kDedupLater>
                 : k_team<MODE, W, WEIGHTED, 256, 128, kBlockCap, kBlockMax, 0>;
  auto k_b2 = dd ? k_team<MODE, W, WEIGHTED, 256, 256, kBlock2Cap, kBlock2Max, kDedupLater>
                 : k_team<MODE, W, WEIGHTED, 256, 256, kBlock2Cap, kBlock2Max, 0>;
  auto k_bg = dd ? k_team<MODE, W, WEIGHTED, kMidThreads, kMidThreads, kBigCap, kBigMax, kDedupLater>
                 : k_team<MODE, W, WEIGHTED, kMidThreads, kMidThreads, kBigCap, kBigMax, 0>;
  static std::atomic<uint64_t> init{0};
  once_per_device(init, [&] {
    allow_smem(k_team<MODE, W, WEIGHTED, 256, 32, kWarpTabCap, kWarpTabMax, kDedupLater>, wtab_smem);
    allow_smem(k_team<MODE, W, WEIGHTED, 256, 32, kWarpTabCap, kWarpTabMax, 0>, wtab_smem);
    allow_smem(k_team<MODE, W, WEIGHTED, 256, 128, kBlockCap, kBlockMax, kDedupLater>, block_smem);
    allow_smem(k_team<MODE, W, WEIGHTED, 256, 128, kBlockCap, kBlockMax, 0>, block_smem);
    allow_smem(k_team<MODE, W, WEIGHTED, 256, 256, kBlock2Cap, kBlock2Max, kDedupLater>, block2_smem);
    allow_smem(k_team<MODE, W, WEIGHTED, 256, 256, kBlock2Cap, kBlock2Max, 0>, block2_smem);
    allow_smem(k_team<MODE, W, WEIGHTED, kMidThreads, kMidThreads, kBigCap, kBigMax, kDedupLater>, big_smem);
    allow_smem(k_team<MODE, W, WEIGHTED, kMidThreads, kMidThreads, kBigCap, kBigMax, 0>, big_smem);
    allow_smem(k_cluster<MODE, W, WEIGHTED>, cluster_smem);
    if constexpr (!WEIGHTED) {
      allow_smem(k_wide<MODE, W, true, true>, wide_bytes(true));
      allow_smem(k_wide<MODE, W, false, true>, wide_bytes(false));
      allow_smem(k_wide<MODE, W, false, true, true>, wide_bytes(false));
      allow_smem(k_wide<MODE, W, false, false>, wide_bytes(false));
    }
    allow_smem(k_hub_accum<MODE, W, WEIGHTED, 1>, hub_smem);
    allow_smem(k_hub_accum<MODE, W, WEIGHTED, 0>, hub_smem);
  });
  int launches = 0;
  cudaStream_t ts = s;  // the current tier's stream
  // A team kernel's launch (full kTeamBatch batches: see launch_group).
  auto team_launch = [&](auto kernel, int threads, int teams, uint32_t max_batch, size_t smem,
                         const uint32_t* list, uint32_t count, bool counter) {
    // A tier of at most one row per team of one CTA per SM (a few stray long rows of a
    // small graph) takes one row per batch: its rows are too few to be neighbours, and a
    // full batch would be one team's serial chain of row latencies (SBM-100K: 10 rows of
    // degree > 32, 25 us per pass as one batch).
    const uint32_t bsz = (small_tier_batch() && count <= uint32_t(teams) * sms) ? 1u : max_batch;
    if (counter) NULPA_CUDA(cudaMemsetAsync(c.work, 0, sizeof(unsigned int), ts));
    kernel<<<resident_grid(kernel, threads, smem, count, teams * bsz, sms), threads, smem, ts>>>(
        c, list, count, bsz);
  };
  // Tier groups (see concurrent_mode): [T_THREAD, T_WARP] and [T_WTAB, T_HUB]. A group
  // with two or more tiers to run goes side by side on the fork's streams when `fk` is
  // given; each of its tiers then has its own work counter (c.work[t]).
  auto runs = [&](int t) {
    return (t == T_HUB ? p.n_hubs != 0 : p.count[t] != 0) && (tiers >> t & 1u) != 0;
  };
  int n_low = 0, n_high = 0;
  uint32_t low_ro = 0xFFFFFFFFu;  // positions above every register tier that runs
  for (int t = T_THREAD; t <= T_HUB; ++t)
    if (runs(t)) {
      if (t <= T_WARP) {
        ++n_low;
        low_ro = std::min(low_ro, p.ro_end[t]);
      } else {
        ++n_high;
      }
    }
  const bool conc_low = fk && (fk->groups & 1u) && n_low >= 2;
  const bool conc_high = fk && (fk->groups & 2u) && n_high >= 2;
  unsigned int* const work0 = c.work;
  bool conc = false;    // the current tier runs beside the others of its group
  auto tier = [&](int t) {
    conc = t <= T_WARP ? conc_low : conc_high;
    ts = conc ? fk->enter(t) : s;
    c.work = conc ? work0 + t : work0;
    c.ctr = ctr + t * C_COUNT;
    const bool ro = t < Plan::kLists && ro_labels() && p.ro_end[T_HUB] != 0;
    // Read-only labels must not be written during the launch: beside other tiers that
    // is only the prefix above the whole register group (and nothing for the table
    // group, whose hub tier sits at the top).
    c.ro_end = !ro ? 0u : !conc ? p.ro_end[t] : t <= T_WARP ? low_ro : 0u;
    c.ro_lo = (ro && !conc && ro_labels_low()) ? p.ro_lo[t] : 0xFFFFFFFFu;
    prof.begin(t, ts);
  };
  if (conc_low) fk->fork(s);
  if (p.count[T_THREAD] && (tiers >> T_THREAD & 1u)) {
    tier(T_THREAD);
    if (p.thread_max <= 8 && MODE == kAsync && p.chunked_thread && p.chunk_L) {
      // the graph's chunk-major range: one thread per chunk of chunk_L entries
      const unsigned gc = grid_for((p.count[T_THREAD] + p.chunk_L - 1) / p.chunk_L, 256, ~0u);
      // (default: the degree-<=4 walk where the range allows it, lattices)
      const int want = chunk_rows() ? chunk_rows() : (p.chunk_dmax <= 4 ? 24 : 14);
      const int rows = (want >= 20 && p.chunk_dmax > 4) ? 14 : want;
      switch (rows) {
        case 24:  // rows of degree <= 4 (lattices): 4-entry registers, 4 rows, prefetched targets
          k_chunk_walk<MODE, W, WEIGHTED, 4, 4, true><<<gc, 256, 0, ts>>>(
              c, p.count[T_THREAD], p.chunk_lo, p.chunk_L);
          break;
        case 28:  // ... 8 rows
          k_chunk_walk<MODE, W, WEIGHTED, 4, 8, true><<<gc, 256, 0, ts>>>(
              c, p.count[T_THREAD], p.chunk_lo, p.chunk_L);
          break;
        case 34:  // degree <= 4, 4 rows, prefetched targets, held to 6 CTAs per SM
          k_chunk_walk<MODE, W, WEIGHTED, 4, 4, true, 6><<<gc, 256, 0, ts>>>(
              c, p.count[T_THREAD], p.chunk_lo, p.chunk_L);
          break;
        case 32:  // ... 2 rows
          k_chunk_walk<MODE, W, WEIGHTED, 4, 2, true, 6><<<gc, 256, 0, ts>>>(
              c, p.count[T_THREAD], p.chunk_lo, p.chunk_L);
          break;
        case 1:
          k_thread<MODE, W, WEIGHTED, 8, true><<<gc, 256, 0, ts>>>(
              c, p.list[T_THREAD], p.count[T_THREAD], p.chunk_lo, p.chunk_L);
          break;
        case 2:
          k_chunk_walk<MODE, W, WEIGHTED, 8, 2><<<gc, 256, 0, ts>>>(c, p.count[T_THREAD],
                                                                     p.chunk_lo, p.chunk_L);
          break;
        case 4:
          k_chunk_walk<MODE, W, WEIGHTED, 8, 4><<<gc, 256, 0, ts>>>(c, p.count[T_THREAD],
                                                                     p.chunk_lo, p.chunk_L);
          break;
        case 8:
          k_chunk_walk<MODE, W, WEIGHTED, 8, 8><<<gc, 256, 0, ts>>>(c, p.count[T_THREAD],
                                                                     p.chunk_lo, p.chunk_L);
          break;
        case 18:  // 8 rows, next row's targets prefetched
          k_chunk_walk<MODE, W, WEIGHTED, 8, 8, true><<<gc, 256, 0, ts>>>(
              c, p.count[T_THREAD], p.chunk_lo, p.chunk_L);
          break;
        default:  // 14: 4 rows, next row's targets prefetched
          k_chunk_walk<MODE, W, WEIGHTED, 8, 4, true><<<gc, 256, 0, ts>>>(
              c, p.count[T_THREAD], p.chunk_lo, p.chunk_L);
      }
    } else if (p.thread_max <= 8 && MODE == kAsync && p.chunked_thread)
      // chunks of >= kMinChunk vertices per thread (a short chunk propagates little)
      k_thread<MODE, W, WEIGHTED, 8, true>
          <<<resident_grid(k_thread<MODE, W, WEIGHTED, 8, true>, 256, 0, p.count[T_THREAD],
                           256 * kMinChunk, sms),
             256, 0, ts>>>(c, p.list[T_THREAD], p.count[T_THREAD]);
    else if (p.thread_max <= 8 && thread_q())
      k_thread_q<MODE, W, WEIGHTED, 8>
          <<<resident_grid(k_thread_q<MODE, W, WEIGHTED, 8>, 256, 0, p.count[T_THREAD], 256 * 4, sms),
             256, 0, ts>>>(c, p.list[T_THREAD], p.count[T_THREAD]);
    else if (p.thread_max <= 8 && thread_pair())
      k_thread<MODE, W, WEIGHTED, 8, false, 2>
          <<<resident_grid(k_thread<MODE, W, WEIGHTED, 8, false, 2>, 256, 0, p.count[T_THREAD], 512, sms),
             256, 0, ts>>>(c, p.list[T_THREAD], p.count[T_THREAD]);
    else if (p.thread_max <= 8)
      k_thread<MODE, W, WEIGHTED, 8>
          <<<resident_grid(k_thread<MODE, W, WEIGHTED, 8>, 256, 0, p.count[T_THREAD], 256, sms),
             256, 0, ts>>>(c, p.list[T_THREAD], p.count[T_THREAD]);
    else
      k_thread<MODE, W, WEIGHTED, 16>
          <<<resident_grid(k_thread<MODE, W, WEIGHTED, 16>, 256, 0, p.count[T_THREAD], 256, sms),
             256, 0, ts>>>(c, p.list[T_THREAD], p.count[T_THREAD]);
    prof.end(T_THREAD, ts);
    ++launches;
  }
  if (p.count[T_HALF] && (tiers >> T_HALF & 1u)) {
    tier(T_HALF);
    launch_group<MODE, W, WEIGHTED, 16>(c, p.list[T_HALF], p.count[T_HALF], ts, sms);
    prof.end(T_HALF, ts);
    ++launches;
  }
  if (p.count[T_WARP] && (tiers >> T_WARP & 1u)) {
    tier(T_WARP);
    launch_group<MODE, W, WEIGHTED, 32>(c, p.list[T_WARP], p.count[T_WARP], ts, sms);
    prof.end(T_WARP, ts);
    ++launches;
  }
  if (conc_low) fk->join(s);
  if (conc_high) fk->fork(s);
  // Hub accumulation beside the table tiers (concurrent_mode 5/6): k_hub_select claims the
  // hubs and k_hub_accum/sweep fill their tables on the hub stream while team32 .. wide run
  // on `s`; the hubs' labels are written only after the join (k_hub_decide), so no other
  // tier sees a hub label change during its launch and every read-only range stays valid.
  // (The accumulation reads labels the table tiers are writing: an async read of an older
  // label, re-examined through the hub's flag, which the writer clears, lpa.cpp:161-163.)
  const bool hub_beside = fk && (fk->groups & 4u) && !conc_high && runs(T_HUB);
  HubCtx h = p.hub_ctx();
  h.stop = c.stop;
  const unsigned gi =
      p.n_hubs ? resident_grid(k_hub_accum<MODE, W, WEIGHTED, 1>, kBlockThreads, hub_smem, p.n_items, 1, sms) : 1u;
  const unsigned gh = grid_for(p.n_hubs, 256, 1024);
  const unsigned gs = grid_for(p.n_sitems, 1, sms * 8);
  auto hub_gather = [&](const PassCtx& hc, cudaStream_t hs) {
    int l = 3;
    k_hub_select<MODE><<<gh, 256, 0, hs>>>(hc, h);
    if (hc.fresh)  // first pass: labels mostly distinct, no in-warp dedupe (see k_team)
      k_hub_accum<MODE, W, WEIGHTED, 0><<<gi, kBlockThreads, hub_smem, hs>>>(hc, h);
    else
      k_hub_accum<MODE, W, WEIGHTED, 1><<<gi, kBlockThreads, hub_smem, hs>>>(hc, h);
    k_hub_sweep<W, WEIGHTED><<<gs, kBlockThreads, 0, hs>>>(h);
    if constexpr (sizeof(VBits<W>) == 8) {
      k_hub_sweep_key_f64<kPacked<WEIGHTED>><<<gs, kBlockThreads, 0, hs>>>(h);
      ++l;
    }
    return l;
  };
  auto hub_finish = [&](const PassCtx& hc, cudaStream_t hs) {
    int l = 1;
    k_hub_decide<MODE, W, WEIGHTED><<<gh, 256, 0, hs>>>(hc, h);
    if (MODE == kAsync && hc.wake) {
      k_hub_wake<<<gi, kBlockThreads, 0, hs>>>(hc, h);
      ++l;
    }
    return l;
  };
  PassCtx chub = c;
  if (hub_beside) {
    fk->fork(s);
    cudaStream_t hs = fk->enter(T_HUB);
    chub.ctr = ctr + T_HUB * C_COUNT;
    chub.work = work0;
    chub.ro_end = (ro_labels() && p.ro_end[T_HUB] != 0) ? p.ro_end[T_HUB] : 0u;
    chub.ro_lo = 0xFFFFFFFFu;
    prof.begin(T_HUB, hs);
    launches += hub_gather(chub, hs);
    prof.end(T_HUB, hs);
  }
  if (p.count[T_WTAB] && (tiers >> T_WTAB & 1u)) {
    tier(T_WTAB);
    team_launch(k_wt, 256, 8, kTeamBatch<32>, wtab_smem, p.list[T_WTAB], p.count[T_WTAB], false);
    prof.end(T_WTAB, ts);
    ++launches;
  }
  if (p.count[T_BLOCK] && (tiers >> T_BLOCK & 1u)) {
    tier(T_BLOCK);
    team_launch(k_b1, 256, 2, kTeamBatch<128>, block_smem, p.list[T_BLOCK], p.count[T_BLOCK], false);
    prof.end(T_BLOCK, ts);
    ++launches;
  }
  if (p.count[T_BLOCK2] && (tiers >> T_BLOCK2 & 1u)) {
    tier(T_BLOCK2);
    team_launch(k_b2, 256, 1, kTeamBatch<256>, block2_smem, p.list[T_BLOCK2], p.count[T_BLOCK2], true);
    prof.end(T_BLOCK2, ts);
    ++launches;
  }
  if (p.count[T_BIG] && (tiers >> T_BIG & 1u)) {
    tier(T_BIG);
    team_launch(k_bg, kMidThreads, 1, kTeamBatch<kMidThreads>, big_smem, p.list[T_BIG], p.count[T_BIG],
                true);
    prof.end(T_BIG, ts);
    ++launches;
  }
  if (p.count[T_CLUSTER] && (tiers >> T_CLUSTER & 1u)) {
    tier(T_CLUSTER);
    NULPA_CUDA(cudaMemsetAsync(c.work, 0, sizeof(unsigned int), ts));
    // persistent clusters pull vertices from c.work; grid a multiple of the cluster size
    const unsigned gc = std::max<unsigned>(kClusterSize, (sms / kClusterSize) * kClusterSize);
    if constexpr (WEIGHTED)
      k_cluster<MODE, W, WEIGHTED><<<gc, kBigThreads, cluster_smem, ts>>>(c, p.list[T_CLUSTER],
                                                                        p.count[T_CLUSTER]);
    else
      launch_wide<MODE, W>(p, c, ts, sms);
    prof.end(T_CLUSTER, ts);
    ++launches;
  }
  if (p.n_hubs && (tiers >> T_HUB & 1u)) {
    if (hub_beside) {
      fk->join(s);  // the hub tables are complete: decide and wake after the table tiers
      launches += hub_finish(chub, s);
    } else {
      tier(T_HUB);
      launches += hub_gather(c, ts);
      launches += hub_finish(c, ts);
      prof.end(T_HUB, ts);
    }
  }
  if (conc_high) fk->join(s);
  NULPA_CUDA(cudaGetLastError());
  return launches;
}

template <int MODE>
int dispatch_pass(const Plan& p, const PassCtx& c, unsigned long long* ctr, int value_bytes,
                  cudaStream_t s, int sms, Prof& prof, unsigned tiers = ~0u, Fork* fk = nullptr) {
  const bool weighted = c.g.w != nullptr;
  if (value_bytes == 8)
    return weighted ? launch_pass<MODE, double, true>(p, c, ctr, s, sms, prof, tiers, fk)
                    : launch_pass<MODE, double, false>(p, c, ctr, s, sms, prof, tiers, fk);
  return weighted ? launch_pass<MODE, float, true>(p, c, ctr, s, sms, prof, tiers, fk)
                  : launch_pass<MODE, float, false>(p, c, ctr, s, sms, prof, tiers, fk);
}

// ParallelAsync first pass, long rows first: every tier of degree > block_max runs
// the table-free identity rule (k_first_pass_list; all of them read identity
// labels), then the lower tiers run in place and see those moves.
int long_rows_first_pass(const Plan& p, PassCtx c, unsigned long long* ctr, int value_bytes,
                         cudaStream_t s, int sms, Prof& prof, int first_tier = T_BLOCK2) {
  int launches = 0;
  for (int t = T_HUB; t >= first_tier; --t) {
    if (!p.count[t]) continue;
    c.ctr = ctr + t * C_COUNT;
    prof.begin(t, s);
    k_first_pass_list<kAsync><<<grid_for(p.count[t], 256, sms * 8), 256, 0, s>>>(c, p.list[t],
                                                                                p.count[t]);
    prof.end(t, s);
    ++launches;
  }
  NULPA_CUDA(cudaGetLastError());
  const unsigned low = (1u << first_tier) - 1u;  // the tiers below first_tier
  return launches + dispatch_pass<kAsync>(p, c, ctr, value_bytes, s, sms, prof, low);
}

template <typename W, bool WEIGHTED>
void launch_sequential(const PassCtx& c, void* gtab, cudaStream_t s) {
  constexpr size_t smem = kHubCap * Table<kPacked<WEIGHTED>, W>::kSlotBytes;
  static std::atomic<uint64_t> init{0};
  once_per_device(init, [&] { allow_smem(k_sequential<W, WEIGHTED>, smem); });
  k_sequential<W, WEIGHTED><<<1, kBlockThreads, smem, s>>>(c, gtab);
  NULPA_CUDA(cudaGetLastError());
}

void validate_opts(const nulpa_graph* g, const nulpa_opts& o) {
  // validate_config, lpa.cpp:317-326 — identical messages.
  if (g->n == 0) throw Error(NULPA_EINVAL, "label propagation requires a non-empty graph");
  if (!(o.tolerance > 0.0 && o.tolerance <= 1.0))
    throw Error(NULPA_EINVAL, "tolerance must lie in (0, 1]");
  if (o.max_iterations < 1) throw Error(NULPA_EINVAL, "max-iterations must be >= 1");
  if (o.pl_period < 0) throw Error(NULPA_EINVAL, "pl-period must be >= 0");
  if (o.cc_period < 0) throw Error(NULPA_EINVAL, "cc-period must be >= 0");
  if (o.switch_degree < 2) throw Error(NULPA_EINVAL, "switch-degree must be >= 2");
  if (o.workers < 0) throw Error(NULPA_EINVAL, "workers must be >= 0");
  if (o.exec < 0 || o.exec > 2) throw Error(NULPA_EINVAL, "unknown execution mode");
  if (o.strategy < 0 || o.strategy > 3) throw Error(NULPA_EINVAL, "unknown probe strategy");
}

struct Stream {
  cudaStream_t s = nullptr;
  Stream() { NULPA_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~Stream() {
    if (s) cudaStreamDestroy(s);
  }
};

template <typename T>
struct DBuf {
  T* p = nullptr;
  DBuf() = default;
  explicit DBuf(size_t n) : p(dalloc<T>(n)) {}
  ~DBuf() { dfree(p); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(DBuf&& o) noexcept {
    std::swap(p, o.p);
    return *this;
  }
};

// Pinned host counters. Buffers are recycled through a per-thread free list:
// cudaHostAlloc / cudaFreeHost on every call cost milliseconds (and can stall on
// the driver's unmap), far more than the counters they carry.
struct Pinned {
  unsigned long long* p = nullptr;
  size_t cap = 0;
  explicit Pinned(size_t count = C_COUNT) {
    auto& fl = free_list();
    for (size_t k = 0; k < fl.size(); ++k)
      if (fl[k].second >= count) {
        p = fl[k].first;
        cap = fl[k].second;
        fl.erase(fl.begin() + k);
        return;
      }
    NULPA_CUDA(cudaHostAlloc(&p, count * sizeof(unsigned long long), cudaHostAllocDefault));
    cap = count;
  }
  ~Pinned() {
    if (p) free_list().emplace_back(p, cap);
  }
  Pinned(const Pinned&) = delete;
  Pinned& operator=(const Pinned&) = delete;
  static std::vector<std::pair<unsigned long long*, size_t>>& free_list() {
    static thread_local std::vector<std::pair<unsigned long long*, size_t>> fl;
    return fl;
  }
};

// cross_check (lpa.cpp:338-360) on the device; returns the revert count.
// Arrays in position order.
uint64_t device_cross_check(nulpa_graph* g, uint32_t* lab, const uint32_t* prev, uint8_t* flags,
                            unsigned long long* d_aux, unsigned long long* h_aux, cudaStream_t s,
                            int sms, uint64_t* launches = nullptr) {
  const uint32_t n = g->n;
  DBuf<uint8_t> r0(n), r1(n);
  NULPA_CUDA(cudaMemsetAsync(r0.p, 0, n, s));
  uint8_t* rin = r0.p;
  uint8_t* rout = r1.p;
  const unsigned gb = grid_for(n, 256, sms * 8);
  for (uint32_t round = 0; round <= n; ++round) {
    NULPA_CUDA(cudaMemsetAsync(d_aux, 0, sizeof(unsigned long long), s));
    k_cc_round<<<gb, 256, 0, s>>>(lab, prev, rin, rout, n, d_aux, g->perm, g->inv);
    NULPA_CUDA(cudaGetLastError());
    if (launches) ++*launches;
    NULPA_CUDA(cudaMemcpyAsync(h_aux, d_aux, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    NULPA_CUDA(cudaStreamSynchronize(s));
    std::swap(rin, rout);
    if (*h_aux == 0) break;
  }
  Graph dg{g->offsets, g->targets, g->weights, n};
  NULPA_CUDA(cudaMemsetAsync(d_aux, 0, sizeof(unsigned long long), s));
  k_cc_apply<<<grid_for(n, 256, sms * 8), 256, 0, s>>>(dg, lab, prev, rin, flags, d_aux);
  NULPA_CUDA(cudaGetLastError());
  if (launches) ++*launches;
  NULPA_CUDA(cudaMemcpyAsync(h_aux, d_aux, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  return *h_aux;
}

}  // namespace

void run_lpa(nulpa_graph* g, const nulpa_opts& o, const nulpa_tuning* tuning,
             uint32_t* labels_host, uint32_t* labels_dev_out, nulpa_stats* st) {
  Trace tr("run_lpa");
  validate_opts(g, o);
  use_device(g->device);
  std::lock_guard<std::recursive_mutex> plan_lock(g->plan_mu);
  const auto t_setup = std::chrono::steady_clock::now();
  Stream stream;
  cudaStream_t s = stream.s;
  const int sms = sm_count();
  const int vbytes = o.precision == 64 ? 8 : 4;
  const uint32_t n = g->n;
  Plan* p = get_plan(g, resolve_tiers(o.switch_degree, tuning), vbytes, s);

  DBuf<uint32_t> lab0(n), lab1, prev, changed;
  DBuf<uint8_t> flags(n);
  constexpr int kCtr = kTiers * C_COUNT;
  // Passes are enqueued kBatch at a time behind a device-side pass guard (k_decide) and
  // their counters read back once per batch, so a small graph's run is not one host
  // round trip per pass. Cross-check (a host-driven fixpoint) and Sequential mode keep
  // one read-back per pass.
  const bool batched = o.cc_period == 0 && o.exec != NULPA_EXEC_SEQUENTIAL &&
                       !(tuning && tuning->unbatched);
  const int kBatch = batched ? std::max(1, std::min(o.max_iterations, batch_passes())) : 1;
  const int blocks = batched ? o.max_iterations : 1;  // one counter block per pass
  DBuf<unsigned long long> ctr(size_t(kCtr) * blocks);
  DBuf<unsigned int> work(kTiers);  // work counters of the team / wide tiers (one per tier)
  // Tier streams for side-by-side tiers (concurrent_mode), leased for the whole run.
  const int cmode = concurrent_mode();
  Fork* fk = nullptr;
  std::unique_lock<std::mutex> fork_lock;
  const unsigned groups = cmode == 1 || (cmode == 2 && n <= (1u << 22)) ? 3u
                          : cmode == 2 || cmode == 3 ? 1u : cmode == 4 ? 2u
                          : cmode == 5 ? 5u : cmode == 6 ? 4u : 0u;
  if (groups) {
    Fork& f = Fork::of_device(g->device);
    fork_lock = std::unique_lock<std::mutex>(f.mu, std::try_to_lock);
    if (fork_lock.owns_lock()) {
      f.init();
      f.groups = groups;
      fk = &f;
    }
  }
  DBuf<unsigned int> stop(1);
  Pinned hc(size_t(kCtr) * blocks + 1);
  unsigned long long* hstop = hc.p + size_t(kCtr) * blocks;
  NULPA_CUDA(cudaMemsetAsync(ctr.p, 0, size_t(kCtr) * blocks * sizeof(unsigned long long), s));
  NULPA_CUDA(cudaMemsetAsync(stop.p, 0, sizeof(unsigned), s));
  if (o.exec == NULPA_EXEC_SYNCHRONOUS) {
    lab1 = DBuf<uint32_t>(n);
    changed = DBuf<uint32_t>(n);
  }
  if (o.cc_period > 0) prev = DBuf<uint32_t>(n);
  DBuf<unsigned char> seq_tab;  // global table for Sequential rows beyond shared memory
  if (o.exec == NULPA_EXEC_SEQUENTIAL) {
    const uint64_t cap = pow2_ceil(2 * std::max<uint32_t>(g->max_degree, 1));
    if (cap > static_cast<uint64_t>(kHubCap)) seq_tab = DBuf<unsigned char>(cap * (4 + 8));
  }
  // per-tier CUDA events, one set per pass of a batch
  std::vector<Prof> profs(kBatch);
  const bool prof_on = tuning && tuning->profile;
  for (Prof& pf : profs) {
    pf.on = prof_on;
    if (prof_on)
      for (auto& e : pf.ev) {
        NULPA_CUDA(cudaEventCreate(&e[0]));
        NULPA_CUDA(cudaEventCreate(&e[1]));
      }
  }
  tr.mark("plan + buffers");
  L2Window l2win(s, lab0.p, n);
  k_init<<<grid_for(n, 256, sms * 8), 256, 0, s>>>(lab0.p, flags.p, g->offsets, n, g->perm);
  NULPA_CUDA(cudaGetLastError());
  NULPA_CUDA(cudaStreamSynchronize(s));
  const double setup_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t_setup).count();

  cudaEvent_t ev0, ev1;
  NULPA_CUDA(cudaEventCreate(&ev0));
  NULPA_CUDA(cudaEventCreate(&ev1));
  NULPA_CUDA(cudaEventRecord(ev0, s));

  const Graph dg{g->offsets, g->targets, g->weights, n};
  // Table-free first pass from identity labels (k_first_pass): unit weights and
  // strictly ascending rows make every neighbour label unique.
  const bool identity_first =
      g->rows_simple && g->weights == nullptr && !(tuning && tuning->no_identity_first);
  int iterations = 0, pl_iterations = 0;
  bool converged = false;
  uint64_t cc_reverts = 0, tot_v = 0, tot_e = 0, tot_w = 0, launches = 0;
  double tier_ms[kTiers] = {0}, tier_bytes[kTiers] = {0};
  uint64_t tier_edges[kTiers] = {0};
  uint32_t tier_passes[kTiers] = {0};
  const double edge_bytes = g->weights ? 12.0 : 8.0;
  uint32_t* cur = lab0.p;
  uint32_t* nxt = lab1.p;

  // Host bookkeeping of one finished pass from its counter block (returns dN).
  auto absorb = [&](const unsigned long long* blk, Prof& pf, bool pl, uint64_t reverted) {
    uint64_t raw_dn = 0;
    for (int t = 0; t < kTiers; ++t) {
      const unsigned long long* k = blk + t * C_COUNT;
      if (k[C_FAIL])
        throw Error(NULPA_EINTERNAL, "hashtable insertion failed (capacity invariant violated)");
      raw_dn += k[C_DN];
      tot_v += k[C_PROC_V];
      tot_e += k[C_PROC_E];
      tot_w += k[C_WAKE_E];
      tier_edges[t] += k[C_PROC_E];
      // SURVEY §8d per tier: flag sweep over the tier's list (1 B), row bounds
      // + own label of processed vertices (12 B), target + neighbour label
      // (+ weight) per scanned edge, label write per change, wake store per
      // neighbour of a changed vertex.
      const double list_len = t < Plan::kLists ? p->count[t] : 0.0;
      tier_bytes[t] += list_len + 12.0 * k[C_PROC_V] + edge_bytes * k[C_PROC_E] +
                       4.0 * k[C_DN] + double(k[C_WAKE_E]);
      if (pf.used[t]) {
        ++tier_passes[t];
        if (pf.on) {
          float tms = 0.f;
          NULPA_CUDA(cudaEventElapsedTime(&tms, pf.ev[t][0], pf.ev[t][1]));
          tier_ms[t] += tms;
        }
      }
    }
    const uint64_t dn = raw_dn - reverted;
    cc_reverts += reverted;
    if (st && st->delta_n) st->delta_n[iterations] = dn;
    ++iterations;
    if (pl) ++pl_iterations;
    return dn;
  };

  for (int iter = 0; iter < o.max_iterations; ++iter) {
    const bool pick_less = o.pl_period > 0 && iter % o.pl_period == 0;
    const bool check = o.cc_period > 0 && iter % o.cc_period == 0;
    if (check) NULPA_CUDA(cudaMemcpyAsync(prev.p, cur, n * 4ull, cudaMemcpyDeviceToDevice, s));
    const bool was_pl = iter > 0 && o.pl_period > 0 && (iter - 1) % o.pl_period == 0;
    if (!o.prune || (was_pl && !pick_less)) NULPA_CUDA(cudaMemsetAsync(flags.p, 0, n, s));
    unsigned long long* ctr_it = ctr.p + size_t(kCtr) * (batched ? iter : 0);
    unsigned long long* ctr_other = ctr_it + T_OTHER * C_COUNT;
    if (!batched) NULPA_CUDA(cudaMemsetAsync(ctr_it, 0, kCtr * sizeof(unsigned long long), s));
    Prof& prof = profs[iter % kBatch];
    for (bool& u : prof.used) u = false;

    // Neighbour wake-ups are dead stores when the next pass resets every flag
    // (or there is no next pass) and no reader inside this pass can see them
    // (Synchronous wakes after the pass; an async pass that started from
    // all-zero flags only wakes vertices whose flag is already 0 or that were
    // already examined). Skipping them leaves every result unchanged.
    const bool this_reset = iter == 0 || !o.prune || (was_pl && !pick_less);
    const bool next_pl = o.pl_period > 0 && (iter + 1) % o.pl_period == 0;
    const bool next_reset = iter + 1 >= o.max_iterations || !o.prune || (pick_less && !next_pl);
    const bool wake = !(next_reset && (this_reset || o.exec == NULPA_EXEC_SYNCHRONOUS));

    PassCtx c;
    c.g = dg;
    c.flags = flags.p;
    c.ctr = ctr_it;
    c.stop = batched ? stop.p : nullptr;
    c.pick_less = pick_less ? 1 : 0;
    c.strategy = o.strategy;
    c.changed = nullptr;
    c.changed_n = ctr_other + C_NCHANGED;
    c.wake = wake ? 1 : 0;
    c.work = work.p;
    c.vid = g->perm;
    c.pos = g->inv;
    c.fresh = iter == 0 ? 1 : 0;
    c.hints = iter > 0 ? 1 : 0;
    // Synchronous only: there the identity first pass is exactly the reference's.
    // (Under ParallelAsync it is a legal schedule too, but it replaces the in-place
    // first pass, whose early label flooding converges R-MAT one pass sooner and
    // which the reference's low-tier-first KATs rely on, test_lpa.cpp:256-267.)
    const bool first_async = o.exec == NULPA_EXEC_PARALLEL_ASYNC && tuning &&
                             tuning->async_first_pass == 1;
    if (iter == 0 && identity_first && (o.exec == NULPA_EXEC_SYNCHRONOUS || first_async)) {
      // Labels are still the identity: the table-free first pass (k_first_pass).
      c.lab_in = cur;
      c.lab_out = o.exec == NULPA_EXEC_SYNCHRONOUS ? nxt : cur;
      c.ctr = ctr_it + T_THREAD * C_COUNT;
      c.changed = (o.exec == NULPA_EXEC_SYNCHRONOUS && wake) ? changed.p : nullptr;
      if (o.exec == NULPA_EXEC_SYNCHRONOUS)
        NULPA_CUDA(cudaMemcpyAsync(nxt, cur, n * 4ull, cudaMemcpyDeviceToDevice, s));
      prof.begin(T_THREAD, s);
      if (o.exec == NULPA_EXEC_SYNCHRONOUS)
        k_first_pass<kSync><<<grid_for(n, 256, sms * 8), 256, 0, s>>>(c, 0, n);
      else
        k_first_pass<kAsync><<<grid_for(n, 256, sms * 8), 256, 0, s>>>(c, 0, n);
      prof.end(T_THREAD, s);
      ++launches;
      NULPA_CUDA(cudaGetLastError());
      if (o.exec == NULPA_EXEC_SYNCHRONOUS) {
        if (wake) {
          k_wake_list<<<grid_for(n, kBlockThreads / 32, sms * 8), kBlockThreads, 0, s>>>(
              dg, flags.p, changed.p, ctr_other + C_NCHANGED, ctr_other, c.stop);
          ++launches;
        }
        std::swap(cur, nxt);
      }
    } else if (o.exec == NULPA_EXEC_PARALLEL_ASYNC && iter == 0 && identity_first && tuning &&
               tuning->async_first_pass >= 2) {
      // 2: degree > block_max first, 3: the wide and hub tiers first, 4: hubs first
      c.lab_in = cur;
      c.lab_out = cur;
      const int ft = tuning->async_first_pass == 2 ? T_BLOCK2
                     : tuning->async_first_pass == 3 ? T_CLUSTER : T_HUB;
      launches += long_rows_first_pass(*p, c, ctr_it, vbytes, s, sms, prof, ft);
    } else if (o.exec == NULPA_EXEC_PARALLEL_ASYNC) {
      c.lab_in = cur;
      c.lab_out = cur;
      launches += dispatch_pass<kAsync>(*p, c, ctr_it, vbytes, s, sms, prof, ~0u, fk);
    } else if (o.exec == NULPA_EXEC_SYNCHRONOUS) {
      // sync_move (lpa.cpp:70-100): frozen snapshot `cur`, staged writes to `nxt`,
      // wake-ups after the joint application.
      NULPA_CUDA(cudaMemcpyAsync(nxt, cur, n * 4ull, cudaMemcpyDeviceToDevice, s));
      c.lab_in = cur;
      c.lab_out = nxt;
      c.changed = wake ? changed.p : nullptr;
      launches += dispatch_pass<kSync>(*p, c, ctr_it, vbytes, s, sms, prof, ~0u, fk);
      if (wake) {
        prof.begin(T_OTHER, s);
        k_wake_list<<<grid_for(n, kBlockThreads / 32, sms * 8), kBlockThreads, 0, s>>>(
            dg, flags.p, changed.p, ctr_other + C_NCHANGED, ctr_other, c.stop);
        prof.end(T_OTHER, s);
        ++launches;
        NULPA_CUDA(cudaGetLastError());
      }
      std::swap(cur, nxt);
    } else {
      c.lab_in = cur;
      c.lab_out = cur;
      c.ctr = ctr_other;
      prof.begin(T_OTHER, s);
      if (vbytes == 8) {
        if (dg.w)
          launch_sequential<double, true>(c, seq_tab.p, s);
        else
          launch_sequential<double, false>(c, seq_tab.p, s);
      } else {
        if (dg.w)
          launch_sequential<float, true>(c, seq_tab.p, s);
        else
          launch_sequential<float, false>(c, seq_tab.p, s);
      }
      prof.end(T_OTHER, s);
      ++launches;
    }
    if (batched) {
      k_decide<<<1, 32, 0, s>>>(ctr_it, n, o.tolerance, pick_less ? 1 : 0, iter, stop.p);
      ++launches;
      NULPA_CUDA(cudaGetLastError());
      // read back once per batch: the guard and the batch's counter blocks
      const int first = iterations;
      if ((iter + 1) % kBatch == 0 || iter + 1 == o.max_iterations) {
        NULPA_CUDA(cudaMemcpyAsync(hc.p + size_t(kCtr) * first, ctr.p + size_t(kCtr) * first,
                                   size_t(kCtr) * (iter + 1 - first) * sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, s));
        NULPA_CUDA(cudaMemcpyAsync(hstop, stop.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
        *hstop = 0;
        NULPA_CUDA(cudaStreamSynchronize(s));
        const unsigned sv = static_cast<unsigned>(*hstop & 0xFFFFFFFFull);
        const int last = sv ? static_cast<int>(sv) : iter + 1;  // passes that ran
        for (int it = first; it < last; ++it) {
          const bool pl = o.pl_period > 0 && it % o.pl_period == 0;
          absorb(hc.p + size_t(kCtr) * it, profs[it % kBatch], pl, 0);
        }
        if (sv) {
          converged = true;
          break;
        }
      }
      continue;
    }
    uint64_t reverted = 0;
    if (check)
      reverted = device_cross_check(g, cur, prev.p, flags.p, ctr_other + C_AUX,
                                    hc.p + T_OTHER * C_COUNT + C_AUX, s, sms, &launches);
    NULPA_CUDA(cudaMemcpyAsync(hc.p, ctr_it, kCtr * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s));
    NULPA_CUDA(cudaStreamSynchronize(s));
    const uint64_t dn = absorb(hc.p, prof, pick_less, reverted);
    if (!pick_less && static_cast<double>(dn) / n < o.tolerance) {
      converged = true;
      break;
    }
  }
  NULPA_CUDA(cudaEventRecord(ev1, s));
  NULPA_CUDA(cudaEventSynchronize(ev1));
  float ms = 0.f;
  NULPA_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  for (Prof& pf : profs)
    if (pf.on)
      for (auto& e : pf.ev) {
        cudaEventDestroy(e[0]);
        cudaEventDestroy(e[1]);
      }

  tr.mark("loop");
  // Results leave in vertex order (layout.cu).
  if (labels_dev_out) to_vertices_u32(g, cur, labels_dev_out, s);
  if (labels_host) {
    const uint32_t* src = cur;
    if (g->perm) {
      if (labels_dev_out) {
        src = labels_dev_out;
      } else {
        if (!nxt) lab1 = DBuf<uint32_t>(n);
        uint32_t* tmp = cur == lab0.p ? lab1.p : lab0.p;
        to_vertices_u32(g, cur, tmp, s);
        src = tmp;
      }
    }
    NULPA_CUDA(cudaMemcpyAsync(labels_host, src, n * 4ull, cudaMemcpyDeviceToHost, s));
  }
  NULPA_CUDA(cudaStreamSynchronize(s));
  tr.mark("labels out");
  if (st) {
    st->iterations = iterations;
    st->converged = converged ? 1 : 0;
    st->pl_iterations = pl_iterations;
    st->reserved = 0;
    st->cc_reverts = cc_reverts;
    st->elapsed_seconds = ms * 1e-3;
    st->processed_vertices = tot_v;
    st->processed_edges = tot_e;
    st->wake_edges = tot_w;
    double total = 0.0;
    for (int t = 0; t < kTiers; ++t) {
      st->tier_ms[t] = tier_ms[t];
      st->tier_bytes[t] = tier_bytes[t];
      st->tier_edges[t] = tier_edges[t];
      st->tier_passes[t] = tier_passes[t];
      total += tier_bytes[t];
    }
    st->algorithmic_bytes = static_cast<uint64_t>(total);
    st->setup_seconds = setup_s;
    st->kernel_launches = launches;
  }
}

uint64_t run_sync_step(nulpa_graph* g, const uint32_t* lab_in_dev, int pick_less, int strategy,
                       int precision, uint32_t* lab_out_dev) {
  use_device(g->device);
  std::lock_guard<std::recursive_mutex> plan_lock(g->plan_mu);
  if (strategy < 0 || strategy > 3) throw Error(NULPA_EINVAL, "unknown probe strategy");
  Stream stream;
  cudaStream_t s = stream.s;
  const int sms = sm_count();
  const int vbytes = precision == 64 ? 8 : 4;
  Plan* p = get_plan(g, resolve_tiers(32, nullptr), vbytes, s);
  constexpr int kCtr = kTiers * C_COUNT;
  DBuf<unsigned long long> ctr(kCtr);
  Pinned hc(kCtr);
  NULPA_CUDA(cudaMemsetAsync(ctr.p, 0, kCtr * sizeof(unsigned long long), s));
  // Labels arrive and leave in vertex order; the pass runs in position order.
  DBuf<uint32_t> pin, pout;
  const uint32_t* in_p = lab_in_dev;
  uint32_t* out_p = lab_out_dev;
  if (g->perm) {
    pin = DBuf<uint32_t>(g->n);
    pout = DBuf<uint32_t>(g->n);
    to_positions_u32(g, lab_in_dev, pin.p, s);
    in_p = pin.p;
    out_p = pout.p;
  }
  NULPA_CUDA(cudaMemcpyAsync(out_p, in_p, g->n * 4ull, cudaMemcpyDeviceToDevice, s));
  PassCtx c;
  c.g = Graph{g->offsets, g->targets, g->weights, g->n};
  c.vid = g->perm;
  c.pos = g->inv;
  c.lab_in = in_p;
  c.lab_out = out_p;
  c.flags = nullptr;
  c.ctr = ctr.p;
  c.changed = nullptr;
  c.changed_n = ctr.p + T_OTHER * C_COUNT + C_NCHANGED;
  c.pick_less = pick_less ? 1 : 0;
  c.strategy = strategy;
  c.wake = 0;
  DBuf<unsigned int> work(2);
  c.work = work.p;
  Prof prof;
  dispatch_pass<kSync>(*p, c, ctr.p, vbytes, s, sms, prof);
  if (g->perm) to_vertices_u32(g, out_p, lab_out_dev, s);
  NULPA_CUDA(cudaMemcpyAsync(hc.p, ctr.p, kCtr * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  uint64_t dn = 0;
  for (int t = 0; t < kTiers; ++t) {
    if (hc.p[t * C_COUNT + C_FAIL])
      throw Error(NULPA_EINTERNAL, "hashtable insertion failed (capacity invariant violated)");
    dn += hc.p[t * C_COUNT + C_DN];
  }
  return dn;
}

// Vertex-order device arrays (labels and flags updated in place).
uint64_t run_cross_check(nulpa_graph* g, uint32_t* lab_dev, const uint32_t* prev_dev,
                         uint8_t* flags_dev) {
  use_device(g->device);
  Stream stream;
  cudaStream_t s = stream.s;
  DBuf<unsigned long long> aux(1);
  Pinned hc;
  if (!g->perm)
    return device_cross_check(g, lab_dev, prev_dev, flags_dev, aux.p, hc.p, s, sm_count());
  const uint32_t n = g->n;
  DBuf<uint32_t> l(n), pv(n);
  DBuf<uint8_t> f(n);
  to_positions_u32(g, lab_dev, l.p, s);
  to_positions_u32(g, prev_dev, pv.p, s);
  to_positions_u8(g, flags_dev, f.p, s);
  const uint64_t r = device_cross_check(g, l.p, pv.p, f.p, aux.p, hc.p, s, sm_count());
  to_vertices_u32(g, l.p, lab_dev, s);
  to_vertices_u8(g, f.p, flags_dev, s);
  NULPA_CUDA(cudaStreamSynchronize(s));
  return r;
}

}  // namespace nulpa

// ---- pass-level session over a vertex range (multi-GPU partition) ------------

struct nulpa_session {
  nulpa_graph* g = nullptr;
  nulpa_opts o{};
  nulpa::Plan* plan = nullptr;
  uint32_t lo = 0, hi = 0;
  uint32_t* labels = nullptr;  // caller device array [n] (replicated)
  uint8_t* flags = nullptr;    // caller device array [n]
  nulpa::DBuf<uint32_t> staging, changed;
  nulpa::DBuf<uint32_t> snapshot;  // labels[lo, hi) at the start of the last pass
  nulpa::DBuf<unsigned long long> ctr;
  nulpa::DBuf<unsigned int> work{2};
  nulpa::Pinned hc{nulpa::dev::kTiers * nulpa::dev::C_COUNT};
  nulpa::Stream stream;
  int sms = 148, vbytes = 4;
  cudaStream_t ext = nullptr;   // caller's stream (nulpa_session_set_stream; may be the
  bool has_ext = false;         // legacy default stream 0), else `stream`
  bool fresh = false;           // labels are the identity (after nulpa_session_init)
  bool identity_first = false;  // graph allows the table-free first pass
  uint64_t passes = 0;          // passes since nulpa_session_init
  ~nulpa_session() { delete plan; }
};

namespace nulpa {
namespace {
__global__ void k_copy_range(const uint32_t* src, uint32_t* dst, uint32_t lo, uint32_t hi) {
  for (uint32_t i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// Changed-only exchange: (position, label) pairs of the range's changed labels,
// compacted with one atomic per warp, then padded with kEmpty pairs up to `cap`.
__global__ void k_pack_changes(const uint32_t* lab, const uint32_t* snap, uint32_t lo, uint32_t hi,
                               uint32_t* out, uint32_t cap, unsigned* count) {
  const uint32_t span = hi - lo, bound = (span + 31u) & ~31u;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < bound; t += gridDim.x * blockDim.x) {
    const bool ch = t < span && lab[lo + t] != snap[t];
    const unsigned m = __ballot_sync(dev::kFull, ch);
    if (!m) continue;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    unsigned b = 0;
    if (lane == leader) b = atomicAdd(count, static_cast<unsigned>(__popc(m)));
    b = __shfl_sync(dev::kFull, b, leader) + __popc(m & ((1u << lane) - 1u));
    if (ch && b < cap) {
      out[2ull * b] = lo + t;
      out[2ull * b + 1] = lab[lo + t];
    }
  }
}

__global__ void k_pad_changes(uint32_t* out, uint32_t cap, const unsigned* count) {
  const uint32_t first = min(*count, cap);
  for (uint32_t k = first + blockIdx.x * blockDim.x + threadIdx.x; k < cap; k += gridDim.x * blockDim.x) {
    out[2ull * k] = dev::kEmpty;
    out[2ull * k + 1] = dev::kEmpty;
  }
}

__global__ void k_apply_changes(uint32_t* lab, const uint32_t* in, uint64_t pairs) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < pairs;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t p = in[2 * k];
    if (p != dev::kEmpty) lab[p] = in[2 * k + 1];
  }
}

__global__ void k_edge_bounds(const uint64_t* off, uint32_t n, uint32_t parts, uint32_t* bounds) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > parts) return;
  if (p == 0) {
    bounds[0] = 0;
    return;
  }
  if (p == parts) {
    bounds[parts] = n;
    return;
  }
  // smallest v with off[v] >= p * m2 / parts (edge-balanced 1-D split)
  const uint64_t target = (off[n] * p) / parts;
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (off[mid] >= target)
      hi = mid;
    else
      lo = mid + 1;
  }
  bounds[p] = lo;
}
}  // namespace

void session_pass(nulpa_session* ss, int pick_less, int wake, nulpa_pass_info* info) {
  using namespace dev;
  nulpa_graph* g = ss->g;
  cudaStream_t s = ss->has_ext ? ss->ext : ss->stream.s;
  constexpr int kCtr = kTiers * C_COUNT;
  NULPA_CUDA(cudaMemsetAsync(ss->ctr.p, 0, kCtr * sizeof(unsigned long long), s));
  PassCtx c;
  c.g = Graph{g->offsets, g->targets, g->weights, g->n};
  c.flags = ss->flags;
  c.ctr = ss->ctr.p;
  c.pick_less = pick_less ? 1 : 0;
  c.strategy = ss->o.strategy;
  c.changed = nullptr;
  unsigned long long* other = ss->ctr.p + T_OTHER * C_COUNT;
  c.changed_n = other + C_NCHANGED;
  c.wake = wake ? 1 : 0;
  c.work = ss->work.p;
  c.vid = g->perm;
  c.pos = g->inv;
  c.fresh = ss->fresh ? 1 : 0;
  c.hints = ss->passes > 0 ? 1 : 0;  // hints written by this session's earlier passes
  ++ss->passes;
  Prof prof;
  cudaEvent_t e0, e1;
  NULPA_CUDA(cudaEventCreate(&e0));
  NULPA_CUDA(cudaEventCreate(&e1));
  // the range's labels before the pass (nulpa_session_pack_changes diffs against it)
  if (ss->hi > ss->lo)
    NULPA_CUDA(cudaMemcpyAsync(ss->snapshot.p, ss->labels + ss->lo, (ss->hi - ss->lo) * 4ull,
                               cudaMemcpyDeviceToDevice, s));
  NULPA_CUDA(cudaEventRecord(e0, s));
  uint64_t launches = 0;
  const bool first =
      ss->fresh && ss->identity_first && ss->o.exec == NULPA_EXEC_SYNCHRONOUS;  // see run_lpa
  ss->fresh = false;
  if (first && ss->o.exec == NULPA_EXEC_PARALLEL_ASYNC) {
    c.lab_in = ss->labels;
    c.lab_out = ss->labels;
    c.ctr = ss->ctr.p + T_THREAD * C_COUNT;
    k_first_pass<kAsync><<<grid_for(ss->hi - ss->lo, 256, ss->sms * 8), 256, 0, s>>>(c, ss->lo,
                                                                                   ss->hi);
    ++launches;
  } else if (ss->o.exec == NULPA_EXEC_PARALLEL_ASYNC) {
    c.lab_in = ss->labels;
    c.lab_out = ss->labels;
    launches += dispatch_pass<kAsync>(*ss->plan, c, ss->ctr.p, ss->vbytes, s, ss->sms, prof);
  } else {
    // Synchronous: decisions from the replicated snapshot into `staging`, applied to
    // the owned range after the pass, then the deferred wake (lpa.cpp:92-98).
    NULPA_CUDA(cudaMemcpyAsync(ss->staging.p, ss->labels, g->n * 4ull, cudaMemcpyDeviceToDevice, s));
    c.lab_in = ss->labels;
    c.lab_out = ss->staging.p;
    c.changed = wake ? ss->changed.p : nullptr;
    if (first) {
      c.ctr = ss->ctr.p + T_THREAD * C_COUNT;
      k_first_pass<kSync><<<grid_for(ss->hi - ss->lo, 256, ss->sms * 8), 256, 0, s>>>(c, ss->lo,
                                                                                    ss->hi);
      ++launches;
    } else {
      launches += dispatch_pass<kSync>(*ss->plan, c, ss->ctr.p, ss->vbytes, s, ss->sms, prof);
    }
    k_copy_range<<<grid_for(ss->hi - ss->lo, 256, ss->sms * 8), 256, 0, s>>>(
        ss->staging.p, ss->labels, ss->lo, ss->hi);
    ++launches;
    if (wake) {
      k_wake_list<<<grid_for(ss->hi - ss->lo, kBlockThreads / 32, ss->sms * 8), kBlockThreads,
                    0, s>>>(c.g, ss->flags, ss->changed.p, other + C_NCHANGED, other);
      ++launches;
    }
    NULPA_CUDA(cudaGetLastError());
  }
  NULPA_CUDA(cudaEventRecord(e1, s));
  NULPA_CUDA(cudaMemcpyAsync(ss->hc.p, ss->ctr.p, kCtr * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  float ms = 0.f;
  NULPA_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  nulpa_pass_info r{};
  for (int t = 0; t < kTiers; ++t) {
    const unsigned long long* k = ss->hc.p + t * C_COUNT;
    if (k[C_FAIL])
      throw Error(NULPA_EINTERNAL, "hashtable insertion failed (capacity invariant violated)");
    r.changed += k[C_DN];
    r.processed_vertices += k[C_PROC_V];
    r.processed_edges += k[C_PROC_E];
    r.wake_edges += k[C_WAKE_E];
  }
  r.device_ms = ms;
  r.kernel_launches = launches;
  if (info) *info = r;
}

}  // namespace nulpa

// ---- C ABI ---------------------------------------------------------------------------

using namespace nulpa;

namespace {

struct HostGraph {
  nulpa_graph* g = nullptr;
  HostGraph(const nulpa_csr* csr, int device) {
    const int rc = nulpa_graph_upload(csr, device, &g);
    if (rc != NULPA_OK) throw Error(rc, nulpa_last_error());
  }
  // lpa(): the run's plan is built while the targets cross PCIe.
  HostGraph(const nulpa_csr* csr, const nulpa_opts& o, const nulpa_tuning* tuning) {
    const TierBounds tb = resolve_tiers(o.switch_degree, tuning);
    g = upload_graph(csr, o.device, &tb, o.precision == 64 ? 8 : 4);
  }
  ~HostGraph() {
    if (g) nulpa_graph_free(g);
  }
};

template <typename T>
struct DevArray {
  T* p = nullptr;
  size_t n = 0;
  DevArray(size_t count) : p(dalloc<T>(count)), n(count) {}
  ~DevArray() { dfree(p); }
  void upload(const T* h) {
    if (n) NULPA_CUDA(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice));
  }
  void download(T* h) const {
    if (n) NULPA_CUDA(cudaMemcpy(h, p, n * sizeof(T), cudaMemcpyDeviceToHost));
  }
};

}  // namespace

extern "C" {

void nulpa_default_opts(nulpa_opts* o) {
  o->tolerance = 0.05;
  o->max_iterations = 20;
  o->pl_period = 4;
  o->cc_period = 0;
  o->strategy = NULPA_PROBE_QUADRATIC_DOUBLE;
  o->switch_degree = 32;
  o->precision = 32;
  o->exec = NULPA_EXEC_PARALLEL_ASYNC;
  o->workers = 0;
  o->seed = 0;
  o->prune = 1;
  o->device = 0;
}

int nulpa_run_graph(nulpa_graph* g, const nulpa_opts* opts, const nulpa_tuning* tuning,
                    uint32_t* labels_host, uint32_t* labels_device, nulpa_stats* stats) {
  return guarded([&] {
    if (!g || !opts) throw Error(NULPA_EINVAL, "null argument");
    run_lpa(g, *opts, tuning, labels_host, labels_device, stats);
  });
}

int nulpa_run(const nulpa_csr* csr, const nulpa_opts* opts, const nulpa_tuning* tuning,
              uint32_t* labels_out, nulpa_stats* stats) {
  return guarded([&] {
    if (!opts) throw Error(NULPA_EINVAL, "null options");
    check_host_csr(csr);
    nulpa_graph probe;  // validate before any device work (lpa.cpp:363)
    probe.n = csr->n;
    validate_opts(&probe, *opts);
    Trace tr("nulpa_run");
    HostGraph hg(csr, *opts, tuning);
    tr.mark("upload");
    run_lpa(hg.g, *opts, tuning, labels_out, nullptr, stats);
    tr.mark("run_lpa");
  });
}

int nulpa_sync_step_graph(nulpa_graph* g, const uint32_t* in, int pick_less, int strategy,
                          int precision, uint32_t* out, uint64_t* changed) {
  return guarded([&] {
    if (!g) throw Error(NULPA_EINVAL, "null graph");
    const uint64_t dn = run_sync_step(g, in, pick_less, strategy, precision, out);
    if (changed) *changed = dn;
  });
}

int nulpa_sync_step(const nulpa_csr* csr, const uint32_t* labels_in, int pick_less, int strategy,
                    int precision, uint32_t* labels_out, uint64_t* changed) {
  return guarded([&] {
    check_host_csr(csr);
    HostGraph hg(csr, default_device());
    DevArray<uint32_t> in(csr->n), out(csr->n);
    in.upload(labels_in);
    const uint64_t dn = run_sync_step(hg.g, in.p, pick_less, strategy, precision, out.p);
    out.download(labels_out);
    if (changed) *changed = dn;
  });
}

int nulpa_cross_check(const nulpa_csr* csr, uint32_t* labels, const uint32_t* prev,
                      uint8_t* flags, uint64_t* reverted) {
  return guarded([&] {
    check_host_csr(csr);
    HostGraph hg(csr, default_device());
    const uint32_t n = csr->n;
    DevArray<uint32_t> l(n), pv(n);
    DevArray<uint8_t> f(n);
    l.upload(labels);
    pv.upload(prev);
    f.upload(flags);
    const uint64_t r = run_cross_check(hg.g, l.p, pv.p, f.p);
    l.download(labels);
    f.download(flags);
    if (reverted) *reverted = r;
  });
}

int nulpa_partition_by_degree(const nulpa_csr* csr, uint32_t switch_degree, uint32_t* low,
                              uint64_t* n_low, uint32_t* high, uint64_t* n_high) {
  return guarded([&] {
    // partition_by_degree, lpa.cpp:330-336 (same message), over the input's ids:
    // only the offsets are needed.
    if (switch_degree < 2) throw Error(NULPA_EINVAL, "switch-degree must be >= 2");
    check_host_csr(csr);
    use_device(default_device());
    const uint32_t n = csr->n;
    Stream stream;
    DevArray<uint64_t> off(uint64_t(n) + 1);
    off.upload(csr->offsets);
    DevArray<uint32_t> d_low(n + 1), d_high(n + 1);
    uint64_t nl = 0, nh = 0;
    partition_two_way(off.p, n, switch_degree, d_low.p, d_high.p, &nl, &nh, stream.s);
    if (nl) NULPA_CUDA(cudaMemcpy(low, d_low.p, nl * 4, cudaMemcpyDeviceToHost));
    if (nh) NULPA_CUDA(cudaMemcpy(high, d_high.p, nh * 4, cudaMemcpyDeviceToHost));
    *n_low = nl;
    *n_high = nh;
  });
}

}  // extern "C"

extern "C" {

int nulpa_graph_edge_ranges(nulpa_graph* g, uint32_t parts, uint32_t* bounds) {
  return guarded([&] {
    if (!g || parts == 0) throw Error(NULPA_EINVAL, "bad partition request");
    use_device(g->device);
    DBuf<uint32_t> d(parts + 1);
    k_edge_bounds<<<(parts + 256) / 256, 256>>>(g->offsets, g->n, parts, d.p);
    NULPA_CUDA(cudaGetLastError());
    NULPA_CUDA(cudaMemcpy(bounds, d.p, (parts + 1) * 4ull, cudaMemcpyDeviceToHost));
  });
}

int nulpa_session_create(nulpa_graph* g, const nulpa_opts* opts, const nulpa_tuning* tuning,
                         uint32_t v_begin, uint32_t v_end, uint32_t* labels_dev,
                         uint8_t* flags_dev, nulpa_session** out) {
  return guarded([&] {
    if (!g || !opts || !labels_dev || !flags_dev) throw Error(NULPA_EINVAL, "null argument");
    validate_opts(g, *opts);
    if (opts->exec == NULPA_EXEC_SEQUENTIAL)
      throw Error(NULPA_EINVAL, "sequential mode cannot be partitioned across devices");
    if (v_begin > v_end || v_end > g->n) throw Error(NULPA_EINVAL, "vertex range out of bounds");
    use_device(g->device);
    auto* ss = new nulpa_session();
    try {
      ss->g = g;
      ss->o = *opts;
      ss->lo = v_begin;
      ss->hi = v_end;
      ss->labels = labels_dev;
      ss->flags = flags_dev;
      ss->sms = sm_count();
      ss->vbytes = opts->precision == 64 ? 8 : 4;
      ss->identity_first =
          g->rows_simple && g->weights == nullptr && !(tuning && tuning->no_identity_first);
      ss->plan = build_plan(g, resolve_tiers(opts->switch_degree, tuning), ss->vbytes,
                            ss->stream.s, v_begin, v_end);
      ss->ctr = DBuf<unsigned long long>(dev::kTiers * dev::C_COUNT);
      ss->snapshot = DBuf<uint32_t>(uint64_t(v_end - v_begin) + 1);
      if (opts->exec == NULPA_EXEC_SYNCHRONOUS) {
        ss->staging = DBuf<uint32_t>(g->n);
        ss->changed = DBuf<uint32_t>(uint64_t(v_end - v_begin) + 1);
      }
    } catch (...) {
      delete ss;
      throw;
    }
    *out = ss;
  });
}

int nulpa_session_init(nulpa_session* ss) {
  return guarded([&] {
    if (!ss) throw Error(NULPA_EINVAL, "null session");
    use_device(ss->g->device);
    cudaStream_t st = ss->has_ext ? ss->ext : ss->stream.s;
    k_init<<<grid_for(ss->g->n, 256, ss->sms * 8), 256, 0, st>>>(
        ss->labels, ss->flags, ss->g->offsets, ss->g->n, ss->g->perm);
    NULPA_CUDA(cudaGetLastError());
    NULPA_CUDA(cudaStreamSynchronize(st));
    ss->fresh = true;
    ss->passes = 0;
  });
}

int nulpa_session_pass(nulpa_session* ss, int pick_less, int wake, nulpa_pass_info* info) {
  return guarded([&] {
    if (!ss) throw Error(NULPA_EINVAL, "null session");
    use_device(ss->g->device);
    session_pass(ss, pick_less, wake, info);
  });
}

int nulpa_session_set_stream(nulpa_session* ss, void* stream) {
  return guarded([&] {
    if (!ss) throw Error(NULPA_EINVAL, "null session");
    ss->ext = static_cast<cudaStream_t>(stream);
    ss->has_ext = true;
  });
}

int nulpa_session_pack_changes(nulpa_session* ss, uint32_t* out_dev, uint32_t cap, void* stream) {
  return guarded([&] {
    if (!ss || (cap && !out_dev)) throw Error(NULPA_EINVAL, "null argument");
    use_device(ss->g->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned* cnt = ss->work.p + 1;
    NULPA_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned), st));
    const uint32_t span = ss->hi - ss->lo;
    if (span)
      k_pack_changes<<<grid_for(span, 256, ss->sms * 8), 256, 0, st>>>(
          ss->labels, ss->snapshot.p, ss->lo, ss->hi, out_dev, cap, cnt);
    if (cap) k_pad_changes<<<grid_for(cap, 256, ss->sms * 4), 256, 0, st>>>(out_dev, cap, cnt);
    NULPA_CUDA(cudaGetLastError());
  });
}

int nulpa_session_apply_changes(nulpa_session* ss, const uint32_t* in_dev, uint64_t pairs,
                                void* stream) {
  return guarded([&] {
    if (!ss || (pairs && !in_dev)) throw Error(NULPA_EINVAL, "null argument");
    use_device(ss->g->device);
    if (pairs)
      k_apply_changes<<<grid_for(pairs, 256, ss->sms * 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
          ss->labels, in_dev, pairs);
    NULPA_CUDA(cudaGetLastError());
  });
}

int nulpa_session_free(nulpa_session* ss) {
  return guarded([&] {
    if (ss) {
      cudaSetDevice(ss->g->device);
      delete ss;
    }
  });
}

}  // extern "C"
