// Device primitives shared by the nulpa kernels (sm_100a).
//
// The per-vertex open-addressing hashtable (reference: hashtable.hpp:16-185)
// is re-designed for the GPU: power-of-two capacity so the slot index is a
// mask instead of a 64-bit `%`, Fibonacci start slot, and the reference's
// hybrid quadratic-double advance (idx += step; step = 2*step + h2(key)) for
// the first `cap` probes followed by a +1 completeness sweep — the same
// "strategy budget, then sweep" structure as hashtable.hpp:126-147. Keys are
// claimed with atomicCAS and values accumulated with atomicAdd (the
// reference's `shared` branch, hashtable.hpp:110-118) because every table is
// filled by a whole warp or CTA. Placement is never observable in results:
// the argmax (hashtable.hpp:163-185) is order-independent.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace nulpa {
namespace dev {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr unsigned kFull = 0xFFFFFFFFu;

enum Mode : int { kAsync = 0, kSync = 1 };

// Device counters (u64), zeroed per pass.
enum Counter : int {
  C_DN = 0,        // label changes
  C_PROC_V = 1,    // processed (examined) vertices
  C_PROC_E = 2,    // edges scanned by processed vertices
  C_WAKE_E = 3,    // neighbour wake stores
  C_FAIL = 4,      // hashtable insert failures (must stay 0)
  C_NCHANGED = 5,  // length of the changed-vertex list (sync mode; "other" slot)
  C_AUX = 6,       // cross-check scratch ("other" slot)
  C_COUNT = 8
};
// One C_COUNT block of counters per tier: 0 thread, 1 warp, 2 block, 3 hub, 4 other.
constexpr int kTiers = 5;

struct Graph {
  const uint64_t* __restrict__ off;
  const uint32_t* __restrict__ tgt;
  const float* __restrict__ w;  // nullptr = unit weights
  uint32_t n;
};

struct PassCtx {
  Graph g;
  const uint32_t* lab_in;   // neighbour labels are read here (async: == lab_out)
  uint32_t* lab_out;        // decisions are written here
  uint8_t* flags;           // pruning flags; nullptr = examine everything, no flags
  unsigned long long* ctr;  // Counter array
  uint32_t* changed;        // sync mode: changed-vertex list for the deferred wake
  unsigned long long* changed_n;  // its length
  int pick_less;
  int strategy;
};

// Tier geometry.
constexpr int kWarpCap = 1024;    // per-warp table slots (deg <= 512 at load <= 1/2)
constexpr int kWarpTier = 512;
constexpr int kBlockCap = 8192;   // per-CTA table slots (deg <= 4096 at load <= 1/2)
constexpr int kBlockTier = 4096;
constexpr int kHubChunk = 4096;   // edges per hub work item (<= kBlockCap / 2)
constexpr int kBlockThreads = 256;


// Hub-tier tables and work items (k_hub_* in lpa_kernels.cuh).
struct HubCtx {
  const uint32_t* hub_v;      // [H] vertex ids
  const uint64_t* tab_off;    // [H] slot offset into keys/vals
  const uint32_t* tab_cap;    // [H] power-of-two capacity
  const uint64_t* occ_off;    // [H] offset into occ
  uint32_t* occ_n;            // [H] occupied-slot counts
  uint32_t* occ;              // occupied-slot lists
  uint32_t* keys;             // global table keys (kEmpty when idle)
  void* vals;                 // global table values (W)
  unsigned long long* best;   // [H] packed argmax (float) / value bits (double)
  uint32_t* best_k;           // [H] min key among maxima (double path)
  uint8_t* active;            // [H]
  uint8_t* changed;           // [H]
  const uint32_t* item_hub;   // [I] hub index of each work item
  const uint32_t* item_start; // [I] first edge of the item within the hub row
  uint32_t n_hubs;
  uint32_t n_items;
};

// ---- memory access helpers -------------------------------------------------

// Async mode reads neighbour labels that other SMs may be writing in place:
// load through L2 (ld.global.cg) so a stale L1 line is never reused within a
// pass. Sync mode reads an immutable snapshot through the read-only path.
template <int MODE>
__device__ __forceinline__ uint32_t load_label(const uint32_t* p) {
  if constexpr (MODE == kAsync)
    return __ldcg(p);
  else
    return __ldg(p);
}

__device__ __forceinline__ uint8_t load_flag(const uint8_t* p) { return __ldcg(p); }

template <typename W, bool WEIGHTED>
__device__ __forceinline__ W edge_weight(const Graph& g, uint64_t e) {
  if constexpr (WEIGHTED)
    return static_cast<W>(__ldg(g.w + e));
  else
    return W(1);
}

// ---- (value, key) argmax with ties to the smaller key -----------------------
// ht_better, hashtable.hpp:163-169. kEmpty marks "no candidate".
template <typename W>
struct Best {
  W v;
  uint32_t k;
};

template <typename W>
__device__ __forceinline__ void best_merge(Best<W>& a, W v, uint32_t k) {
  if (k == kEmpty) return;
  if (a.k == kEmpty || v > a.v || (v == a.v && k < a.k)) {
    a.v = v;
    a.k = k;
  }
}

template <typename W, int WIDTH = 32>
__device__ __forceinline__ Best<W> warp_best(Best<W> b) {
#pragma unroll
  for (int o = WIDTH / 2; o > 0; o >>= 1) {
    const W ov = __shfl_xor_sync(kFull, b.v, o, WIDTH);
    const uint32_t ok = __shfl_xor_sync(kFull, b.k, o, WIDTH);
    best_merge(b, ov, ok);
  }
  return b;
}

// Sum of `w` over the lanes in `peers` in ascending lane order (= ascending
// neighbour order, the reference's accumulation order). All 32 lanes call it.
template <typename W>
__device__ __forceinline__ W peer_sum(W w, unsigned peers) {
  W s = W(0);
#pragma unroll 4
  for (int b = 0; b < 32; ++b) {
    const W wb = __shfl_sync(kFull, w, b);
    if ((peers >> b) & 1u) s += wb;
  }
  return s;
}

// ---- open-addressing table ----------------------------------------------------

__device__ __forceinline__ uint32_t hash_start(uint32_t key) { return key * 0x9E3779B1u; }
__device__ __forceinline__ uint32_t hash_step(uint32_t key) {
  uint32_t h = key ^ (key >> 15);
  h *= 0x85EBCA6Bu;
  return (h ^ (h >> 13)) | 1u;
}

// Advance the probe index (hashtable.hpp:134-147 advance rules) — strategy
// numbering matches labelprop::ProbeStrategy.
__device__ __forceinline__ void probe_advance(int strategy, uint32_t& idx, uint32_t& step,
                                              uint32_t h2) {
  switch (strategy) {
    case 0: idx += 1; break;                       // Linear
    case 1: idx += step; step *= 2; break;         // Quadratic
    case 2: idx += h2; break;                      // DoubleHash (fixed odd step)
    default: idx += step; step = 2 * step + h2;    // QuadraticDouble
  }
}

// Accumulate (key, v) into a table of `cap` (power of two) slots that several
// threads fill concurrently. `occ`/`occ_n` (optional) record each newly
// claimed slot so the table can be swept and cleared sparsely.
// Returns false only if every slot is taken by other keys.
template <typename W>
__device__ __forceinline__ bool ht_add(uint32_t* keys, W* vals, uint32_t cap, int strategy,
                                       uint32_t key, W v, uint32_t* occ = nullptr,
                                       uint32_t* occ_n = nullptr) {
  const uint32_t mask = cap - 1;
  const uint32_t h2 = hash_step(key);
  uint32_t idx = hash_start(key) >> (__clz(cap) + 1);  // top log2(cap) bits
  if (cap == 1) idx = 0;
  uint32_t step = 1;
  for (uint32_t t = 0; t < 2 * cap; ++t) {
    const uint32_t s = idx & mask;
    uint32_t cur = *((volatile uint32_t*)(keys + s));
    if (cur == kEmpty) {
      cur = atomicCAS(keys + s, kEmpty, key);
      if (cur == kEmpty) {
        atomicAdd(vals + s, v);
        if (occ) occ[atomicAdd(occ_n, 1u)] = s;
        return true;
      }
    }
    if (cur == key) {
      atomicAdd(vals + s, v);
      return true;
    }
    if (t + 1 >= cap)
      idx += 1;  // completeness sweep
    else
      probe_advance(strategy, idx, step, h2);
  }
  return false;
}

// Smallest power of two >= x (x >= 1).
__host__ __device__ __forceinline__ uint32_t pow2_ceil(uint32_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// ---- counter aggregation ---------------------------------------------------------

__device__ __forceinline__ void warp_add_counter(unsigned long long* ctr, int which,
                                                 unsigned long long v) {
  // Every lane of the warp must call this.
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(ctr + which, v);
}

}  // namespace dev
}  // namespace nulpa
