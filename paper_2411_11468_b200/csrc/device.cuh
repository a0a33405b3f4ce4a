// Device primitives shared by the nulpa kernels (sm_100a).
//
// The per-vertex open-addressing hashtable (reference: hashtable.hpp:16-185)
// is re-designed for the GPU:
//  * power-of-two capacity, so the slot index is a mask instead of the
//    reference's 64-bit `idx % p1`;
//  * Fibonacci start slot and the reference's hybrid quadratic-double advance
//    (idx += step; step = 2*step + h2(key)) for the first `cap` probes, then a
//    +1 completeness sweep — the "strategy budget, then sweep" structure of
//    hashtable.hpp:126-147 (all four ProbeStrategy advances are selectable);
//  * unit-weight graphs (the common case) use ONE 64-bit word per slot,
//    (key << 32) | count, read with one load by the argmax sweep; a key is
//    claimed by a 32-bit CAS on the key half and counted by a 32-bit atomicAdd
//    on the count half (both native shared-memory atomics). Weighted graphs use
//    split key / value arrays with CAS + atomicAdd (the reference's `shared`
//    branch, hashtable.hpp:110-118).
// Placement is never observable in results: the argmax (higher value, ties to
// the smaller key; hashtable.hpp:163-185) is order-independent. Warp argmax
// uses two redux.sync instructions on order-preserving value bits.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

namespace nulpa {
namespace dev {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr unsigned long long kEmptyWord = 0xFFFFFFFF00000000ull;  // packed slot: key EMPTY, count 0

enum Mode : int { kAsync = 0, kSync = 1 };

// Device counters (u64), zeroed per pass. One C_COUNT block per tier.
enum Counter : int {
  C_DN = 0,        // label changes
  C_PROC_V = 1,    // processed (examined) vertices
  C_PROC_E = 2,    // edges scanned by processed vertices
  C_WAKE_E = 3,    // neighbour wake stores
  C_FAIL = 4,      // hashtable insert failures (must stay 0)
  C_NCHANGED = 5,  // length of the changed-vertex list (sync mode; "other" block)
  C_AUX = 6,       // cross-check scratch ("other" block)
  C_COUNT = 8
};

// Degree tiers.
enum Tier : int {
  T_THREAD = 0,   // deg <= thread_max (<= 16): one thread per vertex
  T_HALF = 1,     // deg <= 16: half a warp per vertex, register dedup
  T_WARP = 2,     // deg <= 32: one warp per vertex, register dedup
  T_WTAB = 3,     // deg <= 256: a 32-thread team per vertex, shared-memory table
  T_BLOCK = 4,    // deg <= 1024: a 128-thread team per vertex
  T_BLOCK2 = 5,   // deg <= 4096: a 256-thread team per vertex
  T_BIG = 6,      // deg <= 12288: one 1024-thread CTA per vertex, 128 KB shared table
  T_CLUSTER = 7,  // deg <= 98304: one 8-CTA cluster per vertex, table distributed over DSMEM
  T_HUB = 8,      // larger: (hub, chunk) items, shared pre-aggregation + global table
  T_OTHER = 9,    // deferred wake, cross-check, sequential
  kTiers = 10
};

constexpr int kBlockThreads = 256;
constexpr int kWarpTabMax = 256;    // T_WTAB degree bound
constexpr int kWarpTabCap = 512;    // per-team slots (load <= 1/2)
constexpr int kBlockMax = 1024;     // T_BLOCK degree bound
constexpr int kBlockCap = 2048;     // per-team slots (load <= 1/2)
constexpr int kBlock2Max = 4096;    // T_BLOCK2 degree bound
constexpr int kBlock2Cap = 8192;    // per-team slots (load <= 1/2)
constexpr int kHubCap = 4096;       // hub pre-aggregation slots per CTA
constexpr int kBigThreads = 1024;   // wide-row CTAs (k_wide, k_cluster)
#ifndef NULPA_MID_THREADS
#define NULPA_MID_THREADS 512
#define NULPA_MID_CAP 8192
#define NULPA_MID_MAX 6144
#endif
// T_BIG: one CTA per vertex, two CTAs per SM (measured 37.3 -> 18.7 ms per R27 run
// for degree 1025-6144 against one 1024-thread CTA per SM; the 6145-12288 rows then
// run on the wide tier).
constexpr int kMidThreads = NULPA_MID_THREADS;
constexpr int kBigCap = NULPA_MID_CAP;  // its table (64 KB packed)
constexpr int kBigMax = NULPA_MID_MAX;  // load <= 3/4
constexpr int kClusterSize = 8;     // portable cluster size
constexpr int kClusterCap = 16384;  // slots per CTA of the cluster
constexpr int kClusterMax = kClusterSize * kClusterCap * 3 / 4;  // 98304, load <= 3/4
// Wide tier (k_wide): CTA size and shared-table slots. 512 threads with an 8K-slot table
// (two independent CTAs per SM, up to 6144 labels per phase, up to 16 bucketed phases);
// measured at R-MAT 27 on one B200: wide tier 29.9 -> 27.0 ms per run against one
// 1024-thread CTA per SM with 16K slots (-DNULPA_WIDE_THREADS=1024 -DNULPA_WIDE_CAP=16384
// -DNULPA_WIDE_BUCKETS=8): while one CTA sits in a barrier or its argmax sweep, the
// other's label gathers keep the SM's loads in flight.
#ifndef NULPA_WIDE_BUCKETS
#define NULPA_WIDE_BUCKETS 16
#endif
#ifndef NULPA_WIDE_THREADS
#define NULPA_WIDE_THREADS 512
#endif
#ifndef NULPA_WIDE_CAP
#define NULPA_WIDE_CAP 8192
#endif
constexpr int kWideThreads = NULPA_WIDE_THREADS;
constexpr int kWideCap = NULPA_WIDE_CAP;
constexpr int kWideCtasPerSm = 1024 / NULPA_WIDE_THREADS;  // resident CTAs per SM (regs <= 64)
// u32 per wide-tier CTA: the row snapshot, or the buckets of phases 1..NULPA_WIDE_BUCKETS-1
constexpr uint32_t kWideScratch = (NULPA_WIDE_BUCKETS - 1) * uint32_t(kClusterMax);
constexpr int kHubChunk = 2048;     // edges per hub work item (<= kBlockCap / 2)
constexpr int kHubSweep = 8192;     // table slots per hub sweep item

struct Graph {
  const uint64_t* __restrict__ off;
  const uint32_t* __restrict__ tgt;
  const float* __restrict__ w;  // nullptr = unit weights
  uint32_t n;
};

struct PassCtx {
  Graph g;
  const uint32_t* lab_in;         // neighbour labels are read here (async: == lab_out)
  uint32_t* lab_out;              // decisions are written here
  uint8_t* flags;                 // pruning flags; nullptr = examine everything
  unsigned long long* ctr;        // this tier's Counter block
  uint32_t* changed;              // sync mode: changed-vertex list for the deferred wake
  unsigned long long* changed_n;  // its length
  int pick_less;
  int strategy;
  int wake;                       // store neighbour wake-ups (0 when provably dead, see engine.cu)
  unsigned int* work;             // dynamic work counter (cluster tier)
  const uint32_t* vid = nullptr;  // position -> vertex id (layout.cu); nullptr = identity
  const uint32_t* pos = nullptr;  // vertex id -> position; nullptr = identity
  int fresh = 0;                  // labels are still the identity (first pass of a run)
  int hints = 0;                  // the wide tier's per-row hints come from this run's
                                  // previous pass (k_wide; 0: ignore them)
  // Pass guard (batched runs, engine.cu): set on the device once the run has converged;
  // every pass kernel enqueued after that returns at once. nullptr = unguarded.
  const unsigned* stop = nullptr;
  // Positions [0, ro_end) hold labels no thread writes during this launch (async mode): in
  // position order they are the vertices of the higher-degree tiers, which run in later
  // launches. Their gathers take the L1-cached read-only path (graph.cu: tier_ro_bounds).
  uint32_t ro_end = 0;
  // ... and so do positions [ro_lo, n): the lower-degree tiers, which ran in earlier launches.
  uint32_t ro_lo = 0xFFFFFFFFu;
};

// Vertex id stored at position p (label values are vertex ids).
__device__ __forceinline__ uint32_t vertex_id(const uint32_t* vid, uint32_t p) {
  return vid ? __ldg(vid + p) : p;
}
__device__ __forceinline__ uint32_t position_of(const uint32_t* pos, uint32_t v) {
  return pos ? __ldg(pos + v) : v;
}

// Hub-tier tables and work items (k_hub_* in lpa_kernels.cuh).
struct HubCtx {
  const uint32_t* hub_v;      // [H] vertex ids
  const uint64_t* tab_off;    // [H] slot offset into the global table
  const uint32_t* tab_cap;    // [H] power-of-two capacity
  void* tab;                  // packed words (unit weights) or keys (split)
  void* tab_vals;             // split tables: values
  unsigned long long* best;   // [H] packed argmax (value bits << 32 | ~key), or double bits
  uint32_t* best_k;           // [H] min key among maxima (double path)
  uint8_t* active;            // [H]
  uint8_t* changed;           // [H]
  const uint32_t* item_hub;   // [I] hub index of each work item
  const uint32_t* item_start; // [I] first edge of the item within the hub row
  const uint32_t* sitem_hub;  // [S] hub index of each table-sweep item
  const uint32_t* sitem_start;// [S] first slot of the sweep item
  uint32_t n_hubs;
  uint32_t n_items;
  uint32_t n_sitems;
  const unsigned* stop = nullptr;  // pass guard (PassCtx::stop)
};

// True once a batched run has converged: the kernel has nothing to do (uniform).
__device__ __forceinline__ bool stopped(const unsigned* stop) {
  return stop != nullptr && __ldcg(stop) != 0u;
}

// ---- memory access helpers -------------------------------------------------

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Adjacency is streamed once per pass: bypass L1 and evict first from L2 so it
// does not push the re-read label array out of the 126 MB L2.
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

// ---- the asynchronous label / flag protocol (lpa.cpp:44-60) --------------------------
// The reference makes every label and flag access seq_cst so that "a stale read is
// always re-examined": a vertex j that claims itself (flags[j] = 1) and then reads a
// neighbour's label, and a neighbour i that stores a new label and then reads flags[j]
// to wake j, must not BOTH read the old value (store buffering). On the GPU the labels
// and flags that other SMs read and write during a pass are accessed with relaxed
// device-scope operations (morally strong in the PTX memory model; they bypass L1, so
// no stale line is reused), and a fence.sc.gpu separates each claim store from the
// label loads that depend on it and each label store from its wake loads. Either the
// claimer's loads see the new label, or the changer's flag load sees the claim and
// wakes j. One fence per claimed batch and per changed vertex. (The asm statements are
// volatile, so the compiler keeps them in program order around the fence.)
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v));
}
__device__ __forceinline__ uint8_t ld_relaxed(const uint8_t* p) {
  uint16_t v;
  asm volatile("ld.relaxed.gpu.global.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return static_cast<uint8_t>(v);
}
__device__ __forceinline__ void st_relaxed(uint8_t* p, uint8_t v) {
  asm volatile("st.relaxed.gpu.global.u8 [%0], %1;" ::"l"(p), "h"(static_cast<uint16_t>(v)));
}
#ifndef NULPA_NO_FENCE
__device__ __forceinline__ void fence_sc() { asm volatile("fence.sc.gpu;" ::: "memory"); }
#else  // (cost measurement only: drops the a18 ordering)
__device__ __forceinline__ void fence_sc() {}
#endif

// Async mode reads neighbour labels that other SMs may be writing in place (relaxed,
// device scope). Sync mode reads an immutable snapshot through the read-only path.
template <int MODE>
__device__ __forceinline__ uint32_t load_label(const uint32_t* p) {
  if constexpr (MODE == kAsync)
    return ld_relaxed(p);
  else
    return __ldg(p);
}

__device__ __forceinline__ uint8_t load_flag(const uint8_t* p) { return ld_relaxed(p); }

// Neighbour label at position j: labels that cannot change during this launch (j < ro_end:
// a later tier's vertices) come through the read-only, L1-cached path — the hottest
// labels of a power-law graph, shared by every warp on the SM — the rest by the relaxed
// device-scope load of the async protocol.
template <int MODE, typename Ctx>
__device__ __forceinline__ uint32_t gather_label(const Ctx& c, uint32_t j) {
  if constexpr (MODE == kAsync)
    return (j < c.ro_end || j >= c.ro_lo) ? __ldg(c.lab_in + j) : ld_relaxed(c.lab_in + j);
  else
    return __ldg(c.lab_in + j);
}

template <typename W, bool WEIGHTED>
__device__ __forceinline__ W edge_weight(const Graph& g, uint64_t e) {
  if constexpr (WEIGHTED)
    return static_cast<W>(__ldg(g.w + e));
  else
    return W(1);
}

// ---- TMA bulk copies (cp.async.bulk, 1-D) with an mbarrier --------------------------
// Row slices of the adjacency are staged into shared memory by the copy engine: one
// thread arms the stage's mbarrier with the byte count and issues the bulk copy; every
// consumer waits on the barrier's phase parity. The copy needs 16-byte alignment of
// both addresses and of the size, so a slice is widened to whole 4-entry groups.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
// Make barrier initialisation visible to the async (copy-engine) proxy.
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Arm `bar` for `bytes` and start the bulk copy global -> shared (evict-first in L2: the
// targets stream once per pass).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
// Complete the barrier's phase without a copy (an empty stage).
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// ---- (value, key) argmax, ties to the smaller key (ht_better, hashtable.hpp:163-169) ----
// Candidate values travel as order-preserving u32 bits (integer counts, or the
// bits of non-negative fp32 sums); fp64 sums travel as doubles.
template <typename W>
using VBits = std::conditional_t<sizeof(W) == 8, double, uint32_t>;

template <typename W>
__device__ __forceinline__ VBits<W> to_vbits(W v) {
  if constexpr (sizeof(W) == 8)
    return v;
  else
    return __float_as_uint(static_cast<float>(v));
}

template <typename V>
struct Best {
  V v;
  uint32_t k;  // kEmpty = no candidate
};

template <typename V>
__device__ __forceinline__ void best_merge(Best<V>& a, V v, uint32_t k) {
  if (k == kEmpty) return;
  if (a.k == kEmpty || v > a.v || (v == a.v && k < a.k)) {
    a.v = v;
    a.k = k;
  }
}

// Argmax over the lanes in `mask` (every lane in `mask` calls it with the same mask).
__device__ __forceinline__ Best<uint32_t> warp_best(Best<uint32_t> b, unsigned mask = kFull) {
  // values are < 2^31 for counts and non-negative floats; +1 makes "none" the minimum
  const uint32_t v = b.k == kEmpty ? 0u : b.v + 1u;
  const uint32_t mv = __reduce_max_sync(mask, v);
  const uint32_t mk = __reduce_min_sync(mask, (v == mv && b.k != kEmpty) ? b.k : kEmpty);
  return Best<uint32_t>{mv ? mv - 1u : 0u, mk};
}

__device__ __forceinline__ Best<double> warp_best(Best<double> b, unsigned = kFull) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(kFull, b.v, o);
    const uint32_t ok = __shfl_xor_sync(kFull, b.k, o);
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

// ---- probing ------------------------------------------------------------------

__device__ __forceinline__ uint32_t hash_start(uint32_t key, uint32_t cap) {
  return cap == 1 ? 0u : (key * 0x9E3779B1u) >> (__clz(cap) + 1);  // top log2(cap) bits
}
__device__ __forceinline__ uint32_t hash_step(uint32_t key) {
  uint32_t h = key ^ (key >> 15);
  h *= 0x85EBCA6Bu;
  return (h ^ (h >> 13)) | 1u;
}

// Advance rules of hashtable.hpp:134-147 (strategy numbering = labelprop::ProbeStrategy).
__device__ __forceinline__ void probe_advance(int strategy, uint32_t& idx, uint32_t& step,
                                              uint32_t h2) {
  switch (strategy) {
    case 0: idx += 1; break;                       // Linear
    case 1: idx += step; step *= 2; break;         // Quadratic
    case 2: idx += h2; break;                      // DoubleHash (fixed odd step)
    default: idx += step; step = 2 * step + h2;    // QuadraticDouble
  }
}

// Unit-weight tables count in u32, exactly. The reference's fp32 values (ValuePrecision
// Bits32) add 1.0f per occurrence, and an fp32 sum of ones stops growing at 2^24
// (16777216 + 1 rounds back to 16777216, ties to even), so a label repeated more than
// 2^24 times in one row compares as 2^24 there. The argmax sees the count the reference
// would: min(count, 2^24). (Integer counts compare like the bits of their float values.)
__device__ __forceinline__ uint32_t fp32_count(uint32_t count) { return min(count, 16777216u); }

// Insert results: 0 = failed (table full), 1 = counted into an existing key,
// 2 = claimed a new slot. The slot index is returned through *slot.
template <bool PACKED, typename W>
struct Table;

// Unit weights in GLOBAL memory (hub tables): one 64-bit word per slot,
// (key << 32) | count. A new key is claimed together with its count by one
// 64-bit CAS, an existing key is counted by one 64-bit atomicAdd (both native on
// global memory; the count never carries into the key half).
template <typename W>
struct Table<true, W> {
  unsigned long long* w;
  static constexpr size_t kSlotBytes = 8;
  __device__ __forceinline__ void bind(void* base, uint32_t) {
    w = static_cast<unsigned long long*>(base);
  }
  __device__ __forceinline__ void bind_split(void* base, void*) {
    w = static_cast<unsigned long long*>(base);
  }
  __device__ __forceinline__ void clear_slot(uint32_t s) { w[s] = kEmptyWord; }
  __device__ __forceinline__ int add(uint32_t cap, int strategy, uint32_t key, W v,
                                     uint32_t* slot) {
    const uint32_t cnt = static_cast<uint32_t>(v);
    const unsigned long long mine = (static_cast<unsigned long long>(key) << 32) | cnt;
    const uint32_t mask = cap - 1;
    uint32_t idx = hash_start(key, cap), step = 1, h2 = 0;
    for (uint32_t t = 0; t < 2 * cap; ++t) {
      const uint32_t s = idx & mask;
      unsigned long long cur = *((volatile unsigned long long*)(w + s));
      if (cur == kEmptyWord) {
        cur = atomicCAS(w + s, kEmptyWord, mine);
        if (cur == kEmptyWord) {
          *slot = s;
          return 2;
        }
      }
      if (static_cast<uint32_t>(cur >> 32) == key) {
        atomicAdd(w + s, static_cast<unsigned long long>(cnt));
        *slot = s;
        return 1;
      }
      if (t == 0) h2 = hash_step(key);  // second hash only after a collision
      if (t + 1 >= cap)
        idx += 1;  // completeness sweep
      else
        probe_advance(strategy, idx, step, h2);
    }
    return 0;
  }
  __device__ __forceinline__ void read(uint32_t s, uint32_t& key, VBits<W>& v) const {
    const unsigned long long x = w[s];
    key = static_cast<uint32_t>(x >> 32);
    if constexpr (sizeof(W) == 8)
      v = static_cast<double>(static_cast<uint32_t>(x));
    else
      v = fp32_count(static_cast<uint32_t>(x));
  }
  __device__ __forceinline__ W value(uint32_t s) const {
    return static_cast<W>(static_cast<uint32_t>(w[s]));
  }
};

// Weighted: split key / value arrays, CAS on the key then atomicAdd on the value.
template <typename W>
struct Table<false, W> {
  uint32_t* k;
  W* v;
  static constexpr size_t kSlotBytes = 4 + sizeof(W);
  // base holds `cap_slots` keys followed by `cap_slots` values
  __device__ __forceinline__ void bind(void* base, uint32_t cap_slots) {
    k = static_cast<uint32_t*>(base);
    v = reinterpret_cast<W*>(static_cast<unsigned char*>(base) + cap_slots * sizeof(uint32_t));
  }
  __device__ __forceinline__ void bind_split(void* keys, void* vals) {
    k = static_cast<uint32_t*>(keys);
    v = static_cast<W*>(vals);
  }
  __device__ __forceinline__ void clear_slot(uint32_t s) {
    k[s] = kEmpty;
    v[s] = W(0);
  }
  __device__ __forceinline__ int add(uint32_t cap, int strategy, uint32_t key, W val,
                                     uint32_t* slot) {
    const uint32_t mask = cap - 1, h2 = hash_step(key);
    uint32_t idx = hash_start(key, cap), step = 1;
    for (uint32_t t = 0; t < 2 * cap; ++t) {
      const uint32_t s = idx & mask;
      uint32_t cur = *((volatile uint32_t*)(k + s));
      if (cur == kEmpty) {
        cur = atomicCAS(k + s, kEmpty, key);
        if (cur == kEmpty) {
          atomicAdd(v + s, val);
          *slot = s;
          return 2;
        }
      }
      if (cur == key) {
        atomicAdd(v + s, val);
        *slot = s;
        return 1;
      }
      if (t + 1 >= cap)
        idx += 1;
      else
        probe_advance(strategy, idx, step, h2);
    }
    return 0;
  }
  __device__ __forceinline__ void read(uint32_t s, uint32_t& key, VBits<W>& val) const {
    key = k[s];
    val = to_vbits<W>(v[s]);
  }
  __device__ __forceinline__ W value(uint32_t s) const { return v[s]; }
};

// Unit-weight table in the CTA's OWN shared memory (team and hub-chunk
// tables): same slot format and probe sequence as Table<true, W>, but with
// 32-bit shared-window addresses (no generic-pointer conversion in the loop),
// the first probe inlined and the collision walk kept out of the common path.
template <typename W>
struct SmemTable {
  uint32_t base;  // shared-window address of slot 0
  static constexpr size_t kSlotBytes = 8;
  __device__ __forceinline__ void bind(void* p, uint32_t) {
    base = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  }
  __device__ __forceinline__ uint32_t ld_key(uint32_t s) const {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + s * 8u + 4u) : "memory");
    return v;
  }
  __device__ __forceinline__ uint32_t cas_key(uint32_t s, uint32_t key) const {
    uint32_t old;
    asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;"
                 : "=r"(old)
                 : "r"(base + s * 8u + 4u), "r"(kEmpty), "r"(key)
                 : "memory");
    return old;
  }
  __device__ __forceinline__ void add_count(uint32_t s, uint32_t cnt) const {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(base + s * 8u), "r"(cnt) : "memory");
  }
  __device__ __forceinline__ void clear_slot(uint32_t s) {
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(base + s * 8u), "l"(kEmptyWord) : "memory");
  }
  __device__ __forceinline__ void read(uint32_t s, uint32_t& key, VBits<W>& v) const {
    unsigned long long x;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(x) : "r"(base + s * 8u) : "memory");
    key = static_cast<uint32_t>(x >> 32);
    if constexpr (sizeof(W) == 8)
      v = static_cast<double>(static_cast<uint32_t>(x));
    else
      v = fp32_count(static_cast<uint32_t>(x));
  }
  __device__ __forceinline__ W value(uint32_t s) const {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + s * 8u) : "memory");
    return static_cast<W>(v);
  }
  // Claim-or-find `key` and add `val`: 2 = claimed a new slot, 1 = existing key,
  // 0 = table full.
  __device__ __forceinline__ int add(uint32_t cap, int strategy, uint32_t key, W val,
                                     uint32_t* slot) {
    const uint32_t cnt = static_cast<uint32_t>(val);
    const uint32_t mask = cap - 1;
    uint32_t idx = hash_start(key, cap);
    uint32_t s = idx & mask;
    uint32_t cur = ld_key(s);
    int r = 1;
    if (cur == kEmpty) {
      cur = cas_key(s, key);
      if (cur == kEmpty) {
        cur = key;
        r = 2;
      }
    }
    if (__builtin_expect(cur == key, 1)) {
      add_count(s, cnt);
      *slot = s;
      return r;
    }
    return strategy == 3 ? add_collided<3>(cap, key, cnt, idx, slot)
                         : add_collided<-1>(cap, key, cnt, idx, slot, strategy);
  }
  // Probe walk after a first-probe collision; STRAT = 3 (QuadraticDouble, the
  // default) is specialised, -1 dispatches on `strategy` at run time.
  template <int STRAT>
  __device__ __forceinline__ int add_collided(uint32_t cap, uint32_t key, uint32_t cnt,
                                              uint32_t idx, uint32_t* slot, int strategy = 3) {
    if constexpr (STRAT >= 0) strategy = STRAT;
    const uint32_t mask = cap - 1, h2 = hash_step(key);
    uint32_t step = 1;
    probe_advance(strategy, idx, step, h2);
    for (uint32_t t = 1; t < 2 * cap; ++t) {
      const uint32_t s = idx & mask;
      uint32_t cur = ld_key(s);
      int r = 1;
      if (cur == kEmpty) {
        cur = cas_key(s, key);
        if (cur == kEmpty) {
          cur = key;
          r = 2;
        }
      }
      if (cur == key) {
        add_count(s, cnt);
        *slot = s;
        return r;
      }
      if (t + 1 >= cap)
        idx += 1;  // completeness sweep
      else
        probe_advance(strategy, idx, step, h2);
    }
    return 0;
  }
};

// Smallest power of two >= x (x >= 1).
__host__ __device__ __forceinline__ uint32_t pow2_ceil(uint32_t x) {
#ifdef __CUDA_ARCH__
  return x <= 1 ? 1u : 1u << (32 - __clz(x - 1));
#else
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
#endif
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
