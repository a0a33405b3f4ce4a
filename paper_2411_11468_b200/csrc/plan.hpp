// Per-graph execution plan: degree tiers and hub tables.
#pragma once

#include <cstdint>

#include "internal.hpp"
#include "device.cuh"

namespace nulpa {

struct Plan {
  uint32_t thread_max = 0, warp_max = 0, block_max = 0, schedule = 1;
  uint32_t* wide_scratch = nullptr;  // [SMs x wide_stride] row snapshots / phase buckets of the wide tier
  uint32_t wide_stride = 0;          // u32 per CTA: (NULPA_WIDE_BUCKETS - 1) x the tier's max degree
  uint32_t* wide_hint = nullptr;     // [count[T_CLUSTER]] distinct labels each row held in its last pass
  // Per tier: positions [0, ro_end[t]) belong to higher-degree buckets than any vertex of
  // tier t (position layout, whole-graph plans; 0 otherwise). T_HUB: n (the hub
  // accumulate kernels write no label).
  uint32_t ro_end[dev::kTiers] = {};
  uint32_t ro_lo[dev::kTiers] = {};  // positions [ro_lo[t], n) belong to lower-degree buckets
  uint32_t v_lo = 0, v_hi = 0;  // vertex range the tiers cover
  uint64_t m2 = 0;              // the graph's target count (TMA windows stay inside it)
  int value_bytes = 4;  // hashtable value width the hub tables were sized for
  // Tier vertex lists (ascending id unless scrambled), indexed by dev::Tier;
  // list[T_HUB] holds the hubs.
  static constexpr int kLists = dev::T_HUB + 1;
  uint32_t* list[kLists] = {};
  uint32_t count[kLists] = {};
  // Thread tier walked in contiguous chunks (ParallelAsync): schedule 4, chosen when
  // the tier carries most of the graph's edges (lattice / road-like inputs).
  bool chunked_thread = false;
  // ... over the graph's chunk-major low range (nulpa_graph::chunk_*): the walk computes
  // its positions (chunk_lo + column start + chunk index) instead of reading the list.
  uint32_t chunk_lo = 0, chunk_L = 0, chunk_dmax = 0;
  bool weighted = false;  // hub tables: packed 64-bit words (unit weights) or split
  // Hub tier.
  uint32_t n_hubs = 0, n_items = 0;
  uint32_t n_sitems = 0;
  uint64_t table_slots = 0;
  uint64_t* tab_off = nullptr;
  uint32_t* tab_cap = nullptr;
  uint32_t* sitem_hub = nullptr;
  uint32_t* sitem_start = nullptr;
  void* tab = nullptr;       // packed words, or keys (weighted)
  void* tab_vals = nullptr;  // weighted: values
  unsigned long long* best = nullptr;
  uint32_t* best_k = nullptr;
  uint8_t* active = nullptr;
  uint8_t* changed = nullptr;
  uint32_t* item_hub = nullptr;
  uint32_t* item_start = nullptr;
  double build_seconds = 0.0;

  dev::HubCtx hub_ctx() const {
    dev::HubCtx h;
    h.hub_v = list[dev::T_HUB];
    h.tab_off = tab_off;
    h.tab_cap = tab_cap;
    h.sitem_hub = sitem_hub;
    h.sitem_start = sitem_start;
    h.n_sitems = n_sitems;
    h.tab = tab;
    h.tab_vals = tab_vals;
    h.best = best;
    h.best_k = best_k;
    h.active = active;
    h.changed = changed;
    h.item_hub = item_hub;
    h.item_start = item_start;
    h.n_hubs = n_hubs;
    h.n_items = n_items;
    return h;
  }
  ~Plan();
};

struct TierBounds {
  uint32_t thread_max, warp_max, block_max;
  uint32_t schedule;  // 1 ascending id, 2 scrambled
};

// Resolve the tier bounds from LpaConfig.switch_degree and the tuning struct.
TierBounds resolve_tiers(uint32_t switch_degree, const nulpa_tuning* tuning);

// Build (or reuse the cached) plan of a resident graph over all vertices.
Plan* get_plan(nulpa_graph* g, const TierBounds& tb, int value_bytes, cudaStream_t s);
// Build an uncached plan over the vertex range [v_lo, v_hi) (caller owns it).
Plan* build_plan(nulpa_graph* g, const TierBounds& tb, int value_bytes, cudaStream_t s,
                 uint32_t v_lo, uint32_t v_hi);

int sm_count();

// Host CSR -> resident graph (nulpa_graph_upload). With `tb`, the plan for
// (tb, value_bytes) is built while the targets stream in (nulpa_run).
nulpa_graph* upload_graph(const nulpa_csr* csr, int device, const TierBounds* tb = nullptr,
                          int value_bytes = 4);

}  // namespace nulpa
