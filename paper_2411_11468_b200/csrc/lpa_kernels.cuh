// ν-LPA pass kernels for sm_100a, one per degree tier.
//
// Reference hot path (paths relative to /root/reference/proj):
//   parallel_move scalar path   src/lpa.cpp:139-165
//   parallel_move team path     src/lpa.cpp:169-230
//   sync_move                   src/lpa.cpp:70-100
//   lpa_move (Sequential)       include/labelprop/lpa.hpp:123-145
//   detail::scan_candidate      include/labelprop/lpa.hpp:92-111
//   ht_accumulate/ht_max_key    include/labelprop/hashtable.hpp:96-185
//
// Every kernel applies the same per-vertex rule: skip if flagged, mark
// processed, pick the neighbour label of greatest total weight (self-loops
// skipped, ties to the smaller label), move if (pick_less ? c* < cur : c* !=
// cur), then wake every neighbour (async: inline; sync: deferred to
// k_wake_list after the joint application, lpa.cpp:92-98).
//
// Tiers (device.cuh), each list ascending by vertex id like partition_by_degree
// (or hashed, tuning.schedule = 2):
//   k_thread    deg <= 8/16   one thread per vertex, labels in registers, O(d^2) count
//                             in neighbour order (bit-identical to the reference sums)
//   k_group<16> deg <= 16     half a warp per vertex, __match_any_sync dedup, redux argmax
//   k_group<32> deg <= 32     one warp per vertex, same
//   k_wtab      deg <= 256    one warp per vertex, per-warp shared-memory table
//   k_block     deg <= 2048   one CTA per vertex, shared-memory table
//   k_hub_*     larger        (hub, 2048-edge chunk) items: shared-memory pre-aggregation,
//                             flush into a per-hub global table, sparse argmax over the
//                             occupied-slot list (packed 64-bit atomicMax), decide, wake
#pragma once

#include <cooperative_groups.h>

#include "device.cuh"

namespace nulpa {
namespace dev {

// ---- shared epilogue ----------------------------------------------------------

// Apply the move rule for vertex i (lpa.cpp:157-164 / :87-90). Returns true if
// the label changed. Called by exactly one thread per vertex.
// FENCE = false: the caller issues the fence itself (once for several label stores).
template <int MODE, bool FENCE = true>
__device__ __forceinline__ bool apply_move(const PassCtx& c, uint32_t i, uint32_t cand) {
  if (cand == kEmpty) return false;
  const uint32_t cur = (MODE == kAsync) ? ld_relaxed(c.lab_out + i) : __ldg(c.lab_in + i);
  const bool allowed = c.pick_less ? (cand < cur) : (cand != cur);
  if (!allowed) return false;
  if constexpr (MODE == kAsync) {
    st_relaxed(c.lab_out + i, cand);
    if (FENCE && c.wake) fence_sc();  // the label store before the wake loads (a18)
  } else {
    c.lab_out[i] = cand;
    if (c.changed) c.changed[atomicAdd(c.changed_n, 1ull)] = i;
  }
  return true;
}

// Wake neighbour j (flags[j] = 0, lpa.cpp:163). The store is skipped when the
// flag already reads 0: hubs are woken by millions of neighbours per pass, and a
// load of a hot byte is far cheaper than a partial-sector store to it.
__device__ __forceinline__ void wake_vertex(uint8_t* flags, uint32_t j) {
  if (load_flag(flags + j)) st_relaxed(flags + j, uint8_t(0));
}

// Wake the neighbours in entries [e0, e1) of the row at `lo`, thread `tid` of `T`: U
// targets, then their U flags, are in flight before any store. (The flag accesses are
// volatile asm, so a plain loop of wake_vertex would wait out one target load and one flag
// load per neighbour.)
template <int U = 4, typename Off>
__device__ __forceinline__ void wake_row(uint8_t* flags, const uint32_t* __restrict__ tgt, Off lo,
                                         uint32_t e0, uint32_t e1, uint32_t tid, uint32_t T,
                                         uint64_t pol) {
  for (uint32_t b = e0 + tid; b < e1; b += T * U) {
    uint32_t j[U];
    uint8_t f[U];
#pragma unroll
    for (int u = 0; u < U; ++u) j[u] = b + u * T < e1 ? ld_stream(tgt + lo + b + u * T, pol) : kEmpty;
#pragma unroll
    for (int u = 0; u < U; ++u) f[u] = j[u] != kEmpty ? load_flag(flags + j[u]) : uint8_t(0);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (f[u]) st_relaxed(flags + j[u], uint8_t(0));
  }
}

// Wake the neighbours of every row of a warp's batch whose bit is set in `chg` (lane k
// holds row k's `lo` and `d`): the rows' entries are walked as one stream, 32 * U at a
// time (lane f takes the f-th entry, its row found by a search over the lanes' prefix
// sums), so short rows do not leave lanes idle. All 32 lanes call it.
template <int U = 4>
__device__ __forceinline__ void warp_wake_rows(uint8_t* flags, const uint32_t* __restrict__ tgt,
                                               uint64_t lo, uint32_t d, unsigned chg, uint64_t pol) {
  const int lane = threadIdx.x & 31;
  const uint32_t dm = (chg >> lane & 1u) ? d : 0u;
  uint32_t pre = dm;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(kFull, pre, o);
    if (lane >= o) pre += x;
  }
  const uint32_t excl = pre - dm, total = __shfl_sync(kFull, pre, 31);
  for (uint32_t f0 = 0; f0 < total; f0 += 32 * U) {
    uint32_t j[U];
    uint8_t fl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t f = f0 + u * 32 + lane;
      int r = 0;  // the last lane whose rows start at or before entry f
#pragma unroll
      for (int st = 16; st > 0; st >>= 1)
        if (__shfl_sync(kFull, excl, r + st) <= f) r += st;
      const uint64_t lo_r = __shfl_sync(kFull, lo, r);
      const uint32_t ex_r = __shfl_sync(kFull, excl, r);
      j[u] = f < total ? ld_stream(tgt + lo_r + (f - ex_r), pol) : kEmpty;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) fl[u] = j[u] != kEmpty ? load_flag(flags + j[u]) : uint8_t(0);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (fl[u]) st_relaxed(flags + j[u], uint8_t(0));
  }
}

// Check-and-set the processed flag (lpa.cpp:143-144). Returns true to skip.
// The caller fences (claim_fence) before loading the labels the decision depends on.
__device__ __forceinline__ bool claim_vertex(const PassCtx& c, uint32_t i) {
  if (!c.flags) return false;
  if (load_flag(c.flags + i)) return true;
  st_relaxed(c.flags + i, uint8_t(1));
  return false;
}

// fence.sc between this thread's claims and the label loads that follow them (a18).
// Only async passes with pruning can race a claim against a wake.
template <int MODE>
__device__ __forceinline__ void claim_fence(const PassCtx& c) {
  if (MODE == kAsync && c.flags) fence_sc();
}

// Apply the move rule given the vertex's current label `cur` (read when the
// vertex was claimed: only this vertex's own thread ever writes it).
template <int MODE, bool FENCE = true>
__device__ __forceinline__ bool apply_move_cur(const PassCtx& c, uint32_t i, uint32_t cand,
                                               uint32_t cur) {
  if (cand == kEmpty) return false;
  const bool allowed = c.pick_less ? (cand < cur) : (cand != cur);
  if (!allowed) return false;
  if constexpr (MODE == kAsync) {
    st_relaxed(c.lab_out + i, cand);
    if (FENCE && c.wake) fence_sc();  // the label store before the wake loads (a18)
  } else {
    c.lab_out[i] = cand;
    if (c.changed) c.changed[atomicAdd(c.changed_n, 1ull)] = i;
  }
  return true;
}

// Per-vertex prologue for a batch of up to 32 list entries, one per lane: the
// list entry, the claim (lpa.cpp:143-144), the row bounds and the current
// label are fetched for 32 vertices at once, so their load latencies overlap
// instead of being paid one vertex after another.
struct Meta {
  uint32_t i, d, cur;
  uint64_t lo;
  bool act;
};

template <int MODE>
__device__ __forceinline__ Meta fetch_meta(const PassCtx& c, const uint32_t* __restrict__ list,
                                           uint32_t t, uint32_t count) {
  Meta m{0u, 0u, 0u, 0ull, false};
  if (t < count) {
    m.i = __ldg(list + t);
    m.act = !claim_vertex(c, m.i);
    if (m.act) {
      m.lo = __ldg(c.g.off + m.i);
      m.d = static_cast<uint32_t>(__ldg(c.g.off + m.i + 1) - m.lo);
      m.cur = (MODE == kAsync) ? ld_relaxed(c.lab_out + m.i) : __ldg(c.lab_in + m.i);
    }
  }
  claim_fence<MODE>(c);  // (consumers of the batch synchronise with this thread first)
  return m;
}

// fetch_meta for a whole warp (all 32 lanes call it, lane k takes entry t = base + k).
// When the batch's 32 list entries are 32 consecutive positions (tier lists are position
// ranges, scrambled at most in 32-position blocks), the row bounds come from ONE
// coalesced 256-byte read of off[i0 .. i0+31] plus one 8-byte read by lane 31:
// off[i + 1] is the next lane's off[i] (NULPA_VEC_META; otherwise two loads per lane).
#ifndef NULPA_VEC_META
#define NULPA_VEC_META 0
#endif
template <int MODE>
__device__ __forceinline__ Meta fetch_meta_warp(const PassCtx& c, const uint32_t* __restrict__ list,
                                                uint32_t t, uint32_t count) {
  if constexpr (!NULPA_VEC_META) {
    return fetch_meta<MODE>(c, list, t, count);
  } else {
    const int lane = threadIdx.x & 31;
    Meta m{0u, 0u, 0u, 0ull, false};
    const bool in = t < count;
    m.i = in ? __ldg(list + t) : 0u;
    const uint32_t i0 = __shfl_sync(kFull, m.i, 0);
    const bool run = __all_sync(kFull, !in || m.i == i0 + static_cast<uint32_t>(lane));
    m.act = in && !claim_vertex(c, m.i);
    if (run) {
      const uint64_t o = in ? __ldg(c.g.off + m.i) : 0ull;
      uint64_t o1 = __shfl_down_sync(kFull, o, 1);
      if (lane == 31 && in) o1 = __ldg(c.g.off + m.i + 1);
      // (a lane past `count` has in == false; the last in-range lane below it loads its own)
      if (in && lane < 31 && t + 1 >= count) o1 = __ldg(c.g.off + m.i + 1);
      if (m.act) {
        m.lo = o;
        m.d = static_cast<uint32_t>(o1 - o);
      }
    } else if (m.act) {
      m.lo = __ldg(c.g.off + m.i);
      m.d = static_cast<uint32_t>(__ldg(c.g.off + m.i + 1) - m.lo);
    }
    if (m.act) m.cur = (MODE == kAsync) ? ld_relaxed(c.lab_out + m.i) : __ldg(c.lab_in + m.i);
    claim_fence<MODE>(c);
    return m;
  }
}

__device__ __forceinline__ Meta shfl_meta(const Meta& m, int src) {
  Meta r;
  r.i = __shfl_sync(kFull, m.i, src);
  r.d = __shfl_sync(kFull, m.d, src);
  r.cur = __shfl_sync(kFull, m.cur, src);
  r.lo = __shfl_sync(kFull, m.lo, src);
  r.act = __shfl_sync(kFull, m.act ? 1 : 0, src) != 0;
  return r;
}

template <bool WEIGHTED>
constexpr bool kPacked = !WEIGHTED;  // unit weights -> packed 64-bit slots

// ---- tier: thread per vertex ---------------------------------------------------

// CHUNKED (ParallelAsync, schedule 4): thread k walks the contiguous list slice
// [k*L, (k+1)*L) in order, as each of the reference's workers walks its chunk
// (lpa.cpp:139-165), instead of the grid-stride interleave.
// V: list entries a thread takes per iteration (grid-stride walk only): their claims
// share one fence and their row, target and label loads are issued together.
// cm_L != 0 (CHUNKED): the tier is the graph's chunk-major range at cm_lo (layout.cu
// chunk_major) with chunks of cm_L entries: entry r of chunk k sits at column r, row k,
// i.e. at cm_lo + r*q + min(r, rem) + k for count = q*cm_L + rem, and the grid must
// cover every chunk.
template <int MODE, typename W, bool WEIGHTED, int DMAX, bool CHUNKED = false, int V = 1>
__global__ void __launch_bounds__(256) k_thread(PassCtx c, const uint32_t* __restrict__ list,
                                                uint32_t count, uint32_t cm_lo = 0,
                                                uint32_t cm_L = 0) {
  static_assert(!CHUNKED || V == 1, "a chunk walk takes its entries one at a time");
  if (stopped(c.stop)) return;
  unsigned long long n_v = 0, n_e = 0, n_dn = 0, n_w = 0;
  const uint64_t pol = policy_evict_first();
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t L = CHUNKED ? (cm_L ? cm_L : (count + stride - 1) / stride) : 0u;
  const uint32_t cq = (CHUNKED && cm_L) ? count / cm_L : 0u;
  const uint32_t crem = (CHUNKED && cm_L) ? count % cm_L : 0u;
  const uint32_t t_end = CHUNKED ? min(count, (tid + 1) * L) : count;
  const uint32_t step = CHUNKED ? 1u : stride;
  for (uint32_t t = CHUNKED ? tid * L : tid; t < t_end; t += step * V) {
    uint32_t iv[V], d[V];
    uint64_t lo[V];
    bool act[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const uint32_t tv = t + v * step;
      act[v] = tv < t_end;
      if (CHUNKED && cm_L) {
        const uint32_t r = tv - tid * L;
        iv[v] = act[v] ? cm_lo + r * cq + min(r, crem) + tid : 0u;
      } else {
        iv[v] = act[v] ? __ldg(list + tv) : 0u;
      }
      if (act[v]) act[v] = !claim_vertex(c, iv[v]);
    }
    claim_fence<MODE>(c);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      lo[v] = act[v] ? __ldg(c.g.off + iv[v]) : 0ull;
      d[v] = act[v] ? static_cast<uint32_t>(__ldg(c.g.off + iv[v] + 1) - lo[v]) : 0u;
    }
    uint32_t nb[V][DMAX];
    uint32_t lab[V][DMAX];
    W wt[V][DMAX];
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int k = 0; k < DMAX; ++k)
        nb[v][k] = (k < d[v]) ? ld_stream(c.g.tgt + lo[v] + k, pol) : iv[v];
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int k = 0; k < DMAX; ++k) {
        const bool valid = k < d[v] && nb[v][k] != iv[v];  // self-loops skipped (lpa.hpp:102)
        lab[v][k] = valid ? gather_label<MODE>(c, nb[v][k]) : kEmpty;
        wt[v][k] = valid ? edge_weight<W, WEIGHTED>(c.g, lo[v] + k) : W(0);
      }
    // The V rows' label stores share one fence before their wake loads (a18).
    bool chg[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      chg[v] = false;
      if (!act[v]) continue;
      // Per-label total in neighbour order (bit-identical to the reference's
      // sequential accumulation, even for non-integer weights), then argmax.
      Best<VBits<W>> b{VBits<W>(0), kEmpty};
#pragma unroll
      for (int k = 0; k < DMAX; ++k) {
        W sum = W(0);
#pragma unroll
        for (int m = 0; m < DMAX; ++m) sum += (lab[v][m] == lab[v][k]) ? wt[v][m] : W(0);
        best_merge(b, to_vbits<W>(sum), lab[v][k]);
      }
      ++n_v;
      n_e += d[v];
      chg[v] = apply_move<MODE, false>(c, iv[v], b.k);
      n_dn += chg[v];
    }
    if (MODE == kAsync && c.wake) {
      bool any = false;
#pragma unroll
      for (int v = 0; v < V; ++v) any |= chg[v];
      if (any) fence_sc();
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (!chg[v]) continue;
        uint8_t f[DMAX];  // every flag load in flight before the first store
#pragma unroll
        for (int k = 0; k < DMAX; ++k) f[k] = k < d[v] ? load_flag(c.flags + nb[v][k]) : uint8_t(0);
#pragma unroll
        for (int k = 0; k < DMAX; ++k)
          if (f[k]) st_relaxed(c.flags + nb[v][k], uint8_t(0));
        n_w += d[v];
      }
    }
  }
  warp_add_counter(c.ctr, C_PROC_V, n_v);
  warp_add_counter(c.ctr, C_PROC_E, n_e);
  warp_add_counter(c.ctr, C_DN, n_dn);
  warp_add_counter(c.ctr, C_WAKE_E, n_w);
}

// Thread per vertex, Q rows per thread iteration with the protocol's fences amortised:
// the Q claims share one fence, the Q rows are then decided one after another (one row's
// loads in registers at a time), and their label stores share one fence before the
// warp wakes every changed row of the iteration as one stream (warp_wake_rows).
template <int MODE, typename W, bool WEIGHTED, int DMAX, int Q = 4>
__global__ void __launch_bounds__(256) k_thread_q(PassCtx c, const uint32_t* __restrict__ list,
                                                  uint32_t count) {
  if (stopped(c.stop)) return;
  unsigned long long n_v = 0, n_e = 0, n_dn = 0, n_w = 0;
  const uint64_t pol = policy_evict_first();
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  // every lane of a warp runs the same number of iterations (warp-wide wake-ups)
  const uint32_t span = ((count + 31u) & ~31u);
  for (uint32_t t = tid; t - (tid & 31u) < span; t += stride * Q) {
    uint32_t iq[Q];
    bool aq[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const uint32_t tv = t + q * stride;
      aq[q] = tv < count;
      iq[q] = aq[q] ? __ldg(list + tv) : 0u;
      if (aq[q]) aq[q] = !claim_vertex(c, iq[q]);
    }
    claim_fence<MODE>(c);
    bool stored = false;
    unsigned chg = 0;  // bit q: row q of this thread changed label
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      if (!aq[q]) continue;
      const uint32_t i = iq[q];
      const uint64_t lo = __ldg(c.g.off + i);
      const uint32_t d = static_cast<uint32_t>(__ldg(c.g.off + i + 1) - lo);
      uint32_t nb[DMAX], lab[DMAX];
      W wt[DMAX];
#pragma unroll
      for (int k = 0; k < DMAX; ++k) nb[k] = (k < d) ? ld_stream(c.g.tgt + lo + k, pol) : i;
#pragma unroll
      for (int k = 0; k < DMAX; ++k) {
        const bool valid = k < d && nb[k] != i;  // self-loops skipped (lpa.hpp:102)
        lab[k] = valid ? gather_label<MODE>(c, nb[k]) : kEmpty;
        wt[k] = valid ? edge_weight<W, WEIGHTED>(c.g, lo + k) : W(0);
      }
      // per-label total in neighbour order (bit-identical sums), then argmax
      Best<VBits<W>> b{VBits<W>(0), kEmpty};
#pragma unroll
      for (int k = 0; k < DMAX; ++k) {
        W sum = W(0);
#pragma unroll
        for (int m = 0; m < DMAX; ++m) sum += (lab[m] == lab[k]) ? wt[m] : W(0);
        best_merge(b, to_vbits<W>(sum), lab[k]);
      }
      ++n_v;
      n_e += d;
      if (apply_move<MODE, false>(c, i, b.k)) {
        ++n_dn;
        stored = true;
        chg |= 1u << q;
        if (MODE == kAsync && c.wake) n_w += d;
      }
    }
    if (MODE == kAsync && c.wake && __any_sync(kFull, chg != 0)) {
      if (stored) fence_sc();  // this thread's label stores before any wake load (a18)
      __syncwarp();
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const bool mine = chg >> q & 1u;
        const unsigned rows = __ballot_sync(kFull, mine);
        if (!rows) continue;
        uint64_t lo = 0;
        uint32_t d = 0;
        if (mine) {
          lo = __ldg(c.g.off + iq[q]);
          d = static_cast<uint32_t>(__ldg(c.g.off + iq[q] + 1) - lo);
        }
        warp_wake_rows<4>(c.flags, c.g.tgt, lo, d, rows, pol);
      }
    }
  }
  warp_add_counter(c.ctr, C_PROC_V, n_v);
  warp_add_counter(c.ctr, C_PROC_E, n_e);
  warp_add_counter(c.ctr, C_DN, n_dn);
  warp_add_counter(c.ctr, C_WAKE_E, n_w);
}

// Chunk walk over the graph's chunk-major range (layout.cu chunk_major), Q rows of a
// thread's chunk per iteration: their claims share one fence, their row bounds are loaded
// together, the rows are decided one after another in chunk order (each row's loads
// follow the previous row's label store, so the walk sees its own moves as k_thread's
// does), and their label stores share one fence before this thread wakes the changed
// rows' neighbours. Thread k's rows sit at cm_lo + r*q + min(r, rem) + k: every load is
// coalesced across the warp.
// PF: the next row's targets are loaded while this row's labels are in flight (targets
// never change), so a row's chain is one label round trip.
// MINB: resident CTAs of 256 threads per SM the register budget is held to (the layout's
// walk threads per SM, layout.cu chunk_major: 4 for ranges of degree <= 8, 6 for <= 4).
template <int MODE, typename W, bool WEIGHTED, int DMAX, int Q = 4, bool PF = false, int MINB = 4>
__global__ void __launch_bounds__(256, MINB) k_chunk_walk(PassCtx c, uint32_t count, uint32_t cm_lo,
                                                          uint32_t cm_L) {
  if (stopped(c.stop)) return;
  unsigned long long n_v = 0, n_e = 0, n_dn = 0, n_w = 0;
  const uint64_t pol = policy_evict_first();
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t cq = count / cm_L, crem = count % cm_L;
  // entries of this thread's chunk: cm_L for k < cq, crem for k == cq, none above
  const uint32_t len = k < cq ? cm_L : (k == cq ? crem : 0u);
  for (uint32_t r0 = 0; r0 < len; r0 += Q) {
    uint32_t iq[Q];
    bool aq[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const uint32_t r = r0 + q;
      aq[q] = r < len;
      iq[q] = cm_lo + r * cq + min(r, crem) + k;
      if (aq[q]) aq[q] = !claim_vertex(c, iq[q]);
    }
    claim_fence<MODE>(c);
    uint64_t lq[Q];
    uint32_t dq[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      lq[q] = aq[q] ? __ldg(c.g.off + iq[q]) : 0ull;
      dq[q] = aq[q] ? static_cast<uint32_t>(__ldg(c.g.off + iq[q] + 1) - lq[q]) : 0u;
    }
    unsigned chg = 0;  // bit q: row q changed label
    uint32_t nn[DMAX];  // PF: the next active row's targets
    auto row_targets = [&](int q, uint32_t (&dst)[DMAX]) {
#pragma unroll
      for (int e = 0; e < DMAX; ++e)
        dst[e] = (aq[q] && e < dq[q]) ? ld_stream(c.g.tgt + lq[q] + e, pol) : iq[q];
    };
    if (PF) row_targets(0, nn);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      uint32_t nb[DMAX], lab[DMAX];
      if constexpr (PF) {
#pragma unroll
        for (int e = 0; e < DMAX; ++e) nb[e] = nn[e];
        if (q + 1 < Q) row_targets(q + 1, nn);  // (before this row's gathers, in flight with them)
      }
      if (!aq[q]) continue;
      const uint32_t i = iq[q];
      const uint64_t lo = lq[q];
      const uint32_t d = dq[q];
      W wt[DMAX];
      if constexpr (!PF) {
#pragma unroll
        for (int e = 0; e < DMAX; ++e) nb[e] = (e < d) ? ld_stream(c.g.tgt + lo + e, pol) : i;
      }
#pragma unroll
      for (int e = 0; e < DMAX; ++e) {
        const bool valid = e < d && nb[e] != i;  // self-loops skipped (lpa.hpp:102)
        lab[e] = valid ? gather_label<MODE>(c, nb[e]) : kEmpty;
        wt[e] = valid ? edge_weight<W, WEIGHTED>(c.g, lo + e) : W(0);
      }
      // per-label total in neighbour order (bit-identical sums), then argmax
      Best<VBits<W>> b{VBits<W>(0), kEmpty};
#pragma unroll
      for (int e = 0; e < DMAX; ++e) {
        W sum = W(0);
#pragma unroll
        for (int m = 0; m < DMAX; ++m) sum += (lab[m] == lab[e]) ? wt[m] : W(0);
        best_merge(b, to_vbits<W>(sum), lab[e]);
      }
      ++n_v;
      n_e += d;
      if (apply_move<MODE, false>(c, i, b.k)) {
        ++n_dn;
        chg |= 1u << q;
        if (MODE == kAsync && c.wake) n_w += d;
      }
    }
    if (MODE == kAsync && c.wake && chg) {
      fence_sc();  // this thread's label stores before any wake load (a18)
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        if (!(chg >> q & 1u)) continue;
        uint32_t nb[DMAX];
        uint8_t f[DMAX];  // every flag load in flight before the first store
#pragma unroll
        for (int e = 0; e < DMAX; ++e) nb[e] = e < dq[q] ? ld_stream(c.g.tgt + lq[q] + e, pol) : 0u;
#pragma unroll
        for (int e = 0; e < DMAX; ++e) f[e] = e < dq[q] ? load_flag(c.flags + nb[e]) : uint8_t(0);
#pragma unroll
        for (int e = 0; e < DMAX; ++e)
          if (f[e]) st_relaxed(c.flags + nb[e], uint8_t(0));
      }
    }
  }
  warp_add_counter(c.ctr, C_PROC_V, n_v);
  warp_add_counter(c.ctr, C_PROC_E, n_e);
  warp_add_counter(c.ctr, C_DN, n_dn);
  warp_add_counter(c.ctr, C_WAKE_E, n_w);
}

// ---- tier: G lanes per vertex, register dedup -------------------------------------

template <typename V, int G>
__device__ __forceinline__ Best<V> group_best(Best<V> b, unsigned gmask) {
  if constexpr (std::is_same_v<V, uint32_t>) {
    return warp_best(b, gmask);
  } else {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(kFull, b.v, o, G);
      const uint32_t ok = __shfl_xor_sync(kFull, b.k, o, G);
      best_merge(b, ov, ok);
    }
    return b;
  }
}

// S steps of a warp's batch are loaded at once: the targets of all S steps, then their
// labels (S independent loads in flight per lane), then the S steps are decided one
// after another. The batch prologue (claims, row bounds, current labels of 32 list
// entries) is shared through shared memory.
// `bsz` (8, 16 or 32) list entries per warp batch: 32 on large tiers; small graphs use
// shorter batches so that more warps share the tier (a warp walks its batch's steps one
// after another, each step a target and a label load latency).
template <int MODE, typename W, bool WEIGHTED, int G, int S = 8>
__global__ void __launch_bounds__(256) k_group(PassCtx c, const uint32_t* __restrict__ list,
                                               uint32_t count, uint32_t bsz = 32) {
  if (stopped(c.stop)) return;
  constexpr int kPer = 32 / G;           // vertices per warp step
  const int kSteps = static_cast<int>(bsz) / kPer;  // steps per batch
  static_assert((32 / kPer) % S == 0, "steps per chunk (S > 1 runs 32-entry batches)");
  const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G, wid = threadIdx.x >> 5;
  const unsigned gmask = (G == 32) ? kFull : (((1u << G) - 1u) << (sub * G));
  __shared__ Meta s_meta[8][32];
  const uint64_t pol = policy_evict_first();
  unsigned long long n_v = 0, n_e = 0, n_dn = 0, n_w = 0;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  if (S > 1) bsz = 32;
  for (uint32_t base = gw * bsz; base < count; base += nw * bsz) {
    s_meta[wid][lane] = fetch_meta_warp<MODE>(c, list, base + lane, min(count, base + bsz));
    __syncwarp();  // every lane's claim (and its fence) before any lane's label loads
    // Async wake-ups are deferred to the end of the batch: every lane that stored a label
    // fences once, then the warp wakes the changed rows' neighbours as one stream.
    unsigned chg_bits = 0;
    bool stored = false;
    // S == 1: the next step's target is loaded while this step's label is in flight
    // (targets never change, so this adds no staleness)
    auto step_target = [&](int st) -> uint32_t {
      const Meta& m = s_meta[wid][st * kPer + sub];
      return (m.act && gl < m.d) ? ld_stream(c.g.tgt + m.lo + gl, pol) : m.i;
    };
    uint32_t jn = (S == 1 && kSteps > 0) ? step_target(0) : 0u;
#pragma unroll 1
    for (int c0 = 0; c0 < kSteps; c0 += S) {
      uint32_t j[S], lab[S];
      W w[S];
#pragma unroll
      for (int k = 0; k < S; ++k) j[k] = S == 1 ? jn : step_target(c0 + k);
#pragma unroll
      for (int k = 0; k < S; ++k) {
        const Meta& m = s_meta[wid][(c0 + k) * kPer + sub];
        const bool valid = m.act && gl < m.d && j[k] != m.i;
        lab[k] = valid ? gather_label<MODE>(c, j[k]) : kEmpty;
        w[k] = valid ? edge_weight<W, WEIGHTED>(c.g, m.lo + gl) : W(0);
      }
      if (S == 1 && c0 + 1 < kSteps) jn = step_target(c0 + 1);
      // Async, S > 1: the labels of all S steps were loaded before any of them was
      // decided, so step k patches in the moves of this chunk's earlier steps (a lane
      // whose neighbour is one of those vertices takes its new label): every step sees
      // the batch's earlier moves exactly as the one-step-at-a-time walk does.
      uint32_t pv[S][kPer], pl[S][kPer];
#pragma unroll
      for (int k = 0; k < S; ++k) {
        const Meta m = s_meta[wid][(c0 + k) * kPer + sub];
        if constexpr (MODE == kAsync && S > 1) {
          uint32_t x = lab[k];
#pragma unroll
          for (int q = 0; q < k; ++q)
#pragma unroll
            for (int r = 0; r < kPer; ++r)
              if (j[k] == pv[q][r] && pl[q][r] != kEmpty && x != kEmpty) x = pl[q][r];
          lab[k] = x;
        }
        const unsigned peers = __match_any_sync(kFull, lab[k]) & gmask;
        W sm;
        if constexpr (WEIGHTED)
          sm = peer_sum(w[k], peers);
        else
          sm = static_cast<W>(__popc(peers));
        Best<VBits<W>> b{VBits<W>(0), kEmpty};
        if (lab[k] != kEmpty && (__ffs(peers) - 1) == lane) b = Best<VBits<W>>{to_vbits<W>(sm), lab[k]};
        b = group_best<VBits<W>, G>(b, gmask);
        bool ch = false;
        if (m.act && gl == 0) {
          ch = apply_move_cur<MODE, false>(c, m.i, b.k, m.cur);
          stored |= ch;
          ++n_v;
          n_e += m.d;
          n_dn += ch;
          if (MODE == kAsync && ch && c.wake) n_w += m.d;
        }
        if (MODE == kAsync) {
          const unsigned bl = __ballot_sync(kFull, ch);
#pragma unroll
          for (int q = 0; q < kPer; ++q)
            if (bl >> (q * G) & 1u) chg_bits |= 1u << ((c0 + k) * kPer + q);
          if constexpr (S > 1) {
#pragma unroll
            for (int r = 0; r < kPer; ++r) {  // lane r * G decided vertex r of this step
              pv[k][r] = __shfl_sync(kFull, m.i, r * G);
              pl[k][r] = __shfl_sync(kFull, ch ? b.k : kEmpty, r * G);
            }
          }
        }
      }
    }
    if (MODE == kAsync && c.wake && chg_bits) {
      if (stored) fence_sc();  // this lane's label stores before any wake load (a18)
      __syncwarp();
      const Meta& me = s_meta[wid][lane];
      warp_wake_rows<4>(c.flags, c.g.tgt, me.lo, me.d, chg_bits, pol);
    }
    __syncwarp();  // s_meta is rewritten by the next batch
  }
  warp_add_counter(c.ctr, C_PROC_V, n_v);
  warp_add_counter(c.ctr, C_PROC_E, n_e);
  warp_add_counter(c.ctr, C_DN, n_dn);
  warp_add_counter(c.ctr, C_WAKE_E, n_w);
}

// ---- cooperative gather + insert -------------------------------------------------
// Team tables are kept EMPTY between vertices: every newly claimed slot is
// appended to an occupancy list (one shared atomic per warp), and the argmax
// sweep reads and resets only the occupied slots. Per-vertex table work is
// therefore O(distinct labels), not O(capacity).

// Append the slots claimed in this warp round to the occupancy list.
__device__ __forceinline__ void occ_append(bool claimed, uint32_t slot, uint16_t* occ,
                                           unsigned* occ_n) {
  const unsigned m = __ballot_sync(kFull, claimed);
  if (!m) return;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  unsigned base = 0;
  if (lane == leader) base = atomicAdd(occ_n, static_cast<unsigned>(__popc(m)));
  base = __shfl_sync(kFull, base, leader);
  if (claimed) occ[base + __popc(m & ((1u << lane) - 1u))] = static_cast<uint16_t>(slot);
}

// One round of a team gather: each lane holds one edge (or none), dedups its
// label against the warp with __match_any_sync, and the lowest lane of each
// label group adds the group's weight to the table. All 32 lanes call it.
template <typename W, bool WEIGHTED, typename Tab>
__device__ __forceinline__ void gather_insert(const PassCtx& c, uint32_t lab, W w, Tab& tab,
                                              uint32_t cap, uint16_t* occ, unsigned* occ_n,
                                              unsigned long long& fails) {
  const unsigned peers = __match_any_sync(kFull, lab);
  W s;
  if constexpr (WEIGHTED)
    s = peer_sum(w, peers);
  else
    s = static_cast<W>(__popc(peers));
  const int lane = threadIdx.x & 31;
  int r = -1;
  uint32_t slot = 0;
  if (lab != kEmpty && (__ffs(peers) - 1) == lane) {
    r = tab.add(cap, c.strategy, lab, s, &slot);
    if (r == 0) ++fails;
  }
  if (occ) occ_append(r == 2, slot, occ, occ_n);
}

// U rounds of a team gather at once, unit weights, the CTA's own shared table:
// the same result as U calls of gather_insert, but every step is issued for all
// U rounds before the next step (U match_any, then U first probes, U claims, U
// count adds, one occupancy append), so the rounds' latency chains overlap
// instead of running back to back. `live` has bit u set when round u holds at
// least one of the warp's edges (warp-uniform). All 32 lanes call it.
template <int U, typename W, int DEDUP = 1>
__device__ __forceinline__ void gather_insert_multi(const PassCtx& c, const uint32_t (&lab)[U],
                                                    unsigned live, SmemTable<W>& tab,
                                                    uint32_t cap, uint16_t* occ, unsigned* occ_n,
                                                    unsigned long long& fails) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t mask = cap - 1;
  unsigned peers[U];
  uint32_t idx[U], cur[U];
  bool lead[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (!(live >> u & 1u)) {
      peers[u] = 0u;
    } else if constexpr (DEDUP == 1) {
      peers[u] = __match_any_sync(kFull, lab[u]);
    } else {
      peers[u] = 1u << lane;
    }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    lead[u] = lab[u] != kEmpty && (peers[u] & lt) == 0u && peers[u] != 0u;
    idx[u] = hash_start(lab[u], cap);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    cur[u] = lead[u] ? tab.ld_key(idx[u] & mask) : 0u;
  }
  int r[U];
  uint32_t slot[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    slot[u] = idx[u] & mask;
    r[u] = -1;
    if (lead[u]) {
      r[u] = 1;
      if (cur[u] == kEmpty) {
        cur[u] = tab.cas_key(slot[u], lab[u]);
        if (cur[u] == kEmpty) {
          cur[u] = lab[u];
          r[u] = 2;
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (!lead[u]) continue;
    if (cur[u] == lab[u]) {
      tab.add_count(slot[u], __popc(peers[u]));
    } else {  // first-probe collision: the probe walk (rare)
      r[u] = c.strategy == 3
                 ? tab.template add_collided<3>(cap, lab[u], __popc(peers[u]), idx[u], &slot[u])
                 : tab.template add_collided<-1>(cap, lab[u], __popc(peers[u]), idx[u], &slot[u],
                                                 c.strategy);
      if (r[u] == 0) ++fails;
    }
  }
  // One occupancy append for every slot claimed in the U rounds.
  if (occ == nullptr) return;  // (hub chunk tables are swept whole)
  unsigned m[U], tot = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    m[u] = __ballot_sync(kFull, r[u] == 2);
    tot += __popc(m[u]);
  }
  if (tot == 0) return;
  unsigned b = 0;
  if (lane == 0) b = atomicAdd(occ_n, tot);
  b = __shfl_sync(kFull, b, 0);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (r[u] == 2) occ[b + __popc(m[u] & lt)] = static_cast<uint16_t>(slot[u]);
    b += __popc(m[u]);
  }
}

// Gather edges [e0, e1) of vertex i (U edges per thread in flight) into `tab`.
// `T` threads cooperate; all of them call it with the same bounds.
template <int MODE, typename W, bool WEIGHTED, typename Tab, int U = 4, int DEDUP = 1>
__device__ __forceinline__ void team_gather(const PassCtx& c, uint32_t i, uint64_t lo,
                                            uint32_t e0, uint32_t e1, Tab& tab, uint32_t cap,
                                            uint32_t tid, uint32_t T, uint64_t pol,
                                            uint16_t* occ, unsigned* occ_n,
                                            unsigned long long& fails) {
  for (uint32_t base = e0; base < e1; base += T * U) {
    uint32_t j[U], lab[U];
    W w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t e = base + u * T + tid;
      j[u] = e < e1 ? ld_stream(c.g.tgt + lo + e, pol) : i;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t e = base + u * T + tid;
      const bool valid = e < e1 && j[u] != i;
      lab[u] = valid ? gather_label<MODE>(c, j[u]) : kEmpty;
      w[u] = valid ? edge_weight<W, WEIGHTED>(c.g, lo + e) : W(0);
    }
    // Skip warp-rounds with no edge at all (warp-uniform test): short rows do not
    // pay for the unrolled tail.
    const uint32_t wbase = base + (tid & ~31u);
    if constexpr (std::is_same_v<Tab, SmemTable<W>>) {
      unsigned live = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) live |= (wbase + u * T < e1 ? 1u : 0u) << u;
      gather_insert_multi<U, W, DEDUP>(c, lab, live, tab, cap, occ, occ_n, fails);
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (wbase + u * T < e1)
          gather_insert<W, WEIGHTED>(c, lab[u], w[u], tab, cap, occ, occ_n, fails);
    }
  }
}

// Argmax over the occupied slots [tid, n_occ) step T; resets them as it goes.
template <typename W, typename Tab>
__device__ __forceinline__ Best<VBits<W>> occ_argmax_reset(Tab& tab, const uint16_t* occ,
                                                          unsigned n_occ, uint32_t tid,
                                                          uint32_t T) {
  Best<VBits<W>> b{VBits<W>(0), kEmpty};
  for (uint32_t p = tid; p < n_occ; p += T) {
    const uint32_t s = occ[p];
    uint32_t k;
    VBits<W> v;
    tab.read(s, k, v);
    best_merge(b, v, k);
    tab.clear_slot(s);
  }
  return b;
}

// ---- block-wide helpers ------------------------------------------------------------

template <typename V>
__device__ __forceinline__ Best<V> block_best(Best<V> b, Best<V>* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  b = warp_best(b);
  if (lane == 0) red[warp] = b;
  __syncthreads();
  if (warp == 0) {
    Best<V> r = lane < static_cast<int>(blockDim.x >> 5) ? red[lane] : Best<V>{V(0), kEmpty};
    r = warp_best(r);
    if (lane == 0) red[0] = r;
  }
  __syncthreads();
  return red[0];
}

// Table capacity for a row of degree d: load <= 1/4 where the team's fixed
// table allows it (fewer first-probe collisions), never above 1/2 for the
// <= 256-thread teams or 3/4 for the 128 KB tables (always a power of two).
template <int CAP>
__device__ __forceinline__ uint32_t table_cap(uint32_t d) {
  const uint32_t want = pow2_ceil(4 * d);
  if constexpr (CAP <= kBlock2Cap)
    return min(want, static_cast<uint32_t>(CAP));  // CAP >= 2 * MAXD
  else
    return max(min(want, static_cast<uint32_t>(CAP)), pow2_ceil(d + d / 3 + 1));
}

template <typename Tab, int CAP, int MAXD>
constexpr size_t block_bytes() {
  return size_t(CAP) * Tab::kSlotBytes + size_t(MAXD) * sizeof(uint16_t);
}

// ---- tier: TEAM threads per vertex, several teams per CTA ---------------------------
// A CTA of CTA_THREADS threads holds CTA_THREADS / TEAM independent teams; each
// team owns one vertex at a time and its own shared table + occupancy list, and
// synchronises on its own named barrier (bar.sync id, TEAM), so teams never wait
// for each other. The team size is matched to the degree band (about 4-8 edges
// per thread) so no round of the gather runs mostly-idle lanes.
__device__ __forceinline__ void team_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int TEAM, typename V>
__device__ __forceinline__ Best<V> team_best(Best<V> b, Best<V>* red, int team_tid, int bar,
                                             unsigned* reset = nullptr) {
  // `reset` (optional): zeroed once every team thread is past its reads of it
  // (the occupancy count of the sweep that produced b), ordered before return.
  b = warp_best(b);
  if constexpr (TEAM == 32) {
    if (reset) {
      __syncwarp();
      if (team_tid == 0) *reset = 0;
      __syncwarp();
    }
    return b;
  } else {
    const int w = team_tid >> 5, lane = team_tid & 31;
    if (lane == 0) red[w] = b;
    team_sync(bar, TEAM);
    if (reset && team_tid == 0) *reset = 0;
    if (w == 0) {
      Best<V> r = lane < TEAM / 32 ? red[lane] : Best<V>{V(0), kEmpty};
      r = warp_best(r);
      if (lane == 0) red[0] = r;
    }
    team_sync(bar, TEAM);
    return red[0];
  }
}

#ifndef NULPA_TEAM_U
#define NULPA_TEAM_U 4
#endif
constexpr int kTeamU = NULPA_TEAM_U;  // gather rounds in flight per team thread

template <int TEAM>
constexpr uint32_t kTeamBatch = TEAM <= 32 ? 32u : (TEAM <= 128 ? 16u : 4u);

#ifndef NULPA_TEAM_PREFETCH
#define NULPA_TEAM_PREFETCH 0
#endif
// 1: the next vertex's first-round targets and labels; 2: its targets only (no staleness)
constexpr int kTeamPrefetch = NULPA_TEAM_PREFETCH;

// First gather round of the row in `m` (edges [0, T * U)): targets into j, labels into lab.
template <int MODE, int U>
__device__ __forceinline__ void round_load(const PassCtx& c, const Meta& m, uint32_t base,
                                           uint32_t tid, uint32_t T, uint64_t pol, uint32_t (&j)[U],
                                           uint32_t (&lab)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t e = base + u * T + tid;
    j[u] = e < m.d ? ld_stream(c.g.tgt + m.lo + e, pol) : m.i;
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t e = base + u * T + tid;
    lab[u] = (e < m.d && j[u] != m.i) ? gather_label<MODE>(c, j[u]) : kEmpty;
  }
}

template <typename Tab, int CAP, int MAXD>
constexpr size_t team_bytes() {
  return size_t(CAP) * Tab::kSlotBytes + size_t(MAXD) * sizeof(uint16_t);
}

// DEDUP: merge equal labels inside a warp (__match_any_sync) before the table
// insert. It pays once labels have collapsed; in the first pass of a run almost
// every label is distinct and the table's own claim/add handles the few repeats
// for less (launch_pass picks the variant per pass).
#ifndef NULPA_TEAM_MINB
#define NULPA_TEAM_MINB 4  // resident 256-thread team CTAs per SM (registers <= 64)
#endif
template <int MODE, typename W, bool WEIGHTED, int CTA_THREADS, int TEAM, int CAP, int MAXD,
          int DEDUP = 1>
__global__ void __launch_bounds__(CTA_THREADS, CTA_THREADS <= 256 ? NULPA_TEAM_MINB : (CTA_THREADS == 512 ? 2 : 1))
    k_team(PassCtx c, const uint32_t* __restrict__ list, uint32_t count,
           uint32_t bsz = kTeamBatch<TEAM>) {
  if (stopped(c.stop)) return;
  static_assert(CTA_THREADS % TEAM == 0 && TEAM % 32 == 0, "team shape");
  constexpr int kTeams = CTA_THREADS / TEAM;
  using Tab = std::conditional_t<kPacked<WEIGHTED>, SmemTable<W>, Table<false, W>>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Best<VBits<W>> s_red[kTeams][TEAM / 32 > 0 ? TEAM / 32 : 1];
  __shared__ unsigned s_occ_n[kTeams];
  const int team = threadIdx.x / TEAM, ttid = threadIdx.x % TEAM;
  const int bar = 1 + team;  // named barrier 0 is __syncthreads
  unsigned char* base = smem_raw + size_t(team) * team_bytes<Tab, CAP, MAXD>();
  Tab tab;
  tab.bind(base, CAP);
  uint16_t* occ = reinterpret_cast<uint16_t*>(base + size_t(CAP) * Tab::kSlotBytes);
  auto sync = [&]() {
    if constexpr (TEAM == 32)
      __syncwarp();
    else
      team_sync(bar, TEAM);
  };
  for (uint32_t s = ttid; s < CAP; s += TEAM) tab.clear_slot(s);  // once per lifetime
  if (ttid == 0) s_occ_n[team] = 0;
  sync();
  const uint64_t pol = policy_evict_first();
  unsigned long long n_v = 0, n_e = 0, n_dn = 0, n_w = 0, fails = 0;
  // Teams take kBatch list entries at a time: the team's first warp fetches the
  // batch prologue (claims, row bounds, current labels) for all of them at once.
  // Larger teams own fewer, longer rows per batch (load balance at the tail).
  // kBatch entries per team batch at most; `bsz` (<= kBatch) at run time: a tier too small
  // to give every resident team a full batch uses shorter ones (more teams busy, a shorter
  // per-team chain of vertices).
  constexpr uint32_t kBatch = kTeamBatch<TEAM>;
  bsz = min(max(bsz, 1u), kBatch);
  __shared__ Meta s_meta[TEAM > 32 ? kTeams : 1][kBatch];
  const uint32_t nteams = gridDim.x * kTeams;
  // Teams of >= 256 threads own long rows: they pull batches from a work
  // counter (c.work, zeroed before the launch) so the tier's tail stays balanced;
  // smaller teams take batches grid-stride.
  constexpr bool kDynamic = TEAM >= 256;
  __shared__ uint32_t s_base[kTeams];
  auto next_base = [&](uint32_t cur) -> uint32_t {
    if constexpr (kDynamic) {
      if (ttid == 0) s_base[team] = atomicAdd(c.work, bsz);
      sync();
      const uint32_t b = s_base[team];
      sync();
      return b;
    } else {
      return cur + nteams * bsz;
    }
  };
  uint32_t first = (blockIdx.x * kTeams + team) * bsz;
  if constexpr (kDynamic) first = next_base(0);
  for (uint32_t base = first; base < count; base = next_base(base)) {
    Meta mine{};
    const uint32_t lim = min(count, base + bsz);
    if constexpr (TEAM == 32)
      mine = fetch_meta_warp<MODE>(c, list, base + ttid, lim);
    else if (ttid < kBatch)
      mine = fetch_meta<MODE>(c, list, base + ttid, lim);
    if constexpr (TEAM > 32) {
      if (ttid < kBatch) s_meta[team][ttid] = mine;
    }
    sync();  // the batch's claims (and fences) before the team's label loads
    const uint32_t nb = min(bsz, count - base);
    // Cross-vertex prefetch (unit weights): the first gather round of the batch's next
    // active vertex is loaded while this one is finished — its targets are requested
    // before this vertex's table inserts, its labels before this vertex's argmax, move
    // and wake-ups — so a team waits on roughly one memory latency per vertex instead
    // of two. (The early reads are a legal asynchronous schedule: the vertex was
    // claimed, and fenced, before any of them.)
    constexpr bool kPF = kPacked<WEIGHTED> && kTeamPrefetch != 0;
    constexpr uint32_t kRound = uint32_t(TEAM) * kTeamU;  // row entries of one gather round
    unsigned act_mask = 0;
    if constexpr (kPF && TEAM == 32) act_mask = __ballot_sync(kFull, mine.act);
    auto next_active = [&](uint32_t v) -> uint32_t {  // first active entry after v, or nb
      if constexpr (TEAM == 32) {
        const unsigned rest = v >= 31 ? 0u : (act_mask & (~0u << (v + 1)));
        return rest ? min(nb, static_cast<uint32_t>(__ffs(rest) - 1)) : nb;
      } else {
        uint32_t k = v + 1;
        while (k < nb && !s_meta[team][k].act) ++k;
        return k;
      }
    };
    uint32_t pf_j[kTeamU], pf_l[kTeamU];
    uint32_t pf_v = nb;  // entry whose first round is in pf_l (nb = none)
    unsigned chg_bits = 0;  // entries of the batch whose label changed
    for (uint32_t v = 0; v < nb; ++v) {
      Meta m;
      if constexpr (TEAM == 32)
        m = shfl_meta(mine, v);
      else
        m = s_meta[team][v];
      if (!m.act) continue;  // uniform over the team
      const uint32_t cap = table_cap<CAP>(m.d);
      // Two team barriers per vertex: after the gather, and inside team_best
      // (which also re-arms the occupancy count for the next vertex; the sweep
      // has cleared the table by then).
      if constexpr (kPF) {
        uint32_t lab0[kTeamU];
        if (pf_v == v && kTeamPrefetch == 2) {
#pragma unroll
          for (int u = 0; u < kTeamU; ++u) {
            const uint32_t e = u * TEAM + ttid;
            lab0[u] = (e < m.d && pf_j[u] != m.i) ? gather_label<MODE>(c, pf_j[u]) : kEmpty;
          }
        } else if (pf_v == v) {
#pragma unroll
          for (int u = 0; u < kTeamU; ++u) lab0[u] = pf_l[u];
        } else {
          round_load<MODE>(c, m, 0, ttid, TEAM, pol, pf_j, lab0);
        }
        // the next vertex's first-round targets, in flight during this vertex's inserts
        pf_v = next_active(v);
        Meta mn{};
        if (pf_v < nb) {
          if constexpr (TEAM == 32)
            mn = shfl_meta(mine, pf_v);
          else
            mn = s_meta[team][pf_v];
#pragma unroll
          for (int u = 0; u < kTeamU; ++u) {
            const uint32_t e = u * TEAM + ttid;
            pf_j[u] = e < mn.d ? ld_stream(c.g.tgt + mn.lo + e, pol) : mn.i;
          }
        }
        {
          const uint32_t wb = ttid & ~31u;
          unsigned live = 0;
#pragma unroll
          for (int u = 0; u < kTeamU; ++u) live |= (wb + u * TEAM < m.d ? 1u : 0u) << u;
          gather_insert_multi<kTeamU, W, DEDUP>(c, lab0, live, tab, cap, occ, &s_occ_n[team], fails);
        }
        if (m.d > kRound)
          team_gather<MODE, W, WEIGHTED, Tab, kTeamU, DEDUP>(c, m.i, m.lo, kRound, m.d, tab, cap, ttid,
                                                               TEAM, pol, occ, &s_occ_n[team], fails);
        // the next vertex's first-round labels, in flight during this vertex's argmax
        if (kTeamPrefetch == 1 && pf_v < nb) {
#pragma unroll
          for (int u = 0; u < kTeamU; ++u) {
            const uint32_t e = u * TEAM + ttid;
            pf_l[u] = (e < mn.d && pf_j[u] != mn.i) ? gather_label<MODE>(c, pf_j[u]) : kEmpty;
          }
        }
      } else {
        team_gather<MODE, W, WEIGHTED, Tab, kTeamU, DEDUP>(c, m.i, m.lo, 0, m.d, tab, cap, ttid, TEAM,
                                                             pol, occ, &s_occ_n[team], fails);
      }
      sync();
      Best<VBits<W>> b = occ_argmax_reset<W>(tab, occ, s_occ_n[team], ttid, TEAM);
      b = team_best<TEAM>(b, s_red[team], ttid, bar, &s_occ_n[team]);
      // Every thread holds b and m.cur, so every thread knows the move (the
      // rule of apply_move_cur); thread 0 writes it.
      const bool changed = b.k != kEmpty && (c.pick_less ? b.k < m.cur : b.k != m.cur);
      if (ttid == 0) {
        apply_move_cur<MODE, false>(c, m.i, b.k, m.cur);
        ++n_v;
        n_e += m.d;
        n_dn += changed;
        if (MODE == kAsync && changed && c.wake) n_w += m.d;
      }
      if (MODE == kAsync && changed) chg_bits |= 1u << v;
    }
    // Async wake-ups of the batch's changed rows, deferred to here: thread 0 fences its
    // label stores once (a18), then the team wakes the rows' neighbours.
    if (MODE == kAsync && c.wake && chg_bits) {
      if (ttid == 0) fence_sc();
      sync();
      if constexpr (TEAM == 32) {
        warp_wake_rows<4>(c.flags, c.g.tgt, mine.lo, mine.d, chg_bits, pol);
      } else {
        for (unsigned bits = chg_bits; bits; bits &= bits - 1) {
          const Meta& mw = s_meta[team][__ffs(bits) - 1];
          wake_row<4>(c.flags, c.g.tgt, mw.lo, 0u, mw.d, ttid, TEAM, pol);
        }
      }
    }
    if constexpr (TEAM > 32) sync();  // s_meta is rewritten by the next batch
  }
  warp_add_counter(c.ctr, C_PROC_V, n_v);
  warp_add_counter(c.ctr, C_PROC_E, n_e);
  warp_add_counter(c.ctr, C_DN, n_dn);
  warp_add_counter(c.ctr, C_WAKE_E, n_w);
  warp_add_counter(c.ctr, C_FAIL, fails);
}

// ---- tier: 8-CTA cluster per vertex, table distributed over DSMEM --------------------
// A thread-block cluster owns one hub at a time (vertices are pulled from a
// work counter). The hub's table is split over the cluster's shared memories:
// slot owner = a second hash of the label, so every label lives in exactly one
// CTA; inserts (and occupancy-list appends) go to the owner's shared memory
// through DSMEM atomics. Each CTA streams 1/8 of the row, sweeps its own
// occupied slots, and rank 0 merges the eight partial argmaxes. No global-memory
// table, no DRAM traffic for aggregation.
__device__ __forceinline__ uint32_t owner_of(uint32_t key) {
  return ((key ^ (key >> 16)) * 0x7FEB352Du) >> (32 - 3);  // 3 = log2(kClusterSize)
}

template <typename Tab>
constexpr size_t cluster_bytes() {
  return size_t(kClusterCap) * Tab::kSlotBytes + size_t(kClusterCap) * sizeof(uint16_t);
}

template <int MODE, typename W, bool WEIGHTED>
__global__ void __cluster_dims__(kClusterSize, 1, 1) __launch_bounds__(kBigThreads)
    k_cluster(PassCtx c, const uint32_t* __restrict__ list, uint32_t count) {
  if (stopped(c.stop)) return;
  namespace cg = cooperative_groups;
  static_assert(kClusterSize == 8, "owner_of assumes 8 ranks");
  using Tab = Table<kPacked<WEIGHTED>, W>;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tab local;
  local.bind(smem_raw, kClusterCap);
  uint16_t* occ = reinterpret_cast<uint16_t*>(smem_raw + size_t(kClusterCap) * Tab::kSlotBytes);
  __shared__ uint32_t s_item;
  __shared__ int s_flag, s_changed;
  __shared__ unsigned s_occ_n;
  __shared__ Best<VBits<W>> red[32];
  __shared__ Best<VBits<W>> part[kClusterSize];
  for (uint32_t s = threadIdx.x; s < kClusterCap; s += blockDim.x) local.clear_slot(s);  // once
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31;
  unsigned long long n_v = 0, n_e = 0, n_dn = 0, n_w = 0, fails = 0;
  for (;;) {
    if (threadIdx.x == 0) {
      s_occ_n = 0;
      if (rank == 0) s_item = atomicAdd(c.work, 1u);
    }
    cl.sync();                                                   // (A) item published
    const uint32_t t = *cl.map_shared_rank(&s_item, 0);
    if (t >= count) break;  // uniform over the cluster; the final sync below keeps rank 0's
                            // shared memory alive until every rank has read s_item
    const uint32_t i = __ldg(list + t);
    if (rank == 0 && threadIdx.x == 0) {
      s_flag = claim_vertex(c, i) ? 1 : 0;
      claim_fence<MODE>(c);
    }
    const uint64_t lo = __ldg(c.g.off + i);
    const uint32_t d = static_cast<uint32_t>(__ldg(c.g.off + i + 1) - lo);
    const uint32_t cap = pow2_ceil(d + d / 3 + 1) / kClusterSize;  // per-rank partition
    cl.sync();                                                   // (B) flag visible
    if (*cl.map_shared_rank(&s_flag, 0)) continue;
    // Stream this rank's slice of the row; warp dedup; insert at the owner rank.
    const uint32_t e0 = static_cast<uint32_t>((uint64_t(d) * rank) / kClusterSize);
    const uint32_t e1 = static_cast<uint32_t>((uint64_t(d) * (rank + 1)) / kClusterSize);
    constexpr int U = 4;
    for (uint32_t base = e0; base < e1; base += blockDim.x * U) {
      uint32_t j[U], lab[U];
      W w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t e = base + u * blockDim.x + threadIdx.x;
        j[u] = e < e1 ? ld_stream(c.g.tgt + lo + e, pol) : i;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t e = base + u * blockDim.x + threadIdx.x;
        const bool valid = e < e1 && j[u] != i;
        lab[u] = valid ? gather_label<MODE>(c, j[u]) : kEmpty;
        w[u] = valid ? edge_weight<W, WEIGHTED>(c.g, lo + e) : W(0);
      }
      const uint32_t wbase = base + (threadIdx.x & ~31u);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (wbase + u * blockDim.x >= e1) break;  // warp-uniform: no edge left for this warp
        const unsigned peers = __match_any_sync(kFull, lab[u]);
        W s;
        if constexpr (WEIGHTED)
          s = peer_sum(w[u], peers);
        else
          s = static_cast<W>(__popc(peers));
        if (lab[u] != kEmpty && (__ffs(peers) - 1) == lane) {
          const uint32_t own = owner_of(lab[u]);
          unsigned char* rbase = cl.map_shared_rank(smem_raw, own);
          Tab remote;
          remote.bind(rbase, kClusterCap);
          uint32_t slot;
          const int r = remote.add(cap, c.strategy, lab[u], s, &slot);
          if (r == 0) {
            ++fails;
          } else if (r == 2) {
            const unsigned pos = atomicAdd(cl.map_shared_rank(&s_occ_n, own), 1u);
            reinterpret_cast<uint16_t*>(rbase + size_t(kClusterCap) * Tab::kSlotBytes)[pos] =
                static_cast<uint16_t>(slot);
          }
        }
      }
    }
    cl.sync();                                                   // (C) all inserts landed
    Best<VBits<W>> b = occ_argmax_reset<W>(local, occ, s_occ_n, threadIdx.x, blockDim.x);
    b = block_best(b, red);
    if (threadIdx.x == 0) *cl.map_shared_rank(&part[rank], 0) = b;
    cl.sync();                                                   // (D) partial argmaxes at rank 0
    if (rank == 0 && threadIdx.x == 0) {
      Best<VBits<W>> f{VBits<W>(0), kEmpty};
      for (int r = 0; r < kClusterSize; ++r) best_merge(f, part[r].v, part[r].k);
      s_changed = apply_move<MODE>(c, i, f.k) ? 1 : 0;
      ++n_v;
      n_e += d;
      n_dn += s_changed;
      if (MODE == kAsync && s_changed && c.wake) n_w += d;
    }
    cl.sync();                                                   // (E) decision visible
    if (MODE == kAsync && c.wake && *cl.map_shared_rank(&s_changed, 0))
      wake_row<4>(c.flags, c.g.tgt, lo, e0, e1, threadIdx.x, blockDim.x, pol);
  }
  cl.sync();
  warp_add_counter(c.ctr, C_PROC_V, n_v);
  warp_add_counter(c.ctr, C_PROC_E, n_e);
  warp_add_counter(c.ctr, C_DN, n_dn);
  warp_add_counter(c.ctr, C_WAKE_E, n_w);
  warp_add_counter(c.ctr, C_FAIL, fails);
}

// ---- tier: wide rows, one 1024-thread CTA per vertex, label-partitioned phases --------
// Rows of kBigMax < d <= kClusterMax (unit weights). The CTA's 16K-slot shared
// table holds at most kWideLimit distinct labels, so a row with more distinct
// labels is aggregated in P phases over a hash partition of the labels: phase 0
// gathers the row, inserts the labels with phase_of(label, P) == 0 and appends every
// other label to its phase's bucket in the CTA's scratch (L2-resident); phase q
// streams bucket q. Each phase sweeps the table into a running (max count, min label)
// and clears it. The argmax over all phases is exact (each label lives in exactly one
// phase). The first pass from identity labels (every label distinct) starts at
// P = ceil(d / kWideLimit); other passes start at P = 1 and double P when the table
// overflows (past kWideBuckets phases the row re-streams an in-order snapshot,
// filtering by phase). No cluster barriers, no remote atomics, and every SM owns its
// own vertex.
#ifndef NULPA_WIDE_LIMIT
#define NULPA_WIDE_LIMIT (NULPA_WIDE_CAP / 4 * 3)
#endif
constexpr uint32_t kWideLimit = NULPA_WIDE_LIMIT;
#ifndef NULPA_WIDE_FRESH_P1
#define NULPA_WIDE_FRESH_P1 0  // 1: the first pass also starts at one phase (overflow vote on)
#endif  // distinct labels per phase (load <= 3/4)

__device__ __forceinline__ uint32_t phase_of(uint32_t key, uint32_t P) {
  const uint32_t h = (key ^ (key >> 16)) * 0x7FEB352Du;
  return static_cast<uint32_t>((static_cast<uint64_t>(h) * P) >> 32);
}

// Phase buckets of the wide tier: bucket q (1 <= q < P) of a P-phase row holds up to
// d labels at scratch + (q - 1) * d, so no label distribution can overfill one.
constexpr uint32_t kWideBuckets = NULPA_WIDE_BUCKETS;  // P <= this is bucketed; larger P re-streams in order
static_assert((kWideBuckets - 1) * uint64_t(kClusterMax) <= kWideScratch,
              "wide scratch holds every bucket layout");

constexpr size_t wide_table_bytes() {
  return size_t(kWideCap) * 8 + size_t(kWideCap) * sizeof(uint16_t);
}
#ifndef NULPA_WIDE_U
#define NULPA_WIDE_U 4
#endif
constexpr uint32_t kWideChunk = kWideThreads * NULPA_WIDE_U;  // row entries per gather round
constexpr uint32_t kWideStage = kWideChunk + 8;  // one TMA stage (widened to 16-byte groups)
// STAGED kernels add two TMA stages of row targets after the table.
constexpr size_t wide_bytes(bool staged = false) {
  return wide_table_bytes() + (staged ? 2 * size_t(kWideStage) * sizeof(uint32_t) : 0);
}

// STAGED: phase 0 streams the row's targets into shared memory with TMA bulk copies,
// two chunks ahead of the label gather (mbarrier per stage). PREFETCH: the labels of
// round r + 1 are gathered before round r is inserted, so the dependent label loads are
// in flight while the table atomics of the previous round run.
// DEEP (with PREFETCH, not STAGED): the targets of round r + 2 are loaded while round r is
// inserted, so the label gather of round r + 1 never waits on its targets.
template <int MODE, typename W, bool STAGED = true, bool PREFETCH = true, bool DEEP = false>
__global__ void __launch_bounds__(kWideThreads, kWideCtasPerSm) k_wide(PassCtx c, const uint32_t* __restrict__ list,
                                                         uint32_t count, int fresh,
                                                         uint32_t* __restrict__ scratch,
                                                         uint32_t stride, uint64_t m2,
                                                         uint32_t* __restrict__ hint) {
  if (stopped(c.stop)) return;
  // This CTA's row snapshot / phase buckets (L2-resident): phase 0 of a multi-phase
  // vertex writes the labels of later phases here; those phases stream them back.
  uint32_t* snap = scratch + size_t(blockIdx.x) * stride;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemTable<W> tab;
  tab.bind(smem_raw, kWideCap);
  uint16_t* occ = reinterpret_cast<uint16_t*>(smem_raw + size_t(kWideCap) * 8);
  uint32_t* stage = reinterpret_cast<uint32_t*>(smem_raw + wide_table_bytes());
  __shared__ uint32_t s_item;
  __shared__ int s_flag, s_over;
  __shared__ unsigned s_occ_n;
  __shared__ unsigned s_bcnt[kWideBuckets];
  __shared__ Best<VBits<W>> red[32];
  __shared__ __align__(8) uint64_t s_bar[2];
  constexpr uint32_t kWideBatch = 4;  // vertices per work-counter fetch (batched prologue)
  __shared__ Meta s_meta[kWideBatch];
  for (uint32_t x = threadIdx.x; x < kWideCap; x += blockDim.x) tab.clear_slot(x);  // once
  if (STAGED && threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_init_fence();
  }
  const uint64_t pol = policy_evict_first();
  unsigned long long n_v = 0, n_e = 0, n_dn = 0, n_w = 0, fails = 0;
  constexpr int U = NULPA_WIDE_U;  // gather rounds in flight per thread
  constexpr uint32_t CH = kWideChunk;
  uint32_t par = 0;  // phase parity of each TMA stage (bit b), identical in every thread
  // The 16-byte-group window [a0, a1) of chunk k of the row at `lo` (degree d) that a
  // bulk copy can move; entries past m2 & ~3 (the array's last partial group) are read
  // from global memory instead.
  auto window = [&](uint64_t lo, uint32_t d, uint32_t k, uint64_t& a0, uint64_t& a1) {
    const uint64_t g0 = lo + uint64_t(k) * CH;
    const uint64_t g1 = lo + min(uint64_t(d), uint64_t(k + 1) * CH);
    a0 = g0 & ~3ull;
    a1 = min((g1 + 3) & ~3ull, m2 & ~3ull);
  };
  auto issue = [&](uint64_t lo, uint32_t d, uint32_t k) {  // thread 0 only
    uint64_t a0, a1;
    window(lo, d, k, a0, a1);
    uint64_t* bar = &s_bar[k & 1];
    if (a1 > a0)
      tma_load_1d(stage + (k & 1) * kWideStage, c.g.tgt + a0, static_cast<uint32_t>(a1 - a0) * 4u,
                  bar, pol);
    else
      mbar_arrive(bar);
  };
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(c.work, kWideBatch);
    __syncthreads();
    const uint32_t t0 = s_item;
    if (t0 >= count) break;
    if (threadIdx.x < kWideBatch) s_meta[threadIdx.x] = fetch_meta<MODE>(c, list, t0 + threadIdx.x, count);
    __syncthreads();
    const uint32_t nb = min(kWideBatch, count - t0);
    for (uint32_t vb = 0; vb < nb; ++vb) {
    const Meta m = s_meta[vb];
    if (!m.act) continue;  // (uniform; s_meta is rewritten only after the next fetch barrier)
    const uint32_t i = m.i;
    const uint64_t lo = m.lo;
    const uint32_t d = m.d;
    // Phases: from identity labels every label is distinct, P = ceil(d / limit). Later
    // passes start from the distinct-label count the row held in its previous pass (labels
    // only merge as a run goes on), so neither the per-round overflow vote nor a restart is
    // needed unless the row is near the limit (or has no history: P = 1 with the vote).
    const uint32_t h = (fresh || !c.hints) ? 0u : hint[t0 + vb];
    uint32_t P = (fresh && !NULPA_WIDE_FRESH_P1) ? (d + kWideLimit - 1) / kWideLimit
                                                 : max(1u, (h + kWideLimit - 1) / kWideLimit);
    const bool known = !fresh && h != 0u && h <= kWideLimit / 2;  // far below the limit: no vote
    uint32_t distinct = 0;  // (thread 0) labels aggregated over the phases of this row
    // Bucketed phases: phase 0 gathers the row once and appends every label of a
    // later phase to that phase's bucket in the CTA's L2 scratch, so phase q > 0
    // streams only its own labels (d label reads in all, not P * d).
    Best<VBits<W>> best{VBits<W>(0), kEmpty};  // running result (thread 0)
    for (uint32_t ph = 0; ph < P; ++ph) {
      const bool use_b = P > 1 && P <= kWideBuckets;
      if (threadIdx.x == 0) {
        s_occ_n = 0;
        s_over = 0;
        if (ph == 0)
          for (uint32_t b = 0; b < kWideBuckets; ++b) s_bcnt[b] = 0;
      }
      __syncthreads();
      // A phase can only overflow when it may hold more than kWideLimit labels.
      const uint32_t len = (use_b && ph > 0) ? s_bcnt[ph] : d;
      const uint32_t nch = (len + CH - 1) / CH;
      // Early stop (a per-round block vote) only where a row may hold more distinct
      // labels than the phase takes and the phase re-streams the whole row. Bucketed
      // phases run to the end: a full table (rare) still flags s_over and restarts.
      const bool may_overflow = !use_b && !known && (len > kWideLimit || P > 1);
      const uint32_t cap = P == 1 ? min(static_cast<uint32_t>(kWideCap), pow2_ceil(2 * d))
                                  : static_cast<uint32_t>(kWideCap);
      const uint32_t* src = use_b ? snap + size_t(ph - 1) * d : snap;
      const bool from_row = ph == 0;  // phase 0 gathers targets -> labels; later phases stream labels
      if (STAGED && from_row && threadIdx.x == 0 && nch > 0) {
        issue(lo, d, 0);
        if (nch > 1) issue(lo, d, 1);
      }
      uint32_t jq[U];  // DEEP: the targets of the next round to gather
      auto load_targets = [&](uint32_t k) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t e = k * CH + u * kWideThreads + threadIdx.x;
          jq[u] = e < d ? ld_stream(c.g.tgt + lo + e, pol) : i;
        }
      };
      if (DEEP && from_row && nch > 0) load_targets(0);
      // Gather round k into lab[] (issues the loads; the values are consumed later).
      auto gather = [&](uint32_t k, uint32_t (&lab)[U]) {
        const uint32_t base = k * CH;
        if (DEEP && from_row) {
#pragma unroll
          for (int u = 0; u < U; ++u) lab[u] = jq[u] != i ? gather_label<MODE>(c, jq[u]) : kEmpty;
          if (k + 1 < nch) load_targets(k + 1);
        } else if (from_row) {
          uint32_t j[U];
          if constexpr (STAGED) {
            const uint32_t b = k & 1;
            mbar_wait(&s_bar[b], (par >> b) & 1u);
            par ^= 1u << b;
            uint64_t a0, a1;
            window(lo, d, k, a0, a1);
            const uint32_t* buf = stage + b * kWideStage;
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t e = base + u * kWideThreads + threadIdx.x;
              const uint64_t gi = lo + e;
              j[u] = e < d ? (gi < a1 ? buf[gi - a0] : ld_stream(c.g.tgt + gi, pol)) : i;
            }
          } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t e = base + u * kWideThreads + threadIdx.x;
              j[u] = e < d ? ld_stream(c.g.tgt + lo + e, pol) : i;
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) lab[u] = j[u] != i ? gather_label<MODE>(c, j[u]) : kEmpty;
          if constexpr (STAGED) {
            __syncthreads();  // every thread has read stage k & 1: refill it with chunk k + 2
            if (threadIdx.x == 0 && k + 2 < nch) issue(lo, d, k + 2);
          }
        } else {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t e = base + u * kWideThreads + threadIdx.x;
            lab[u] = e < len ? __ldcg(src + e) : kEmpty;
          }
        }
      };
      uint32_t cur[U], nxt[U];
      if (nch > 0) gather(0, cur);
      uint32_t k = 0;
      for (; k < nch; ++k) {
        if (PREFETCH && k + 1 < nch) gather(k + 1, nxt);
        const uint32_t base = k * CH;
        if (from_row) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t e = base + u * kWideThreads + threadIdx.x;
            if (P > 1 && !use_b && e < d) snap[e] = cur[u];
          }
          if (use_b) {
            const int lane = threadIdx.x & 31;
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t q = cur[u] != kEmpty ? phase_of(cur[u], P) : 0u;
              const unsigned peers = __match_any_sync(kFull, q);
              unsigned at = 0;
              const int leader = __ffs(peers) - 1;
              if (q != 0 && lane == leader) at = atomicAdd(&s_bcnt[q], __popc(peers));
              at = __shfl_sync(kFull, at, leader) + __popc(peers & ((1u << lane) - 1u));
              if (q != 0) {
                snap[size_t(q - 1) * d + at] = cur[u];
                cur[u] = kEmpty;
              }
            }
          }
        }
        if (!use_b) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (P > 1 && cur[u] != kEmpty && phase_of(cur[u], P) != ph) cur[u] = kEmpty;
        }
        const uint32_t wbase = base + (threadIdx.x & ~31u);
        unsigned live = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) live |= (wbase + u * kWideThreads < len ? 1u : 0u) << u;
        unsigned long long f = 0;
        gather_insert_multi<U, W, 0>(c, cur, live, tab, cap, occ, &s_occ_n, f);
        if (f) s_over = 1;  // table full: treat as overflow
        // Stop early once the phase holds too many distinct labels: one barrier
        // with a block-wide OR (uniform result). Thread 0's read of the occupancy
        // count may miss appends still in flight; the vote is a heuristic, while
        // exactness rests on s_over (a failed insert) alone.
        if (may_overflow) {
          const unsigned occ_now = *static_cast<volatile unsigned*>(&s_occ_n);
          if (__syncthreads_or(f != 0 || (threadIdx.x == 0 && occ_now > kWideLimit))) {
            if (threadIdx.x == 0) s_over = 1;
            break;
          }
        }
        if (k + 1 < nch) {
          if constexpr (!PREFETCH) gather(k + 1, nxt);
#pragma unroll
          for (int u = 0; u < U; ++u) cur[u] = nxt[u];
        }
      }
      if (STAGED && from_row) {
        // an early stop leaves issued chunks unconsumed: complete their phases so every
        // stage's parity stays in step (chunks k+1 .. min(nch-1, g+2) for the last
        // gathered round g = k + PREFETCH)
        const uint32_t g = PREFETCH ? min(k + 1, nch - 1) : k;
        for (uint32_t q = g + 1; q < nch && q <= g + 2; ++q) {
          mbar_wait(&s_bar[q & 1], (par >> (q & 1)) & 1u);
          par ^= 1u << (q & 1);
        }
      }
      __syncthreads();
      const bool over = s_over != 0;  // (a bucketed phase 0 past kWideLimit is still exact)
      if (threadIdx.x == 0) distinct += s_occ_n;
      Best<VBits<W>> b = occ_argmax_reset<W>(tab, occ, s_occ_n, threadIdx.x, blockDim.x);
      b = block_best(b, red);  // (ends with a barrier: the table is clear again)
      if (over) {
        // restart with twice as many phases (at least enough for all-distinct rows)
        P = max(2 * P, (d + kWideLimit - 1) / kWideLimit);
        ph = static_cast<uint32_t>(-1);
        best = Best<VBits<W>>{VBits<W>(0), kEmpty};
        distinct = 0;
        continue;
      }
      if (threadIdx.x == 0) best_merge(best, b.v, b.k);
    }
    if (threadIdx.x == 0) {
      hint[t0 + vb] = max(distinct, 1u);
      s_flag = apply_move_cur<MODE>(c, i, best.k, m.cur) ? 1 : 0;
      ++n_v;
      n_e += d;
      n_dn += s_flag;
      if (MODE == kAsync && s_flag && c.wake) n_w += d;
    }
    __syncthreads();
    if (MODE == kAsync && c.wake && s_flag) wake_row<4>(c.flags, c.g.tgt, lo, 0u, d, threadIdx.x, blockDim.x, pol);
    __syncthreads();
    }
  }
  warp_add_counter(c.ctr, C_PROC_V, n_v);
  warp_add_counter(c.ctr, C_PROC_E, n_e);
  warp_add_counter(c.ctr, C_DN, n_dn);
  warp_add_counter(c.ctr, C_WAKE_E, n_w);
  warp_add_counter(c.ctr, C_FAIL, fails);
}

// ---- first pass from identity labels -------------------------------------------------
// run_engine starts from labels[i] = i (lpa.cpp:250). On a graph whose rows hold
// distinct, ascending targets with unit weights, every neighbour label then
// occurs exactly once, so scan_candidate's argmax (all counts 1, ties to the
// smaller key) is simply the smallest neighbour id other than i: the first or
// second entry of the sorted row. The pass needs no table at all. Synchronous
// mode gets the reference's exact first pass; ParallelAsync gets the legal
// schedule in which every first-pass read precedes every write.
template <int MODE>
__global__ void __launch_bounds__(256) k_first_pass(PassCtx c, uint32_t v_lo, uint32_t v_hi) {
  unsigned long long n_v = 0, n_e = 0, n_dn = 0, n_w = 0;
  const uint32_t bound = v_lo + ((v_hi - v_lo + 31u) & ~31u);
  for (uint32_t i = v_lo + blockIdx.x * blockDim.x + threadIdx.x; i < bound;
       i += gridDim.x * blockDim.x) {
    if (i >= v_hi) continue;
    if (claim_vertex(c, i)) continue;
    const uint64_t lo = __ldg(c.g.off + i);
    const uint32_t d = static_cast<uint32_t>(__ldg(c.g.off + i + 1) - lo);
    if (d == 0) continue;
    uint32_t cand = __ldg(c.g.tgt + lo);
    if (cand == i) cand = d > 1 ? __ldg(c.g.tgt + lo + 1) : kEmpty;  // self-loop skipped
    if (cand != kEmpty) cand = vertex_id(c.vid, cand);  // rows keep the input's in-row order
    const uint32_t own = vertex_id(c.vid, i);           // identity labels: label = vertex id
    ++n_v;
    n_e += d > 1 ? 2 : 1;
    const bool allowed = cand != kEmpty && (c.pick_less ? cand < own : cand != own);
    if (!allowed) continue;
    c.lab_out[i] = cand;
    ++n_dn;
    if (MODE == kSync && c.changed) c.changed[atomicAdd(c.changed_n, 1ull)] = i;
    if (MODE == kAsync && c.wake) {
      fence_sc();  // the label store before the wake loads (a18)
      wake_row<4>(c.flags, c.g.tgt, lo, 0u, d, 0u, 1u, policy_evict_first());
      n_w += d;
    }
  }
  warp_add_counter(c.ctr, C_PROC_V, n_v);
  warp_add_counter(c.ctr, C_PROC_E, n_e);
  warp_add_counter(c.ctr, C_DN, n_dn);
  warp_add_counter(c.ctr, C_WAKE_E, n_w);
}

// The same table-free rule over a tier list (used for the long-row tiers at the
// start of a ParallelAsync run: they are processed first, all of them reading
// identity labels, before the lower tiers run in place).
template <int MODE>
__global__ void __launch_bounds__(256) k_first_pass_list(PassCtx c, const uint32_t* __restrict__ list,
                                                         uint32_t count) {
  unsigned long long n_v = 0, n_e = 0, n_dn = 0;
  const uint32_t bound = (count + 31u) & ~31u;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < bound; t += gridDim.x * blockDim.x) {
    if (t >= count) continue;
    const uint32_t i = __ldg(list + t);
    if (claim_vertex(c, i)) continue;
    const uint64_t lo = __ldg(c.g.off + i);
    const uint32_t d = static_cast<uint32_t>(__ldg(c.g.off + i + 1) - lo);
    if (d == 0) continue;
    uint32_t cand = __ldg(c.g.tgt + lo);
    if (cand == i) cand = d > 1 ? __ldg(c.g.tgt + lo + 1) : kEmpty;  // self-loop skipped
    if (cand != kEmpty) cand = vertex_id(c.vid, cand);
    const uint32_t own = vertex_id(c.vid, i);
    ++n_v;
    n_e += d > 1 ? 2 : 1;
    const bool allowed = cand != kEmpty && (c.pick_less ? cand < own : cand != own);
    if (!allowed) continue;
    c.lab_out[i] = cand;
    ++n_dn;
  }
  warp_add_counter(c.ctr, C_PROC_V, n_v);
  warp_add_counter(c.ctr, C_PROC_E, n_e);
  warp_add_counter(c.ctr, C_DN, n_dn);
}

// ---- tier: hubs, global tables -------------------------------------------------------

template <int MODE>
__global__ void k_hub_select(PassCtx c, HubCtx h) {
  if (stopped(c.stop)) return;
  unsigned long long n_v = 0, n_e = 0;
  const uint32_t bound = (h.n_hubs + 31u) & ~31u;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < bound;
       x += gridDim.x * blockDim.x) {
    if (x >= h.n_hubs) continue;
    const uint32_t i = h.hub_v[x];
    const bool skip = claim_vertex(c, i);
    h.active[x] = skip ? 0 : 1;
    if (!skip) {
      ++n_v;
      n_e += c.g.off[i + 1] - c.g.off[i];
    }
  }
  warp_add_counter(c.ctr, C_PROC_V, n_v);
  warp_add_counter(c.ctr, C_PROC_E, n_e);
}

template <typename Tab, typename W, bool PACKED>
__device__ __forceinline__ void bind_hub_table(Tab& g, const HubCtx& h, uint32_t x) {
  if constexpr (PACKED)
    g.bind_split(static_cast<unsigned long long*>(h.tab) + h.tab_off[x], nullptr);
  else
    g.bind_split(static_cast<uint32_t*>(h.tab) + h.tab_off[x],
                 static_cast<W*>(h.tab_vals) + h.tab_off[x]);
}

// Accumulate one (hub, chunk) item: pre-aggregate the chunk in shared memory,
// then flush each distinct label once into the hub's global table (swept densely
// afterwards by k_hub_sweep).
#ifndef NULPA_FLUSH_U
#define NULPA_FLUSH_U 4
#endif
template <int MODE, typename W, bool WEIGHTED, int DEDUP = 1>
__global__ void __launch_bounds__(kBlockThreads) k_hub_accum(PassCtx c, HubCtx h) {
  if (stopped(c.stop)) return;
  using Tab = std::conditional_t<kPacked<WEIGHTED>, SmemTable<W>, Table<false, W>>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned s_occ_n;
  Tab tab;
  tab.bind(smem_raw, kHubCap);
  // The chunk table is kept empty between items: its occupied slots are listed
  // (as in the team tables) and the flush reads and resets only those.
  uint16_t* socc = reinterpret_cast<uint16_t*>(smem_raw + size_t(kHubCap) * Tab::kSlotBytes);
  for (uint32_t s = threadIdx.x; s < kHubCap; s += blockDim.x) tab.clear_slot(s);  // once
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31;
  unsigned long long fails = 0;
  for (uint32_t it = blockIdx.x; it < h.n_items; it += gridDim.x) {
    const uint32_t x = h.item_hub[it];
    if (!h.active[x]) continue;  // uniform across the CTA
    const uint32_t i = h.hub_v[x];
    const uint64_t lo = __ldg(c.g.off + i);
    const uint32_t d = static_cast<uint32_t>(__ldg(c.g.off + i + 1) - lo);
    const uint32_t e0 = h.item_start[it];
    const uint32_t e1 = min(d, e0 + kHubChunk);
    const uint32_t cap = kHubCap;
    if (threadIdx.x == 0) s_occ_n = 0;
    __syncthreads();
    team_gather<MODE, W, WEIGHTED, Tab, kTeamU, DEDUP>(c, i, lo, e0, e1, tab, cap, threadIdx.x,
                                                      blockDim.x, pol, socc, &s_occ_n, fails);
    __syncthreads();
    Table<kPacked<WEIGHTED>, W> g;  // the hub's global table (swept densely, k_hub_sweep)
    bind_hub_table<Table<kPacked<WEIGHTED>, W>, W, kPacked<WEIGHTED>>(g, h, x);
    const uint32_t gcap = h.tab_cap[x];
    const uint32_t n_occ = s_occ_n;
    uint32_t p0 = 0;
    if constexpr (kPacked<WEIGHTED>) {
      // Packed (unit-weight) tables: kFlushU claims in flight per thread. Each is a
      // CAS of (key, count) into the label's first slot, which either claims it or
      // returns the resident key (then one fire-and-forget add); only a collision
      // takes the probe walk.
      constexpr uint32_t kFlushU = NULPA_FLUSH_U;
      const uint32_t mask = gcap - 1;
      for (; p0 + kFlushU * blockDim.x <= n_occ; p0 += kFlushU * blockDim.x) {
        uint32_t sl[kFlushU], key[kFlushU], cnt[kFlushU];
        unsigned long long old[kFlushU];
#pragma unroll
        for (uint32_t u = 0; u < kFlushU; ++u) {
          sl[u] = socc[p0 + u * blockDim.x + threadIdx.x];
          VBits<W> vb;
          tab.read(sl[u], key[u], vb);
          cnt[u] = static_cast<uint32_t>(tab.value(sl[u]));
        }
#pragma unroll
        for (uint32_t u = 0; u < kFlushU; ++u)
          old[u] = atomicCAS(g.w + (hash_start(key[u], gcap) & mask), kEmptyWord,
                             (static_cast<unsigned long long>(key[u]) << 32) | cnt[u]);
#pragma unroll
        for (uint32_t u = 0; u < kFlushU; ++u) {
          if (old[u] != kEmptyWord) {
            if (static_cast<uint32_t>(old[u] >> 32) == key[u]) {
              atomicAdd(g.w + (hash_start(key[u], gcap) & mask),
                        static_cast<unsigned long long>(cnt[u]));
            } else {
              uint32_t gslot;
              if (g.add(gcap, c.strategy, key[u], W(cnt[u]), &gslot) == 0) ++fails;
            }
          }
          tab.clear_slot(sl[u]);
        }
      }
    }
    for (uint32_t p = p0 + threadIdx.x; p < n_occ; p += blockDim.x) {
      const uint32_t sl = socc[p];
      uint32_t k;
      VBits<W> vb;
      tab.read(sl, k, vb);
      uint32_t gslot;
      if (g.add(gcap, c.strategy, k, tab.value(sl), &gslot) == 0) ++fails;
      tab.clear_slot(sl);
    }
    __syncthreads();
  }
  warp_add_counter(c.ctr, C_FAIL, fails);
}

// Dense argmax over each active hub's table, (hub, kHubSweep-slot) items: the
// slots are read and reset in order (coalesced), so a pass costs two streams over
// the hub tables instead of one random access per distinct label (the first pass
// from identity labels fills the tables with ~one label per edge).
template <typename W, bool WEIGHTED>
__global__ void __launch_bounds__(kBlockThreads) k_hub_sweep(HubCtx h) {
  if (stopped(h.stop)) return;
  using Tab = Table<kPacked<WEIGHTED>, W>;
  __shared__ Best<VBits<W>> red[32];
  for (uint32_t it = blockIdx.x; it < h.n_sitems; it += gridDim.x) {
    const uint32_t x = h.sitem_hub[it];
    if (!h.active[x]) continue;  // (uniform) untouched tables stay empty
    const uint32_t s0 = h.sitem_start[it];
    const uint32_t s1 = min(h.tab_cap[x], s0 + kHubSweep);
    Tab g;
    bind_hub_table<Tab, W, kPacked<WEIGHTED>>(g, h, x);
    Best<VBits<W>> b{VBits<W>(0), kEmpty};
    for (uint32_t sl = s0 + threadIdx.x; sl < s1; sl += blockDim.x) {
      uint32_t k;
      VBits<W> v;
      g.read(sl, k, v);
      if (k == kEmpty) continue;
      best_merge(b, v, k);
      if constexpr (sizeof(VBits<W>) == 4) g.clear_slot(sl);
    }
    b = block_best(b, red);
    if (threadIdx.x == 0 && b.k != kEmpty) {
      if constexpr (sizeof(VBits<W>) == 4) {
        // (value bits, ~key): a larger value wins, then a smaller key.
        atomicMax(h.best + x, (static_cast<unsigned long long>(b.v) << 32) |
                                  static_cast<unsigned long long>(~b.k));
      } else {
        atomicMax(h.best + x, static_cast<unsigned long long>(__double_as_longlong(b.v)));
      }
    }
    __syncthreads();
  }
}

// fp64 values only: the smallest key among slots holding the maximum value (dense,
// like k_hub_sweep); resets the slots. PACKED = unit weights, where the hub table is
// (key << 32 | count) words; otherwise split key / double arrays.
template <bool PACKED>
__global__ void __launch_bounds__(kBlockThreads) k_hub_sweep_key_f64(HubCtx h) {
  if (stopped(h.stop)) return;
  using Tab = Table<PACKED, double>;
  for (uint32_t it = blockIdx.x; it < h.n_sitems; it += gridDim.x) {
    const uint32_t x = h.sitem_hub[it];
    if (!h.active[x]) continue;
    const uint32_t s0 = h.sitem_start[it];
    const uint32_t s1 = min(h.tab_cap[x], s0 + kHubSweep);
    Tab g;
    bind_hub_table<Tab, double, PACKED>(g, h, x);
    const double bestv = __longlong_as_double(static_cast<long long>(h.best[x]));
    for (uint32_t sl = s0 + threadIdx.x; sl < s1; sl += blockDim.x) {
      uint32_t k;
      double v;
      g.read(sl, k, v);
      if (k == kEmpty) continue;
      if (v == bestv) atomicMin(h.best_k + x, k);
      g.clear_slot(sl);
    }
  }
}

template <int MODE, typename W, bool WEIGHTED>
__global__ void k_hub_decide(PassCtx c, HubCtx h) {
  if (stopped(c.stop)) return;
  unsigned long long n_dn = 0;
  const uint32_t bound = (h.n_hubs + 31u) & ~31u;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < bound;
       x += gridDim.x * blockDim.x) {
    if (x >= h.n_hubs) continue;
    uint8_t ch = 0;
    if (h.active[x]) {
      uint32_t cand = kEmpty;  // stays kEmpty when the row held only self-loops
      if constexpr (sizeof(VBits<W>) == 4) {
        if (h.best[x] != 0) cand = ~static_cast<uint32_t>(h.best[x] & 0xFFFFFFFFull);
      } else {
        cand = h.best_k[x];
      }
      ch = apply_move<MODE>(c, h.hub_v[x], cand) ? 1 : 0;
      n_dn += ch;
    }
    h.changed[x] = ch;
    h.best[x] = 0;
    h.best_k[x] = kEmpty;
  }
  warp_add_counter(c.ctr, C_DN, n_dn);
}

// Async wake for changed hubs, one chunk per work item.
__global__ void __launch_bounds__(kBlockThreads) k_hub_wake(PassCtx c, HubCtx h) {
  if (stopped(c.stop)) return;
  unsigned long long n_w = 0;
  const uint64_t pol = policy_evict_first();
  for (uint32_t it = blockIdx.x; it < h.n_items; it += gridDim.x) {
    const uint32_t x = h.item_hub[it];
    if (!h.changed[x]) continue;
    const uint32_t i = h.hub_v[x];
    const uint64_t lo = c.g.off[i];
    const uint32_t d = static_cast<uint32_t>(c.g.off[i + 1] - lo);
    const uint32_t e0 = h.item_start[it];
    const uint32_t e1 = min(d, e0 + kHubChunk);
    wake_row<4>(c.flags, c.g.tgt, lo, e0, e1, threadIdx.x, blockDim.x, pol);
    if (threadIdx.x == 0) n_w += e1 - e0;
  }
  warp_add_counter(c.ctr, C_WAKE_E, n_w);
}

// ---- sync-mode deferred wake (lpa.cpp:97-98) -----------------------------------------

__global__ void __launch_bounds__(kBlockThreads) k_wake_list(Graph g, uint8_t* flags,
                                                             const uint32_t* list,
                                                             const unsigned long long* count_p,
                                                             unsigned long long* ctr,
                                                             const unsigned* stop = nullptr) {
  if (stopped(stop)) return;
  const uint32_t count = static_cast<uint32_t>(*count_p);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + warp, nw = gridDim.x * (blockDim.x >> 5);
  unsigned long long n_w = 0;
  for (uint32_t t = gw; t < count; t += nw) {
    const uint32_t i = list[t];
    const uint64_t lo = g.off[i], hi = g.off[i + 1];
    wake_row<4>(flags, g.tgt, lo, 0u, static_cast<uint32_t>(hi - lo), lane, 32u, policy_evict_first());
    if (lane == 0) n_w += hi - lo;
  }
  warp_add_counter(ctr, C_WAKE_E, n_w);
}

// ---- Sequential mode (lpa_move, lpa.hpp:123-145) -----------------------------------------
// One CTA walks the vertices in ascending id order with in-place updates; each
// vertex's scan is CTA-parallel. Exact reference semantics on the GPU (no CPU
// fallback); slow by construction — a compatibility mode, not the hot path.
template <typename W, bool WEIGHTED>
__global__ void __launch_bounds__(kBlockThreads) k_sequential(PassCtx c, void* gtab) {
  using Tab = Table<kPacked<WEIGHTED>, W>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Best<VBits<W>> red[32];
  __shared__ int s_flag;
  unsigned long long n_v = 0, n_e = 0, n_dn = 0, n_w = 0, fails = 0;
  for (uint32_t v = 0; v < c.g.n; ++v) {
    const uint32_t i = position_of(c.pos, v);  // ascending vertex id (lpa.hpp:129)
    if (threadIdx.x == 0) {
      int skip = 1;
      if (!c.flags[i]) {
        c.flags[i] = 1;
        skip = (c.g.off[i + 1] == c.g.off[i]) ? 1 : 0;
      }
      s_flag = skip;
    }
    __syncthreads();
    const int skip = s_flag;
    __syncthreads();
    if (skip) continue;
    const uint64_t lo = c.g.off[i];
    const uint32_t d = static_cast<uint32_t>(c.g.off[i + 1] - lo);
    const uint32_t cap = pow2_ceil(2 * d);
    Tab tab;
    if (cap <= static_cast<uint32_t>(kHubCap))
      tab.bind(smem_raw, kHubCap);
    else
      tab.bind(gtab, cap);
    for (uint32_t s = threadIdx.x; s < cap; s += blockDim.x) tab.clear_slot(s);
    __syncthreads();
    if constexpr (WEIGHTED) {
      // Each label's weights are added in neighbour order, one rounding at a time,
      // as the reference's plain accumulation does (hashtable.hpp:119-125): warp 0
      // walks the row in 32-edge chunks; the lowest lane of each label group claims
      // (or finds) the slot with its own weight, then adds its peers' weights in
      // ascending lane order. Different labels touch different slots.
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        for (uint32_t base = 0; base < d; base += 32) {
          const uint32_t e = base + lane;
          const uint32_t j = e < d ? c.g.tgt[lo + e] : i;
          const bool valid = e < d && j != i;
          const uint32_t lab = valid ? c.lab_out[j] : kEmpty;
          const W w = valid ? edge_weight<W, WEIGHTED>(c.g, lo + e) : W(0);
          const unsigned peers = __match_any_sync(kFull, lab);
          const bool lead = lab != kEmpty && (__ffs(peers) - 1) == lane;
          uint32_t slot = 0;
          if (lead && tab.add(cap, c.strategy, lab, w, &slot) == 0) ++fails;
          W acc = lead ? tab.value(slot) : W(0);
          for (int b = 0; b < 32; ++b) {
            const W wb = __shfl_sync(kFull, w, b);
            if (lead && b != lane && ((peers >> b) & 1u)) acc += wb;
          }
          if (lead) tab.v[slot] = acc;
          __syncwarp();
        }
      }
    } else {
      for (uint32_t base = 0; base < d; base += blockDim.x) {
        const uint32_t e = base + threadIdx.x;
        const uint32_t j = e < d ? c.g.tgt[lo + e] : i;
        const bool valid = e < d && j != i;
        const uint32_t lab = valid ? c.lab_out[j] : kEmpty;
        gather_insert<W, WEIGHTED>(c, lab, W(1), tab, cap, nullptr, nullptr, fails);
      }
    }
    __syncthreads();
    Best<VBits<W>> b{VBits<W>(0), kEmpty};
    for (uint32_t s = threadIdx.x; s < cap; s += blockDim.x) {
      uint32_t k;
      VBits<W> v;
      tab.read(s, k, v);
      best_merge(b, v, k);
    }
    b = block_best(b, red);
    if (threadIdx.x == 0) {
      int ch = 0;
      if (b.k != kEmpty) {
        const uint32_t cur = c.lab_out[i];
        if (c.pick_less ? (b.k < cur) : (b.k != cur)) {
          c.lab_out[i] = b.k;
          ch = 1;
        }
      }
      s_flag = ch;
      ++n_v;
      n_e += d;
      n_dn += ch;
    }
    __syncthreads();
    if (s_flag) {
      for (uint32_t e = threadIdx.x; e < d; e += blockDim.x) c.flags[c.g.tgt[lo + e]] = 0;
      if (threadIdx.x == 0) n_w += d;
    }
    __syncthreads();
  }
  warp_add_counter(c.ctr, C_PROC_V, n_v);
  warp_add_counter(c.ctr, C_PROC_E, n_e);
  warp_add_counter(c.ctr, C_DN, n_dn);
  warp_add_counter(c.ctr, C_WAKE_E, n_w);
  warp_add_counter(c.ctr, C_FAIL, fails);
}

// ---- cross-check (lpa.cpp:338-360) ---------------------------------------------------------
// The reference scans i ascending and reads labels[c*] (c* < i) after earlier
// reverts. revert(i) = changed(i) && i > c_i && final(c_i) != c_i with
// final(v) = revert(v) ? prev[v] : lab[v]: a recursion on strictly smaller ids,
// solved by Jacobi rounds until no flag moves (depth-bounded).
// Arrays are in position order; label values (and the i > c* rule) are vertex ids.
__global__ void k_cc_round(const uint32_t* lab, const uint32_t* prev, const uint8_t* r_in,
                           uint8_t* r_out, uint32_t n, unsigned long long* moved,
                           const uint32_t* vid, const uint32_t* pos) {
  unsigned long long mv = 0;
  const uint32_t bound = (n + 31u) & ~31u;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < bound;
       i += gridDim.x * blockDim.x) {
    if (i >= n) continue;
    const uint32_t ci = lab[i];
    uint8_t r = 0;
    if (ci != prev[i] && vertex_id(vid, i) > ci) {
      const uint32_t pc = position_of(pos, ci);
      const uint32_t fc = r_in[pc] ? prev[pc] : lab[pc];
      r = fc != ci ? 1 : 0;
    }
    if (r != r_in[i]) ++mv;
    r_out[i] = r;
  }
  warp_add_counter(moved, 0, mv);
}

__global__ void k_cc_apply(Graph g, uint32_t* lab, const uint32_t* prev, const uint8_t* r,
                           uint8_t* flags, unsigned long long* reverted) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + warp, nw = gridDim.x * (blockDim.x >> 5);
  unsigned long long nrev = 0;
  // Warp-per-32-vertex blocks so the neighbour wake is warp-cooperative.
  for (uint32_t base = gw * 32; base < g.n; base += nw * 32) {
    const uint32_t i = base + lane;
    unsigned mine = (i < g.n && r[i]) ? 1u : 0u;
    if (mine) {
      lab[i] = prev[i];
      flags[i] = 0;
      ++nrev;
    }
    unsigned m = __ballot_sync(kFull, mine);
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t v = base + b;
      const uint64_t lo = g.off[v], hi = g.off[v + 1];
      wake_row<4>(flags, g.tgt, lo, 0u, static_cast<uint32_t>(hi - lo), lane, 32u, policy_evict_first());
    }
  }
  warp_add_counter(reverted, 0, nrev);
}

}  // namespace dev
}  // namespace nulpa
