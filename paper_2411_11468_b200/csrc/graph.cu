// Device CSR residency and the per-graph execution plan (degree tiers).
//
// CsrGraph (graph.hpp:53-84, graph.cpp:165-178) becomes a device-resident
// structure: offsets u64[n+1], targets u32[m2], weights f32[m2] — weights are
// elided when every weight is 1.0f, so unit-weight graphs move 8 bytes per
// scanned edge instead of 12. partition_by_degree (lpa.cpp:330-336) becomes a
// four-way device tiering built once per graph (K1 in SURVEY §2.2).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "internal.hpp"
#include "layout.hpp"
#include "plan.hpp"

#ifndef NULPA_BLOCK2_SPLIT
#define NULPA_BLOCK2_SPLIT dev::kBlockMax  // rows above block_max go to the 1024-thread CTA tier
#endif

namespace nulpa {

namespace {
thread_local std::string g_last_error;

struct DegreeOf {
  const uint64_t* off;
  __host__ __device__ uint32_t operator()(uint32_t i) const {
    return static_cast<uint32_t>(off[i + 1] - off[i]);
  }
};

struct DegInRange {
  const uint64_t* off;
  uint64_t lo, hi;
  __host__ __device__ bool operator()(uint32_t i) const {
    const uint64_t d = off[i + 1] - off[i];
    return d >= lo && d <= hi;
  }
};

struct IsUnit {
  __host__ __device__ uint32_t operator()(float w) const { return w == 1.0f ? 0u : 1u; }
};

struct ToDouble {
  __host__ __device__ double operator()(float w) const { return static_cast<double>(w); }
};

__global__ void k_gather_degrees(const uint32_t* list, const uint64_t* off, uint32_t count,
                                 uint32_t* deg) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < count; t += gridDim.x * blockDim.x)
    deg[t] = static_cast<uint32_t>(off[list[t] + 1] - off[list[t]]);
}

__global__ void k_fill_u64(unsigned long long* p, uint64_t count, unsigned long long v) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < count;
       t += (uint64_t)gridDim.x * blockDim.x)
    p[t] = v;
}

__global__ void k_check_offsets(const uint64_t* off, uint32_t n, uint64_t m2, unsigned* bad) {
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (off[i + 1] < off[i]) atomicOr(bad, 1u);
  if (blockIdx.x == 0 && threadIdx.x == 0 && (off[0] != 0 || off[n] != m2)) atomicOr(bad, 2u);
}

// Rows are "simple" when targets strictly ascend inside every row: count all
// descents tgt[e] >= tgt[e+1] and the ones that sit exactly at a row start.
__global__ void k_count_descents(const uint32_t* tgt, uint64_t m2, unsigned long long* cnt) {
  unsigned long long c = 0;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e + 1 < m2;
       e += (uint64_t)gridDim.x * blockDim.x)
    c += tgt[e] >= tgt[e + 1];
  if (c) atomicAdd(cnt, c);
}

__global__ void k_count_boundary_descents(const uint64_t* off, const uint32_t* tgt, uint32_t n,
                                          unsigned long long* cnt) {
  unsigned long long c = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t lo = off[i];
    if (lo > 0 && off[i + 1] > lo) c += tgt[lo - 1] >= tgt[lo];
  }
  if (c) atomicAdd(cnt, c);
}

__global__ void k_check_targets(const uint32_t* tgt, uint64_t m2, uint32_t n, unsigned* bad) {
  for (uint64_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m2;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if (tgt[e] >= n) atomicOr(bad, 4u);
}
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }
const std::string& last_error() { return g_last_error; }

void use_device(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    (void)cudaGetLastError();
    throw Error(NULPA_ECUDA, std::string("no CUDA device available (nulpa has no CPU fallback): ") +
                                 cudaGetErrorString(e));
  }
  if (device < 0 || device >= count)
    throw Error(NULPA_EINVAL, "CUDA device " + std::to_string(device) + " out of range");
  NULPA_CUDA(cudaSetDevice(device));
  // Device buffers come from the stream-ordered pool, which keeps freed memory
  // mapped so repeated lpa() calls (new graph, plan, labels each time) neither
  // re-map multi-GB arrays nor trim the pool at every synchronisation point.
  // NULPA_POOL_KEEP_GB caps what stays cached (default: everything).
  static thread_local int configured = -1;
  if (configured != device) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      const char* env = std::getenv("NULPA_POOL_KEEP_GB");
      uint64_t keep = env ? std::strtoull(env, nullptr, 10) << 30 : ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    (void)cudaGetLastError();
    configured = device;
  }
}

int default_device() {
  if (const char* e = std::getenv("NULPA_DEVICE")) return std::atoi(e);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    (void)cudaGetLastError();
    dev = 0;
  }
  return dev;
}

// Allocations are stream-ordered on the legacy stream; every buffer is freed only
// after the work that used it has been synchronised.
static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

Trace::Trace(const char* sc) : on(std::getenv("NULPA_TRACE") != nullptr), scope(sc) {
  t0 = last = on ? now_s() : 0.0;
}

Trace::~Trace() { mark("exit"); }

void Trace::mark(const char* what) {
  if (!on) return;
  const double t = now_s();
  std::fprintf(stderr, "[nulpa trace] %s: %-24s +%8.3f ms (at %8.3f ms)\n", scope, what,
               (t - last) * 1e3, (t - t0) * 1e3);
  last = t;
}

void* dmalloc(size_t bytes) {
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 16, 0);
  if (e == cudaSuccess) e = cudaStreamSynchronize(0);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    throw Error(e == cudaErrorMemoryAllocation ? NULPA_ENOMEM : NULPA_ECUDA,
                "cudaMallocAsync(" + std::to_string(bytes) + " bytes): " + cudaGetErrorString(e));
  }
  return p;
}

void dfree(void* p) {
  if (p) cudaFreeAsync(p, 0);
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

void check_host_csr(const nulpa_csr* csr) {
  if (!csr) throw Error(NULPA_EINVAL, "null CSR");
  if (!csr->offsets) throw Error(NULPA_EINVAL, "inconsistent CSR arrays");
  if (csr->offsets[0] != 0 || csr->offsets[csr->n] != csr->m2)
    throw Error(NULPA_EINVAL, "inconsistent CSR arrays");
  if (csr->m2 > 0 && !csr->targets) throw Error(NULPA_EINVAL, "inconsistent CSR arrays");
}

// Reductions over the resident arrays: max degree, 2m, unit-weight detection,
// structural validation (offsets monotone, targets < n).
void finalize_graph(nulpa_graph* g, cudaStream_t s, bool relayout) {
  const uint32_t n = g->n;
  unsigned* d_bad = dalloc<unsigned>(1);
  uint32_t* d_max = dalloc<uint32_t>(1);
  double* d_sum = dalloc<double>(1);
  uint32_t* d_nonunit = dalloc<uint32_t>(1);
  NULPA_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(unsigned), s));
  k_check_offsets<<<256, 256, 0, s>>>(g->offsets, n, g->m2, d_bad);
  if (g->m2) k_check_targets<<<1024, 256, 0, s>>>(g->targets, g->m2, n, d_bad);
  NULPA_CUDA(cudaGetLastError());
  unsigned bad = 0;
  NULPA_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  if (bad) {
    dfree(d_bad);
    dfree(d_max);
    dfree(d_sum);
    dfree(d_nonunit);
    throw Error(NULPA_EINVAL, bad & 4u ? "CSR target id out of range" : "inconsistent CSR arrays");
  }
  uint32_t maxd = 0;
  if (n > 0) {
    auto degs = cub::TransformInputIterator<uint32_t, DegreeOf, cub::CountingInputIterator<uint32_t>>(
        cub::CountingInputIterator<uint32_t>(0), DegreeOf{g->offsets});
    size_t tb = 0;
    NULPA_CUDA(cub::DeviceReduce::Max(nullptr, tb, degs, d_max, n, s));
    void* tmp = dmalloc(tb);
    NULPA_CUDA(cub::DeviceReduce::Max(tmp, tb, degs, d_max, n, s));
    NULPA_CUDA(cudaMemcpyAsync(&maxd, d_max, sizeof maxd, cudaMemcpyDeviceToHost, s));
    NULPA_CUDA(cudaStreamSynchronize(s));
    dfree(tmp);
  }
  g->max_degree = maxd;
  double total = static_cast<double>(g->m2);
  if (g->weights && g->m2) {
    auto wd = cub::TransformInputIterator<double, ToDouble, const float*>(g->weights, ToDouble{});
    auto nu = cub::TransformInputIterator<uint32_t, IsUnit, const float*>(g->weights, IsUnit{});
    size_t tb1 = 0, tb2 = 0;
    NULPA_CUDA(cub::DeviceReduce::Sum(nullptr, tb1, wd, d_sum, g->m2, s));
    NULPA_CUDA(cub::DeviceReduce::Sum(nullptr, tb2, nu, d_nonunit, g->m2, s));
    void* tmp = dmalloc(std::max(tb1, tb2));
    NULPA_CUDA(cub::DeviceReduce::Sum(tmp, tb1, wd, d_sum, g->m2, s));
    NULPA_CUDA(cudaMemcpyAsync(&total, d_sum, sizeof total, cudaMemcpyDeviceToHost, s));
    uint32_t nonunit = 0;
    NULPA_CUDA(cub::DeviceReduce::Sum(tmp, tb2, nu, d_nonunit, g->m2, s));
    NULPA_CUDA(cudaMemcpyAsync(&nonunit, d_nonunit, sizeof nonunit, cudaMemcpyDeviceToHost, s));
    NULPA_CUDA(cudaStreamSynchronize(s));
    dfree(tmp);
    if (nonunit == 0) {
      // Every weight is 1.0f: drop the array (results are identical, 4 B/edge saved).
      if (g->owns) dfree(g->weights);
      g->weights = nullptr;
    }
  }
  g->total_2m = total;
  // Strictly ascending rows (no duplicate targets) enable the identity first pass.
  g->rows_simple = true;
  if (g->m2 > 1) {
    unsigned long long* d_c = dalloc<unsigned long long>(2);
    NULPA_CUDA(cudaMemsetAsync(d_c, 0, 16, s));
    k_count_descents<<<2048, 256, 0, s>>>(g->targets, g->m2, d_c);
    k_count_boundary_descents<<<1024, 256, 0, s>>>(g->offsets, g->targets, n, d_c + 1);
    NULPA_CUDA(cudaGetLastError());
    unsigned long long h[2] = {0, 0};
    NULPA_CUDA(cudaMemcpyAsync(h, d_c, 16, cudaMemcpyDeviceToHost, s));
    NULPA_CUDA(cudaStreamSynchronize(s));
    dfree(d_c);
    g->rows_simple = h[0] == h[1];
  }
  dfree(d_bad);
  dfree(d_max);
  dfree(d_sum);
  dfree(d_nonunit);
  // Position-order residency (layout.cu); rows_simple above refers to the input
  // numbering, in which the in-row order is kept.
  if (relayout) relayout_graph(g, s);
}

void partition_two_way(const uint64_t* off, uint32_t n, uint32_t sw, uint32_t* low,
                       uint32_t* high, uint64_t* n_low, uint64_t* n_high, cudaStream_t s) {
  uint64_t* d_num = dalloc<uint64_t>(1);
  cub::CountingInputIterator<uint32_t> ids(0);
  size_t tb = 0;
  NULPA_CUDA(cub::DeviceSelect::If(nullptr, tb, ids, low, d_num, static_cast<uint64_t>(n),
                        DegInRange{off, 0, sw - 1ull}, s));
  void* tmp = dmalloc(tb);
  NULPA_CUDA(cub::DeviceSelect::If(tmp, tb, ids, low, d_num, static_cast<uint64_t>(n),
                        DegInRange{off, 0, sw - 1ull}, s));
  NULPA_CUDA(cudaMemcpyAsync(n_low, d_num, 8, cudaMemcpyDeviceToHost, s));
  NULPA_CUDA(cub::DeviceSelect::If(tmp, tb, ids, high, d_num, static_cast<uint64_t>(n),
                        DegInRange{off, sw, ~0ull}, s));
  NULPA_CUDA(cudaMemcpyAsync(n_high, d_num, 8, cudaMemcpyDeviceToHost, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  dfree(tmp);
  dfree(d_num);
}

// ro_end per tier: the first position whose degree bucket (ceil(log2 deg), the layout's
// key) is at most bmax[t]. Position order is by bucket, descending, so every earlier
// position holds a vertex of a higher-degree tier.
__global__ void k_ro_bounds(const uint64_t* off, uint32_t n, const int* bmax, int k, uint32_t* out) {
  const int t = threadIdx.x;
  if (t >= k) return;
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    const uint64_t d = off[mid + 1] - off[mid];
    const int b = d == 0 ? -1 : (d == 1 ? 0 : 64 - __clzll(d - 1));
    if (b <= bmax[t])
      hi = mid;
    else
      lo = mid + 1;
  }
  out[t] = lo;
}

__global__ void k_hash_keys(const uint32_t* ids, uint32_t count, uint32_t* keys, int shift) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < count; t += gridDim.x * blockDim.x) {
    uint32_t x = (ids[t] >> shift) * 0x9E3779B1u;
    x ^= x >> 16;
    x *= 0x85EBCA6Bu;
    x ^= x >> 13;
    keys[t] = x;
  }
}

// Reorder a vertex list by a hash of (id >> shift): a fixed pseudo-random
// permutation of 2^shift-id blocks; the stable sort keeps ascending order inside
// a block, so shift > 0 keeps the rows of neighbouring ids together.
void scramble_list(uint32_t* list, uint32_t count, cudaStream_t s, int shift = 0) {
  if (count < 2) return;
  uint32_t* k0 = dalloc<uint32_t>(count);
  uint32_t* k1 = dalloc<uint32_t>(count);
  uint32_t* v1 = dalloc<uint32_t>(count);
  k_hash_keys<<<256, 256, 0, s>>>(list, count, k0, shift);
  cub::DoubleBuffer<uint32_t> keys(k0, k1), vals(list, v1);
  size_t tb = 0;
  NULPA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, vals, count, 0, 32, s));
  void* tmp = dmalloc(tb);
  NULPA_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, vals, count, 0, 32, s));
  if (vals.Current() != list)
    NULPA_CUDA(cudaMemcpyAsync(list, vals.Current(), count * 4ull, cudaMemcpyDeviceToDevice, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  dfree(tmp);
  dfree(k0);
  dfree(k1);
  dfree(v1);
}

Plan::~Plan() {
  for (auto* p : list) dfree(p);
  dfree(tab_off);
  dfree(tab_cap);
  dfree(sitem_hub);
  dfree(sitem_start);
  dfree(tab);
  dfree(tab_vals);
  dfree(best);
  dfree(best_k);
  dfree(active);
  dfree(changed);
  dfree(item_hub);
  dfree(item_start);
  dfree(wide_scratch);
  dfree(wide_hint);
}

TierBounds resolve_tiers(uint32_t switch_degree, const nulpa_tuning* t) {
  // Thread tier: deg < switch_degree (the reference's scalar path), capped by
  // the register table of k_thread (16 entries). The half-warp and warp
  // register tiers cover the rest up to 32; then the per-warp table tier
  // (<= 256), the per-CTA table tier (<= 2048) and the hub tier.
  uint32_t tmax = (t && t->thread_max_degree) ? t->thread_max_degree : 8u;
  tmax = std::min<uint32_t>(tmax, 16u);
  if (switch_degree >= 2) tmax = std::min<uint32_t>(tmax, switch_degree - 1);
  uint32_t wmax = (t && t->warp_max_degree) ? t->warp_max_degree : uint32_t(dev::kWarpTabMax);
  wmax = std::max<uint32_t>(std::min<uint32_t>(wmax, dev::kWarpTabMax), 32u);
  uint32_t bmax = (t && t->block_max_degree) ? t->block_max_degree : uint32_t(dev::kBlockMax);
  bmax = std::max<uint32_t>(std::min<uint32_t>(bmax, dev::kBlockMax), wmax);
  const uint32_t sched = (t && t->schedule) ? t->schedule : 4u;  // default: see nulpa.h
  return {tmax, wmax, bmax, sched};
}

Plan* get_plan(nulpa_graph* g, const TierBounds& tb, int value_bytes, cudaStream_t s) {
  if (g->plan && g->plan->thread_max == tb.thread_max && g->plan->warp_max == tb.warp_max &&
      g->plan->block_max == tb.block_max && g->plan->schedule == tb.schedule &&
      g->plan->value_bytes == value_bytes && g->plan->v_lo == 0 && g->plan->v_hi == g->n)
    return g->plan;
  delete g->plan;
  g->plan = nullptr;
  g->plan = build_plan(g, tb, value_bytes, s, 0, g->n);
  return g->plan;
}

Plan* build_plan(nulpa_graph* g, const TierBounds& tb, int value_bytes, cudaStream_t s,
                 uint32_t v_lo, uint32_t v_hi) {
  const auto t0 = std::chrono::steady_clock::now();
  Plan* p = new Plan();
  try {
    p->thread_max = tb.thread_max;
    p->warp_max = tb.warp_max;
    p->block_max = tb.block_max;
    p->schedule = tb.schedule;
    p->value_bytes = value_bytes;
    p->v_lo = v_lo;
    p->v_hi = v_hi;
    p->m2 = g->m2;
    const uint32_t span = v_hi - v_lo;
    p->weighted = g->weights != nullptr;
    const uint64_t tm = tb.thread_max;
    const uint64_t bounds[Plan::kLists][2] = {
        {1, tm},                                        // T_THREAD
        {tm + 1, 16},                                   // T_HALF (empty if tm >= 16)
        {std::max<uint64_t>(tm, 16) + 1, 32},           // T_WARP
        {33, tb.warp_max},                              // T_WTAB
        {uint64_t(tb.warp_max) + 1, tb.block_max},      // T_BLOCK
        {uint64_t(tb.block_max) + 1, NULPA_BLOCK2_SPLIT},   // T_BLOCK2
        {uint64_t(NULPA_BLOCK2_SPLIT) + 1, dev::kBigMax},   // T_BIG
        {uint64_t(dev::kBigMax) + 1, dev::kClusterMax},  // T_CLUSTER
        {uint64_t(dev::kClusterMax) + 1, ~0ull}};        // T_HUB
    uint64_t* d_num = dalloc<uint64_t>(1);
    uint32_t* scratch = dalloc<uint32_t>(uint64_t(span) + 1);
    size_t tbytes = 0;
    cub::CountingInputIterator<uint32_t> ids(v_lo);
    NULPA_CUDA(cub::DeviceSelect::If(nullptr, tbytes, ids, scratch, d_num, static_cast<uint64_t>(span),
                          DegInRange{g->offsets, 1, 1}, s));
    void* tmp = dmalloc(tbytes);
    for (int t = 0; t < Plan::kLists; ++t) {
      NULPA_CUDA(cub::DeviceSelect::If(tmp, tbytes, ids, scratch, d_num, static_cast<uint64_t>(span),
                            DegInRange{g->offsets, bounds[t][0], bounds[t][1]}, s));
      uint64_t cnt = 0;
      NULPA_CUDA(cudaMemcpyAsync(&cnt, d_num, sizeof cnt, cudaMemcpyDeviceToHost, s));
      NULPA_CUDA(cudaStreamSynchronize(s));
      p->list[t] = dalloc<uint32_t>(cnt + 1);
      p->count[t] = static_cast<uint32_t>(cnt);
      if (cnt)
        NULPA_CUDA(cudaMemcpyAsync(p->list[t], scratch, cnt * 4, cudaMemcpyDeviceToDevice, s));
    }
    NULPA_CUDA(cudaStreamSynchronize(s));
    dfree(tmp);
    dfree(d_num);
    dfree(scratch);
    // Scrambled visit order (ParallelAsync only: any interleaving is a valid
    // asynchronous schedule; Synchronous/Sequential results do not depend on it).
    // Tiers up to degree block_max are scrambled in 32-position blocks.
    if (tb.schedule == 4 && p->count[dev::T_THREAD]) {
      // Edges of the thread tier: when they are most of the graph, the tier is walked
      // in contiguous chunks (k_thread CHUNKED) from an unscrambled list.
      const uint32_t m = p->count[dev::T_THREAD];
      auto degs = cub::TransformInputIterator<uint32_t, DegreeOf, const uint32_t*>(
          p->list[dev::T_THREAD], DegreeOf{g->offsets});
      unsigned long long* d_sum = dalloc<unsigned long long>(1);
      size_t tb2 = 0;
      NULPA_CUDA(cub::DeviceReduce::Sum(nullptr, tb2, degs, d_sum, m, s));
      void* t2 = dmalloc(tb2);
      NULPA_CUDA(cub::DeviceReduce::Sum(t2, tb2, degs, d_sum, m, s));
      unsigned long long e = 0;
      NULPA_CUDA(cudaMemcpyAsync(&e, d_sum, 8, cudaMemcpyDeviceToHost, s));
      NULPA_CUDA(cudaStreamSynchronize(s));
      dfree(t2);
      dfree(d_sum);
      p->chunked_thread = 2 * e >= g->m2;
      // The graph stores exactly this tier chunk-major (layout.cu chunk_major): the walk
      // reads it coalesced.
      if (p->chunked_thread && g->chunk_n && v_lo == 0 && v_hi == g->n && tb.thread_max == 8 &&
          m == g->chunk_n) {
        p->chunk_lo = g->chunk_lo;
        p->chunk_L = g->chunk_L;
        p->chunk_dmax = g->chunk_dmax;
      }
    }
    if (tb.schedule == 4) {  // as 3, except a chunk-walked thread tier stays unscrambled
      for (int t = p->chunked_thread ? dev::T_HALF : dev::T_THREAD; t <= dev::T_WARP; ++t)
        scramble_list(p->list[t], p->count[t], s, 5);
    }
    if (tb.schedule == 3) {  // the register tiers (<= 32) scrambled, position order above
      for (int t = dev::T_THREAD; t <= dev::T_WARP; ++t) scramble_list(p->list[t], p->count[t], s, 5);
    }
    if (tb.schedule == 2) {
      // 32-position blocks: a warp's batch of 32 list entries stays contiguous
      // (coalesced prologue loads), the block order is pseudo-random. The
      // long-row tiers (>= 1025) keep position order: their vertices then run
      // largest degree bucket first, which balances the tier's tail.
      for (int t = dev::T_THREAD; t <= dev::T_BLOCK; ++t) scramble_list(p->list[t], p->count[t], s, 5);
    }

    // Read-only label prefixes (PassCtx::ro_end), position layout and whole-graph plans.
    if (g->perm && v_lo == 0 && v_hi == g->n && g->n > 0) {
      // bm[t]: the bucket of tier t's highest degree (prefix bound); bm[kLists + t]: one
      // below the bucket of its lowest degree (suffix bound; every degree there is smaller).
      auto bucket = [](uint64_t d) { return d <= 1 ? 0 : (d >= (1ull << 40) ? 64 : 64 - __builtin_clzll(d - 1)); };
      int bm[2 * Plan::kLists];
      for (int t = 0; t < Plan::kLists; ++t) {
        bm[t] = bucket(bounds[t][1]);
        bm[Plan::kLists + t] = bounds[t][0] <= 1 ? -1 : bucket(bounds[t][0]) - 1;
      }
      int* d_bm = dalloc<int>(2 * Plan::kLists);
      uint32_t* d_out = dalloc<uint32_t>(2 * Plan::kLists);
      NULPA_CUDA(cudaMemcpyAsync(d_bm, bm, sizeof bm, cudaMemcpyHostToDevice, s));
      k_ro_bounds<<<1, 64, 0, s>>>(g->offsets, g->n, d_bm, 2 * Plan::kLists, d_out);
      NULPA_CUDA(cudaGetLastError());
      uint32_t out[2 * Plan::kLists];
      NULPA_CUDA(cudaMemcpyAsync(out, d_out, sizeof out, cudaMemcpyDeviceToHost, s));
      NULPA_CUDA(cudaStreamSynchronize(s));
      // Inside a chunk-major low range (degrees 1..8, buckets 0..3, not sorted) a bucket
      // bound below 3 has no position: take the range's edges (fewer read-only labels).
      if (g->chunk_n)
        for (int x = 0; x < 2 * Plan::kLists; ++x)
          if (bm[x] >= 0 && bm[x] < 3) out[x] = x < Plan::kLists ? g->chunk_lo : g->chunk_lo + g->chunk_n;
      for (int t = 0; t < Plan::kLists; ++t) {
        p->ro_end[t] = out[t];
        p->ro_lo[t] = out[Plan::kLists + t];
      }
      dfree(d_bm);
      dfree(d_out);
      p->ro_end[dev::T_HUB] = g->n;  // hub accumulation writes no label
    }
    // Wide tier (k_wide): per resident CTA, room for the buckets of phases
    // 1..kWideBuckets-1 of its longest possible row (or one in-order snapshot).
    if (p->count[dev::T_CLUSTER] && !p->weighted) {
      // (a non-empty wide tier means max_degree > kBigMax; anything else is stale)
      const uint32_t dmax = g->max_degree > uint32_t(dev::kBigMax)
                                ? std::min<uint32_t>(g->max_degree, dev::kClusterMax)
                                : uint32_t(dev::kClusterMax);
      p->wide_stride = (NULPA_WIDE_BUCKETS - 1) * dmax;
      // (one region per resident CTA: k_wide's grid is at most kWideCtasPerSm per SM)
      p->wide_scratch = dalloc<uint32_t>(uint64_t(sm_count()) * dev::kWideCtasPerSm * p->wide_stride);
      p->wide_hint = dalloc<uint32_t>(p->count[dev::T_CLUSTER]);
      NULPA_CUDA(cudaMemsetAsync(p->wide_hint, 0, p->count[dev::T_CLUSTER] * 4ull, s));
    }
    // Hub tier: per-hub global tables and (hub, chunk) work items. Hub counts
    // are small (vertices of degree > block_max), so the layout is built on
    // the host.
    const uint32_t H = p->count[dev::T_HUB];
    p->n_hubs = H;
    std::vector<uint32_t> hdeg(H);
    if (H) {
      uint32_t* d_deg = dalloc<uint32_t>(H);
      k_gather_degrees<<<256, 256, 0, s>>>(p->list[dev::T_HUB], g->offsets, H, d_deg);
      NULPA_CUDA(cudaGetLastError());
      NULPA_CUDA(cudaMemcpyAsync(hdeg.data(), d_deg, H * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
      NULPA_CUDA(cudaStreamSynchronize(s));
      dfree(d_deg);
    }
    std::vector<uint64_t> toff(H);
    std::vector<uint32_t> tcap(H), ihub, istart, shub, sstart;
    uint64_t slots = 0;
    for (uint32_t x = 0; x < H; ++x) {
      const uint32_t d = hdeg[x];
      const uint32_t cap = dev::pow2_ceil(d + d / 2 + 1);  // load factor <= 2/3
      toff[x] = slots;
      tcap[x] = cap;
      slots += cap;
      for (uint32_t e = 0; e < d; e += dev::kHubChunk) {
        ihub.push_back(x);
        istart.push_back(e);
      }
      for (uint32_t sl = 0; sl < cap; sl += dev::kHubSweep) {
        shub.push_back(x);
        sstart.push_back(sl);
      }
    }
    p->n_items = static_cast<uint32_t>(ihub.size());
    p->n_sitems = static_cast<uint32_t>(shub.size());
    p->table_slots = slots;
    // (+1 entries so every array is non-empty and the memsets below stay in bounds)
    p->tab_off = dalloc<uint64_t>(H + 1);
    p->tab_cap = dalloc<uint32_t>(H + 1);
    p->best = dalloc<unsigned long long>(H + 1);
    p->best_k = dalloc<uint32_t>(H + 1);
    p->active = dalloc<uint8_t>(H + 1);
    p->changed = dalloc<uint8_t>(H + 1);
    if (p->weighted) {
      p->tab = dalloc<uint32_t>(slots + 1);
      p->tab_vals = dmalloc(slots * value_bytes + 16);
    } else {
      p->tab = dalloc<unsigned long long>(slots + 1);
    }
    p->item_hub = dalloc<uint32_t>(p->n_items + 1);
    p->item_start = dalloc<uint32_t>(p->n_items + 1);
    p->sitem_hub = dalloc<uint32_t>(p->n_sitems + 1);
    p->sitem_start = dalloc<uint32_t>(p->n_sitems + 1);
    if (H) {
      NULPA_CUDA(cudaMemcpy(p->tab_off, toff.data(), H * 8, cudaMemcpyHostToDevice));
      NULPA_CUDA(cudaMemcpy(p->tab_cap, tcap.data(), H * 4, cudaMemcpyHostToDevice));
      NULPA_CUDA(cudaMemcpy(p->sitem_hub, shub.data(), shub.size() * 4, cudaMemcpyHostToDevice));
      NULPA_CUDA(cudaMemcpy(p->sitem_start, sstart.data(), sstart.size() * 4, cudaMemcpyHostToDevice));
      NULPA_CUDA(cudaMemcpy(p->item_hub, ihub.data(), ihub.size() * 4, cudaMemcpyHostToDevice));
      NULPA_CUDA(cudaMemcpy(p->item_start, istart.data(), istart.size() * 4, cudaMemcpyHostToDevice));
    }
    NULPA_CUDA(cudaMemsetAsync(p->best, 0, H * 8 + 8, s));
    NULPA_CUDA(cudaMemsetAsync(p->best_k, 0xFF, H * 4 + 4, s));
    NULPA_CUDA(cudaMemsetAsync(p->changed, 0, H + 1, s));
    if (p->weighted) {
      NULPA_CUDA(cudaMemsetAsync(p->tab, 0xFF, slots * 4 + 4, s));
      NULPA_CUDA(cudaMemsetAsync(p->tab_vals, 0, slots * value_bytes + 16, s));
    } else {
      k_fill_u64<<<1024, 256, 0, s>>>(static_cast<unsigned long long*>(p->tab), slots + 1,
                                      dev::kEmptyWord);
      NULPA_CUDA(cudaGetLastError());
    }
    NULPA_CUDA(cudaStreamSynchronize(s));
    // Edge totals of the lower tiers (for reporting).
    // (computed lazily by callers that need them; hubs are exact above)
  } catch (...) {
    delete p;
    throw;
  }
  p->build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return p;
}

}  // namespace nulpa

// ---- C ABI: resident graph ------------------------------------------------------

using namespace nulpa;

namespace nulpa {
nulpa_graph* upload_graph(const nulpa_csr* csr, int device, const TierBounds* tb,
                          int value_bytes) {
  check_host_csr(csr);
  use_device(device);
  auto* g = new nulpa_graph();
  try {
    g->device = device;
    g->n = csr->n;
    g->m2 = csr->m2;
    g->owns = true;
    if (can_upload_pipelined(csr)) {
      std::function<void()> plan_now;
      if (tb)
        plan_now = [&] {
          cudaStream_t sp = nullptr;
          NULPA_CUDA(cudaStreamCreateWithFlags(&sp, cudaStreamNonBlocking));
          try {
            get_plan(g, *tb, value_bytes, sp);
          } catch (...) {
            cudaStreamDestroy(sp);
            throw;
          }
          cudaStreamDestroy(sp);
        };
      upload_pipelined(csr, g, plan_now);
      // a weight array dropped as all-unit after the plan was built: plan again later
      if (g->plan && g->plan->weighted != (g->weights != nullptr)) {
        delete g->plan;
        g->plan = nullptr;
      }
      return g;
    }
    g->offsets = dalloc<uint64_t>(uint64_t(csr->n) + 1);
    g->targets = dalloc<uint32_t>(csr->m2);
    NULPA_CUDA(cudaMemcpy(g->offsets, csr->offsets, (uint64_t(csr->n) + 1) * 8,
                          cudaMemcpyHostToDevice));
    if (csr->m2)
      NULPA_CUDA(cudaMemcpy(g->targets, csr->targets, csr->m2 * 4, cudaMemcpyHostToDevice));
    if (csr->weights && csr->m2) {
      g->weights = dalloc<float>(csr->m2);
      NULPA_CUDA(cudaMemcpy(g->weights, csr->weights, csr->m2 * 4, cudaMemcpyHostToDevice));
    }
    finalize_graph(g, 0);
  } catch (...) {
    nulpa_graph_free(g);
    throw;
  }
  return g;
}
}  // namespace nulpa

extern "C" {

const char* nulpa_last_error(void) { return nulpa::last_error().c_str(); }

int nulpa_version(void) { return 1; }

int nulpa_device_count(int* count) {
  return guarded([&] {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}


int nulpa_graph_upload(const nulpa_csr* csr, int device, nulpa_graph** out) {
  return guarded([&] {
    if (!out) throw Error(NULPA_EINVAL, "null argument");
    *out = upload_graph(csr, device);
  });
}

int nulpa_graph_wrap_device(const nulpa_csr* csr, int device, nulpa_graph** out) {
  return guarded([&] {
    if (!csr || !csr->offsets || (csr->m2 && !csr->targets))
      throw Error(NULPA_EINVAL, "inconsistent CSR arrays");
    use_device(device);
    auto* g = new nulpa_graph();
    g->device = device;
    g->n = csr->n;
    g->m2 = csr->m2;
    g->owns = false;
    g->offsets = const_cast<uint64_t*>(csr->offsets);
    g->targets = const_cast<uint32_t*>(csr->targets);
    g->weights = const_cast<float*>(csr->weights);
    try {
      finalize_graph(g, 0);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int nulpa_graph_free(nulpa_graph* g) {
  return guarded([&] {
    if (!g) return;
    cudaSetDevice(g->device);
    delete g->plan;
    if (g->owns) {
      dfree(g->offsets);
      dfree(g->targets);
      dfree(g->weights);
    }
    dfree(g->perm);
    dfree(g->inv);
    delete g;
  });
}

int nulpa_graph_info(const nulpa_graph* g, uint32_t* n, uint64_t* m2, uint32_t* max_degree,
                     int* weighted) {
  return guarded([&] {
    if (!g) throw Error(NULPA_EINVAL, "null graph");
    if (n) *n = g->n;
    if (m2) *m2 = g->m2;
    if (max_degree) *max_degree = g->max_degree;
    if (weighted) *weighted = g->weights ? 1 : 0;
  });
}

int nulpa_graph_device_csr(const nulpa_graph* g, nulpa_csr* out) {
  return guarded([&] {
    if (!g) throw Error(NULPA_EINVAL, "null graph");
    out->n = g->n;
    out->reserved = 0;
    out->m2 = g->m2;
    out->offsets = g->offsets;
    out->targets = g->targets;
    out->weights = g->weights;
  });
}

int nulpa_graph_download(const nulpa_graph* g, uint64_t* offsets, uint32_t* targets,
                         float* weights) {
  return guarded([&] {
    if (!g) throw Error(NULPA_EINVAL, "null graph");
    use_device(g->device);
    download_vertex_order(g, offsets, targets, g->weights ? weights : nullptr);
    if (weights && !g->weights) std::fill(weights, weights + g->m2, 1.0f);
  });
}

}  // extern "C"
