// Degree-bucketed vertex layout of the resident CSR (device CSR residency,
// SURVEY §8a row a17).
//
// Label gathers are the path's random reads: one u32 per scanned edge, at the
// position of the neighbour. On power-law inputs (R-MAT, web) about 10% of the
// vertices are the endpoints of 90% of the edges, but under the input's vertex
// numbering those hot labels are scattered — one useful 4-byte label per 32-byte
// sector — so the working set of hot sectors is 8x the hot labels and overflows
// the 126 MB L2 at scale 27. The resident graph therefore stores its rows in
// POSITION order: vertices are grouped by degree bucket (ceil(log2(deg)),
// largest first, isolated vertices last) and kept in ascending id order inside
// a bucket, which packs the hot labels into a few tens of MB and keeps the
// natural locality of lattice-like inputs.
//
// Only storage moves. A label VALUE is still the id of the vertex it came from
// (labels are vertex ids: lpa.cpp:250, the Pick-Less rule lpa.cpp:159 and the
// smaller-key tie-break hashtable.hpp:163-169 compare them), so every result is
// the same as in the input numbering:
//   perm[p] = vertex id stored at position p,  inv[v] = position of vertex v.
// Labels cross the C ABI in vertex order and are permuted at the boundary.
// In-row neighbour order is preserved (the thread tier's bit-identical
// summation order and the identity first pass depend on it).
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif
#include <mutex>
#include <thread>
#include <type_traits>
#include <vector>

#include "internal.hpp"
#include "layout.hpp"

namespace nulpa {

namespace {

std::atomic<int> g_default_layout{NULPA_LAYOUT_DEGREE_BUCKETS};

// 0..32 for deg >= 1 (bucket b holds 2^(b-1) < deg <= 2^b), isolated vertices last.
__device__ __forceinline__ uint32_t layout_key(uint64_t deg) {
  if (deg == 0) return 40u;
  const uint32_t b = deg == 1 ? 0u : 64u - static_cast<uint32_t>(__clzll(deg - 1));
  return 33u - b;  // larger degree -> smaller key -> earlier position
}

__global__ void k_layout_keys(const uint64_t* off, uint32_t n, uint8_t* keys, uint32_t* ids) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    keys[v] = static_cast<uint8_t>(layout_key(off[v + 1] - off[v]));
    ids[v] = v;
  }
}

__global__ void k_invert(const uint32_t* perm, uint32_t n, uint32_t* inv) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    inv[perm[p]] = p;
}

struct RowDegree {
  const uint64_t* off;
  const uint32_t* src_row;
  __host__ __device__ uint64_t operator()(uint32_t r) const {
    const uint32_t s = src_row[r];
    return off[s + 1] - off[s];
  }
};

// dst row r <- src row src_row[r], every target t translated to map[t], for
// rows [r0, n). A warp owns 32 consecutive destination rows: a lane copies its
// own row when it is short; longer rows are copied by the whole warp, one at a
// time (rows here are <= kLongRow, so a warp's share stays bounded).
__global__ void __launch_bounds__(256) k_permute_rows(const uint64_t* __restrict__ src_off,
                                                      const uint32_t* __restrict__ src_tgt,
                                                      const float* __restrict__ src_w,
                                                      const uint32_t* __restrict__ src_row,
                                                      const uint32_t* __restrict__ map,
                                                      const uint64_t* __restrict__ dst_off,
                                                      uint32_t* __restrict__ dst_tgt,
                                                      float* __restrict__ dst_w, uint32_t r0,
                                                      uint32_t n) {
  constexpr uint32_t kShort = 8;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t base = r0 + gw * 32; base < n; base += nw * 32) {
    const uint32_t r = base + lane;
    uint64_t slo = 0, dlo = 0;
    uint32_t d = 0;
    if (r < n) {
      const uint32_t s = src_row[r];
      slo = src_off[s];
      d = static_cast<uint32_t>(src_off[s + 1] - slo);
      dlo = dst_off[r];
    }
    if (d <= kShort) {
      for (uint32_t e = 0; e < d; ++e) {
        dst_tgt[dlo + e] = map[src_tgt[slo + e]];
        if (src_w) dst_w[dlo + e] = src_w[slo + e];
      }
    }
    unsigned long_rows = __ballot_sync(0xFFFFFFFFu, d > kShort);
    while (long_rows) {
      const int b = __ffs(long_rows) - 1;
      long_rows &= long_rows - 1;
      const uint64_t bs = __shfl_sync(0xFFFFFFFFu, slo, b);
      const uint64_t bd = __shfl_sync(0xFFFFFFFFu, dlo, b);
      const uint32_t bdeg = __shfl_sync(0xFFFFFFFFu, d, b);
      for (uint32_t e = lane; e < bdeg; e += 32) {
        dst_tgt[bd + e] = map[src_tgt[bs + e]];
        if (src_w) dst_w[bd + e] = src_w[bs + e];
      }
    }
  }
}

// The long-row prefix [0, P) of a bucketed layout (rows of more than kLongRow
// entries, up to millions): edge-balanced — every warp owns kSpan consecutive
// destination entries, finds its first row by binary search and walks rows.
constexpr uint32_t kLongRow = 256;
constexpr uint64_t kSpan = 4096;

__global__ void __launch_bounds__(256) k_permute_long_rows(
    const uint64_t* __restrict__ src_off, const uint32_t* __restrict__ src_tgt,
    const float* __restrict__ src_w, const uint32_t* __restrict__ src_row,
    const uint32_t* __restrict__ map, const uint64_t* __restrict__ dst_off,
    uint32_t* __restrict__ dst_tgt, float* __restrict__ dst_w, uint32_t P) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * uint64_t(blockDim.x)) >> 5;
  const uint64_t E = dst_off[P];
  for (uint64_t e0 = gw * kSpan; e0 < E; e0 += nw * kSpan) {
    const uint64_t e1 = min(E, e0 + kSpan);
    uint32_t lo = 0, hi = P;  // dst_off[lo] <= e0 < dst_off[hi]
    while (hi - lo > 1) {
      const uint32_t mid = lo + (hi - lo) / 2;
      if (dst_off[mid] <= e0)
        lo = mid;
      else
        hi = mid;
    }
    uint32_t r = lo;
    for (uint64_t e = e0; e < e1; ++r) {
      const uint64_t row_end = min(dst_off[r + 1], e1);
      const uint64_t sb = src_off[src_row[r]] + (e - dst_off[r]);
      const uint32_t len = static_cast<uint32_t>(row_end - e);
      for (uint32_t k = lane; k < len; k += 32) {
        dst_tgt[e + k] = map[src_tgt[sb + k]];
        if (src_w) dst_w[e + k] = src_w[sb + k];
      }
      e = row_end;
    }
  }
}

struct LongRow {
  const uint64_t* off;
  __host__ __device__ uint32_t operator()(uint32_t v) const {
    return off[v + 1] - off[v] > kLongRow ? 1u : 0u;
  }
};

template <typename T>
__global__ void k_gather(const T* __restrict__ src, const uint32_t* __restrict__ idx, uint32_t n,
                         T* __restrict__ dst) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

unsigned blocks_for(uint64_t work) {
  const uint64_t b = (work + 255) / 256;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(b, 148ull * 16)));
}

// Build dst_off (exclusive scan of the permuted row degrees) and the rows.
// `long_prefix` = number of leading destination rows longer than kLongRow (the
// bucketed layout puts them first; 0 when unknown).
void permute_csr(const uint64_t* src_off, const uint32_t* src_tgt, const float* src_w,
                 const uint32_t* src_row, const uint32_t* map, uint32_t n, uint64_t m2,
                 uint64_t* dst_off, uint32_t* dst_tgt, float* dst_w, cudaStream_t s,
                 uint32_t long_prefix = 0) {
  NULPA_CUDA(cudaMemsetAsync(dst_off, 0, sizeof(uint64_t), s));
  if (n > 0) {
    auto degs = cub::TransformInputIterator<uint64_t, RowDegree, cub::CountingInputIterator<uint32_t>>(
        cub::CountingInputIterator<uint32_t>(0), RowDegree{src_off, src_row});
    size_t tb = 0;
    NULPA_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, degs, dst_off + 1, n, s));
    void* tmp = dmalloc(tb);
    NULPA_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, degs, dst_off + 1, n, s));
    if (m2 && long_prefix)
      k_permute_long_rows<<<148 * 8, 256, 0, s>>>(src_off, src_tgt, src_w, src_row, map,
                                                  dst_off, dst_tgt, dst_w, long_prefix);
    if (m2 && long_prefix < n)
      k_permute_rows<<<blocks_for(uint64_t(n - long_prefix) / 8 + 1), 256, 0, s>>>(
          src_off, src_tgt, src_w, src_row, map, dst_off, dst_tgt, dst_w, long_prefix, n);
    NULPA_CUDA(cudaGetLastError());
    NULPA_CUDA(cudaStreamSynchronize(s));
    dfree(tmp);
  }
}

// ---- pipelined upload: the host CSR streamed in row chunks, each chunk scattered
// straight into position order while the next one is in flight ----------------------

// Short rows (degree <= kLongRow) of the input rows [v_a, v_b), whose targets sit in
// `stage` (stage[0] is entry off[v_a]). Validates every target (< n) and counts
// in-row descents (rows_simple) on the way.
__global__ void __launch_bounds__(256) k_scatter_short(
    const uint64_t* __restrict__ off, const uint32_t* __restrict__ stage, uint32_t v_a,
    uint32_t v_b, const uint32_t* __restrict__ inv, const uint64_t* __restrict__ dst_off,
    uint32_t* __restrict__ dst_tgt, uint32_t n, unsigned* bad, unsigned long long* desc,
    const float* __restrict__ wstage, float* __restrict__ dst_w, unsigned long long* nonunit) {
  constexpr uint32_t kShort = 8;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint64_t e_base = off[v_a];
  unsigned long long nd = 0, nnu = 0;
  unsigned nbad = 0;
  for (uint32_t base = v_a + gw * 32; base < v_b; base += nw * 32) {
    const uint32_t v = base + lane;
    uint64_t slo = 0, dlo = 0;
    uint32_t d = 0;
    if (v < v_b) {
      slo = off[v] - e_base;
      d = static_cast<uint32_t>(off[v + 1] - off[v]);
      if (d > kLongRow) d = 0;  // k_scatter_long
      if (d) dlo = dst_off[inv[v]];
    }
    if (d <= kShort) {
      uint32_t prev = 0;
      for (uint32_t e = 0; e < d; ++e) {
        const uint32_t t = stage[slo + e];
        nbad |= t >= n;
        nd += e > 0 && prev >= t;
        prev = t;
        dst_tgt[dlo + e] = t < n ? inv[t] : 0u;
        if (wstage) {
          const float w = wstage[slo + e];
          nnu += w != 1.0f;
          dst_w[dlo + e] = w;
        }
      }
    }
    unsigned long_rows = __ballot_sync(0xFFFFFFFFu, d > kShort);
    while (long_rows) {
      const int b = __ffs(long_rows) - 1;
      long_rows &= long_rows - 1;
      const uint64_t bs = __shfl_sync(0xFFFFFFFFu, slo, b);
      const uint64_t bd = __shfl_sync(0xFFFFFFFFu, dlo, b);
      const uint32_t bdeg = __shfl_sync(0xFFFFFFFFu, d, b);
      for (uint32_t e = lane; e < bdeg; e += 32) {
        const uint32_t t = stage[bs + e];
        nbad |= t >= n;
        nd += e > 0 && stage[bs + e - 1] >= t;
        dst_tgt[bd + e] = t < n ? inv[t] : 0u;
        if (wstage) {
          const float w = wstage[bs + e];
          nnu += w != 1.0f;
          dst_w[bd + e] = w;
        }
      }
    }
  }
  if (nbad) atomicOr(bad, 4u);
  if (nd) atomicAdd(desc, nd);
  if (nnu) atomicAdd(nonunit, nnu);
}

// [la, lb): the entries of the long-row list L (ascending input ids) inside [v_a, v_b).
__global__ void k_long_range(const uint32_t* L, uint32_t nL, uint32_t v_a, uint32_t v_b,
                             uint32_t* out) {
  uint32_t lo = 0, hi = nL;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) / 2;
    if (L[mid] < v_a) lo = mid + 1; else hi = mid;
  }
  out[0] = lo;
  hi = nL;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) / 2;
    if (L[mid] < v_b) lo = mid + 1; else hi = mid;
  }
  out[1] = lo;
}

// Long rows of the chunk, edge-balanced: warps own kSpan entries of the stream of
// the chunk's long-row entries (LP = exclusive prefix of the long rows' degrees).
__global__ void __launch_bounds__(256) k_scatter_long(
    const uint64_t* __restrict__ off, const uint32_t* __restrict__ stage, uint32_t v_a,
    const uint32_t* __restrict__ L, const uint64_t* __restrict__ LP, const uint32_t* range,
    const uint32_t* __restrict__ inv, const uint64_t* __restrict__ dst_off,
    uint32_t* __restrict__ dst_tgt, uint32_t n, unsigned* bad, unsigned long long* desc,
    const float* __restrict__ wstage, float* __restrict__ dst_w, unsigned long long* nonunit) {
  const int lane = threadIdx.x & 31;
  const uint32_t la = range[0], lb = range[1];
  if (la >= lb) return;
  const uint64_t E0 = LP[la], E1 = LP[lb];
  const uint64_t e_base = off[v_a];
  const uint64_t gw = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * uint64_t(blockDim.x)) >> 5;
  unsigned long long nd = 0, nnu = 0;
  unsigned nbad = 0;
  for (uint64_t s0 = E0 + gw * kSpan; s0 < E1; s0 += nw * kSpan) {
    const uint64_t s1 = min(E1, s0 + kSpan);
    uint32_t lo = la, hi = lb;  // LP[lo] <= s0 < LP[hi]
    while (hi - lo > 1) {
      const uint32_t mid = lo + (hi - lo) / 2;
      if (LP[mid] <= s0) lo = mid; else hi = mid;
    }
    for (uint64_t cur = s0, k = lo; cur < s1; ++k) {
      const uint32_t v = L[k];
      const uint64_t row_end = min(LP[k + 1], s1);
      const uint64_t r0 = cur - LP[k];  // offset inside the row
      const uint64_t src = off[v] - e_base + r0;
      const uint64_t dst = dst_off[inv[v]] + r0;
      const uint32_t len = static_cast<uint32_t>(row_end - cur);
      for (uint32_t x = lane; x < len; x += 32) {
        const uint32_t t = stage[src + x];
        nbad |= t >= n;
        nd += (r0 + x) > 0 && stage[src + x - 1] >= t;
        dst_tgt[dst + x] = t < n ? inv[t] : 0u;
        if (wstage) {
          const float w = wstage[src + x];
          nnu += w != 1.0f;
          dst_w[dst + x] = w;
        }
      }
      cur = row_end;
    }
  }
  if (nbad) atomicOr(bad, 4u);
  nd = __reduce_add_sync(0xFFFFFFFFu, static_cast<unsigned>(nd));
  if (lane == 0 && nd) atomicAdd(desc, nd);
  if (nnu) atomicAdd(nonunit, nnu);
}

struct LongDeg {
  const uint64_t* off;
  const uint32_t* L;
  __host__ __device__ uint64_t operator()(uint32_t k) const { return off[L[k] + 1] - off[L[k]]; }
};

struct DegreeOfRow {
  const uint64_t* off;
  __host__ __device__ uint32_t operator()(uint32_t v) const {
    return static_cast<uint32_t>(off[v + 1] - off[v]);
  }
};

__global__ void k_offsets_ok(const uint64_t* off, uint32_t n, uint64_t m2, unsigned* bad) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (off[i + 1] < off[i]) atomicOr(bad, 1u);
  if (blockIdx.x == 0 && threadIdx.x == 0 && (off[0] != 0 || off[n] != m2)) atomicOr(bad, 2u);
}

}  // namespace

int default_layout() { return g_default_layout.load(); }

void build_perm(const uint64_t* off, uint32_t n, uint32_t** perm_out, uint32_t** inv_out,
                cudaStream_t s, nulpa_graph* g);

namespace {

// ---- pageable host sources (the C++ drop-in's std::vector storage) ------------------
// cudaMemcpyAsync from pageable memory is staged by the driver through a small pinned
// buffer at a fraction of the link rate. Pageable chunks are instead copied by all host
// threads into a pinned ring (two buffers per array, kept across calls) and sent from
// there, the copy of chunk k+1 overlapping the DMA of chunk k. A chunk whose weights are
// all 1.0f is not sent at all (filled on the device): unit-weight graphs that arrive with
// an explicit weight array, as every labelprop::CsrGraph does, cost no weight traffic.

bool is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

struct PinnedRing {
  std::mutex mu;
  void* buf[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t cap = 0;  // bytes per buffer
  void* get(int k, size_t bytes) {  // (called with mu held)
    if (bytes > cap) {
      for (void*& b : buf)
        if (b) {
          cudaFreeHost(b);
          b = nullptr;
        }
      cap = bytes;
    }
    if (!buf[k]) NULPA_CUDA(cudaHostAlloc(&buf[k], cap, cudaHostAllocDefault));
    return buf[k];
  }
};
PinnedRing& pinned_ring() {
  static PinnedRing r;
  return r;
}

unsigned copy_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return std::max(1u, std::min(h ? h : 1u, 32u));
}

// Copy into the pinned staging ring with non-temporal stores (NULPA_STREAM_COPY=1, read
// once; off by default): the ring is read only by the DMA engine, so memcpy's
// read-for-ownership of its lines is host memory traffic spent for nothing. Measured on the
// GPU boxes' hosts (drop-in, R27, s per step): 1.20 / 1.80 / 1.02 / 1.08 with it against
// 1.28 / 1.16 / 1.31 / 1.01 without — box noise larger than any effect, so memcpy stays.
inline bool stream_copy_on() {
  static const bool m = [] {
    const char* e = std::getenv("NULPA_STREAM_COPY");
    return e ? std::atoi(e) != 0 : false;
  }();
  return m;
}

void host_copy(void* dst, const void* src, size_t bytes) {
#if defined(__x86_64__)
  if (stream_copy_on()) {
    char* d = static_cast<char*>(dst);
    const char* s = static_cast<const char*>(src);
    const size_t head = std::min(bytes, (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15);
    std::memcpy(d, s, head);
    d += head;
    s += head;
    bytes -= head;
    const size_t n64 = bytes / 64;
    for (size_t i = 0; i < n64; ++i, d += 64, s += 64) {
      const __m128i v0 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s));
      const __m128i v1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 16));
      const __m128i v2 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 32));
      const __m128i v3 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 48));
      _mm_stream_si128(reinterpret_cast<__m128i*>(d), v0);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + 16), v1);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + 32), v2);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + 48), v3);
    }
    std::memcpy(d, s, bytes - n64 * 64);
    _mm_sfence();  // the streamed stores are visible before the DMA is enqueued
    return;
  }
#endif
  std::memcpy(dst, src, bytes);
}

// dst[0, count) = src[0, count) on all host threads; returns true when every element
// equals `unit` (checked only when check_unit).
template <typename T>
bool parallel_copy(T* dst, const T* src, uint64_t count, bool check_unit, T unit) {
  const unsigned t = static_cast<unsigned>(std::min<uint64_t>(copy_threads(), count / 65536 + 1));
  std::atomic<bool> all_unit{true};
  auto work = [&](unsigned k) {
    const uint64_t a = count * k / t, b = count * (k + 1) / t;
    if (dst) host_copy(dst + a, src + a, (b - a) * sizeof(T));
    if (check_unit) {
      bool u = true;
      uint64_t i = a;
#if defined(__x86_64__)
      if constexpr (std::is_same_v<T, float>) {
        // four lanes per compare, the exit tested once per 256 elements (the scalar loop's
        // per-element early exit kept it well below the host memory bandwidth)
        const __m128 uv = _mm_set1_ps(unit);
        for (; u && i + 256 <= b; i += 256) {
          int bad = 0;
          for (int k = 0; k < 256; k += 4)
            bad |= _mm_movemask_ps(_mm_cmpneq_ps(_mm_loadu_ps(src + i + k), uv));
          u = bad == 0;
        }
      }
#endif
      for (; i < b && u; ++i) u = src[i] == unit;
      if (!u) all_unit = false;
    }
  };
  std::vector<std::thread> pool;
  for (unsigned k = 1; k < t; ++k) pool.emplace_back(work, k);
  work(0);
  for (auto& th : pool) th.join();
  return all_unit.load();
}

__global__ void k_fill_f32(float* p, uint64_t count, float v) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x)
    p[i] = v;
}

}  // namespace

bool can_upload_pipelined(const nulpa_csr* csr) {
  return default_layout() == NULPA_LAYOUT_DEGREE_BUCKETS && csr->n >= 2 && csr->m2 > 0;
}

namespace {
struct ToDoubleW {
  __host__ __device__ double operator()(float w) const { return static_cast<double>(w); }
};
}  // namespace

// Host CSR (unit weights) -> resident position-order graph. The offsets go first
// (the permutation needs only degrees); the targets then stream in row chunks of
// ~256 MB on one stream while the previous chunk is validated and scattered into
// position order on another, so the relayout and the structural checks hide behind
// the PCIe transfer.
void upload_pipelined(const nulpa_csr* csr, nulpa_graph* g,
                      const std::function<void()>& while_streaming) {
  // Entries per staging buffer (NULPA_UPLOAD_CHUNK overrides it: the tests force
  // many small chunks and rows longer than a chunk).
  uint64_t kChunk = 64ull << 20;
  if (const char* e = std::getenv("NULPA_UPLOAD_CHUNK")) kChunk = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
  const uint32_t n = csr->n;
  const uint64_t m2 = csr->m2;
  cudaStream_t sa = nullptr, sb = nullptr;
  cudaEvent_t ready[2] = {}, freed[2] = {};
  uint64_t* src_off = nullptr;
  uint32_t* stage[2] = {nullptr, nullptr};
  float* wstage[2] = {nullptr, nullptr};
  uint64_t stage_cap[2] = {0, 0};
  const bool weighted = csr->weights != nullptr;
  unsigned long long* d_nonunit = nullptr;
  uint32_t *L = nullptr, *range = nullptr;
  uint64_t* LP = nullptr;
  unsigned* d_bad = nullptr;
  unsigned long long* d_desc = nullptr;
  uint32_t* d_max = nullptr;
  void* tmp = nullptr;
  auto cleanup = [&]() {
    if (sa) cudaStreamSynchronize(sa);
    if (sb) cudaStreamSynchronize(sb);
    dfree(src_off);
    dfree(stage[0]);
    dfree(stage[1]);
    dfree(wstage[0]);
    dfree(wstage[1]);
    dfree(d_nonunit);
    dfree(L);
    dfree(LP);
    dfree(range);
    dfree(d_bad);
    dfree(d_desc);
    dfree(d_max);
    dfree(tmp);
    for (int k = 0; k < 2; ++k) {
      if (ready[k]) cudaEventDestroy(ready[k]);
      if (freed[k]) cudaEventDestroy(freed[k]);
    }
    if (sa) cudaStreamDestroy(sa);
    if (sb) cudaStreamDestroy(sb);
  };
  try {
    NULPA_CUDA(cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking));
    NULPA_CUDA(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      NULPA_CUDA(cudaEventCreateWithFlags(&ready[k], cudaEventDisableTiming));
      NULPA_CUDA(cudaEventCreateWithFlags(&freed[k], cudaEventDisableTiming));
    }
    src_off = dalloc<uint64_t>(uint64_t(n) + 1);
    d_bad = dalloc<unsigned>(1);
    d_desc = dalloc<unsigned long long>(1);
    d_max = dalloc<uint32_t>(1);
    d_nonunit = dalloc<unsigned long long>(1);
    NULPA_CUDA(cudaMemsetAsync(d_nonunit, 0, 8, sb));
    range = dalloc<uint32_t>(2);
    NULPA_CUDA(cudaMemsetAsync(d_bad, 0, 4, sb));
    NULPA_CUDA(cudaMemsetAsync(d_desc, 0, 8, sb));
    NULPA_CUDA(cudaMemcpyAsync(src_off, csr->offsets, (uint64_t(n) + 1) * 8,
                               cudaMemcpyHostToDevice, sb));
    k_offsets_ok<<<blocks_for(n), 256, 0, sb>>>(src_off, n, m2, d_bad);
    NULPA_CUDA(cudaGetLastError());
    unsigned bad = 0;
    NULPA_CUDA(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, sb));
    NULPA_CUDA(cudaStreamSynchronize(sb));
    if (bad) throw Error(NULPA_EINVAL, "inconsistent CSR arrays");
    // Permutation, position-order offsets, the long-row list of the input order.
    build_perm(src_off, n, &g->perm, &g->inv, sb, g);
    g->offsets = dalloc<uint64_t>(uint64_t(n) + 1);
    g->targets = dalloc<uint32_t>(m2);
    if (weighted) g->weights = dalloc<float>(m2);
    NULPA_CUDA(cudaMemsetAsync(g->offsets, 0, 8, sb));
    {
      auto degs = cub::TransformInputIterator<uint64_t, RowDegree, cub::CountingInputIterator<uint32_t>>(
          cub::CountingInputIterator<uint32_t>(0), RowDegree{src_off, g->perm});
      size_t tb = 0;
      NULPA_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, degs, g->offsets + 1, n, sb));
      auto is_long = cub::TransformInputIterator<uint32_t, LongRow, cub::CountingInputIterator<uint32_t>>(
          cub::CountingInputIterator<uint32_t>(0), LongRow{src_off});
      size_t tb2 = 0;
      L = dalloc<uint32_t>(uint64_t(n) + 1);
      NULPA_CUDA(cub::DeviceSelect::Flagged(nullptr, tb2, cub::CountingInputIterator<uint32_t>(0), is_long, L,
                                 range, n, sb));
      auto dg = cub::TransformInputIterator<uint32_t, DegreeOfRow, cub::CountingInputIterator<uint32_t>>(
          cub::CountingInputIterator<uint32_t>(0), DegreeOfRow{src_off});
      size_t tb3 = 0;
      NULPA_CUDA(cub::DeviceReduce::Max(nullptr, tb3, dg, d_max, n, sb));
      tmp = dmalloc(std::max(tb, std::max(tb2, tb3)));
      NULPA_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, degs, g->offsets + 1, n, sb));
      NULPA_CUDA(cub::DeviceSelect::Flagged(tmp, tb2, cub::CountingInputIterator<uint32_t>(0), is_long, L,
                                 range, n, sb));
      NULPA_CUDA(cub::DeviceReduce::Max(tmp, tb3, dg, d_max, n, sb));
      uint32_t nL = 0;
      NULPA_CUDA(cudaMemcpyAsync(&nL, range, 4, cudaMemcpyDeviceToHost, sb));
      NULPA_CUDA(cudaMemcpyAsync(&g->max_degree, d_max, 4, cudaMemcpyDeviceToHost, sb));
      NULPA_CUDA(cudaStreamSynchronize(sb));
      LP = dalloc<uint64_t>(uint64_t(nL) + 1);
      NULPA_CUDA(cudaMemsetAsync(LP, 0, 8, sb));
      if (nL) {
        auto ld = cub::TransformInputIterator<uint64_t, LongDeg, cub::CountingInputIterator<uint32_t>>(
            cub::CountingInputIterator<uint32_t>(0), LongDeg{src_off, L});
        size_t tb4 = 0;
        NULPA_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb4, ld, LP + 1, nL, sb));
        void* tmp4 = dmalloc(tb4);
        NULPA_CUDA(cub::DeviceScan::InclusiveSum(tmp4, tb4, ld, LP + 1, nL, sb));
        NULPA_CUDA(cudaStreamSynchronize(sb));
        dfree(tmp4);
      }
      // Chunk loop: H2D of chunk k on sa overlaps the scatter of chunk k-1 on sb.
      const uint64_t* ho = csr->offsets;
      const bool pageable = is_pageable(csr->targets) || (weighted && is_pageable(csr->weights));
      std::unique_lock<std::mutex> ring_lock(pinned_ring().mu, std::defer_lock);
      cudaEvent_t sent[2] = {};
      if (pageable) {
        ring_lock.lock();
        for (auto& e : sent) NULPA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      }
      auto destroy_sent = [&] {
        for (auto& e : sent)
          if (e) cudaEventDestroy(e);
      };
      uint32_t v_a = 0;
      for (int k = 0; v_a < n; ++k) {
        const int b = k & 1;
        // largest v_b with ho[v_b] - ho[v_a] <= kChunk (at least one row)
        uint32_t lo = v_a + 1, hi = n;
        while (lo < hi) {
          const uint32_t mid = lo + (hi - lo + 1) / 2;
          if (ho[mid] - ho[v_a] <= kChunk) lo = mid; else hi = mid - 1;
        }
        const uint32_t v_b = lo;
        const uint64_t cnt = ho[v_b] - ho[v_a];
        if (cnt > stage_cap[b]) {  // (only a row longer than kChunk grows a buffer)
          NULPA_CUDA(cudaStreamSynchronize(sb));
          dfree(stage[b]);
          dfree(wstage[b]);
          stage[b] = nullptr;
          wstage[b] = nullptr;
          stage_cap[b] = std::max(cnt, kChunk);
          stage[b] = dalloc<uint32_t>(stage_cap[b]);
          if (weighted) wstage[b] = dalloc<float>(stage_cap[b]);
        }
        if (k >= 2) NULPA_CUDA(cudaStreamWaitEvent(sa, freed[b], 0));
        if (cnt && pageable) {
          // pinned ring: wait until buffer b's previous DMA has left, refill it on the
          // host threads, send it
          if (k >= 2) NULPA_CUDA(cudaEventSynchronize(sent[b]));
          uint32_t* pt = static_cast<uint32_t*>(pinned_ring().get(2 * b, kChunk * 4 > cnt * 4 ? kChunk * 4 : cnt * 4));
          parallel_copy<uint32_t>(pt, csr->targets + ho[v_a], cnt, false, 0u);
          NULPA_CUDA(cudaMemcpyAsync(stage[b], pt, cnt * 4, cudaMemcpyHostToDevice, sa));
          if (weighted) {
            const bool unit = parallel_copy<float>(nullptr, csr->weights + ho[v_a], cnt, true, 1.0f);
            if (unit) {
              k_fill_f32<<<blocks_for(cnt), 256, 0, sa>>>(wstage[b], cnt, 1.0f);
              NULPA_CUDA(cudaGetLastError());
            } else {
              float* pw = static_cast<float*>(pinned_ring().get(2 * b + 1, kChunk * 4 > cnt * 4 ? kChunk * 4 : cnt * 4));
              parallel_copy<float>(pw, csr->weights + ho[v_a], cnt, false, 0.0f);
              NULPA_CUDA(cudaMemcpyAsync(wstage[b], pw, cnt * 4, cudaMemcpyHostToDevice, sa));
            }
          }
          NULPA_CUDA(cudaEventRecord(sent[b], sa));
        } else if (cnt) {
          NULPA_CUDA(cudaMemcpyAsync(stage[b], csr->targets + ho[v_a], cnt * 4,
                                     cudaMemcpyHostToDevice, sa));
          if (weighted)
            NULPA_CUDA(cudaMemcpyAsync(wstage[b], csr->weights + ho[v_a], cnt * 4,
                                       cudaMemcpyHostToDevice, sa));
        }
        NULPA_CUDA(cudaEventRecord(ready[b], sa));
        NULPA_CUDA(cudaStreamWaitEvent(sb, ready[b], 0));
        k_long_range<<<1, 1, 0, sb>>>(L, nL, v_a, v_b, range);
        k_scatter_short<<<blocks_for((uint64_t(v_b - v_a) + 7) / 8), 256, 0, sb>>>(
            src_off, stage[b], v_a, v_b, g->inv, g->offsets, g->targets, n, d_bad, d_desc,
            wstage[b], g->weights, d_nonunit);
        if (nL)
          k_scatter_long<<<148 * 4, 256, 0, sb>>>(src_off, stage[b], v_a, L, LP, range, g->inv,
                                                  g->offsets, g->targets, n, d_bad, d_desc,
                                                  wstage[b], g->weights, d_nonunit);
        NULPA_CUDA(cudaGetLastError());
        NULPA_CUDA(cudaEventRecord(freed[b], sb));
        v_a = v_b;
      }
      if (while_streaming) while_streaming();
      if (pageable) {
        NULPA_CUDA(cudaStreamSynchronize(sa));  // the ring is reusable once sa has drained
        destroy_sent();
      }
    }
    unsigned long long desc = 0;
    NULPA_CUDA(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, sb));
    NULPA_CUDA(cudaMemcpyAsync(&desc, d_desc, 8, cudaMemcpyDeviceToHost, sb));
    NULPA_CUDA(cudaStreamSynchronize(sb));
    if (bad) throw Error(NULPA_EINVAL, bad & 4u ? "CSR target id out of range" : "inconsistent CSR arrays");
    g->total_2m = static_cast<double>(m2);
    if (weighted) {
      unsigned long long nonunit = 0;
      NULPA_CUDA(cudaMemcpy(&nonunit, d_nonunit, 8, cudaMemcpyDeviceToHost));
      if (nonunit == 0) {
        // every weight is 1.0f: drop the array (results identical, 4 B/edge saved)
        dfree(g->weights);
        g->weights = nullptr;
      } else {
        double* d_sum = dalloc<double>(1);
        auto wd = cub::TransformInputIterator<double, ToDoubleW, const float*>(g->weights, ToDoubleW{});
        size_t tb = 0;
        NULPA_CUDA(cub::DeviceReduce::Sum(nullptr, tb, wd, d_sum, m2, sb));
        void* t2 = dmalloc(tb);
        NULPA_CUDA(cub::DeviceReduce::Sum(t2, tb, wd, d_sum, m2, sb));
        NULPA_CUDA(cudaMemcpyAsync(&g->total_2m, d_sum, 8, cudaMemcpyDeviceToHost, sb));
        NULPA_CUDA(cudaStreamSynchronize(sb));
        dfree(t2);
        dfree(d_sum);
      }
    }
    g->rows_simple = desc == 0;
    g->layout = NULPA_LAYOUT_DEGREE_BUCKETS;
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

// perm (position -> vertex) and inv (vertex -> position) of the bucketed order,
// from the input's offsets.
int sm_count();

namespace {

// ---- chunk-major low range ----------------------------------------------------------
// On lattice- and road-like graphs the rows of degree <= 8 carry most of the edges, and
// ParallelAsync walks them in contiguous chunks, one chunk per thread, as each reference
// worker walks its slice (lpa.cpp:139-165; k_thread CHUNKED): thread k visits entries
// k*L .. k*L + L - 1 of the range. In bucket order those entries are L positions apart
// across the lanes of a warp, so every load of the walk touches 32 sectors. Storing the
// range chunk-major — entry e = k*L + r at column r, row k — puts lane k's r-th row next
// to lane k+1's: the walk's row bounds, targets, own labels and flags are read coalesced,
// and so are its neighbour labels (a lattice neighbour e +- 1 or e +- width sits in the
// next lane's or the same lane's column). Only positions move; the walk and every result
// stay as they were.
// Column r holds the q + (r < rem) chunks that reach it (range size M = q*L + rem), so it
// starts at r*q + min(r, rem).
constexpr uint32_t kChunkMaxDeg = 8;
constexpr uint32_t kChunkThreadsPerSm = 1024;  // the chunk walk's threads (k_thread: 4 x 256 per SM)
constexpr uint32_t kChunkMin = 32;             // shortest chunk (a short chunk propagates little)

__global__ void k_low_range_stats(const uint64_t* off, uint32_t n, unsigned long long* out) {
  // out[0]: rows of degree > kChunkMaxDeg, out[1]: rows of degree 1..kChunkMaxDeg, out[2]:
  // their entries, out[4]: their largest degree
  unsigned long long hi = 0, lo = 0, e = 0, mx = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint64_t d = off[v + 1] - off[v];
    const bool low = d >= 1 && d <= kChunkMaxDeg;
    hi += d > kChunkMaxDeg;
    lo += low;
    e += low ? d : 0;
    mx = low && d > mx ? d : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    hi += __shfl_xor_sync(0xFFFFFFFFu, hi, o);
    lo += __shfl_xor_sync(0xFFFFFFFFu, lo, o);
    e += __shfl_xor_sync(0xFFFFFFFFu, e, o);
    mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, hi);
    atomicAdd(out + 1, lo);
    atomicAdd(out + 2, e);
    atomicMax(out + 4, mx);
  }
}

// dst[a + j] = src[a + e(j)]: position a + j of the chunk-major range holds bucket-order
// entry e(j) = k*L + r (column r, row k); positions outside the range are copied.
__global__ void k_chunk_transpose(const uint32_t* src, uint32_t* dst, uint32_t n, uint32_t a,
                                  uint32_t M, uint32_t L) {
  const uint32_t q = M / L, rem = M % L;
  const uint64_t wide = uint64_t(rem) * (q + 1);  // positions of the rem taller columns
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    if (p < a || p >= a + M) {
      dst[p] = src[p];
      continue;
    }
    const uint32_t j = p - a;
    uint32_t r, k;
    if (j < wide) {
      r = j / (q + 1);
      k = j % (q + 1);
    } else {
      const uint32_t jj = static_cast<uint32_t>(j - wide);
      r = rem + jj / q;
      k = jj % q;
    }
    dst[p] = src[a + k * L + r];
  }
}

// Walk threads per SM the layout is cut for (NULPA_CHUNK_TPS, read once; default 1024).
inline uint64_t chunk_threads_per_sm() {
  static const uint64_t m = [] {
    const char* e = std::getenv("NULPA_CHUNK_TPS");
    return e ? static_cast<uint64_t>(std::atoi(e)) : uint64_t(kChunkThreadsPerSm);
  }();
  return m;
}

inline bool chunk_major_enabled() {
  static const bool m = [] {
    const char* e = std::getenv("NULPA_CHUNK_MAJOR");
    return e ? std::atoi(e) != 0 : true;
  }();
  return m;
}

// Apply the chunk-major order to the low range of a bucket-order `perm` when that range
// carries at least half of the entries (where the thread tier is walked in chunks,
// graph.cu build_plan) and is large enough for coalescing to matter.
void chunk_major(const uint64_t* off, uint32_t n, uint32_t* perm, cudaStream_t s, nulpa_graph* g) {
  if (!g) return;
  g->chunk_lo = g->chunk_n = g->chunk_L = g->chunk_dmax = 0;
  if (!chunk_major_enabled() || n < 2) return;
  unsigned long long* d = dalloc<unsigned long long>(5);
  NULPA_CUDA(cudaMemsetAsync(d, 0, 5 * sizeof(unsigned long long), s));
  k_low_range_stats<<<blocks_for(n), 256, 0, s>>>(off, n, d);
  NULPA_CUDA(cudaGetLastError());
  NULPA_CUDA(cudaMemcpyAsync(d + 3, off + n, 8, cudaMemcpyDeviceToDevice, s));
  unsigned long long h[5] = {0, 0, 0, 0, 0};
  NULPA_CUDA(cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  dfree(d);
  const uint64_t a = h[0], M = h[1], e = h[2], m2 = h[3];
  const uint64_t T = uint64_t(sm_count()) * chunk_threads_per_sm();
  if (M < (1u << 16) || 2 * e < m2) return;
  // (chunks of at least kChunkMin entries, as the walk's own bound: engine.cu kMinChunk)
  const uint64_t L = std::max<uint64_t>((M + T - 1) / T, kChunkMin);
  uint32_t* tmp = dalloc<uint32_t>(n);
  k_chunk_transpose<<<blocks_for(n), 256, 0, s>>>(perm, tmp, n, static_cast<uint32_t>(a),
                                                  static_cast<uint32_t>(M), static_cast<uint32_t>(L));
  NULPA_CUDA(cudaGetLastError());
  NULPA_CUDA(cudaMemcpyAsync(perm, tmp, uint64_t(n) * 4, cudaMemcpyDeviceToDevice, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  dfree(tmp);
  g->chunk_lo = static_cast<uint32_t>(a);
  g->chunk_n = static_cast<uint32_t>(M);
  g->chunk_L = static_cast<uint32_t>(L);
  g->chunk_dmax = static_cast<uint32_t>(h[4]);
}

}  // namespace

void build_perm(const uint64_t* off, uint32_t n, uint32_t** perm_out, uint32_t** inv_out,
                cudaStream_t s, nulpa_graph* g) {
  uint8_t* k0 = dalloc<uint8_t>(n);
  uint8_t* k1 = dalloc<uint8_t>(n);
  uint32_t* ids = dalloc<uint32_t>(n);
  uint32_t* perm = dalloc<uint32_t>(n);
  k_layout_keys<<<blocks_for(n), 256, 0, s>>>(off, n, k0, ids);
  NULPA_CUDA(cudaGetLastError());
  {
    // Stable LSD radix sort on the 6-bit bucket key: ascending id inside a bucket.
    cub::DoubleBuffer<uint8_t> keys(k0, k1);
    cub::DoubleBuffer<uint32_t> vals(ids, perm);
    size_t tb = 0;
    NULPA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, vals, n, 0, 6, s));
    void* tmp = dmalloc(tb);
    NULPA_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, vals, n, 0, 6, s));
    NULPA_CUDA(cudaStreamSynchronize(s));
    dfree(tmp);
    if (vals.Current() != perm) std::swap(ids, perm);
  }
  dfree(k0);
  dfree(k1);
  dfree(ids);
  chunk_major(off, n, perm, s, g);
  uint32_t* inv = dalloc<uint32_t>(n);
  k_invert<<<blocks_for(n), 256, 0, s>>>(perm, n, inv);
  NULPA_CUDA(cudaGetLastError());
  *perm_out = perm;
  *inv_out = inv;
}

void relayout_graph(nulpa_graph* g, cudaStream_t s) {
  g->layout = NULPA_LAYOUT_IDENTITY;
  g->chunk_lo = g->chunk_n = g->chunk_L = g->chunk_dmax = 0;
  if (default_layout() != NULPA_LAYOUT_DEGREE_BUCKETS || g->n < 2) return;
  const uint32_t n = g->n;
  const uint64_t m2 = g->m2;
  uint32_t *perm = nullptr, *inv = nullptr;
  build_perm(g->offsets, n, &perm, &inv, s, g);
  // Rows longer than kLongRow form a prefix of the position order (their
  // buckets come first): copy them edge-balanced.
  uint32_t long_rows = 0;
  {
    auto is_long = cub::TransformInputIterator<uint32_t, LongRow, cub::CountingInputIterator<uint32_t>>(
        cub::CountingInputIterator<uint32_t>(0), LongRow{g->offsets});
    uint32_t* d_cnt = dalloc<uint32_t>(1);
    size_t tb = 0;
    NULPA_CUDA(cub::DeviceReduce::Sum(nullptr, tb, is_long, d_cnt, n, s));
    void* tmp = dmalloc(tb);
    NULPA_CUDA(cub::DeviceReduce::Sum(tmp, tb, is_long, d_cnt, n, s));
    NULPA_CUDA(cudaMemcpyAsync(&long_rows, d_cnt, 4, cudaMemcpyDeviceToHost, s));
    NULPA_CUDA(cudaStreamSynchronize(s));
    dfree(tmp);
    dfree(d_cnt);
  }
  uint64_t* off = dalloc<uint64_t>(uint64_t(n) + 1);
  uint32_t* tgt = dalloc<uint32_t>(m2);
  float* w = g->weights ? dalloc<float>(m2) : nullptr;
  permute_csr(g->offsets, g->targets, g->weights, perm, inv, n, m2, off, tgt, w, s, long_rows);
  if (g->owns) {
    dfree(g->offsets);
    dfree(g->targets);
    dfree(g->weights);
  }
  g->owns = true;  // the position-order arrays belong to the graph
  g->offsets = off;
  g->targets = tgt;
  g->weights = w;
  g->perm = perm;
  g->inv = inv;
  g->layout = NULPA_LAYOUT_DEGREE_BUCKETS;
}

void to_positions_u32(const nulpa_graph* g, const uint32_t* vtx, uint32_t* pos, cudaStream_t s) {
  if (!g->perm) {
    if (vtx != pos)
      NULPA_CUDA(cudaMemcpyAsync(pos, vtx, g->n * 4ull, cudaMemcpyDeviceToDevice, s));
    return;
  }
  k_gather<uint32_t><<<blocks_for(g->n), 256, 0, s>>>(vtx, g->perm, g->n, pos);
  NULPA_CUDA(cudaGetLastError());
}

void to_vertices_u32(const nulpa_graph* g, const uint32_t* pos, uint32_t* vtx, cudaStream_t s) {
  if (!g->perm) {
    if (vtx != pos)
      NULPA_CUDA(cudaMemcpyAsync(vtx, pos, g->n * 4ull, cudaMemcpyDeviceToDevice, s));
    return;
  }
  k_gather<uint32_t><<<blocks_for(g->n), 256, 0, s>>>(pos, g->inv, g->n, vtx);
  NULPA_CUDA(cudaGetLastError());
}

void to_positions_u8(const nulpa_graph* g, const uint8_t* vtx, uint8_t* pos, cudaStream_t s) {
  if (!g->perm) {
    if (vtx != pos) NULPA_CUDA(cudaMemcpyAsync(pos, vtx, g->n, cudaMemcpyDeviceToDevice, s));
    return;
  }
  k_gather<uint8_t><<<blocks_for(g->n), 256, 0, s>>>(vtx, g->perm, g->n, pos);
  NULPA_CUDA(cudaGetLastError());
}

void to_vertices_u8(const nulpa_graph* g, const uint8_t* pos, uint8_t* vtx, cudaStream_t s) {
  if (!g->perm) {
    if (vtx != pos) NULPA_CUDA(cudaMemcpyAsync(vtx, pos, g->n, cudaMemcpyDeviceToDevice, s));
    return;
  }
  k_gather<uint8_t><<<blocks_for(g->n), 256, 0, s>>>(pos, g->inv, g->n, vtx);
  NULPA_CUDA(cudaGetLastError());
}

void download_vertex_order(const nulpa_graph* g, uint64_t* off_h, uint32_t* tgt_h, float* w_h) {
  const uint32_t n = g->n;
  const uint64_t m2 = g->m2;
  if (!g->perm) {
    if (off_h) NULPA_CUDA(cudaMemcpy(off_h, g->offsets, (uint64_t(n) + 1) * 8, cudaMemcpyDeviceToHost));
    if (tgt_h && m2) NULPA_CUDA(cudaMemcpy(tgt_h, g->targets, m2 * 4, cudaMemcpyDeviceToHost));
    if (w_h && g->weights) NULPA_CUDA(cudaMemcpy(w_h, g->weights, m2 * 4, cudaMemcpyDeviceToHost));
    return;
  }
  cudaStream_t s = 0;
  uint64_t* off = dalloc<uint64_t>(uint64_t(n) + 1);
  uint32_t* tgt = dalloc<uint32_t>(m2);
  float* w = g->weights ? dalloc<float>(m2) : nullptr;
  try {
    // vertex row v <- position row inv[v], targets translated back by perm.
    permute_csr(g->offsets, g->targets, g->weights, g->inv, g->perm, n, m2, off, tgt, w, s);
    if (off_h) NULPA_CUDA(cudaMemcpy(off_h, off, (uint64_t(n) + 1) * 8, cudaMemcpyDeviceToHost));
    if (tgt_h && m2) NULPA_CUDA(cudaMemcpy(tgt_h, tgt, m2 * 4, cudaMemcpyDeviceToHost));
    if (w_h && w) NULPA_CUDA(cudaMemcpy(w_h, w, m2 * 4, cudaMemcpyDeviceToHost));
  } catch (...) {
    dfree(off);
    dfree(tgt);
    dfree(w);
    throw;
  }
  dfree(off);
  dfree(tgt);
  dfree(w);
}

}  // namespace nulpa

using namespace nulpa;

extern "C" {

int nulpa_set_default_layout(int layout) {
  return guarded([&] {
    if (layout != NULPA_LAYOUT_IDENTITY && layout != NULPA_LAYOUT_DEGREE_BUCKETS)
      throw Error(NULPA_EINVAL, "unknown graph layout");
    g_default_layout.store(layout);
  });
}

int nulpa_graph_layout(const nulpa_graph* g, int* layout) {
  return guarded([&] {
    if (!g || !layout) throw Error(NULPA_EINVAL, "null argument");
    *layout = g->layout;
  });
}

int nulpa_graph_labels_to_vertex_order(const nulpa_graph* g, const uint32_t* pos_dev,
                                       uint32_t* vtx_dev) {
  return guarded([&] {
    if (!g || !pos_dev || !vtx_dev) throw Error(NULPA_EINVAL, "null argument");
    if (pos_dev == vtx_dev && g->perm) throw Error(NULPA_EINVAL, "in-place permutation");
    use_device(g->device);
    to_vertices_u32(g, pos_dev, vtx_dev, 0);
    NULPA_CUDA(cudaStreamSynchronize(0));
  });
}

int nulpa_graph_labels_to_position_order(const nulpa_graph* g, const uint32_t* vtx_dev,
                                         uint32_t* pos_dev) {
  return guarded([&] {
    if (!g || !pos_dev || !vtx_dev) throw Error(NULPA_EINVAL, "null argument");
    if (pos_dev == vtx_dev && g->perm) throw Error(NULPA_EINVAL, "in-place permutation");
    use_device(g->device);
    to_positions_u32(g, vtx_dev, pos_dev, 0);
    NULPA_CUDA(cudaStreamSynchronize(0));
  });
}

}  // extern "C"
