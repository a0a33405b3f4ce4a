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

#include <atomic>

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
    cub::DeviceScan::InclusiveSum(nullptr, tb, degs, dst_off + 1, n, s);
    void* tmp = dmalloc(tb);
    cub::DeviceScan::InclusiveSum(tmp, tb, degs, dst_off + 1, n, s);
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

}  // namespace

int default_layout() { return g_default_layout.load(); }

void relayout_graph(nulpa_graph* g, cudaStream_t s) {
  g->layout = NULPA_LAYOUT_IDENTITY;
  if (default_layout() != NULPA_LAYOUT_DEGREE_BUCKETS || g->n < 2) return;
  const uint32_t n = g->n;
  const uint64_t m2 = g->m2;
  uint8_t* k0 = dalloc<uint8_t>(n);
  uint8_t* k1 = dalloc<uint8_t>(n);
  uint32_t* ids = dalloc<uint32_t>(n);
  uint32_t* perm = dalloc<uint32_t>(n);
  k_layout_keys<<<blocks_for(n), 256, 0, s>>>(g->offsets, n, k0, ids);
  NULPA_CUDA(cudaGetLastError());
  {
    // Stable LSD radix sort on the 6-bit bucket key: ascending id inside a bucket.
    cub::DoubleBuffer<uint8_t> keys(k0, k1);
    cub::DoubleBuffer<uint32_t> vals(ids, perm);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, vals, n, 0, 6, s);
    void* tmp = dmalloc(tb);
    cub::DeviceRadixSort::SortPairs(tmp, tb, keys, vals, n, 0, 6, s);
    NULPA_CUDA(cudaStreamSynchronize(s));
    dfree(tmp);
    if (vals.Current() != perm) std::swap(ids, perm);
  }
  dfree(k0);
  dfree(k1);
  dfree(ids);
  uint32_t* inv = dalloc<uint32_t>(n);
  k_invert<<<blocks_for(n), 256, 0, s>>>(perm, n, inv);
  NULPA_CUDA(cudaGetLastError());
  // Rows longer than kLongRow form a prefix of the position order (their
  // buckets come first): copy them edge-balanced.
  uint32_t long_rows = 0;
  {
    auto is_long = cub::TransformInputIterator<uint32_t, LongRow, cub::CountingInputIterator<uint32_t>>(
        cub::CountingInputIterator<uint32_t>(0), LongRow{g->offsets});
    uint32_t* d_cnt = dalloc<uint32_t>(1);
    size_t tb = 0;
    cub::DeviceReduce::Sum(nullptr, tb, is_long, d_cnt, n, s);
    void* tmp = dmalloc(tb);
    cub::DeviceReduce::Sum(tmp, tb, is_long, d_cnt, n, s);
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
