// build_csr on the device: an edge list (u, v, w) in listing
// order becomes the reference's CSR, bit for bit (graph.cpp:186-307):
//
//  * symmetrize: each unordered pair {a, b}, a != b, keeps the direction it was first
//    listed in; listings in that direction merge by summing their weights in listing
//    order (double), listings in the opposite direction are dropped. Self-loops merge by
//    summation and are stored once.
//  * !symmetrize: same-direction duplicates merge (sum in listing order); every directed
//    pair must have its reverse with an equal weight, else ValidationError.
//  * n = n_declared (ids must fit) or max id + 1; rows sorted by target; weights stored
//    as float(sum).
//
// Instead of the reference's hash maps, pairs are grouped by a stable radix sort of
// their 64-bit key (listing order survives inside a group), groups are reduced by one
// thread each in that order (the double sums are the reference's, term for term), and
// the CSR is a second sort of (row, target) keys.
#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "internal.hpp"

namespace nulpa {

namespace {

unsigned blocks(uint64_t work) {
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, 148ull * 16)));
}

constexpr uint64_t kLoopTag = 0xFFFFFFFFFFFFFFFFull;

// key = (min << 32) | max for a != b (symmetrize), (u << 32) | v for the directed build,
// kLoopTag - u for self-loops (sorted after every pair, grouped by u).
__global__ void k_edge_keys(const uint32_t* u, const uint32_t* v, uint64_t ne, int symmetrize,
                            uint64_t* keys, uint64_t* idx) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < ne;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t a = u[e], b = v[e];
    uint64_t k;
    if (a == b)
      k = kLoopTag - a;
    else if (symmetrize)
      k = (uint64_t(min(a, b)) << 32) | max(a, b);
    else
      k = (uint64_t(a) << 32) | b;
    keys[e] = k;
    idx[e] = e;
  }
}

__global__ void k_max_id(const uint32_t* u, const uint32_t* v, uint64_t ne, unsigned* out) {
  uint32_t m = 0;
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < ne;
       e += uint64_t(gridDim.x) * blockDim.x)
    m = max(m, max(u[e], v[e]));
  m = __reduce_max_sync(0xFFFFFFFFu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// One thread per group of equal keys [gs, ge) of the sorted edges: the merged weight,
// summed in listing order. Pairs (symmetrize) count only the first-listed direction.
__global__ void k_reduce_groups(const uint64_t* skeys, const uint64_t* sidx, const uint64_t* gstart,
                                uint64_t ngroups, uint64_t ne, const uint32_t* u, const double* w,
                                int symmetrize, uint64_t* gkey, double* gw) {
  for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < ngroups;
       g += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t gs = gstart[g], ge = g + 1 < ngroups ? gstart[g + 1] : ne;
    const uint64_t k = skeys[gs];
    const bool loop = k > 0xFFFFFFFF00000000ull && (k >> 32) == 0xFFFFFFFFull;
    double s = 0.0;
    if (loop || !symmetrize) {
      for (uint64_t p = gs; p < ge; ++p) s += w ? w[sidx[p]] : 1.0;
    } else {
      const uint32_t lo = static_cast<uint32_t>(k >> 32);
      const bool first_forward = u[sidx[gs]] == lo;  // (min, max) listing order
      for (uint64_t p = gs; p < ge; ++p) {
        const uint64_t e = sidx[p];
        if ((u[e] == lo) == first_forward) s += w ? w[e] : 1.0;
      }
    }
    gkey[g] = k;
    gw[g] = s;
  }
}

__global__ void k_group_starts(const uint64_t* skeys, uint64_t ne, uint64_t* flags) {
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < ne;
       p += uint64_t(gridDim.x) * blockDim.x)
    flags[p] = (p == 0 || skeys[p] != skeys[p - 1]) ? 1u : 0u;
}

// !symmetrize: every directed pair (a, b) needs (b, a) with an equal merged weight.
// Records the smallest offending key.
__global__ void k_check_symmetric(const uint64_t* gkey, const double* gw, uint64_t npairs,
                                  unsigned long long* bad) {
  for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < npairs;
       g += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = gkey[g];
    const uint64_t r = ((k & 0xFFFFFFFFull) << 32) | (k >> 32);
    uint64_t lo = 0, hi = npairs;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      if (gkey[mid] < r) lo = mid + 1; else hi = mid;
    }
    if (lo >= npairs || gkey[lo] != r || gw[lo] != gw[g]) atomicMin(bad, k);
  }
}

// CSR entries: (row << 32 | target) keys with float weights. Symmetrized pairs emit
// both directions; directed pairs (already symmetric) emit their own direction;
// loops emit one entry.
__global__ void k_emit(const uint64_t* gkey, const double* gw, uint64_t ngroups, uint64_t npairs,
                       int symmetrize, uint64_t* ekey, float* ew) {
  for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < ngroups;
       g += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = gkey[g];
    const float wf = static_cast<float>(gw[g]);
    if (g >= npairs) {  // self-loop of vertex kLoopTag - k
      const uint64_t a = kLoopTag - k;
      const uint64_t out = symmetrize ? 2 * npairs + (g - npairs) : npairs + (g - npairs);
      ekey[out] = (a << 32) | a;
      ew[out] = wf;
    } else if (symmetrize) {
      const uint64_t a = k >> 32, b = k & 0xFFFFFFFFull;
      ekey[2 * g] = (a << 32) | b;
      ew[2 * g] = wf;
      ekey[2 * g + 1] = (b << 32) | a;
      ew[2 * g + 1] = wf;
    } else {
      ekey[g] = k;
      ew[g] = wf;
    }
  }
}

__global__ void k_csr_from_keys(const uint64_t* ekey, uint64_t m2, uint32_t n, uint64_t* off,
                                uint32_t* tgt) {
  // offsets: off[r] = first entry with row >= r (binary search per row)
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r <= n;
       r += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t lo = 0, hi = m2;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      if ((ekey[mid] >> 32) < r) lo = mid + 1; else hi = mid;
    }
    off[r] = lo;
  }
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < m2;
       e += uint64_t(gridDim.x) * blockDim.x)
    tgt[e] = static_cast<uint32_t>(ekey[e] & 0xFFFFFFFFull);
}

struct Scratch {
  std::vector<void*> ptrs;
  template <typename T>
  T* get(uint64_t n) {
    T* p = dalloc<T>(n);
    ptrs.push_back(p);
    return p;
  }
  ~Scratch() {
    cudaDeviceSynchronize();
    for (void* p : ptrs) dfree(p);
  }
};

}  // namespace

// Device build_csr. `w` may be null (every weight 1.0); n_declared < 0 means none.
nulpa_graph* build_csr_device(const uint32_t* u_h, const uint32_t* v_h, const double* w_h,
                              uint64_t ne, int64_t n_declared, int symmetrize, int device) {
  use_device(device);
  cudaStream_t s = 0;
  Scratch sc;
  uint32_t* u = sc.get<uint32_t>(ne);
  uint32_t* v = sc.get<uint32_t>(ne);
  double* w = w_h ? sc.get<double>(ne) : nullptr;
  if (ne) {
    NULPA_CUDA(cudaMemcpy(u, u_h, ne * 4, cudaMemcpyHostToDevice));
    NULPA_CUDA(cudaMemcpy(v, v_h, ne * 4, cudaMemcpyHostToDevice));
    if (w) NULPA_CUDA(cudaMemcpy(w, w_h, ne * 8, cudaMemcpyHostToDevice));
  }
  // Vertex count (graph.cpp:188-200, same messages).
  uint64_t n = n_declared >= 0 ? static_cast<uint64_t>(n_declared) : 0;
  if (ne) {
    unsigned* d_max = sc.get<unsigned>(1);
    NULPA_CUDA(cudaMemsetAsync(d_max, 0, 4, s));
    k_max_id<<<blocks(ne), 256, 0, s>>>(u, v, ne, d_max);
    unsigned max_id = 0;
    NULPA_CUDA(cudaMemcpy(&max_id, d_max, 4, cudaMemcpyDeviceToHost));
    if (n_declared >= 0) {
      if (max_id >= static_cast<uint64_t>(n_declared))
        throw Error(NULPA_EINVAL, "vertex id " + std::to_string(max_id) +
                                      " out of range for declared n=" + std::to_string(n_declared));
    } else {
      n = uint64_t(max_id) + 1;
    }
  }
  if (n > 0xFFFFFFFFull) throw Error(NULPA_EINVAL, "vertex count exceeds the 32-bit id space");
  // Group listings by key, keeping listing order inside a group (stable sort).
  uint64_t* keys = sc.get<uint64_t>(ne);
  uint64_t* idx = sc.get<uint64_t>(ne);
  uint64_t* skeys = sc.get<uint64_t>(ne);
  uint64_t* sidx = sc.get<uint64_t>(ne);
  uint64_t ngroups = 0, npairs = 0;
  uint64_t* gkey = nullptr;
  double* gw = nullptr;
  if (ne) {
    k_edge_keys<<<blocks(ne), 256, 0, s>>>(u, v, ne, symmetrize, keys, idx);
    size_t tb = 0;
    NULPA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, skeys, idx, sidx, ne, 0, 64, s));
    void* tmp = sc.get<unsigned char>(tb);
    NULPA_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, skeys, idx, sidx, ne, 0, 64, s));
    // group starts: flags -> exclusive positions via select
    uint64_t* flags = keys;  // reuse
    k_group_starts<<<blocks(ne), 256, 0, s>>>(skeys, ne, flags);
    uint64_t* gstart = idx;  // reuse
    uint64_t* d_n = sc.get<uint64_t>(1);
    size_t tb2 = 0;
    NULPA_CUDA(cub::DeviceSelect::Flagged(nullptr, tb2, cub::CountingInputIterator<uint64_t>(0), flags,
                               gstart, d_n, ne, s));
    void* tmp2 = sc.get<unsigned char>(tb2);
    NULPA_CUDA(cub::DeviceSelect::Flagged(tmp2, tb2, cub::CountingInputIterator<uint64_t>(0), flags, gstart,
                               d_n, ne, s));
    NULPA_CUDA(cudaMemcpy(&ngroups, d_n, 8, cudaMemcpyDeviceToHost));
    gkey = sc.get<uint64_t>(ngroups);
    gw = sc.get<double>(ngroups);
    k_reduce_groups<<<blocks(ngroups), 256, 0, s>>>(skeys, sidx, gstart, ngroups, ne, u, w,
                                                    symmetrize, gkey, gw);
    NULPA_CUDA(cudaGetLastError());
    // groups are sorted by key: pairs first, loops (keys near kLoopTag) last
    std::vector<uint64_t> hk(ngroups);
    NULPA_CUDA(cudaMemcpy(hk.data(), gkey, ngroups * 8, cudaMemcpyDeviceToHost));
    npairs = static_cast<uint64_t>(
        std::lower_bound(hk.begin(), hk.end(), 0xFFFFFFFF00000000ull) - hk.begin());
    if (!symmetrize && npairs) {
      unsigned long long* d_bad = sc.get<unsigned long long>(1);
      NULPA_CUDA(cudaMemset(d_bad, 0xFF, 8));
      k_check_symmetric<<<blocks(npairs), 256, 0, s>>>(gkey, gw, npairs, d_bad);
      unsigned long long bad = 0;
      NULPA_CUDA(cudaMemcpy(&bad, d_bad, 8, cudaMemcpyDeviceToHost));
      if (bad != ~0ull)
        throw Error(NULPA_EINVAL, "input is not symmetric at edge (" + std::to_string(bad >> 32) +
                                      "," + std::to_string(bad & 0xFFFFFFFFull) +
                                      ") and symmetrize is off");
    }
  }
  const uint64_t nloops = ngroups - npairs;
  const uint64_t m2 = (symmetrize ? 2 * npairs : npairs) + nloops;
  auto* g = new nulpa_graph();
  try {
    g->device = device;
    g->n = static_cast<uint32_t>(n);
    g->m2 = m2;
    g->owns = true;
    g->offsets = dalloc<uint64_t>(n + 1);
    g->targets = dalloc<uint32_t>(m2);
    g->weights = dalloc<float>(m2);
    if (m2) {
      uint64_t* ekey = sc.get<uint64_t>(m2);
      float* ew = sc.get<float>(m2);
      uint64_t* ekey2 = sc.get<uint64_t>(m2);
      k_emit<<<blocks(ngroups), 256, 0, s>>>(gkey, gw, ngroups, npairs, symmetrize, ekey, ew);
      size_t tb = 0;
      NULPA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, ekey, ekey2, ew, g->weights, m2, 0, 64, s));
      void* tmp = sc.get<unsigned char>(tb);
      NULPA_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, ekey, ekey2, ew, g->weights, m2, 0, 64, s));
      k_csr_from_keys<<<blocks(n + 1), 256, 0, s>>>(ekey2, m2, static_cast<uint32_t>(n),
                                                     g->offsets, g->targets);
    } else {
      NULPA_CUDA(cudaMemset(g->offsets, 0, (n + 1) * 8));
    }
    NULPA_CUDA(cudaGetLastError());
    NULPA_CUDA(cudaDeviceSynchronize());
    finalize_graph(g, s);
  } catch (...) {
    nulpa_graph_free(g);
    throw;
  }
  return g;
}

}  // namespace nulpa

using namespace nulpa;

extern "C" {

int nulpa_graph_from_edge_list(const uint32_t* u, const uint32_t* v, const double* w,
                               uint64_t ne, int64_t n_declared, int symmetrize, int device,
                               nulpa_graph** out) {
  return guarded([&] {
    if (!out || (ne && (!u || !v))) throw Error(NULPA_EINVAL, "null argument");
    *out = build_csr_device(u, v, w, ne, n_declared, symmetrize, device);
  });
}

}  // extern "C"
