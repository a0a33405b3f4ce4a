// Synthetic inputs built on the device (§8f row 1).
//
// build_csr (graph.cpp:186-307) is an unordered_map build that cannot reach
// billions of entries, so the bench builds its CSR here: emit both directions
// of every undirected draw as a packed (src, dst) key, radix-sort, drop
// duplicates, and cut rows from the sorted keys. The result is exactly the
// CSR build_csr(symmetrize=true) produces for a SIMPLE unit-weight edge list
// (rows sorted by target, self-loops stored once); duplicate draws are
// dropped rather than weight-summed so the graph stays unit-weight (SURVEY
// §7.2 item 6).
#include <cub/cub.cuh>

#include <cmath>
#include <vector>

#include "internal.hpp"

namespace nulpa {
namespace {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Seeded bijection on [0, 2^bits): odd-multiply / add / xorshift rounds.
struct Perm {
  uint32_t bits;
  uint64_t mul[3], add[3];
  __host__ __device__ uint64_t operator()(uint64_t x) const {
    const uint64_t mask = (bits >= 64) ? ~0ull : ((1ull << bits) - 1);
    for (int r = 0; r < 3; ++r) {
      x = (x * mul[r] + add[r]) & mask;
      x ^= x >> (bits / 2 + 1);
    }
    return x;
  }
};

Perm make_perm(uint32_t bits, uint64_t seed) {
  Perm p;
  p.bits = bits;
  for (int r = 0; r < 3; ++r) {
    p.mul[r] = splitmix64(seed * 7 + r) | 1ull;
    p.add[r] = splitmix64(seed * 13 + r + 100);
  }
  return p;
}

// Cycle-walk the power-of-two bijection into [0, n).
__device__ __forceinline__ uint32_t perm_n(const Perm& p, uint32_t v, uint32_t n) {
  uint64_t x = v;
  do {
    x = p(x);
  } while (x >= n);
  return static_cast<uint32_t>(x);
}

constexpr uint64_t kSentinel = ~0ull;

// Graph500 Kronecker draws: A=.57, B=.19, C=.19, D=.05 per level.
__global__ void k_rmat(uint64_t* keys, uint64_t ne, uint32_t scale, uint64_t seed, Perm perm) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < ne;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t u = 0, v = 0;
    uint64_t h = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      if ((l & 1) == 0) h = splitmix64(seed ^ (e * 0x2545F4914F6CDD1Dull) ^ (uint64_t(l) << 56));
      const uint32_t r32 = (l & 1) ? static_cast<uint32_t>(h >> 32) : static_cast<uint32_t>(h);
      const double r = r32 * (1.0 / 4294967296.0);
      const uint64_t ub = r >= 0.76 ? 1 : 0;                       // C or D
      const uint64_t vb = (r >= 0.57 && r < 0.76) || r >= 0.95 ? 1 : 0;  // B or D
      u = (u << 1) | ub;
      v = (v << 1) | vb;
    }
    u = perm(u);
    v = perm(v);
    if (u == v) {
      keys[2 * e] = kSentinel;
      keys[2 * e + 1] = kSentinel;
    } else {
      keys[2 * e] = (u << 32) | v;
      keys[2 * e + 1] = (v << 32) | u;
    }
  }
}

// Chung-Lu endpoints by inverse-CDF search over cumulative weights.
__global__ void k_chung_lu(uint64_t* keys, uint64_t ne, const double* cdf, uint32_t n,
                           uint64_t seed, Perm perm) {
  const double total = cdf[n - 1];
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < ne;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t ends[2];
    for (int k = 0; k < 2; ++k) {
      const uint64_t h = splitmix64(seed ^ (e * 0x9E3779B97F4A7C15ull) ^ (uint64_t(k) << 62));
      const double r = (h >> 11) * (1.0 / 9007199254740992.0) * total;
      uint32_t lo = 0, hi = n - 1;
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (cdf[mid] > r)
          hi = mid;
        else
          lo = mid + 1;
      }
      ends[k] = perm_n(perm, lo, n);
    }
    const uint64_t u = ends[0], v = ends[1];
    if (u == v) {
      keys[2 * e] = kSentinel;
      keys[2 * e + 1] = kSentinel;
    } else {
      keys[2 * e] = (u << 32) | v;
      keys[2 * e + 1] = (v << 32) | u;
    }
  }
}

__global__ void k_edges_to_keys(const uint32_t* u, const uint32_t* v, uint64_t ne, uint64_t* keys) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < ne;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = u[e], b = v[e];
    keys[2 * e] = (a << 32) | b;
    keys[2 * e + 1] = (a == b) ? kSentinel : ((b << 32) | a);  // self-loop stored once
  }
}

// Cut CSR rows out of sorted unique keys (sentinels already removed).
__global__ void k_keys_to_csr(const uint64_t* keys, uint64_t m2, uint32_t n, uint64_t* off,
                              uint32_t* tgt) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m2;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[p];
    const uint64_t src = k >> 32;
    tgt[p] = static_cast<uint32_t>(k);
    // Row starts of every vertex in (previous source, src] are p.
    const uint64_t first = p == 0 ? 0 : (keys[p - 1] >> 32) + 1;
    for (uint64_t v = first; v <= src; ++v) off[v] = p;
    if (p == m2 - 1)
      for (uint64_t v = src + 1; v <= n; ++v) off[v] = m2;
  }
}

__global__ void k_fill_offsets_empty(uint64_t* off, uint32_t n) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= n;
       v += (uint64_t)gridDim.x * blockDim.x)
    off[v] = 0;
}

__global__ void k_grid(uint32_t R, uint32_t C, uint64_t* off, uint32_t* tgt) {
  const uint64_t n = uint64_t(R) * C;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = static_cast<uint32_t>(v / C), c = static_cast<uint32_t>(v % C);
    // Closed-form row start = sum of the degrees of all lower ids.
    const uint64_t horiz = 2ull * (C - 1);  // horizontal entries of one full row
    uint64_t start = 0;
    if (r > 0) {
      start += uint64_t(C) * (R > 1 ? 1 : 0) + horiz;           // row 0
      start += uint64_t(r - 1) * (2ull * C + horiz);             // rows 1 .. r-1
    }
    const uint64_t vert = (r > 0 ? 1 : 0) + (r + 1 < R ? 1 : 0);
    start += uint64_t(c) * vert + (c > 0 ? 2ull * c - 1 : 0);
    off[v] = start;
    uint64_t p = start;
    if (r > 0) tgt[p++] = static_cast<uint32_t>(v - C);
    if (c > 0) tgt[p++] = static_cast<uint32_t>(v - 1);
    if (c + 1 < C) tgt[p++] = static_cast<uint32_t>(v + 1);
    if (r + 1 < R) tgt[p++] = static_cast<uint32_t>(v + C);
    if (v == n - 1) off[n] = p;
  }
}

int blocks_for(uint64_t work) {
  const uint64_t b = (work + 255) / 256;
  return static_cast<int>(b < 65536ull * 8 ? (b ? b : 1) : 65536ull * 8);
}

// Sort 2*ne keys (sentinels for dropped draws), dedup, build a CSR graph.
nulpa_graph* keys_to_graph(uint64_t* keys, uint64_t nkeys, uint32_t n, int device, int end_bit) {
  cudaStream_t s = 0;
  uint64_t* alt = dalloc<uint64_t>(nkeys);
  uint64_t* d_num = dalloc<uint64_t>(1);
  nulpa_graph* g = nullptr;
  try {
    cub::DoubleBuffer<uint64_t> db(keys, alt);
    size_t tb = 0;
    NULPA_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, nkeys, 0, end_bit, s));
    void* tmp = dmalloc(tb);
    NULPA_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, db, nkeys, 0, end_bit, s));
    NULPA_CUDA(cudaGetLastError());
    dfree(tmp);
    uint64_t* sorted = db.Current();
    uint64_t* other = db.Alternate();
    size_t tb2 = 0;
    NULPA_CUDA(cub::DeviceSelect::Unique(nullptr, tb2, sorted, other, d_num, nkeys, s));
    tmp = dmalloc(tb2);
    NULPA_CUDA(cub::DeviceSelect::Unique(tmp, tb2, sorted, other, d_num, nkeys, s));
    NULPA_CUDA(cudaGetLastError());
    dfree(tmp);
    uint64_t nu = 0;
    NULPA_CUDA(cudaMemcpy(&nu, d_num, 8, cudaMemcpyDeviceToHost));
    // Drop the (single, after dedup) sentinel at the tail.
    if (nu) {
      uint64_t last = 0;
      NULPA_CUDA(cudaMemcpy(&last, other + nu - 1, 8, cudaMemcpyDeviceToHost));
      if (last == kSentinel) --nu;
    }
    g = new nulpa_graph();
    g->device = device;
    g->n = n;
    g->m2 = nu;
    g->owns = true;
    g->offsets = dalloc<uint64_t>(uint64_t(n) + 1);
    g->targets = dalloc<uint32_t>(nu);
    if (nu) {
      k_keys_to_csr<<<blocks_for(nu), 256, 0, s>>>(other, nu, n, g->offsets, g->targets);
    } else {
      k_fill_offsets_empty<<<blocks_for(uint64_t(n) + 1), 256, 0, s>>>(g->offsets, n);
    }
    NULPA_CUDA(cudaGetLastError());
    NULPA_CUDA(cudaDeviceSynchronize());
  } catch (...) {
    dfree(alt);
    dfree(d_num);
    if (g) {
      dfree(g->offsets);
      dfree(g->targets);
      delete g;
    }
    throw;
  }
  dfree(alt);
  dfree(d_num);
  finalize_graph(g, s);
  return g;
}

// Packed key layout for keys_to_graph: (src << 32) | dst — compare bits 0..63,
// but when ids fit in `bits` bits only bits [0,32+bits) carry information.
int key_end_bit(uint32_t id_bits) { return static_cast<int>(std::min<uint32_t>(64, 32 + id_bits)); }

}  // namespace
}  // namespace nulpa

using namespace nulpa;

extern "C" {

int nulpa_gen_rmat(uint32_t scale, uint32_t edgefactor, uint64_t seed, int device,
                   nulpa_graph** out) {
  return guarded([&] {
    if (scale < 1 || scale > 31) throw Error(NULPA_EINVAL, "R-MAT scale must lie in [1, 31]");
    use_device(device);
    const uint64_t ne = (uint64_t(1) << scale) * edgefactor;
    uint64_t* keys = dalloc<uint64_t>(2 * ne);
    try {
      k_rmat<<<blocks_for(ne), 256>>>(keys, ne, scale, seed, make_perm(scale, seed));
      NULPA_CUDA(cudaGetLastError());
      // Sentinel (~0) must sort last: compare all 64 bits.
      *out = keys_to_graph(keys, 2 * ne, 1u << scale, device, 64);
    } catch (...) {
      dfree(keys);
      throw;
    }
    dfree(keys);
  });
}

int nulpa_gen_web(uint32_t n, uint64_t edges, double gamma, uint32_t hubs, uint32_t hub_degree,
                  uint64_t seed, int device, nulpa_graph** out) {
  return guarded([&] {
    if (n < 2 || gamma <= 1.0) throw Error(NULPA_EINVAL, "web generator needs n >= 2, gamma > 1");
    use_device(device);
    // Chung-Lu expected degrees w_i ∝ (i + i0)^(-1/(gamma-1)); the first
    // `hubs` ranks are pinned to hub_degree. CDF built on the host (n doubles).
    std::vector<double> w(n);
    const double a = 1.0 / (gamma - 1.0);
    double sum = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
      w[i] = std::pow(double(i) + 10.0, -a);
      sum += w[i];
    }
    const double target_sum = 2.0 * double(edges);
    double hub_sum = 0.0;
    for (uint32_t i = 0; i < std::min(hubs, n); ++i) hub_sum += hub_degree;
    double rest = 0.0;
    for (uint32_t i = std::min(hubs, n); i < n; ++i) rest += w[i];
    const double scale = (target_sum - hub_sum) / rest;
    for (uint32_t i = 0; i < n; ++i) w[i] = i < hubs ? double(hub_degree) : w[i] * scale;
    for (uint32_t i = 1; i < n; ++i) w[i] += w[i - 1];
    double* cdf = dalloc<double>(n);
    uint64_t* keys = nullptr;
    try {
      NULPA_CUDA(cudaMemcpy(cdf, w.data(), n * sizeof(double), cudaMemcpyHostToDevice));
      keys = dalloc<uint64_t>(2 * edges);
      uint32_t bits = 1;
      while ((1ull << bits) < n) ++bits;
      k_chung_lu<<<blocks_for(edges), 256>>>(keys, edges, cdf, n, seed, make_perm(bits, seed));
      NULPA_CUDA(cudaGetLastError());
      dfree(cdf);
      cdf = nullptr;
      *out = keys_to_graph(keys, 2 * edges, n, device, 64);
    } catch (...) {
      dfree(cdf);
      dfree(keys);
      throw;
    }
    dfree(keys);
  });
}

int nulpa_gen_grid(uint32_t rows, uint32_t cols, int device, nulpa_graph** out) {
  return guarded([&] {
    if (rows < 1 || cols < 1 || uint64_t(rows) * cols > 0xFFFFFFFFull)
      throw Error(NULPA_EINVAL, "grid dimensions out of range");
    use_device(device);
    const uint64_t n = uint64_t(rows) * cols;
    const uint64_t m2 = 2ull * (uint64_t(rows) * (cols - 1) + uint64_t(cols) * (rows - 1));
    auto* g = new nulpa_graph();
    g->device = device;
    g->n = static_cast<uint32_t>(n);
    g->m2 = m2;
    g->owns = true;
    try {
      g->offsets = dalloc<uint64_t>(n + 1);
      g->targets = dalloc<uint32_t>(m2);
      k_grid<<<blocks_for(n), 256>>>(rows, cols, g->offsets, g->targets);
      NULPA_CUDA(cudaGetLastError());
      NULPA_CUDA(cudaDeviceSynchronize());
      finalize_graph(g, 0);
    } catch (...) {
      nulpa_graph_free(g);
      throw;
    }
    *out = g;
  });
}

int nulpa_graph_from_edges(const uint32_t* u, const uint32_t* v, uint64_t ne, uint32_t n,
                           int device, nulpa_graph** out) {
  return guarded([&] {
    use_device(device);
    for (uint64_t e = 0; e < ne; ++e)
      if (u[e] >= n || v[e] >= n)
        throw Error(NULPA_EINVAL, "vertex id " + std::to_string(std::max(u[e], v[e])) +
                                      " out of range for declared n=" + std::to_string(n));
    uint32_t* du = dalloc<uint32_t>(ne);
    uint32_t* dv = dalloc<uint32_t>(ne);
    uint64_t* keys = nullptr;
    try {
      NULPA_CUDA(cudaMemcpy(du, u, ne * 4, cudaMemcpyHostToDevice));
      NULPA_CUDA(cudaMemcpy(dv, v, ne * 4, cudaMemcpyHostToDevice));
      keys = dalloc<uint64_t>(2 * ne);
      if (ne) k_edges_to_keys<<<blocks_for(ne), 256>>>(du, dv, ne, keys);
      NULPA_CUDA(cudaGetLastError());
      dfree(du);
      dfree(dv);
      du = dv = nullptr;
      *out = keys_to_graph(keys, 2 * ne, n, device, 64);
    } catch (...) {
      dfree(du);
      dfree(dv);
      dfree(keys);
      throw;
    }
    dfree(keys);
  });
}

}  // extern "C"
