// Modularity and community count on the device (K7 in SURVEY §2.2).
//
// modularity (quality.cpp:21-49): Q = Σ_c [σ_c/2m − (Σ_c/2m)²] with σ_c the
// intra-community stored weight (both directions, self-loops once) and Σ_c the
// summed weighted degree, accumulated in fp64. Rows are scanned with the same
// degree tiers as the LPA pass (thread / warp / hub chunks) so hubs of degree
// 10^6 do not serialise on one warp; each row contributes one fp64 atomic per
// accumulator, then a fold over communities reduces to Q.
// community_stats(...).count (quality.cpp:56-78) = number of distinct labels.
#include <cub/cub.cuh>

#include <vector>

#include "internal.hpp"
#include "layout.hpp"
#include "plan.hpp"

namespace nulpa {

using namespace dev;

namespace {

__global__ void k_check_labels(const uint32_t* lab, uint32_t n, unsigned long long* first_bad) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (lab[i] >= n) atomicMin(first_bad, static_cast<unsigned long long>(i));
}

// Rows of degree <= 32, 32 list entries per warp, edge-parallel: the lanes scan the
// degrees of the batch's rows, then walk the batch's edges 32 at a time (lane f of a
// round takes the f-th edge of the batch, its row found by a 5-step search over the
// lanes' prefix sums). Targets of consecutive rows are read coalesced, each lane does one
// label gather per round, and the partial sums are merged per COMMUNITY across the
// warp (__match_any_sync) before one fp64 atomic pair per community per round.
// SCALAR: `sigma` is one accumulator (modularity needs only the total intra-community
// weight, Σ_c σ_c = Σ_i in_i), summed per thread and added once per warp.
template <bool SCALAR = false>
__global__ void __launch_bounds__(256) k_mod_rows32(Graph g, const uint32_t* lab,
                                                    const uint32_t* list, uint32_t count,
                                                    double* sigma, double* big) {
  const int lane = threadIdx.x & 31;
  double in_acc = 0.0;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t base = gw * 32; base < count; base += nw * 32) {
    const uint32_t t = base + lane;
    uint32_t i = 0, d = 0, ci = kEmpty;
    uint64_t lo = 0;
    if (t < count) {
      i = list[t];
      lo = g.off[i];
      d = static_cast<uint32_t>(g.off[i + 1] - lo);
      ci = lab[i];
    }
    uint32_t pre = d;  // inclusive scan of the degrees
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(kFull, pre, o);
      if (lane >= o) pre += v;
    }
    const uint32_t excl = pre - d;
    const uint32_t total = __shfl_sync(kFull, pre, 31);
    // four 32-entry rounds per step: their targets, then their labels, are in flight
    // together (one round at a time was two dependent latencies per 32 entries)
    constexpr int U = 4;
    for (uint32_t f0 = 0; f0 < total; f0 += 32 * U) {
      uint32_t ci_u[U], lab_u[U];
      uint64_t e_u[U];
      bool valid[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t f = f0 + u * 32 + lane;
        int r = 0;  // the last lane whose row starts at or before edge f
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const uint32_t ex = __shfl_sync(kFull, excl, r + step);
          if (ex <= f) r += step;
        }
        const uint64_t lo_r = __shfl_sync(kFull, lo, r);
        ci_u[u] = __shfl_sync(kFull, ci, r);
        const uint32_t ex_r = __shfl_sync(kFull, excl, r);
        valid[u] = f < total;
        e_u[u] = lo_r + (f - ex_r);
        lab_u[u] = valid[u] ? __ldg(g.tgt + e_u[u]) : 0u;  // (the target, for now)
      }
#pragma unroll
      for (int u = 0; u < U; ++u) lab_u[u] = valid[u] ? __ldg(lab + lab_u[u]) : kEmpty;
#pragma unroll 1
      for (int u = 0; u < U; ++u) {
        double w = 0.0, in = 0.0;
        if (valid[u]) {
          w = g.w ? static_cast<double>(g.w[e_u[u]]) : 1.0;
          if (lab_u[u] == ci_u[u]) in = w;
        }
        const uint32_t key = valid[u] ? ci_u[u] : kEmpty;
        const unsigned peers = __match_any_sync(kFull, key);
        double ks = 0.0, is = 0.0;
        if (g.w) {
          for (int b2 = 0; b2 < 32; ++b2) {  // (uniform loop: every lane shuffles)
            const double wb = __shfl_sync(kFull, w, b2), ib = __shfl_sync(kFull, in, b2);
            if ((peers >> b2) & 1u) {
              ks += wb;
              is += ib;
            }
          }
        } else {
          ks = static_cast<double>(__reduce_add_sync(peers, valid[u] ? 1u : 0u));
          if (!SCALAR) is = static_cast<double>(__reduce_add_sync(peers, in != 0.0 ? 1u : 0u));
        }
        if constexpr (SCALAR) in_acc += in;
        if (key != kEmpty && (__ffs(peers) - 1) == lane) {
          atomicAdd(big + key, ks);
          if (!SCALAR && is != 0.0) atomicAdd(sigma + key, is);
        }
      }
    }
  }
  if constexpr (SCALAR) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) in_acc += __shfl_xor_sync(kFull, in_acc, o);
    if (lane == 0 && in_acc != 0.0) atomicAdd(sigma, in_acc);
  }
}

// k_i and the intra-community weight of edges [e, end) step STRIDE of a row whose vertex
// has label ci: four targets, then their four labels, are in flight per thread (the label
// gathers are random reads; one at a time left the kernel latency-bound). Sums are fp64.
template <int STRIDE>
__device__ __forceinline__ void accumulate_row_slice(const Graph& g, const uint32_t* lab,
                                                     uint32_t ci, uint64_t e, uint64_t end,
                                                     double& ki, double& si) {
  constexpr int U = 4;
  for (; e + (U - 1) * STRIDE < end; e += U * STRIDE) {
    uint32_t j[U], l[U];
#pragma unroll
    for (int u = 0; u < U; ++u) j[u] = __ldg(g.tgt + e + u * STRIDE);
#pragma unroll
    for (int u = 0; u < U; ++u) l[u] = __ldg(lab + j[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double w = g.w ? static_cast<double>(__ldg(g.w + e + u * STRIDE)) : 1.0;
      ki += w;
      if (l[u] == ci) si += w;
    }
  }
  for (; e < end; e += STRIDE) {
    const double w = g.w ? static_cast<double>(__ldg(g.w + e)) : 1.0;
    ki += w;
    if (__ldg(lab + __ldg(g.tgt + e)) == ci) si += w;
  }
}

// Larger rows: one warp per row.
template <bool SCALAR = false>
__global__ void k_mod_warp(Graph g, const uint32_t* lab, const uint32_t* list, uint32_t count,
                           double* sigma, double* big) {
  const int lane = threadIdx.x & 31;
  double in_acc = 0.0;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t t = gw; t < count; t += nw) {
    const uint32_t i = list[t];
    const uint32_t ci = lab[i];
    double ki = 0.0, si = 0.0;
    accumulate_row_slice<32>(g, lab, ci, g.off[i] + lane, g.off[i + 1], ki, si);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ki += __shfl_xor_sync(kFull, ki, o);
      si += __shfl_xor_sync(kFull, si, o);
    }
    if (lane == 0) {
      if constexpr (SCALAR)
        in_acc += si;
      else if (si != 0.0)
        atomicAdd(sigma + ci, si);
      if (ki != 0.0) atomicAdd(big + ci, ki);
    }
  }
  if (SCALAR && lane == 0 && in_acc != 0.0) atomicAdd(sigma, in_acc);
}

// Long rows (> 1024): one CTA per row, so a 10^4..10^5-entry row is not walked by a single
// warp (a warp-per-row walk left the few longest rows of a power-law graph as the tail).
template <bool SCALAR = false>
__global__ void __launch_bounds__(256) k_mod_block(Graph g, const uint32_t* lab,
                                                   const uint32_t* list, uint32_t count,
                                                   double* sigma, double* big) {
  __shared__ double red[2][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double in_acc = 0.0;
  for (uint32_t t = blockIdx.x; t < count; t += gridDim.x) {
    const uint32_t i = list[t];
    const uint32_t ci = lab[i];
    double ki = 0.0, si = 0.0;
    accumulate_row_slice<256>(g, lab, ci, g.off[i] + threadIdx.x, g.off[i + 1], ki, si);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ki += __shfl_xor_sync(kFull, ki, o);
      si += __shfl_xor_sync(kFull, si, o);
    }
    if (lane == 0) {
      red[0][warp] = ki;
      red[1][warp] = si;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double k = 0.0, sm = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        k += red[0][w];
        sm += red[1][w];
      }
      if constexpr (SCALAR)
        in_acc += sm;
      else if (sm != 0.0)
        atomicAdd(sigma + ci, sm);
      if (k != 0.0) atomicAdd(big + ci, k);
    }
    __syncthreads();
  }
  if (SCALAR && threadIdx.x == 0 && in_acc != 0.0) atomicAdd(sigma, in_acc);
}

// Hub rows: one CTA per (hub, chunk) item.
template <bool SCALAR = false>
__global__ void k_mod_hub(Graph g, const uint32_t* lab, HubCtx h, double* sigma, double* big) {
  __shared__ double red[2][32];
  double in_acc = 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t it = blockIdx.x; it < h.n_items; it += gridDim.x) {
    const uint32_t i = h.hub_v[h.item_hub[it]];
    const uint32_t ci = lab[i];
    const uint64_t lo = g.off[i];
    const uint64_t d = g.off[i + 1] - lo;
    const uint64_t e0 = h.item_start[it];
    const uint64_t e1 = min(d, e0 + static_cast<uint64_t>(kHubChunk));
    double ki = 0.0, si = 0.0;
    accumulate_row_slice<256>(g, lab, ci, lo + e0 + threadIdx.x, lo + e1, ki, si);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ki += __shfl_xor_sync(kFull, ki, o);
      si += __shfl_xor_sync(kFull, si, o);
    }
    if (lane == 0) {
      red[0][warp] = ki;
      red[1][warp] = si;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double k = 0.0, s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        k += red[0][w];
        s += red[1][w];
      }
      if constexpr (SCALAR)
        in_acc += s;
      else if (s != 0.0)
        atomicAdd(sigma + ci, s);
      if (k != 0.0) atomicAdd(big + ci, k);
    }
    __syncthreads();
  }
  if (SCALAR && threadIdx.x == 0 && in_acc != 0.0) atomicAdd(sigma, in_acc);
}

// Q = Σ_c [σ_c / 2m − (Σ_c / 2m)²] (quality.cpp:41-47). SCALAR: `sigma` holds Σ_c σ_c.
template <bool SCALAR = false>
__global__ void k_mod_fold(const double* sigma, const double* big, uint32_t n, double two_m,
                           double* q) {
  __shared__ double red[32];
  double acc = 0.0;
  if (SCALAR && blockIdx.x == 0 && threadIdx.x == 0) acc = *sigma / two_m;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const double sg = SCALAR ? 0.0 : sigma[c], bg = big[c];
    if (bg == 0.0 && sg == 0.0) continue;
    const double frac = bg / two_m;
    acc += sg / two_m - frac * frac;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (threadIdx.x == 0) atomicAdd(q, acc);
  }
}

__global__ void k_mark(const uint32_t* lab, uint32_t n, uint8_t* present) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    present[lab[i]] = 1;
}

struct U8ToU64 {
  __host__ __device__ unsigned long long operator()(uint8_t v) const { return v; }
};

void check_labels(nulpa_graph* g, const uint32_t* lab, cudaStream_t s) {
  unsigned long long* d_bad = dalloc<unsigned long long>(1);
  NULPA_CUDA(cudaMemsetAsync(d_bad, 0xFF, 8, s));
  k_check_labels<<<1024, 256, 0, s>>>(lab, g->n, d_bad);
  unsigned long long bad = ~0ull;
  NULPA_CUDA(cudaMemcpyAsync(&bad, d_bad, 8, cudaMemcpyDeviceToHost, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  dfree(d_bad);
  if (bad != ~0ull) {
    uint32_t l = 0;
    NULPA_CUDA(cudaMemcpy(&l, lab + bad, 4, cudaMemcpyDeviceToHost));
    // check_labels, quality.cpp:9-17 — same message.
    throw Error(NULPA_EINVAL, "label " + std::to_string(l) + " of vertex " + std::to_string(bad) +
                                  " is out of range");
  }
}

}  // namespace

// sigma[c] (intra-community stored weight) and big[c] (summed weighted degree) for
// every community c, from position-order labels `lab` (quality.cpp:29-40).
void accumulate_sigma(nulpa_graph* g, const uint32_t* lab, double* sigma, double* big,
                      cudaStream_t s, bool scalar = false) {
  const uint32_t n = g->n;
  std::lock_guard<std::recursive_mutex> plan_lock(g->plan_mu);
  // Any tiering covers every row once: reuse the cached plan when there is one.
  Plan* p = g->plan ? g->plan : get_plan(g, resolve_tiers(32, nullptr), 4, s);
  const Graph dg{g->offsets, g->targets, g->weights, n};
  const int sms = sm_count();
  auto rows32 = scalar ? k_mod_rows32<true> : k_mod_rows32<false>;
  auto warp = scalar ? k_mod_warp<true> : k_mod_warp<false>;
  auto hub = scalar ? k_mod_hub<true> : k_mod_hub<false>;
  auto block = scalar ? k_mod_block<true> : k_mod_block<false>;
  for (int t = T_THREAD; t <= T_WARP; ++t)
    if (p->count[t])
      rows32<<<std::min<uint32_t>((p->count[t] + 255) / 256, sms * 8), 256, 0, s>>>(
          dg, lab, p->list[t], p->count[t], sigma, big);
  for (int t = T_WTAB; t <= T_BLOCK; ++t)  // rows of 33 .. 1024 entries: a warp per row
    if (p->count[t])
      warp<<<std::min<uint32_t>((p->count[t] + 7) / 8, sms * 8), 256, 0, s>>>(
          dg, lab, p->list[t], p->count[t], sigma, big);
  for (int t = T_BLOCK2; t <= T_CLUSTER; ++t)  // longer rows: a CTA per row
    if (p->count[t])
      block<<<std::min<uint32_t>(p->count[t], sms * 8), 256, 0, s>>>(dg, lab, p->list[t],
                                                                      p->count[t], sigma, big);
  if (p->n_items)
    hub<<<std::min<uint32_t>(p->n_items, sms * 4), 256, 0, s>>>(dg, lab, p->hub_ctx(), sigma, big);
  NULPA_CUDA(cudaGetLastError());
}

// `labels` in vertex order (community ids are label values, so only the row
// order changes under the position layout).
double modularity_device(nulpa_graph* g, const uint32_t* labels, cudaStream_t s) {
  check_labels(g, labels, s);
  if (!(g->total_2m > 0.0))
    throw Error(NULPA_EINVAL, "modularity is undefined on a graph without edges");
  const uint32_t n = g->n;
  uint32_t* lab_pos = nullptr;
  const uint32_t* lab = labels;
  if (g->perm) {
    lab_pos = dalloc<uint32_t>(n);
    to_positions_u32(g, labels, lab_pos, s);
    lab = lab_pos;
  }
  // Σ_c per community (n doubles), Σ_c σ_c as one accumulator, Q
  double* big = dalloc<double>(uint64_t(n) + 2);
  double* sigma = big + n;
  double* d_q = big + n + 1;
  NULPA_CUDA(cudaMemsetAsync(big, 0, (uint64_t(n) + 2) * sizeof(double), s));
  accumulate_sigma(g, lab, sigma, big, s, /*scalar=*/true);
  const int sms = sm_count();
  k_mod_fold<true><<<std::min<uint32_t>((n + 255) / 256, sms * 4), 256, 0, s>>>(sigma, big, n,
                                                                                g->total_2m, d_q);
  NULPA_CUDA(cudaGetLastError());
  double q = 0.0;
  NULPA_CUDA(cudaMemcpyAsync(&q, d_q, sizeof q, cudaMemcpyDeviceToHost, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  dfree(big);
  dfree(lab_pos);
  return q;
}

namespace {
__global__ void k_sizes(const uint32_t* lab, uint32_t n, uint32_t* size) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(size + lab[i], 1u);
}
struct Present {
  const uint32_t* size;
  __host__ __device__ bool operator()(uint32_t c) const { return size[c] != 0; }
};
__global__ void k_gather_stats(const uint32_t* comm, uint64_t k, const uint32_t* size,
                               const double* sigma, const double* big, uint32_t* sz_out,
                               double* sg_out, double* bg_out) {
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < k;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t c = comm[t];
    sz_out[t] = size[c];
    sg_out[t] = sigma[c];
    bg_out[t] = big[c];
  }
}
}  // namespace

// community_stats (quality.cpp:56-78): the communities present (ascending label),
// their sizes, sigma and big_sigma, and the histogram size -> number of communities.
// Host outputs; arrays hold at most n entries.
void community_stats_device(nulpa_graph* g, const uint32_t* labels, cudaStream_t s,
                            uint64_t* count, uint32_t* comm_h, double* sigma_h, double* big_h,
                            uint64_t* hist_size_h, uint64_t* hist_count_h, uint64_t* hist_len) {
  check_labels(g, labels, s);
  const uint32_t n = g->n;
  uint32_t* lab_pos = nullptr;
  const uint32_t* lab = labels;
  if (g->perm) {
    lab_pos = dalloc<uint32_t>(n);
    to_positions_u32(g, labels, lab_pos, s);
    lab = lab_pos;
  }
  double* sigma = dalloc<double>(2ull * n + 1);
  double* big = sigma + n;
  uint32_t* size = dalloc<uint32_t>(n);
  uint32_t* comm = dalloc<uint32_t>(n);
  uint32_t* sz = dalloc<uint32_t>(n);
  uint32_t* sz_sorted = dalloc<uint32_t>(n);
  double* sg = dalloc<double>(n);
  double* bg = dalloc<double>(n);
  uint64_t* d_num = dalloc<uint64_t>(1);
  uint32_t* runs = dalloc<uint32_t>(n);
  uint32_t* run_len = dalloc<uint32_t>(n);
  void* tmp = nullptr;
  try {
    NULPA_CUDA(cudaMemsetAsync(sigma, 0, (2ull * n + 1) * sizeof(double), s));
    NULPA_CUDA(cudaMemsetAsync(size, 0, n * 4ull, s));
    accumulate_sigma(g, lab, sigma, big, s);
    k_sizes<<<std::min<uint32_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(lab, n, size);
    size_t t1 = 0, t2 = 0, t3 = 0;
    cub::CountingInputIterator<uint32_t> ids(0);
    // Every cub call uses the same 32-bit item-count type: the temp-storage size
    // queried for one offset type does not cover another.
    NULPA_CUDA(cub::DeviceSelect::If(nullptr, t1, ids, comm, d_num, n, Present{size}, s));
    NULPA_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t2, sz, sz_sorted, n, 0, 32, s));
    NULPA_CUDA(
        cub::DeviceRunLengthEncode::Encode(nullptr, t3, sz_sorted, runs, run_len, d_num, n, s));
    tmp = dmalloc(std::max(t1, std::max(t2, t3)));
    NULPA_CUDA(cub::DeviceSelect::If(tmp, t1, ids, comm, d_num, n, Present{size}, s));
    uint64_t k64 = 0;
    NULPA_CUDA(cudaMemcpyAsync(&k64, d_num, 8, cudaMemcpyDeviceToHost, s));
    NULPA_CUDA(cudaStreamSynchronize(s));
    const uint32_t k = static_cast<uint32_t>(k64);
    if (k) {
      k_gather_stats<<<std::min<uint32_t>((k + 255) / 256, 148 * 8), 256, 0, s>>>(
          comm, k, size, sigma, big, sz, sg, bg);
      NULPA_CUDA(cudaGetLastError());
      NULPA_CUDA(cub::DeviceRadixSort::SortKeys(tmp, t2, sz, sz_sorted, k, 0, 32, s));
      NULPA_CUDA(
          cub::DeviceRunLengthEncode::Encode(tmp, t3, sz_sorted, runs, run_len, d_num, k, s));
    }
    uint64_t nh = 0;
    if (k) NULPA_CUDA(cudaMemcpyAsync(&nh, d_num, 8, cudaMemcpyDeviceToHost, s));
    NULPA_CUDA(cudaStreamSynchronize(s));
    *count = k;
    *hist_len = nh;
    if (k) {
      if (comm_h) NULPA_CUDA(cudaMemcpy(comm_h, comm, k * 4, cudaMemcpyDeviceToHost));
      if (sigma_h) NULPA_CUDA(cudaMemcpy(sigma_h, sg, k * 8, cudaMemcpyDeviceToHost));
      if (big_h) NULPA_CUDA(cudaMemcpy(big_h, bg, k * 8, cudaMemcpyDeviceToHost));
      std::vector<uint32_t> hs(nh), hc(nh);
      NULPA_CUDA(cudaMemcpy(hs.data(), runs, nh * 4, cudaMemcpyDeviceToHost));
      NULPA_CUDA(cudaMemcpy(hc.data(), run_len, nh * 4, cudaMemcpyDeviceToHost));
      for (uint64_t x = 0; x < nh; ++x) {
        if (hist_size_h) hist_size_h[x] = hs[x];
        if (hist_count_h) hist_count_h[x] = hc[x];
      }
    }
  } catch (...) {
    for (void* q : {(void*)lab_pos, (void*)sigma, (void*)size, (void*)comm, (void*)sz,
                    (void*)sz_sorted, (void*)sg, (void*)bg, (void*)d_num, (void*)runs,
                    (void*)run_len, tmp})
      dfree(q);
    throw;
  }
  for (void* q : {(void*)lab_pos, (void*)sigma, (void*)size, (void*)comm, (void*)sz,
                  (void*)sz_sorted, (void*)sg, (void*)bg, (void*)d_num, (void*)runs,
                  (void*)run_len, tmp})
    dfree(q);
}

uint64_t community_count_device(nulpa_graph* g, const uint32_t* lab, cudaStream_t s) {
  check_labels(g, lab, s);
  const uint32_t n = g->n;
  uint8_t* present = dalloc<uint8_t>(n);
  unsigned long long* d_cnt = dalloc<unsigned long long>(1);
  NULPA_CUDA(cudaMemsetAsync(present, 0, n, s));
  k_mark<<<1024, 256, 0, s>>>(lab, n, present);
  auto it = cub::TransformInputIterator<unsigned long long, U8ToU64, const uint8_t*>(present,
                                                                                     U8ToU64{});
  size_t tb = 0;
  NULPA_CUDA(cub::DeviceReduce::Sum(nullptr, tb, it, d_cnt, n, s));
  void* tmp = dmalloc(tb);
  NULPA_CUDA(cub::DeviceReduce::Sum(tmp, tb, it, d_cnt, n, s));
  unsigned long long cnt = 0;
  NULPA_CUDA(cudaMemcpyAsync(&cnt, d_cnt, 8, cudaMemcpyDeviceToHost, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  dfree(tmp);
  dfree(present);
  dfree(d_cnt);
  return cnt;
}

}  // namespace nulpa

using namespace nulpa;

extern "C" {

int nulpa_modularity_graph(nulpa_graph* g, const uint32_t* labels_dev, double* q) {
  return guarded([&] {
    if (!g) throw Error(NULPA_EINVAL, "null graph");
    use_device(g->device);
    *q = modularity_device(g, labels_dev, 0);
  });
}

int nulpa_community_stats_graph(nulpa_graph* g, const uint32_t* labels_dev, uint64_t* count,
                                uint32_t* communities, double* sigma, double* big_sigma,
                                uint64_t* hist_size, uint64_t* hist_count, uint64_t* hist_len) {
  return guarded([&] {
    if (!g || !count || !hist_len) throw Error(NULPA_EINVAL, "null argument");
    use_device(g->device);
    community_stats_device(g, labels_dev, 0, count, communities, sigma, big_sigma, hist_size,
                           hist_count, hist_len);
  });
}

int nulpa_community_stats(const nulpa_csr* csr, const uint32_t* labels, uint64_t* count,
                          uint32_t* communities, double* sigma, double* big_sigma,
                          uint64_t* hist_size, uint64_t* hist_count, uint64_t* hist_len) {
  return guarded([&] {
    check_host_csr(csr);
    if (!count || !hist_len) throw Error(NULPA_EINVAL, "null argument");
    nulpa_graph* g = nullptr;
    int rc = nulpa_graph_upload(csr, default_device(), &g);
    if (rc) throw Error(rc, nulpa_last_error());
    uint32_t* d = nullptr;
    try {
      d = dalloc<uint32_t>(csr->n);
      NULPA_CUDA(cudaMemcpy(d, labels, csr->n * 4ull, cudaMemcpyHostToDevice));
      community_stats_device(g, d, 0, count, communities, sigma, big_sigma, hist_size,
                             hist_count, hist_len);
    } catch (...) {
      dfree(d);
      nulpa_graph_free(g);
      throw;
    }
    dfree(d);
    nulpa_graph_free(g);
  });
}

int nulpa_community_count_graph(nulpa_graph* g, const uint32_t* labels_dev, uint64_t* count) {
  return guarded([&] {
    if (!g) throw Error(NULPA_EINVAL, "null graph");
    use_device(g->device);
    *count = community_count_device(g, labels_dev, 0);
  });
}

int nulpa_modularity(const nulpa_csr* csr, const uint32_t* labels, double* q) {
  return guarded([&] {
    check_host_csr(csr);
    nulpa_graph* g = nullptr;
    int rc = nulpa_graph_upload(csr, default_device(), &g);
    if (rc) throw Error(rc, nulpa_last_error());
    uint32_t* d = nullptr;
    try {
      d = dalloc<uint32_t>(csr->n);
      NULPA_CUDA(cudaMemcpy(d, labels, csr->n * 4ull, cudaMemcpyHostToDevice));
      *q = modularity_device(g, d, 0);
    } catch (...) {
      dfree(d);
      nulpa_graph_free(g);
      throw;
    }
    dfree(d);
    nulpa_graph_free(g);
  });
}

int nulpa_community_count(const nulpa_csr* csr, const uint32_t* labels, uint64_t* count) {
  return guarded([&] {
    check_host_csr(csr);
    nulpa_graph* g = nullptr;
    int rc = nulpa_graph_upload(csr, default_device(), &g);
    if (rc) throw Error(rc, nulpa_last_error());
    uint32_t* d = nullptr;
    try {
      d = dalloc<uint32_t>(csr->n);
      NULPA_CUDA(cudaMemcpy(d, labels, csr->n * 4ull, cudaMemcpyHostToDevice));
      *count = community_count_device(g, d, 0);
    } catch (...) {
      dfree(d);
      nulpa_graph_free(g);
      throw;
    }
    dfree(d);
    nulpa_graph_free(g);
  });
}

}  // extern "C"
