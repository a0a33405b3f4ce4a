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

// Rows of degree <= 32: one thread per row.
__global__ void k_mod_thread(Graph g, const uint32_t* lab, const uint32_t* list, uint32_t count,
                             double* sigma, double* big) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < count; t += gridDim.x * blockDim.x) {
    const uint32_t i = list[t];
    const uint32_t ci = lab[i];
    double ki = 0.0, si = 0.0;
    for (uint64_t e = g.off[i]; e < g.off[i + 1]; ++e) {
      const double w = g.w ? static_cast<double>(g.w[e]) : 1.0;
      ki += w;
      if (lab[g.tgt[e]] == ci) si += w;
    }
    if (si != 0.0) atomicAdd(sigma + ci, si);
    if (ki != 0.0) atomicAdd(big + ci, ki);
  }
}

// Larger rows: one warp per row.
__global__ void k_mod_warp(Graph g, const uint32_t* lab, const uint32_t* list, uint32_t count,
                           double* sigma, double* big) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t t = gw; t < count; t += nw) {
    const uint32_t i = list[t];
    const uint32_t ci = lab[i];
    double ki = 0.0, si = 0.0;
    for (uint64_t e = g.off[i] + lane; e < g.off[i + 1]; e += 32) {
      const double w = g.w ? static_cast<double>(g.w[e]) : 1.0;
      ki += w;
      if (lab[g.tgt[e]] == ci) si += w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ki += __shfl_xor_sync(kFull, ki, o);
      si += __shfl_xor_sync(kFull, si, o);
    }
    if (lane == 0) {
      if (si != 0.0) atomicAdd(sigma + ci, si);
      if (ki != 0.0) atomicAdd(big + ci, ki);
    }
  }
}

// Hub rows: one CTA per (hub, chunk) item.
__global__ void k_mod_hub(Graph g, const uint32_t* lab, HubCtx h, double* sigma, double* big) {
  __shared__ double red[2][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t it = blockIdx.x; it < h.n_items; it += gridDim.x) {
    const uint32_t i = h.hub_v[h.item_hub[it]];
    const uint32_t ci = lab[i];
    const uint64_t lo = g.off[i];
    const uint64_t d = g.off[i + 1] - lo;
    const uint64_t e0 = h.item_start[it];
    const uint64_t e1 = min(d, e0 + static_cast<uint64_t>(kHubChunk));
    double ki = 0.0, si = 0.0;
    for (uint64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const double w = g.w ? static_cast<double>(g.w[lo + e]) : 1.0;
      ki += w;
      if (lab[g.tgt[lo + e]] == ci) si += w;
    }
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
      if (s != 0.0) atomicAdd(sigma + ci, s);
      if (k != 0.0) atomicAdd(big + ci, k);
    }
    __syncthreads();
  }
}

__global__ void k_mod_fold(const double* sigma, const double* big, uint32_t n, double two_m,
                           double* q) {
  __shared__ double red[32];
  double acc = 0.0;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const double sg = sigma[c], bg = big[c];
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
  // Any tiering covers every row once: reuse the cached plan when there is one.
  Plan* p = g->plan ? g->plan : get_plan(g, resolve_tiers(32, nullptr), 4, s);
  double* sigma = dalloc<double>(2ull * n + 1);
  double* big = sigma + n;
  double* d_q = sigma + 2ull * n;
  NULPA_CUDA(cudaMemsetAsync(sigma, 0, (2ull * n + 1) * sizeof(double), s));
  const Graph dg{g->offsets, g->targets, g->weights, n};
  const int sms = sm_count();
  if (p->count[T_THREAD])
    k_mod_thread<<<std::min<uint32_t>((p->count[T_THREAD] + 255) / 256, sms * 8), 256, 0, s>>>(
        dg, lab, p->list[T_THREAD], p->count[T_THREAD], sigma, big);
  for (int t = T_HALF; t <= T_CLUSTER; ++t)
    if (p->count[t])
      k_mod_warp<<<std::min<uint32_t>((p->count[t] + 7) / 8, sms * 8), 256, 0, s>>>(
          dg, lab, p->list[t], p->count[t], sigma, big);
  if (p->n_items)
    k_mod_hub<<<std::min<uint32_t>(p->n_items, sms * 4), 256, 0, s>>>(dg, lab, p->hub_ctx(), sigma,
                                                                      big);
  k_mod_fold<<<std::min<uint32_t>((n + 255) / 256, sms * 4), 256, 0, s>>>(sigma, big, n,
                                                                          g->total_2m, d_q);
  NULPA_CUDA(cudaGetLastError());
  double q = 0.0;
  NULPA_CUDA(cudaMemcpyAsync(&q, d_q, sizeof q, cudaMemcpyDeviceToHost, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  dfree(sigma);
  dfree(lab_pos);
  return q;
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
  cub::DeviceReduce::Sum(nullptr, tb, it, d_cnt, n, s);
  void* tmp = dmalloc(tb);
  cub::DeviceReduce::Sum(tmp, tb, it, d_cnt, n, s);
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
    int rc = nulpa_graph_upload(csr, 0, &g);
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
    int rc = nulpa_graph_upload(csr, 0, &g);
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
