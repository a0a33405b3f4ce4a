// Device side of the partitioned multi-GPU path (no reference counterpart —
// the reference is single-host, lpa.cpp:235-240).
//
//  * nulpa_graph_slice: one rank's resident graph. A 1-D edge-balanced partition of the
//    position order gives rank p the rows [lo, hi); the slice keeps ONLY those rows'
//    targets (global position ids, so labels and flags stay indexed by position in the
//    replicated arrays) plus offsets for every position (rows outside the range are
//    empty). At R-MAT 27 over 8 ranks that is ~2.1 GB of targets per GPU instead of 16.9.
//  * nulpa_session_pack_changes / nulpa_session_apply_changes: the changed-only label
//    exchange. A session snapshots its range at the start of every pass; after the pass
//    the (position, label) pairs that differ are compacted into a fixed-size packet
//    (padded with a sentinel), the packets of all ranks are all-gathered (one NCCL
//    collective), and every rank applies the others' pairs to its replica.
//  * nulpa_community_sums_graph: sigma_c / Sigma_c partial sums over the rows a slice
//    holds (quality.cpp:29-40); summed over ranks (all-reduce) they give the full graph's
//    modularity.
#include <algorithm>

#include "internal.hpp"
#include "plan.hpp"

namespace nulpa {

void accumulate_sigma(nulpa_graph* g, const uint32_t* lab, double* sigma, double* big,
                      cudaStream_t s, bool scalar = false);

namespace {

__global__ void k_slice_offsets(const uint64_t* off, uint32_t n, uint32_t lo, uint32_t hi,
                                uint64_t* out) {
  const uint64_t base = off[lo], top = off[hi];
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v <= n;
       v += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t o = off[v];
    out[v] = (o < base ? base : (o > top ? top : o)) - base;
  }
}

}  // namespace

nulpa_graph* slice_graph(const nulpa_graph* g, uint32_t lo, uint32_t hi) {
  if (lo > hi || hi > g->n) throw Error(NULPA_EINVAL, "vertex range out of bounds");
  use_device(g->device);
  uint64_t range[2];
  NULPA_CUDA(cudaMemcpy(&range[0], g->offsets + lo, 8, cudaMemcpyDeviceToHost));
  NULPA_CUDA(cudaMemcpy(&range[1], g->offsets + hi, 8, cudaMemcpyDeviceToHost));
  auto* s = new nulpa_graph();
  try {
    s->device = g->device;
    s->n = g->n;
    s->m2 = range[1] - range[0];
    s->owns = true;
    s->layout = g->layout;
    s->rows_simple = g->rows_simple;
    s->offsets = dalloc<uint64_t>(uint64_t(g->n) + 1);
    s->targets = dalloc<uint32_t>(s->m2);
    k_slice_offsets<<<std::min<uint64_t>((uint64_t(g->n) + 256) / 256, 148 * 8), 256>>>(
        g->offsets, g->n, lo, hi, s->offsets);
    NULPA_CUDA(cudaGetLastError());
    if (s->m2)
      NULPA_CUDA(cudaMemcpy(s->targets, g->targets + range[0], s->m2 * 4,
                            cudaMemcpyDeviceToDevice));
    if (g->weights) {
      s->weights = dalloc<float>(s->m2);
      if (s->m2)
        NULPA_CUDA(cudaMemcpy(s->weights, g->weights + range[0], s->m2 * 4,
                              cudaMemcpyDeviceToDevice));
    }
    if (g->perm) {
      s->perm = dalloc<uint32_t>(g->n);
      s->inv = dalloc<uint32_t>(g->n);
      NULPA_CUDA(cudaMemcpy(s->perm, g->perm, g->n * 4ull, cudaMemcpyDeviceToDevice));
      NULPA_CUDA(cudaMemcpy(s->inv, g->inv, g->n * 4ull, cudaMemcpyDeviceToDevice));
    }
    finalize_graph(s, 0, /*relayout=*/false);  // already in position order
    s->rows_simple = g->rows_simple;
    s->total_2m = g->total_2m;  // the whole graph's 2m (modularity's normaliser)
  } catch (...) {
    nulpa_graph_free(s);
    throw;
  }
  return s;
}

}  // namespace nulpa

using namespace nulpa;

extern "C" {

int nulpa_graph_slice(nulpa_graph* g, uint32_t v_begin, uint32_t v_end, nulpa_graph** out) {
  return guarded([&] {
    if (!g || !out) throw Error(NULPA_EINVAL, "null argument");
    *out = slice_graph(g, v_begin, v_end);
  });
}

int nulpa_graph_download_raw(const nulpa_graph* g, uint64_t* offsets, uint32_t* targets,
                             float* weights) {
  return guarded([&] {
    if (!g) throw Error(NULPA_EINVAL, "null graph");
    use_device(g->device);
    if (offsets)
      NULPA_CUDA(cudaMemcpy(offsets, g->offsets, (uint64_t(g->n) + 1) * 8, cudaMemcpyDeviceToHost));
    if (targets && g->m2)
      NULPA_CUDA(cudaMemcpy(targets, g->targets, g->m2 * 4, cudaMemcpyDeviceToHost));
    if (weights && g->m2) {
      if (g->weights)
        NULPA_CUDA(cudaMemcpy(weights, g->weights, g->m2 * 4, cudaMemcpyDeviceToHost));
      else
        std::fill(weights, weights + g->m2, 1.0f);
    }
  });
}

int nulpa_graph_download_layout(const nulpa_graph* g, uint32_t* perm, uint32_t* inv,
                                int* rows_simple) {
  return guarded([&] {
    if (!g) throw Error(NULPA_EINVAL, "null graph");
    use_device(g->device);
    if (!g->perm) throw Error(NULPA_EINVAL, "graph has the identity layout");
    if (perm) NULPA_CUDA(cudaMemcpy(perm, g->perm, g->n * 4ull, cudaMemcpyDeviceToHost));
    if (inv) NULPA_CUDA(cudaMemcpy(inv, g->inv, g->n * 4ull, cudaMemcpyDeviceToHost));
    if (rows_simple) *rows_simple = g->rows_simple ? 1 : 0;
  });
}

int nulpa_graph_upload_positioned(const nulpa_csr* csr, const uint32_t* perm,
                                  const uint32_t* inv, int rows_simple, int device,
                                  nulpa_graph** out) {
  return guarded([&] {
    if (!csr || !out || !csr->offsets || (csr->m2 && !csr->targets) || !perm || !inv)
      throw Error(NULPA_EINVAL, "null argument");
    use_device(device);
    auto* g = new nulpa_graph();
    try {
      g->device = device;
      g->n = csr->n;
      g->m2 = csr->m2;
      g->owns = true;
      g->offsets = dalloc<uint64_t>(uint64_t(csr->n) + 1);
      g->targets = dalloc<uint32_t>(csr->m2);
      NULPA_CUDA(cudaMemcpy(g->offsets, csr->offsets, (uint64_t(csr->n) + 1) * 8,
                            cudaMemcpyHostToDevice));
      if (csr->m2)
        NULPA_CUDA(cudaMemcpy(g->targets, csr->targets, csr->m2 * 4, cudaMemcpyHostToDevice));
      if (csr->weights) {
        g->weights = dalloc<float>(csr->m2);
        if (csr->m2)
          NULPA_CUDA(cudaMemcpy(g->weights, csr->weights, csr->m2 * 4, cudaMemcpyHostToDevice));
      }
      g->perm = dalloc<uint32_t>(csr->n);
      g->inv = dalloc<uint32_t>(csr->n);
      NULPA_CUDA(cudaMemcpy(g->perm, perm, csr->n * 4ull, cudaMemcpyHostToDevice));
      NULPA_CUDA(cudaMemcpy(g->inv, inv, csr->n * 4ull, cudaMemcpyHostToDevice));
      g->layout = NULPA_LAYOUT_DEGREE_BUCKETS;
      finalize_graph(g, 0, /*relayout=*/false);  // positioned by the caller
      g->rows_simple = rows_simple != 0;
    } catch (...) {
      nulpa_graph_free(g);
      throw;
    }
    *out = g;
  });
}

int nulpa_community_sums_graph(nulpa_graph* g, const uint32_t* labels_pos_dev, double* sigma_dev,
                               double* big_dev) {
  return guarded([&] {
    if (!g || !labels_pos_dev || !sigma_dev || !big_dev) throw Error(NULPA_EINVAL, "null argument");
    use_device(g->device);
    NULPA_CUDA(cudaMemsetAsync(sigma_dev, 0, g->n * sizeof(double), 0));
    NULPA_CUDA(cudaMemsetAsync(big_dev, 0, g->n * sizeof(double), 0));
    accumulate_sigma(g, labels_pos_dev, sigma_dev, big_dev, 0);
    NULPA_CUDA(cudaStreamSynchronize(0));
  });
}

}  // extern "C"
