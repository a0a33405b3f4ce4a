// Position-order residency of the CSR (layout.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>

#include "internal.hpp"

namespace nulpa {

int default_layout();
// Reorder a freshly built resident graph into degree-bucket position order
// (no-op under NULPA_LAYOUT_IDENTITY); sets g->perm / g->inv / g->layout.
void relayout_graph(nulpa_graph* g, cudaStream_t s);
// pos[p] = vtx[perm[p]]  /  vtx[v] = pos[inv[v]]  (copies under the identity layout).
void to_positions_u32(const nulpa_graph* g, const uint32_t* vtx, uint32_t* pos, cudaStream_t s);
void to_vertices_u32(const nulpa_graph* g, const uint32_t* pos, uint32_t* vtx, cudaStream_t s);
void to_positions_u8(const nulpa_graph* g, const uint8_t* vtx, uint8_t* pos, cudaStream_t s);
void to_vertices_u8(const nulpa_graph* g, const uint8_t* pos, uint8_t* vtx, cudaStream_t s);
// Host CSR upload with the relayout overlapped with the transfer (unit weights,
// bucketed layout); fills offsets/targets/perm/inv/max_degree/total_2m/rows_simple.
// `while_streaming` runs on the host once every chunk copy is queued, i.e. while
// the targets are still crossing PCIe (it may use g->offsets / max_degree / perm).
bool can_upload_pipelined(const nulpa_csr* csr);
void upload_pipelined(const nulpa_csr* csr, nulpa_graph* g,
                      const std::function<void()>& while_streaming = {});
// Download the CSR in the input's vertex numbering.
void download_vertex_order(const nulpa_graph* g, uint64_t* off_h, uint32_t* tgt_h, float* w_h);

}  // namespace nulpa
