// Internal host-side declarations shared by the nulpa translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>

#include "nulpa/nulpa.h"

namespace nulpa {

// Thrown inside the library, caught at the C-ABI edge and turned into a code.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);
const std::string& last_error();

#define NULPA_CUDA(call)                                                                   \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      (void)cudaGetLastError();                                                            \
      throw ::nulpa::Error(e_ == cudaErrorMemoryAllocation ? NULPA_ENOMEM : NULPA_ECUDA,   \
                           std::string(#call) + ": " + cudaGetErrorString(e_));           \
    }                                                                                      \
  } while (0)

// Run `f` and convert exceptions into C-ABI error codes.
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return NULPA_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc& e) {
    set_last_error(std::string("out of memory: ") + e.what());
    return NULPA_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return NULPA_EOTHER;
  }
}

// Select a device, failing loudly when none is usable (no CPU fallback).
void use_device(int device);
// Device for C-ABI calls that take none: NULPA_DEVICE when set (the C++ drop-in's rule),
// else the calling thread's current device.
int default_device();

// Device allocation that throws Error(NULPA_ENOMEM) on failure.
void* dmalloc(size_t bytes);
void dfree(void* p);

template <typename T>
T* dalloc(size_t count) {
  return static_cast<T*>(dmalloc(count * sizeof(T) + (count == 0 ? 16 : 0)));
}

// Host-side phase timestamps on stderr when NULPA_TRACE is set (diagnostics only).
struct Trace {
  explicit Trace(const char* scope);
  ~Trace();
  void mark(const char* what);
  bool on;
  const char* scope;
  double t0, last;
};

struct Plan;
}  // namespace nulpa

// The resident graph (opaque in the C ABI).
struct nulpa_graph {
  int device = 0;
  uint32_t n = 0;
  uint64_t m2 = 0;
  uint64_t* offsets = nullptr;  // device
  uint32_t* targets = nullptr;  // device
  float* weights = nullptr;     // device, nullptr = unit weights
  bool owns = false;
  uint32_t max_degree = 0;
  double total_2m = 0.0;  // sum of stored weights (graph.cpp:170-171)
  bool rows_simple = false;  // every row strictly ascending (no duplicate targets)
  // Position-order layout (layout.cu): the arrays above are stored by position;
  // perm[p] = vertex id at position p, inv[v] = position of vertex v. Both are
  // nullptr under the identity layout (position == vertex id).
  int layout = NULPA_LAYOUT_IDENTITY;
  uint32_t* perm = nullptr;  // device
  uint32_t* inv = nullptr;   // device
  // Chunk-major low range (layout.cu build_perm): positions [chunk_lo, chunk_lo + chunk_n)
  // hold the rows of degree 1..8 transposed for a chunk walk of chunk_n / chunk_L threads
  // (entry e = k * chunk_L + r of the range's bucket order sits at column r, row k).
  // chunk_n = 0: no such range.
  uint32_t chunk_lo = 0, chunk_n = 0, chunk_L = 0;
  uint32_t chunk_dmax = 0;  // the range's largest degree (<= 8)
  nulpa::Plan* plan = nullptr;  // cached tiering (plan.hpp)
  // Held by every call that uses `plan`: the cached plan (and its hub tables and
  // wide-tier scratch) is shared state, so runs on one graph handle are serialised.
  std::recursive_mutex plan_mu;
};

namespace nulpa {
// Validate a host CSR the way CsrGraph's constructor does (graph.cpp:165-172).
void check_host_csr(const nulpa_csr* csr);
// Fill max_degree / total_2m of a resident graph (device reductions), then move it to the
// default layout. `relayout = false` for arrays that are already in position order (a
// rank's row slice, an upload with a given permutation).
void finalize_graph(nulpa_graph* g, cudaStream_t s, bool relayout = true);
// partition_by_degree (lpa.cpp:330-336) on the device: ascending-id lists of
// deg < switch_degree and deg >= switch_degree.
void partition_two_way(const uint64_t* off, uint32_t n, uint32_t switch_degree, uint32_t* low,
                       uint32_t* high, uint64_t* n_low, uint64_t* n_high, cudaStream_t s);
// Device modularity on a resident graph (quality.cu).
double modularity_device(nulpa_graph* g, const uint32_t* labels_dev, cudaStream_t s);
}  // namespace nulpa
