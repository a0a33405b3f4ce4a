// The ν-LPA iteration driver on the device.
//
// run_engine (lpa.cpp:246-315) re-stated for the GPU: identity labels, flags
// set for isolated vertices, Pick-Less on iterations ≡ 0 (mod pl_period),
// cross-check on iterations ≡ 0 (mod cc_period), flags reset on the first
// non-PL pass after a PL pass (or every pass without pruning), ΔN net of
// reverts, convergence iff a non-PL pass changes fewer than tolerance·n
// vertices. One stream; the ΔN/counter read-back is the only per-pass host
// synchronisation. elapsed_seconds covers the loop only (lpa.cpp:269,311),
// measured with CUDA events.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <utility>

#include "internal.hpp"
#include "lpa_kernels.cuh"
#include "plan.hpp"

namespace nulpa {

using namespace dev;

namespace {

__global__ void k_init(uint32_t* lab, uint8_t* flags, const uint64_t* off, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    lab[i] = i;
    if (flags) flags[i] = (off[i + 1] == off[i]) ? 1 : 0;  // isolated: never examined
  }
}

inline unsigned grid_for(uint64_t work, unsigned per_block, unsigned cap) {
  const uint64_t b = (work + per_block - 1) / per_block;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(b, cap)));
}

template <typename K>
void allow_smem(K kernel, size_t bytes) {
  NULPA_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
}

// Optional per-tier CUDA-event timing (tuning.profile).
struct Prof {
  bool on = false;
  cudaEvent_t ev[kTiers][2];
  bool used[kTiers];
  void begin(int t, cudaStream_t s) {
    used[t] = true;
    if (on) cudaEventRecord(ev[t][0], s);
  }
  void end(int t, cudaStream_t s) {
    if (on) cudaEventRecord(ev[t][1], s);
  }
};

// One pass over every tier (SURVEY §3.1 "new B200 stack"). `ctr` holds one
// C_COUNT block per tier. Returns the number of kernels launched.
template <int MODE, typename W, bool WEIGHTED>
int launch_pass(const Plan& p, PassCtx c, unsigned long long* ctr, cudaStream_t s, int sms,
                Prof& prof) {
  constexpr size_t warp_smem = (kBlockThreads / 32) * kWarpCap * (sizeof(uint32_t) + sizeof(W));
  constexpr size_t block_smem = kBlockCap * (sizeof(uint32_t) + sizeof(W));
  static bool init = false;
  if (!init) {
    allow_smem(k_warp<MODE, W, WEIGHTED>, warp_smem);
    allow_smem(k_block<MODE, W, WEIGHTED>, block_smem);
    allow_smem(k_hub_accum<MODE, W, WEIGHTED>, block_smem);
    init = true;
  }
  int launches = 0;
  if (p.count[0]) {
    c.ctr = ctr + 0 * C_COUNT;
    prof.begin(0, s);
    const unsigned gb = grid_for(p.count[0], 256, sms * 8);
    if (p.thread_max <= 8)
      k_thread<MODE, W, WEIGHTED, 8><<<gb, 256, 0, s>>>(c, p.list[0], p.count[0]);
    else
      k_thread<MODE, W, WEIGHTED, 16><<<gb, 256, 0, s>>>(c, p.list[0], p.count[0]);
    prof.end(0, s);
    ++launches;
  }
  if (p.count[1]) {
    c.ctr = ctr + 1 * C_COUNT;
    prof.begin(1, s);
    k_warp<MODE, W, WEIGHTED><<<grid_for(p.count[1], kBlockThreads / 32, sms * 3), kBlockThreads,
                                warp_smem, s>>>(c, p.list[1], p.count[1]);
    prof.end(1, s);
    ++launches;
  }
  if (p.count[2]) {
    c.ctr = ctr + 2 * C_COUNT;
    prof.begin(2, s);
    k_block<MODE, W, WEIGHTED><<<grid_for(p.count[2], 1, sms * 3), kBlockThreads, block_smem, s>>>(
        c, p.list[2], p.count[2]);
    prof.end(2, s);
    ++launches;
  }
  if (p.n_hubs) {
    c.ctr = ctr + 3 * C_COUNT;
    prof.begin(3, s);
    const HubCtx h = p.hub_ctx();
    const unsigned gi = grid_for(p.n_items, 1, sms * 3);
    const unsigned gh = grid_for(p.n_hubs, 256, 1024);
    k_hub_select<MODE><<<gh, 256, 0, s>>>(c, h);
    k_hub_accum<MODE, W, WEIGHTED><<<gi, kBlockThreads, block_smem, s>>>(c, h);
    k_hub_argmax<W><<<gi, kBlockThreads, 0, s>>>(h);
    launches += 3;
    if constexpr (sizeof(W) == 8) {
      k_hub_argmax_key_f64<<<gi, kBlockThreads, 0, s>>>(h);
      ++launches;
    }
    k_hub_decide<MODE, W><<<gh, 256, 0, s>>>(c, h);
    ++launches;
    if (MODE == kAsync && c.flags) {
      k_hub_wake<<<gi, kBlockThreads, 0, s>>>(c, h);
      ++launches;
    }
    prof.end(3, s);
  }
  NULPA_CUDA(cudaGetLastError());
  return launches;
}

template <int MODE>
int dispatch_pass(const Plan& p, const PassCtx& c, unsigned long long* ctr, int value_bytes,
                  cudaStream_t s, int sms, Prof& prof) {
  const bool weighted = c.g.w != nullptr;
  if (value_bytes == 8)
    return weighted ? launch_pass<MODE, double, true>(p, c, ctr, s, sms, prof)
                    : launch_pass<MODE, double, false>(p, c, ctr, s, sms, prof);
  return weighted ? launch_pass<MODE, float, true>(p, c, ctr, s, sms, prof)
                  : launch_pass<MODE, float, false>(p, c, ctr, s, sms, prof);
}

template <typename W, bool WEIGHTED>
void launch_sequential(const PassCtx& c, uint32_t* gkeys, void* gvals, cudaStream_t s) {
  constexpr size_t smem = kBlockCap * (sizeof(uint32_t) + sizeof(W));
  static bool init = false;
  if (!init) {
    allow_smem(k_sequential<W, WEIGHTED>, smem);
    init = true;
  }
  k_sequential<W, WEIGHTED><<<1, kBlockThreads, smem, s>>>(c, gkeys, static_cast<W*>(gvals));
  NULPA_CUDA(cudaGetLastError());
}

void validate_opts(const nulpa_graph* g, const nulpa_opts& o) {
  // validate_config, lpa.cpp:317-326 — identical messages.
  if (g->n == 0) throw Error(NULPA_EINVAL, "label propagation requires a non-empty graph");
  if (!(o.tolerance > 0.0 && o.tolerance <= 1.0))
    throw Error(NULPA_EINVAL, "tolerance must lie in (0, 1]");
  if (o.max_iterations < 1) throw Error(NULPA_EINVAL, "max-iterations must be >= 1");
  if (o.pl_period < 0) throw Error(NULPA_EINVAL, "pl-period must be >= 0");
  if (o.cc_period < 0) throw Error(NULPA_EINVAL, "cc-period must be >= 0");
  if (o.switch_degree < 2) throw Error(NULPA_EINVAL, "switch-degree must be >= 2");
  if (o.workers < 0) throw Error(NULPA_EINVAL, "workers must be >= 0");
  if (o.exec < 0 || o.exec > 2) throw Error(NULPA_EINVAL, "unknown execution mode");
  if (o.strategy < 0 || o.strategy > 3) throw Error(NULPA_EINVAL, "unknown probe strategy");
}

struct Stream {
  cudaStream_t s = nullptr;
  Stream() { NULPA_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~Stream() {
    if (s) cudaStreamDestroy(s);
  }
};

template <typename T>
struct DBuf {
  T* p = nullptr;
  DBuf() = default;
  explicit DBuf(size_t n) : p(dalloc<T>(n)) {}
  ~DBuf() { dfree(p); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(DBuf&& o) noexcept {
    std::swap(p, o.p);
    return *this;
  }
};

struct Pinned {
  unsigned long long* p = nullptr;
  explicit Pinned(size_t count = C_COUNT) {
    NULPA_CUDA(cudaHostAlloc(&p, count * sizeof(unsigned long long), cudaHostAllocDefault));
  }
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};

// cross_check (lpa.cpp:338-360) on the device; returns the revert count.
uint64_t device_cross_check(nulpa_graph* g, uint32_t* lab, const uint32_t* prev, uint8_t* flags,
                            unsigned long long* d_aux, unsigned long long* h_aux, cudaStream_t s,
                            int sms, uint64_t* launches = nullptr) {
  const uint32_t n = g->n;
  DBuf<uint8_t> r0(n), r1(n);
  NULPA_CUDA(cudaMemsetAsync(r0.p, 0, n, s));
  uint8_t* rin = r0.p;
  uint8_t* rout = r1.p;
  const unsigned gb = grid_for(n, 256, sms * 8);
  for (uint32_t round = 0; round <= n; ++round) {
    NULPA_CUDA(cudaMemsetAsync(d_aux, 0, sizeof(unsigned long long), s));
    k_cc_round<<<gb, 256, 0, s>>>(lab, prev, rin, rout, n, d_aux);
    NULPA_CUDA(cudaGetLastError());
    if (launches) ++*launches;
    NULPA_CUDA(cudaMemcpyAsync(h_aux, d_aux, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    NULPA_CUDA(cudaStreamSynchronize(s));
    std::swap(rin, rout);
    if (*h_aux == 0) break;
  }
  Graph dg{g->offsets, g->targets, g->weights, n};
  NULPA_CUDA(cudaMemsetAsync(d_aux, 0, sizeof(unsigned long long), s));
  k_cc_apply<<<grid_for(n, 256, sms * 8), 256, 0, s>>>(dg, lab, prev, rin, flags, d_aux);
  NULPA_CUDA(cudaGetLastError());
  if (launches) ++*launches;
  NULPA_CUDA(cudaMemcpyAsync(h_aux, d_aux, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  return *h_aux;
}

}  // namespace

void run_lpa(nulpa_graph* g, const nulpa_opts& o, const nulpa_tuning* tuning,
             uint32_t* labels_host, uint32_t* labels_dev_out, nulpa_stats* st) {
  validate_opts(g, o);
  use_device(g->device);
  const auto t_setup = std::chrono::steady_clock::now();
  Stream stream;
  cudaStream_t s = stream.s;
  const int sms = sm_count();
  const int vbytes = o.precision == 64 ? 8 : 4;
  const uint32_t n = g->n;
  Plan* p = get_plan(g, resolve_tiers(o.switch_degree, tuning), vbytes, s);

  DBuf<uint32_t> lab0(n), lab1, prev, changed;
  DBuf<uint8_t> flags(n);
  constexpr int kCtr = kTiers * C_COUNT;
  DBuf<unsigned long long> ctr(kCtr);
  unsigned long long* ctr_other = ctr.p + 4 * C_COUNT;
  Pinned hc(kCtr);
  if (o.exec == NULPA_EXEC_SYNCHRONOUS) {
    lab1 = DBuf<uint32_t>(n);
    changed = DBuf<uint32_t>(n);
  }
  if (o.cc_period > 0) prev = DBuf<uint32_t>(n);
  DBuf<uint32_t> seq_keys;
  DBuf<unsigned char> seq_vals;
  if (o.exec == NULPA_EXEC_SEQUENTIAL) {
    const uint64_t cap = pow2_ceil(2 * std::max<uint32_t>(g->max_degree, 1));
    if (cap > static_cast<uint64_t>(kBlockCap)) {
      seq_keys = DBuf<uint32_t>(cap);
      seq_vals = DBuf<unsigned char>(cap * vbytes);
    }
  }
  Prof prof;
  prof.on = tuning && tuning->profile;
  if (prof.on)
    for (auto& e : prof.ev) {
      NULPA_CUDA(cudaEventCreate(&e[0]));
      NULPA_CUDA(cudaEventCreate(&e[1]));
    }
  k_init<<<grid_for(n, 256, sms * 8), 256, 0, s>>>(lab0.p, flags.p, g->offsets, n);
  NULPA_CUDA(cudaGetLastError());
  NULPA_CUDA(cudaStreamSynchronize(s));
  const double setup_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t_setup).count();

  cudaEvent_t ev0, ev1;
  NULPA_CUDA(cudaEventCreate(&ev0));
  NULPA_CUDA(cudaEventCreate(&ev1));
  NULPA_CUDA(cudaEventRecord(ev0, s));

  const Graph dg{g->offsets, g->targets, g->weights, n};
  int iterations = 0, pl_iterations = 0;
  bool converged = false;
  uint64_t cc_reverts = 0, tot_v = 0, tot_e = 0, tot_w = 0, launches = 0;
  double tier_ms[kTiers] = {0}, tier_bytes[kTiers] = {0};
  uint64_t tier_edges[kTiers] = {0};
  uint32_t tier_passes[kTiers] = {0};
  const double edge_bytes = g->weights ? 12.0 : 8.0;
  uint32_t* cur = lab0.p;
  uint32_t* nxt = lab1.p;

  for (int iter = 0; iter < o.max_iterations; ++iter) {
    const bool pick_less = o.pl_period > 0 && iter % o.pl_period == 0;
    const bool check = o.cc_period > 0 && iter % o.cc_period == 0;
    if (check) NULPA_CUDA(cudaMemcpyAsync(prev.p, cur, n * 4ull, cudaMemcpyDeviceToDevice, s));
    const bool was_pl = iter > 0 && o.pl_period > 0 && (iter - 1) % o.pl_period == 0;
    if (!o.prune || (was_pl && !pick_less)) NULPA_CUDA(cudaMemsetAsync(flags.p, 0, n, s));
    NULPA_CUDA(cudaMemsetAsync(ctr.p, 0, kCtr * sizeof(unsigned long long), s));
    for (bool& u : prof.used) u = false;

    PassCtx c;
    c.g = dg;
    c.flags = flags.p;
    c.ctr = ctr.p;
    c.pick_less = pick_less ? 1 : 0;
    c.strategy = o.strategy;
    c.changed = nullptr;
    c.changed_n = ctr_other + C_NCHANGED;
    if (o.exec == NULPA_EXEC_PARALLEL_ASYNC) {
      c.lab_in = cur;
      c.lab_out = cur;
      launches += dispatch_pass<kAsync>(*p, c, ctr.p, vbytes, s, sms, prof);
    } else if (o.exec == NULPA_EXEC_SYNCHRONOUS) {
      // sync_move (lpa.cpp:70-100): frozen snapshot `cur`, staged writes to `nxt`,
      // wake-ups after the joint application.
      NULPA_CUDA(cudaMemcpyAsync(nxt, cur, n * 4ull, cudaMemcpyDeviceToDevice, s));
      c.lab_in = cur;
      c.lab_out = nxt;
      c.changed = changed.p;
      launches += dispatch_pass<kSync>(*p, c, ctr.p, vbytes, s, sms, prof);
      prof.begin(4, s);
      k_wake_list<<<grid_for(n, kBlockThreads / 32, sms * 8), kBlockThreads, 0, s>>>(
          dg, flags.p, changed.p, ctr_other + C_NCHANGED, ctr_other);
      prof.end(4, s);
      ++launches;
      NULPA_CUDA(cudaGetLastError());
      std::swap(cur, nxt);
    } else {
      c.lab_in = cur;
      c.lab_out = cur;
      c.ctr = ctr_other;
      prof.begin(4, s);
      if (vbytes == 8) {
        if (dg.w)
          launch_sequential<double, true>(c, seq_keys.p, seq_vals.p, s);
        else
          launch_sequential<double, false>(c, seq_keys.p, seq_vals.p, s);
      } else {
        if (dg.w)
          launch_sequential<float, true>(c, seq_keys.p, seq_vals.p, s);
        else
          launch_sequential<float, false>(c, seq_keys.p, seq_vals.p, s);
      }
      prof.end(4, s);
      ++launches;
    }
    uint64_t reverted = 0;
    if (check)
      reverted = device_cross_check(g, cur, prev.p, flags.p, ctr_other + C_AUX, hc.p + 4 * C_COUNT + C_AUX,
                                    s, sms, &launches);
    NULPA_CUDA(cudaMemcpyAsync(hc.p, ctr.p, kCtr * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s));
    NULPA_CUDA(cudaStreamSynchronize(s));
    uint64_t raw_dn = 0;
    for (int t = 0; t < kTiers; ++t) {
      const unsigned long long* k = hc.p + t * C_COUNT;
      if (k[C_FAIL])
        throw Error(NULPA_EINTERNAL, "hashtable insertion failed (capacity invariant violated)");
      raw_dn += k[C_DN];
      tot_v += k[C_PROC_V];
      tot_e += k[C_PROC_E];
      tot_w += k[C_WAKE_E];
      tier_edges[t] += k[C_PROC_E];
      // SURVEY §8d per tier: flag sweep over the tier's list (1 B), row bounds
      // + own label of processed vertices (12 B), target + neighbour label
      // (+ weight) per scanned edge, label write per change, wake store per
      // neighbour of a changed vertex.
      const double list_len = t < 4 ? (t < 3 ? p->count[t] : p->n_hubs) : 0.0;
      tier_bytes[t] += list_len + 12.0 * k[C_PROC_V] + edge_bytes * k[C_PROC_E] +
                       4.0 * k[C_DN] + double(k[C_WAKE_E]);
      if (prof.used[t]) {
        ++tier_passes[t];
        if (prof.on) {
          float tms = 0.f;
          NULPA_CUDA(cudaEventElapsedTime(&tms, prof.ev[t][0], prof.ev[t][1]));
          tier_ms[t] += tms;
        }
      }
    }
    const uint64_t dn = raw_dn - reverted;
    cc_reverts += reverted;
    if (st && st->delta_n) st->delta_n[iterations] = dn;
    ++iterations;
    if (pick_less) ++pl_iterations;
    if (!pick_less && static_cast<double>(dn) / n < o.tolerance) {
      converged = true;
      break;
    }
  }
  NULPA_CUDA(cudaEventRecord(ev1, s));
  NULPA_CUDA(cudaEventSynchronize(ev1));
  float ms = 0.f;
  NULPA_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  if (prof.on)
    for (auto& e : prof.ev) {
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }

  if (labels_host)
    NULPA_CUDA(cudaMemcpyAsync(labels_host, cur, n * 4ull, cudaMemcpyDeviceToHost, s));
  if (labels_dev_out)
    NULPA_CUDA(cudaMemcpyAsync(labels_dev_out, cur, n * 4ull, cudaMemcpyDeviceToDevice, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  if (st) {
    st->iterations = iterations;
    st->converged = converged ? 1 : 0;
    st->pl_iterations = pl_iterations;
    st->reserved = 0;
    st->cc_reverts = cc_reverts;
    st->elapsed_seconds = ms * 1e-3;
    st->processed_vertices = tot_v;
    st->processed_edges = tot_e;
    st->wake_edges = tot_w;
    double total = 0.0;
    for (int t = 0; t < kTiers; ++t) {
      st->tier_ms[t] = tier_ms[t];
      st->tier_bytes[t] = tier_bytes[t];
      st->tier_edges[t] = tier_edges[t];
      st->tier_passes[t] = tier_passes[t];
      total += tier_bytes[t];
    }
    st->algorithmic_bytes = static_cast<uint64_t>(total);
    st->setup_seconds = setup_s;
    st->kernel_launches = launches;
  }
}

uint64_t run_sync_step(nulpa_graph* g, const uint32_t* lab_in_dev, int pick_less, int strategy,
                       int precision, uint32_t* lab_out_dev) {
  use_device(g->device);
  if (strategy < 0 || strategy > 3) throw Error(NULPA_EINVAL, "unknown probe strategy");
  Stream stream;
  cudaStream_t s = stream.s;
  const int sms = sm_count();
  const int vbytes = precision == 64 ? 8 : 4;
  Plan* p = get_plan(g, resolve_tiers(32, nullptr), vbytes, s);
  constexpr int kCtr = kTiers * C_COUNT;
  DBuf<unsigned long long> ctr(kCtr);
  Pinned hc(kCtr);
  NULPA_CUDA(cudaMemsetAsync(ctr.p, 0, kCtr * sizeof(unsigned long long), s));
  NULPA_CUDA(cudaMemcpyAsync(lab_out_dev, lab_in_dev, g->n * 4ull, cudaMemcpyDeviceToDevice, s));
  PassCtx c;
  c.g = Graph{g->offsets, g->targets, g->weights, g->n};
  c.lab_in = lab_in_dev;
  c.lab_out = lab_out_dev;
  c.flags = nullptr;
  c.ctr = ctr.p;
  c.changed = nullptr;
  c.changed_n = ctr.p + 4 * C_COUNT + C_NCHANGED;
  c.pick_less = pick_less ? 1 : 0;
  c.strategy = strategy;
  Prof prof;
  dispatch_pass<kSync>(*p, c, ctr.p, vbytes, s, sms, prof);
  NULPA_CUDA(cudaMemcpyAsync(hc.p, ctr.p, kCtr * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s));
  NULPA_CUDA(cudaStreamSynchronize(s));
  uint64_t dn = 0;
  for (int t = 0; t < kTiers; ++t) {
    if (hc.p[t * C_COUNT + C_FAIL])
      throw Error(NULPA_EINTERNAL, "hashtable insertion failed (capacity invariant violated)");
    dn += hc.p[t * C_COUNT + C_DN];
  }
  return dn;
}

uint64_t run_cross_check(nulpa_graph* g, uint32_t* lab_dev, const uint32_t* prev_dev,
                         uint8_t* flags_dev) {
  use_device(g->device);
  Stream stream;
  DBuf<unsigned long long> aux(1);
  Pinned hc;
  return device_cross_check(g, lab_dev, prev_dev, flags_dev, aux.p, hc.p, stream.s, sm_count());
}

}  // namespace nulpa

// ---- C ABI ---------------------------------------------------------------------------

using namespace nulpa;

namespace {

struct HostGraph {
  nulpa_graph* g = nullptr;
  HostGraph(const nulpa_csr* csr, int device) {
    const int rc = nulpa_graph_upload(csr, device, &g);
    if (rc != NULPA_OK) throw Error(rc, nulpa_last_error());
  }
  ~HostGraph() {
    if (g) nulpa_graph_free(g);
  }
};

template <typename T>
struct DevArray {
  T* p = nullptr;
  size_t n = 0;
  DevArray(size_t count) : p(dalloc<T>(count)), n(count) {}
  ~DevArray() { dfree(p); }
  void upload(const T* h) {
    if (n) NULPA_CUDA(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice));
  }
  void download(T* h) const {
    if (n) NULPA_CUDA(cudaMemcpy(h, p, n * sizeof(T), cudaMemcpyDeviceToHost));
  }
};

}  // namespace

extern "C" {

void nulpa_default_opts(nulpa_opts* o) {
  o->tolerance = 0.05;
  o->max_iterations = 20;
  o->pl_period = 4;
  o->cc_period = 0;
  o->strategy = NULPA_PROBE_QUADRATIC_DOUBLE;
  o->switch_degree = 32;
  o->precision = 32;
  o->exec = NULPA_EXEC_PARALLEL_ASYNC;
  o->workers = 0;
  o->seed = 0;
  o->prune = 1;
  o->device = 0;
}

int nulpa_run_graph(nulpa_graph* g, const nulpa_opts* opts, const nulpa_tuning* tuning,
                    uint32_t* labels_host, uint32_t* labels_device, nulpa_stats* stats) {
  return guarded([&] {
    if (!g || !opts) throw Error(NULPA_EINVAL, "null argument");
    run_lpa(g, *opts, tuning, labels_host, labels_device, stats);
  });
}

int nulpa_run(const nulpa_csr* csr, const nulpa_opts* opts, const nulpa_tuning* tuning,
              uint32_t* labels_out, nulpa_stats* stats) {
  return guarded([&] {
    if (!opts) throw Error(NULPA_EINVAL, "null options");
    check_host_csr(csr);
    nulpa_graph probe;  // validate before any device work (lpa.cpp:363)
    probe.n = csr->n;
    validate_opts(&probe, *opts);
    HostGraph hg(csr, opts->device);
    run_lpa(hg.g, *opts, tuning, labels_out, nullptr, stats);
  });
}

int nulpa_sync_step_graph(nulpa_graph* g, const uint32_t* in, int pick_less, int strategy,
                          int precision, uint32_t* out, uint64_t* changed) {
  return guarded([&] {
    if (!g) throw Error(NULPA_EINVAL, "null graph");
    const uint64_t dn = run_sync_step(g, in, pick_less, strategy, precision, out);
    if (changed) *changed = dn;
  });
}

int nulpa_sync_step(const nulpa_csr* csr, const uint32_t* labels_in, int pick_less, int strategy,
                    int precision, uint32_t* labels_out, uint64_t* changed) {
  return guarded([&] {
    check_host_csr(csr);
    HostGraph hg(csr, 0);
    DevArray<uint32_t> in(csr->n), out(csr->n);
    in.upload(labels_in);
    const uint64_t dn = run_sync_step(hg.g, in.p, pick_less, strategy, precision, out.p);
    out.download(labels_out);
    if (changed) *changed = dn;
  });
}

int nulpa_cross_check(const nulpa_csr* csr, uint32_t* labels, const uint32_t* prev,
                      uint8_t* flags, uint64_t* reverted) {
  return guarded([&] {
    check_host_csr(csr);
    HostGraph hg(csr, 0);
    const uint32_t n = csr->n;
    DevArray<uint32_t> l(n), pv(n);
    DevArray<uint8_t> f(n);
    l.upload(labels);
    pv.upload(prev);
    f.upload(flags);
    const uint64_t r = run_cross_check(hg.g, l.p, pv.p, f.p);
    l.download(labels);
    f.download(flags);
    if (reverted) *reverted = r;
  });
}

int nulpa_partition_by_degree(const nulpa_csr* csr, uint32_t switch_degree, uint32_t* low,
                              uint64_t* n_low, uint32_t* high, uint64_t* n_high) {
  return guarded([&] {
    // partition_by_degree, lpa.cpp:330-336 (same message).
    if (switch_degree < 2) throw Error(NULPA_EINVAL, "switch-degree must be >= 2");
    check_host_csr(csr);
    HostGraph hg(csr, 0);
    nulpa_graph* g = hg.g;
    Stream stream;
    DevArray<uint32_t> d_low(g->n + 1), d_high(g->n + 1);
    uint64_t nl = 0, nh = 0;
    partition_two_way(g->offsets, g->n, switch_degree, d_low.p, d_high.p, &nl, &nh, stream.s);
    if (nl) NULPA_CUDA(cudaMemcpy(low, d_low.p, nl * 4, cudaMemcpyDeviceToHost));
    if (nh) NULPA_CUDA(cudaMemcpy(high, d_high.p, nh * 4, cudaMemcpyDeviceToHost));
    *n_low = nl;
    *n_high = nh;
  });
}

}  // extern "C"
