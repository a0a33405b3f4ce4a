/* nulpa — B200-native ν-LPA label propagation: the C-ABI boundary.
 *
 * Plain pointers and sizes only; no torch or C++ types cross this boundary.
 * Every entry point replaces one reference interface (paths relative to
 * /root/reference/proj) and keeps its argument meaning and error behaviour:
 *
 *   nulpa_run              labelprop::lpa(const CsrGraph&, const LpaConfig&)
 *                            include/labelprop/lpa.hpp:84, src/lpa.cpp:362-366
 *   nulpa_sync_step        one sync_move label-choice step from arbitrary labels
 *                            (detail::scan_candidate lpa.hpp:92-111 + lpa.cpp:87-88)
 *   nulpa_modularity       labelprop::modularity  quality.hpp:19, quality.cpp:21-49
 *   nulpa_community_count  labelprop::community_stats(...).count  quality.cpp:56-78
 *   nulpa_cross_check      labelprop::cross_check  lpa.hpp:72-73, lpa.cpp:338-360
 *   nulpa_partition_by_degree  labelprop::partition_by_degree  lpa.hpp:63, lpa.cpp:330-336
 *
 * Error codes (the C++ drop-in in paper_2411_11468_b200/csrc/dropin.cpp maps
 * them back to the reference exceptions, graph.hpp:17-31):
 *   0 ok, 1 invalid argument (ValidationError), 2 out of memory (std::bad_alloc),
 *   3 internal invariant / hashtable failure (InternalError), 4 CUDA error,
 *   5 other. nulpa_last_error() returns the thread-local message.
 *
 * There is no CPU fallback: every compute entry point runs CUDA kernels for
 * sm_100a and fails with code 4 when no CUDA device is usable.
 */
#ifndef NULPA_NULPA_H
#define NULPA_NULPA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NULPA_OK 0
#define NULPA_EINVAL 1
#define NULPA_ENOMEM 2
#define NULPA_EINTERNAL 3
#define NULPA_ECUDA 4
#define NULPA_EOTHER 5
#define NULPA_EFORMAT 6 /* malformed input file (FormatError, graph.hpp:17-19) */

/* Input file formats: labelprop::FileFormat (graph.hpp:86), same values. */
#define NULPA_FORMAT_MATRIX_MARKET 0
#define NULPA_FORMAT_EDGE_LIST 1

/* Probe strategies: labelprop::ProbeStrategy, hashtable.hpp:25 (same values). */
#define NULPA_PROBE_LINEAR 0
#define NULPA_PROBE_QUADRATIC 1
#define NULPA_PROBE_DOUBLE 2
#define NULPA_PROBE_QUADRATIC_DOUBLE 3

/* Exec modes: labelprop::ExecMode, lpa.hpp:20 (same values). */
#define NULPA_EXEC_PARALLEL_ASYNC 0
#define NULPA_EXEC_SEQUENTIAL 1
#define NULPA_EXEC_SYNCHRONOUS 2

/* CSR graph (labelprop::CsrGraph, graph.hpp:53-84): offsets u64[n+1],
 * targets u32[m2], weights f32[m2] or NULL meaning every weight is 1.0f.
 * Rows sorted by target, both directions stored, self-loops stored once.
 * Borrowed: never freed or modified by the library. */
typedef struct nulpa_csr {
  uint32_t n;
  uint32_t reserved;
  uint64_t m2;
  const uint64_t* offsets;
  const uint32_t* targets;
  const float* weights;
} nulpa_csr;

/* labelprop::LpaConfig (lpa.hpp:25-37), field for field, same defaults. */
typedef struct nulpa_opts {
  double tolerance;       /* 0.05 */
  int32_t max_iterations; /* 20 */
  int32_t pl_period;      /* 4; 0 disables pick-less */
  int32_t cc_period;      /* 0; 0 disables cross-check */
  int32_t strategy;       /* NULPA_PROBE_QUADRATIC_DOUBLE */
  uint32_t switch_degree; /* 32: thread-per-vertex below, cooperative at and above */
  int32_t precision;      /* 32 or 64 (hashtable value width) */
  int32_t exec;           /* NULPA_EXEC_PARALLEL_ASYNC */
  int32_t workers;        /* echoed only (no meaning on a GPU) */
  uint64_t seed;          /* echoed only (the reference never uses it either) */
  int32_t prune;          /* 1 */
  int32_t device;         /* CUDA device ordinal (not an LpaConfig field) */
} nulpa_opts;

/* Kernel-tier tuning (not part of LpaConfig). Zero fields take defaults. */
typedef struct nulpa_tuning {
  uint32_t thread_max_degree; /* thread-per-vertex tier upper bound (<= 16) */
  uint32_t warp_max_degree;   /* 32-thread team tier upper bound (<= 256) */
  uint32_t block_max_degree;  /* 128-thread team tier upper bound (<= 1024) */
  uint32_t hub_chunk;         /* edges per CTA work item in the global-table hub tier */
  uint32_t async_first_pass;  /* ParallelAsync pass 0 from identity labels: 0 in place
                                 (default), 1 table-free synchronous first pass
                                 (k_first_pass; a legal schedule, all reads first) */
  uint32_t profile;           /* 1: time each tier with CUDA events (stats.tier_*) */
  uint32_t schedule;          /* ParallelAsync visit order inside each tier:
                                 0 default (= 4), 1 position order (degree buckets,
                                 largest first; ascending id inside a bucket), 2 the
                                 tiers up to block_max scrambled in 32-position blocks,
                                 3 only the register tiers (degree <= 32) scrambled in
                                 32-position blocks, position order above, 4 as 3, but
                                 when the thread tier holds at least half of the edges
                                 (lattice / road-like graphs) each thread walks a
                                 contiguous chunk of it in order, as the reference's
                                 workers walk theirs.
                                 Any order is a valid asynchronous schedule;
                                 Synchronous/Sequential results do not depend on it. */
  uint32_t no_identity_first; /* 1: disable the table-free first pass from identity labels */
  uint32_t unbatched;         /* 1: read the counters back after every pass instead of
                                 enqueueing passes in batches behind the device-side
                                 convergence guard (same results) */
} nulpa_tuning;

#define NULPA_TIERS 10 /* 0 thread, 1 half-warp, 2 warp, 3/4/5 32/128/256-thread teams with
                          shared tables, 6 512-thread CTA per vertex (degree <= 6144), 7 wide
                          rows (one 1024-thread CTA per vertex, label-partitioned phases; an
                          8-CTA DSMEM cluster for weighted graphs), 8 hub (global table),
                          9 other (deferred wake, cross-check, sequential) */

/* labelprop::RunStats (lpa.hpp:39-46) plus device counters for roofline
 * accounting. delta_n must point at >= max_iterations u64 (or be NULL). */
typedef struct nulpa_stats {
  int32_t iterations;
  int32_t converged;
  int32_t pl_iterations;
  int32_t reserved;
  uint64_t cc_reverts;
  double elapsed_seconds; /* iteration loop only, CUDA events (lpa.cpp:269,311) */
  uint64_t* delta_n;      /* caller buffer, delta_n_per_iter */
  /* totals over all passes (SURVEY §8d algorithmic-byte model) */
  uint64_t processed_vertices;
  uint64_t processed_edges;
  uint64_t wake_edges;
  uint64_t algorithmic_bytes;
  double setup_seconds; /* tiering + table allocation before the loop */
  uint64_t kernel_launches;            /* nulpa kernels launched inside the loop */
  double tier_ms[NULPA_TIERS];         /* device time per tier (tuning.profile) */
  double tier_bytes[NULPA_TIERS];      /* algorithmic bytes per tier */
  uint64_t tier_edges[NULPA_TIERS];    /* edges scanned per tier */
  uint32_t tier_passes[NULPA_TIERS];   /* passes in which the tier launched */
  uint32_t reserved2;
} nulpa_stats;

typedef struct nulpa_graph nulpa_graph; /* device-resident CSR */

/* Resident layouts. DEGREE_BUCKETS (the default) stores the rows in POSITION
 * order: vertices grouped by ceil(log2(degree)), largest first, isolated last,
 * ascending id inside a group, so the labels of the high-degree vertices that
 * most edges point at are packed together and stay in L2. Label VALUES are
 * always vertex ids and every label array that crosses this ABI is in vertex
 * order (except the session API below, which works on position-order arrays);
 * results do not depend on the layout. IDENTITY keeps the input numbering. */
#define NULPA_LAYOUT_IDENTITY 0
#define NULPA_LAYOUT_DEGREE_BUCKETS 1

const char* nulpa_last_error(void);
int nulpa_version(void);
void nulpa_default_opts(nulpa_opts* opts);
int nulpa_device_count(int* count);

/* ---- host-buffer entry points (the drop-in boundary) ---------------------- */

/* labelprop::lpa: upload the graph, run, download labels[n]. */
int nulpa_run(const nulpa_csr* csr, const nulpa_opts* opts, const nulpa_tuning* tuning,
              uint32_t* labels_out, nulpa_stats* stats);

/* One synchronous label-choice step over every vertex of degree >= 1 (no
 * pruning flags): out[i] = c* if (pick_less ? c* < in[i] : c* != in[i]) else in[i]. */
int nulpa_sync_step(const nulpa_csr* csr, const uint32_t* labels_in, int pick_less,
                    int strategy, int precision, uint32_t* labels_out, uint64_t* changed);

int nulpa_modularity(const nulpa_csr* csr, const uint32_t* labels, double* q);
int nulpa_community_count(const nulpa_csr* csr, const uint32_t* labels, uint64_t* count);
/* labelprop::community_stats (quality.hpp:32-38, quality.cpp:56-78): the *count
 * communities present (ascending label) with their sigma (intra weight) and big_sigma
 * (total weighted degree), and the size histogram as *hist_len (size, how many) pairs in
 * ascending size. Host arrays of n entries each (any of the five may be NULL). */
int nulpa_community_stats(const nulpa_csr* csr, const uint32_t* labels, uint64_t* count,
                          uint32_t* communities, double* sigma, double* big_sigma,
                          uint64_t* hist_size, uint64_t* hist_count, uint64_t* hist_len);

/* labelprop::cross_check on host arrays (labels and flags updated in place). */
int nulpa_cross_check(const nulpa_csr* csr, uint32_t* labels, const uint32_t* prev,
                      uint8_t* flags, uint64_t* reverted);

/* labelprop::partition_by_degree: low/high must hold n entries each. */
int nulpa_partition_by_degree(const nulpa_csr* csr, uint32_t switch_degree, uint32_t* low,
                              uint64_t* n_low, uint32_t* high, uint64_t* n_high);

/* ---- device-resident graph ------------------------------------------------ */

/* Copy a host CSR to the device (weights that are all 1.0f are elided). */
int nulpa_graph_upload(const nulpa_csr* host_csr, int device, nulpa_graph** out);
/* Borrow device arrays (e.g. from a generator or torch); not freed by us. */
int nulpa_graph_wrap_device(const nulpa_csr* device_csr, int device, nulpa_graph** out);
int nulpa_graph_free(nulpa_graph* g);
int nulpa_graph_info(const nulpa_graph* g, uint32_t* n, uint64_t* m2, uint32_t* max_degree,
                     int* weighted);
/* Layout used by graphs created after this call (process-wide; default
 * NULPA_LAYOUT_DEGREE_BUCKETS). */
int nulpa_set_default_layout(int layout);
int nulpa_graph_layout(const nulpa_graph* g, int* layout);
/* Permute a DEVICE label array between position order and vertex order
 * (out-of-place; a plain copy under the identity layout). */
int nulpa_graph_labels_to_vertex_order(const nulpa_graph* g, const uint32_t* pos_dev,
                                       uint32_t* vtx_dev);
int nulpa_graph_labels_to_position_order(const nulpa_graph* g, const uint32_t* vtx_dev,
                                         uint32_t* pos_dev);
/* Device pointers of the resident arrays, POSITION order (weights NULL when unit). */
int nulpa_graph_device_csr(const nulpa_graph* g, nulpa_csr* out);
/* Download the resident CSR into host buffers in VERTEX order (weights may be NULL). */
int nulpa_graph_download(const nulpa_graph* g, uint64_t* offsets, uint32_t* targets,
                         float* weights);

/* lpa() on a resident graph; labels to host and/or device buffers (NULL = skip). */
int nulpa_run_graph(nulpa_graph* g, const nulpa_opts* opts, const nulpa_tuning* tuning,
                    uint32_t* labels_host, uint32_t* labels_device, nulpa_stats* stats);
/* Sync step on a resident graph; labels are DEVICE pointers. */
int nulpa_sync_step_graph(nulpa_graph* g, const uint32_t* labels_in_dev, int pick_less,
                          int strategy, int precision, uint32_t* labels_out_dev,
                          uint64_t* changed);
/* Modularity on a resident graph; labels is a DEVICE pointer. */
int nulpa_modularity_graph(nulpa_graph* g, const uint32_t* labels_dev, double* q);
int nulpa_community_count_graph(nulpa_graph* g, const uint32_t* labels_dev, uint64_t* count);
/* community_stats on a resident graph; labels is a DEVICE pointer, outputs are host. */
int nulpa_community_stats_graph(nulpa_graph* g, const uint32_t* labels_dev, uint64_t* count,
                                uint32_t* communities, double* sigma, double* big_sigma,
                                uint64_t* hist_size, uint64_t* hist_count, uint64_t* hist_len);

/* ---- synthetic inputs built on the device (bench / tests) ----------------- */

/* Graph500-style R-MAT (A=.57,B=.19,C=.19,D=.05), edgefactor*2^scale draws,
 * seeded vertex permutation, self-loops dropped, symmetrised, deduplicated,
 * unit weights, rows sorted. */
int nulpa_gen_rmat(uint32_t scale, uint32_t edgefactor, uint64_t seed, int device,
                   nulpa_graph** out);
/* rows x cols 4-neighbour lattice, id = r*cols + c, unit weights. */
int nulpa_gen_grid(uint32_t rows, uint32_t cols, int device, nulpa_graph** out);
/* Chung-Lu power-law graph: n vertices, ~edges undirected draws, exponent
 * gamma, the top `hubs` vertices forced to degree ~hub_degree; dedup'd. */
int nulpa_gen_web(uint32_t n, uint64_t edges, double gamma, uint32_t hubs,
                  uint32_t hub_degree, uint64_t seed, int device, nulpa_graph** out);
/* Build a symmetric, deduplicated, sorted CSR from a host edge list on the
 * device (duplicate pairs dropped, unit weights) — for SBM-style inputs. */
int nulpa_graph_from_edges(const uint32_t* u, const uint32_t* v, uint64_t ne, uint32_t n,
                           int device, nulpa_graph** out);

/* ---- graph files and build_csr ----------------------------------- */

/* labelprop::EdgeList (graph.hpp:40-43) as arrays in listing order; n_declared < 0 when
 * the file declares no vertex count. Arrays are malloc'd by the library. */
typedef struct nulpa_edge_list {
  uint64_t ne;
  int64_t n_declared;
  uint32_t* u;
  uint32_t* v;
  double* w;
} nulpa_edge_list;

/* labelprop::load_graph (graph.hpp:95-96, graph.cpp:68-161,180-184): same inputs, same
 * messages; NULPA_EFORMAT for FormatError, NULPA_EINVAL for ValidationError. */
int nulpa_load_edge_list(const char* path, int format, nulpa_edge_list* out);
void nulpa_edge_list_free(nulpa_edge_list* el);
/* labelprop::build_csr (graph.hpp:107, graph.cpp:186-307) on the device, bit-exact:
 * duplicate merging by weight summation in listing order, first-listed direction kept
 * (symmetrize), self-loops once, rows sorted by target. w NULL = every weight 1.0;
 * n_declared < 0 = none. The result is a resident graph (download it for a CsrGraph). */
int nulpa_graph_from_edge_list(const uint32_t* u, const uint32_t* v, const double* w,
                               uint64_t ne, int64_t n_declared, int symmetrize, int device,
                               nulpa_graph** out);
/* load_graph + build_csr. */
int nulpa_graph_load(const char* path, int format, int symmetrize, int device, nulpa_graph** out);
/* labelprop::write_edge_list (graph.hpp:112, graph.cpp:309-325): `u v w` once per
 * undirected edge (u <= v), same bytes and messages. weights NULL = unit. */
int nulpa_write_edge_list(const char* path, const nulpa_csr* csr);
/* labelprop::write_membership (io.hpp:12, io.cpp:9-14): `vertex<TAB>label` lines, the
 * text formatted on `device` from host labels[n]. */
int nulpa_write_membership(const char* path, const uint32_t* labels, uint64_t n, int device);
/* labelprop::read_membership (io.hpp:19, io.cpp:16-56): labels[n] from the TSV; same
 * checks, messages and error kinds (NULPA_EFORMAT / NULPA_EINVAL). */
int nulpa_read_membership(const char* path, uint32_t n, uint32_t* labels);

/* ---- pass-level sessions: the partitioned multi-GPU path --------
 * A session runs single passes over the POSITION range [v_begin, v_end) of a
 * resident graph, on caller-owned DEVICE arrays labels[n] / flags[n] in
 * position order (nulpa_graph_labels_to_vertex_order converts the result) that
 * are replicated across ranks; the caller exchanges the owned label ranges and the
 * wake flags between passes (torch.distributed / NCCL) and drives the
 * run_engine schedule (paper_2411_11468_b200/dist.py). ParallelAsync updates
 * labels in place inside the range; Synchronous stages decisions and applies
 * them to the range after the pass, then wakes neighbours (remote ones too). */
typedef struct nulpa_session nulpa_session;

typedef struct nulpa_pass_info {
  uint64_t changed;            /* label changes in the range */
  uint64_t processed_vertices;
  uint64_t processed_edges;
  uint64_t wake_edges;
  double device_ms;            /* CUDA-event time of the pass */
  uint64_t kernel_launches;
} nulpa_pass_info;

/* Edge-balanced 1-D split of the position order: bounds[0..parts] with
 * offsets[bounds[p]] ~ p*m2/parts. */
int nulpa_graph_edge_ranges(nulpa_graph* g, uint32_t parts, uint32_t* bounds);
int nulpa_session_create(nulpa_graph* g, const nulpa_opts* opts, const nulpa_tuning* tuning,
                         uint32_t v_begin, uint32_t v_end, uint32_t* labels_dev,
                         uint8_t* flags_dev, nulpa_session** out);
/* labels[p] = vertex id at p and flags[p] = (degree == 0) over ALL n positions. */
int nulpa_session_init(nulpa_session* s);
/* wake = 0 skips the neighbour wake-up stores (legal when the caller's schedule
 * resets every flag before the next pass, see engine.cu run_lpa). */
int nulpa_session_pass(nulpa_session* s, int pick_less, int wake, nulpa_pass_info* info);
int nulpa_session_free(nulpa_session* s);
/* Run the session's kernels on `stream` (a cudaStream_t, e.g. the caller's collective
 * stream) instead of its own, so caller work on that stream needs no host sync. */
int nulpa_session_set_stream(nulpa_session* s, void* stream);
/* Changed-only label exchange: after a pass, write the (position, label) pairs of the
 * range's labels that changed in it to out_dev[2*cap], padded with 0xFFFFFFFF pairs
 * (cap >= the pass's changed count); apply_changes writes all-gathered pairs into this
 * rank's replica (0xFFFFFFFF pairs skipped). Both run on `stream` (a cudaStream_t;
 * NULL = the legacy default stream). */
int nulpa_session_pack_changes(nulpa_session* s, uint32_t* out_dev, uint32_t cap, void* stream);
int nulpa_session_apply_changes(nulpa_session* s, const uint32_t* in_dev, uint64_t pairs,
                                void* stream);
/* One rank's graph of a 1-D partition: the rows [v_begin, v_end) of the position order
 * (global position ids as targets), every other row empty, the layout of `g` kept. */
int nulpa_graph_slice(nulpa_graph* g, uint32_t v_begin, uint32_t v_end, nulpa_graph** out);
/* The resident arrays as stored (position order under the degree-bucket layout), no
 * conversion: a slice saved this way re-uploads with NULPA_LAYOUT_IDENTITY as the same
 * position-order rows. NULL arrays are skipped. */
int nulpa_graph_download_raw(const nulpa_graph* g, uint64_t* offsets, uint32_t* targets,
                             float* weights);
/* The position layout of a resident graph: perm[p] = vertex id at position p, inv[v] =
 * position of vertex v (n entries each), and whether every input row was strictly
 * ascending. Fails on an identity-layout graph. */
int nulpa_graph_download_layout(const nulpa_graph* g, uint32_t* perm, uint32_t* inv,
                                int* rows_simple);
/* Upload a host CSR that is ALREADY in position order (e.g. one rank's slice saved with
 * nulpa_graph_download_raw) together with its layout; no relayout, no plan. */
int nulpa_graph_upload_positioned(const nulpa_csr* csr, const uint32_t* perm,
                                  const uint32_t* inv, int rows_simple, int device,
                                  nulpa_graph** out);
/* sigma_c (intra-community stored weight) and Sigma_c (summed weighted degree) over the
 * rows `g` holds, quality.cpp:29-40, into device arrays of n doubles indexed by label;
 * labels are in POSITION order. Summed over a partition's slices they are the graph's. */
int nulpa_community_sums_graph(nulpa_graph* g, const uint32_t* labels_pos_dev, double* sigma_dev,
                               double* big_dev);

#ifdef __cplusplus
}
#endif
#endif
