/* TEST INFRASTRUCTURE — CPU restatement of the reference's ν-LPA hot path.
 *
 * This is the CHECKER for the CUDA product (paper_2411_11468_b200/csrc). Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * It is never called on the product path.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/proj) and says which. Parity pinning: tests/test_oracle.py
 * checks it against the reference's known-answer tests and against the golden
 * vectors in tests/golden/ produced by the reference itself (oracle/_ref).
 */
#ifndef NULPA_ORACLE_H
#define NULPA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Probe strategies, hashtable.hpp:25 (same numbering). */
enum { OR_LINEAR = 0, OR_QUADRATIC = 1, OR_DOUBLE = 2, OR_QUAD_DOUBLE = 3 };
/* Exec modes, lpa.hpp:20 (same numbering). */
enum { OR_PARALLEL = 0, OR_SEQUENTIAL = 1, OR_SYNCHRONOUS = 2 };

typedef struct {
  uint32_t n;
  uint64_t m2;
  const uint64_t* offsets; /* n + 1 */
  const uint32_t* targets; /* m2 */
  const float* weights;    /* m2, or NULL = all 1.0f */
} or_csr;

typedef struct {
  double tolerance;
  int32_t max_iterations;
  int32_t pl_period;
  int32_t cc_period;
  int32_t strategy;
  uint32_t switch_degree;
  int32_t precision_bits; /* 32 or 64 */
  int32_t exec;           /* OR_SEQUENTIAL or OR_SYNCHRONOUS (deterministic modes) */
  int32_t prune;
} or_config;

typedef struct {
  int32_t iterations;
  int32_t converged;
  int32_t pl_iterations;
  int32_t pad;
  uint64_t cc_reverts;
  uint64_t delta_n[256]; /* first min(iterations, 256) entries valid */
} or_stats;

/* geometry_for, hashtable.hpp:41-46. Returns -1 for degree 0. */
int or_geometry(uint64_t degree, uint64_t* p1, uint64_t* p2);

/* ht_accumulate (unshared), hashtable.hpp:96-149, over one region of p1
 * slots. Returns 0 Done, 1 Failed. */
int or_ht_accumulate_f32(uint32_t* keys, float* vals, uint64_t p1, uint64_t p2, int strategy,
                         uint32_t key, float value);
int or_ht_accumulate_f64(uint32_t* keys, double* vals, uint64_t p1, uint64_t p2, int strategy,
                         uint32_t key, double value);

/* Feed `count` inserts into a fresh region and dump it (probe-placement KATs,
 * test_hashtable.cpp:71-107). Returns the number of failed inserts. */
uint64_t or_ht_accumulate_seq(uint64_t p1, uint64_t p2, int strategy, const uint32_t* keys,
                              const float* values, uint64_t count, uint32_t* slot_keys,
                              float* slot_values);

/* ht_max_key over a region, hashtable.hpp:163-185. Returns 0xFFFFFFFF if empty. */
uint32_t or_ht_max_key_f32(const uint32_t* keys, const float* vals, uint64_t p1, float* best);

/* One synchronous label-choice step from arbitrary labels: scan_candidate
 * (lpa.hpp:92-111) against labels_in for every vertex of degree >= 1, then
 * the move rule of sync_move (lpa.cpp:87-88). Returns changed count. */
uint64_t or_sync_step(const or_csr* g, const uint32_t* labels_in, int pick_less, int strategy,
                      int precision_bits, uint32_t* labels_out);

/* lpa() in the deterministic exec modes (Sequential lpa_move lpa.hpp:123-145,
 * Synchronous sync_move lpa.cpp:70-100) driven by run_engine lpa.cpp:246-315.
 * Returns 0 ok, 1 invalid config (validate_config lpa.cpp:317-326),
 * 3 hashtable failure. */
int or_lpa(const or_csr* g, const or_config* cfg, uint32_t* labels_out, or_stats* stats);

/* cross_check, lpa.cpp:338-360 (sequential ascending scan). */
uint64_t or_cross_check(const or_csr* g, uint32_t* labels, const uint32_t* prev, uint8_t* flags);

/* modularity, quality.cpp:21-49. Returns NaN on an edgeless graph. */
double or_modularity(const or_csr* g, const uint32_t* labels);

/* partition_by_degree, lpa.cpp:330-336. Returns n_low. */
uint64_t or_partition_by_degree(const or_csr* g, uint32_t switch_degree, uint32_t* low,
                                uint32_t* high);

#ifdef __cplusplus
}
#endif
#endif
