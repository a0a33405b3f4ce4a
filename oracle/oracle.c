/* TEST INFRASTRUCTURE — CPU restatement of the reference ν-LPA hot path.
 *
 * The checker for the CUDA product, never the product itself: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this file's
 * library (oracle/liboracle.so). Function-by-function restatement of
 * /root/reference/proj (file:line cited per function); pinned against the
 * reference's KATs and the golden vectors in tests/golden/ (tests/test_oracle.py).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define EMPTY 0xFFFFFFFFu

static uint64_t bit_ceil_u64(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

/* hashtable.hpp:41-46: p1 = bit_ceil(d + 1) - 1, p2 = 2 (p1 + 1) - 1. */
int or_geometry(uint64_t degree, uint64_t* p1, uint64_t* p2) {
  if (degree == 0) return -1;
  *p1 = bit_ceil_u64(degree + 1) - 1;
  *p2 = 2 * (*p1 + 1) - 1;
  return 0;
}

/* hashtable.hpp:96-149 (unshared branch :119-125). Probe index starts at the
 * key; the strategy advance applies for the first 2*p1 probes, then +1 for a
 * completeness sweep, giving up after 4*p1 probes. Unsigned 64-bit wrap-around
 * of idx/step matches the reference's std::uint64_t arithmetic. */
#define OR_ACCUMULATE_BODY                                                        \
  const uint64_t max_retries = 4 * p1;                                            \
  const uint64_t budget = 2 * p1;                                                 \
  const uint64_t khash = (uint64_t)key % p2;                                      \
  uint64_t idx = key;                                                             \
  uint64_t step = (strategy == OR_DOUBLE) ? (khash == 0 ? 1 : khash) : 1;         \
  for (uint64_t t = 0; t < max_retries; ++t) {                                    \
    const uint64_t s = idx % p1;                                                  \
    if (keys[s] == key || keys[s] == EMPTY) {                                     \
      keys[s] = key;                                                              \
      vals[s] += value;                                                           \
      return 0;                                                                   \
    }                                                                             \
    if (t + 1 >= budget) {                                                        \
      idx += 1;                                                                   \
      continue;                                                                   \
    }                                                                             \
    switch (strategy) {                                                           \
      case OR_LINEAR: idx += 1; break;                                            \
      case OR_QUADRATIC: idx += step; step *= 2; break;                           \
      case OR_DOUBLE: idx += step; break;                                         \
      default: idx += step; step = 2 * step + khash; break;                       \
    }                                                                             \
  }                                                                               \
  return 1;

int or_ht_accumulate_f32(uint32_t* keys, float* vals, uint64_t p1, uint64_t p2, int strategy,
                         uint32_t key, float value) {
  OR_ACCUMULATE_BODY
}

int or_ht_accumulate_f64(uint32_t* keys, double* vals, uint64_t p1, uint64_t p2, int strategy,
                         uint32_t key, double value) {
  OR_ACCUMULATE_BODY
}

uint64_t or_ht_accumulate_seq(uint64_t p1, uint64_t p2, int strategy, const uint32_t* keys_in,
                              const float* values, uint64_t count, uint32_t* slot_keys,
                              float* slot_values) {
  for (uint64_t s = 0; s < p1; ++s) {
    slot_keys[s] = EMPTY;
    slot_values[s] = 0.0f;
  }
  uint64_t failures = 0;
  for (uint64_t k = 0; k < count; ++k)
    failures += (uint64_t)or_ht_accumulate_f32(slot_keys, slot_values, p1, p2, strategy,
                                               keys_in[k], values[k]);
  return failures;
}

/* ht_better / ht_max_key, hashtable.hpp:163-185: higher value wins, ties go to
 * the smaller key. */
uint32_t or_ht_max_key_f32(const uint32_t* keys, const float* vals, uint64_t p1, float* best) {
  uint32_t bk = EMPTY;
  float bv = 0.0f;
  for (uint64_t s = 0; s < p1; ++s) {
    const uint32_t k = keys[s];
    if (k == EMPTY) continue;
    if (bk == EMPTY || vals[s] > bv || (vals[s] == bv && k < bk)) {
      bk = k;
      bv = vals[s];
    }
  }
  if (best) *best = bv;
  return bk;
}

static uint32_t or_ht_max_key_f64(const uint32_t* keys, const double* vals, uint64_t p1) {
  uint32_t bk = EMPTY;
  double bv = 0.0;
  for (uint64_t s = 0; s < p1; ++s) {
    const uint32_t k = keys[s];
    if (k == EMPTY) continue;
    if (bk == EMPTY || vals[s] > bv || (vals[s] == bv && k < bk)) {
      bk = k;
      bv = vals[s];
    }
  }
  return bk;
}

/* Scratch table large enough for the largest region of the graph. */
typedef struct {
  uint32_t* keys;
  float* v32;
  double* v64;
  int bits;
} scratch;

static int scratch_init(scratch* sc, const or_csr* g, int bits) {
  uint64_t maxdeg = 0;
  for (uint32_t i = 0; i < g->n; ++i) {
    const uint64_t d = g->offsets[i + 1] - g->offsets[i];
    if (d > maxdeg) maxdeg = d;
  }
  const uint64_t cap = bit_ceil_u64(maxdeg + 1);
  sc->bits = bits;
  sc->keys = (uint32_t*)malloc(cap * sizeof(uint32_t));
  sc->v32 = bits == 64 ? NULL : (float*)malloc(cap * sizeof(float));
  sc->v64 = bits == 64 ? (double*)malloc(cap * sizeof(double)) : NULL;
  return sc->keys && (sc->v32 || sc->v64) ? 0 : -1;
}

static void scratch_free(scratch* sc) {
  free(sc->keys);
  free(sc->v32);
  free(sc->v64);
}

/* detail::scan_candidate, lpa.hpp:92-111: clear the region (ht_clear
 * hashtable.hpp:153-159), accumulate (label_of(j), w_ij) for j != i, return the
 * max key. Returns 0 with *cand set, 1 for "no candidate" (only self-loops),
 * 3 for a hashtable failure. */
static int scan_candidate(const or_csr* g, uint32_t i, const uint32_t* label_of, int strategy,
                          scratch* sc, uint32_t* cand) {
  const uint64_t lo = g->offsets[i], hi = g->offsets[i + 1];
  uint64_t p1, p2;
  if (or_geometry(hi - lo, &p1, &p2) != 0) return 1;
  for (uint64_t s = 0; s < p1; ++s) sc->keys[s] = EMPTY;
  if (sc->bits == 64)
    for (uint64_t s = 0; s < p1; ++s) sc->v64[s] = 0.0;
  else
    for (uint64_t s = 0; s < p1; ++s) sc->v32[s] = 0.0f;
  for (uint64_t p = lo; p < hi; ++p) {
    const uint32_t j = g->targets[p];
    if (j == i) continue;
    const float w = g->weights ? g->weights[p] : 1.0f;
    int failed;
    if (sc->bits == 64)
      failed = or_ht_accumulate_f64(sc->keys, sc->v64, p1, p2, strategy, label_of[j], (double)w);
    else
      failed = or_ht_accumulate_f32(sc->keys, sc->v32, p1, p2, strategy, label_of[j], w);
    if (failed) return 3;
  }
  const uint32_t bk = sc->bits == 64 ? or_ht_max_key_f64(sc->keys, sc->v64, p1)
                                     : or_ht_max_key_f32(sc->keys, sc->v32, p1, NULL);
  if (bk == EMPTY) return 1;
  *cand = bk;
  return 0;
}

uint64_t or_sync_step(const or_csr* g, const uint32_t* labels_in, int pick_less, int strategy,
                      int precision_bits, uint32_t* labels_out) {
  scratch sc;
  if (scratch_init(&sc, g, precision_bits) != 0) return UINT64_MAX;
  uint64_t dn = 0;
  for (uint32_t i = 0; i < g->n; ++i) {
    labels_out[i] = labels_in[i];
    uint32_t c;
    if (scan_candidate(g, i, labels_in, strategy, &sc, &c) != 0) continue;
    const int allowed = pick_less ? (c < labels_in[i]) : (c != labels_in[i]);
    if (!allowed) continue;
    labels_out[i] = c;
    ++dn;
  }
  scratch_free(&sc);
  return dn;
}

/* lpa_move, lpa.hpp:123-145: ascending in-place pass; mark processed at scan
 * start, wake every neighbour of a changed vertex. */
static int seq_move(const or_csr* g, uint32_t* labels, uint8_t* flags, int pick_less,
                    int strategy, scratch* sc, uint64_t* dn) {
  *dn = 0;
  for (uint32_t i = 0; i < g->n; ++i) {
    if (flags[i]) continue;
    flags[i] = 1;
    if (g->offsets[i + 1] == g->offsets[i]) continue;
    uint32_t c;
    const int r = scan_candidate(g, i, labels, strategy, sc, &c);
    if (r == 3) return 3;
    if (r != 0) continue;
    const int allowed = pick_less ? (c < labels[i]) : (c != labels[i]);
    if (!allowed) continue;
    labels[i] = c;
    ++*dn;
    for (uint64_t p = g->offsets[i]; p < g->offsets[i + 1]; ++p) flags[g->targets[p]] = 0;
  }
  return 0;
}

/* sync_move, lpa.cpp:70-100: candidates from a frozen snapshot, applied
 * together, wake-ups only after the joint application. */
static int sync_move(const or_csr* g, uint32_t* labels, uint8_t* flags, int pick_less,
                     int strategy, scratch* sc, uint32_t* snapshot, uint32_t* staged_v,
                     uint32_t* staged_c, uint64_t* dn) {
  memcpy(snapshot, labels, (size_t)g->n * sizeof(uint32_t));
  uint64_t ns = 0;
  for (uint32_t i = 0; i < g->n; ++i) {
    if (flags[i]) continue;
    flags[i] = 1;
    if (g->offsets[i + 1] == g->offsets[i]) continue;
    uint32_t c;
    const int r = scan_candidate(g, i, snapshot, strategy, sc, &c);
    if (r == 3) return 3;
    if (r != 0) continue;
    const int allowed = pick_less ? (c < snapshot[i]) : (c != snapshot[i]);
    if (!allowed) continue;
    staged_v[ns] = i;
    staged_c[ns] = c;
    ++ns;
  }
  for (uint64_t k = 0; k < ns; ++k) labels[staged_v[k]] = staged_c[k];
  for (uint64_t k = 0; k < ns; ++k) {
    const uint32_t i = staged_v[k];
    for (uint64_t p = g->offsets[i]; p < g->offsets[i + 1]; ++p) flags[g->targets[p]] = 0;
  }
  *dn = ns;
  return 0;
}

/* cross_check, lpa.cpp:338-360. */
uint64_t or_cross_check(const or_csr* g, uint32_t* labels, const uint32_t* prev, uint8_t* flags) {
  uint64_t reverted = 0;
  for (uint32_t i = 0; i < g->n; ++i) {
    const uint32_t c = labels[i];
    if (c == prev[i]) continue;
    if (labels[c] == c) continue;
    if (i <= c) continue;
    labels[i] = prev[i]; /* the CAS (expected c) always succeeds single-threaded */
    ++reverted;
    flags[i] = 0;
    for (uint64_t p = g->offsets[i]; p < g->offsets[i + 1]; ++p) flags[g->targets[p]] = 0;
  }
  return reverted;
}

/* validate_config, lpa.cpp:317-326. */
static int validate(const or_csr* g, const or_config* c) {
  if (g->n == 0) return 1;
  if (!(c->tolerance > 0.0 && c->tolerance <= 1.0)) return 1;
  if (c->max_iterations < 1) return 1;
  if (c->pl_period < 0 || c->cc_period < 0) return 1;
  if (c->switch_degree < 2) return 1;
  return 0;
}

/* run_engine, lpa.cpp:246-315, for the deterministic exec modes. */
int or_lpa(const or_csr* g, const or_config* cfg, uint32_t* labels, or_stats* st) {
  if (validate(g, cfg)) return 1;
  if (cfg->exec != OR_SEQUENTIAL && cfg->exec != OR_SYNCHRONOUS) return 1;
  const uint32_t n = g->n;
  memset(st, 0, sizeof(*st));
  uint8_t* flags = (uint8_t*)calloc(n, 1);
  uint32_t* prev = (uint32_t*)malloc((size_t)n * 4);
  uint32_t* snap = (uint32_t*)malloc((size_t)n * 4);
  uint32_t* sv = (uint32_t*)malloc((size_t)n * 4);
  uint32_t* sc_c = (uint32_t*)malloc((size_t)n * 4);
  scratch sc;
  int rc = 0;
  if (!flags || !prev || !snap || !sv || !sc_c || scratch_init(&sc, g, cfg->precision_bits)) {
    rc = 2;
    goto out;
  }
  for (uint32_t i = 0; i < n; ++i) {
    labels[i] = i;
    flags[i] = (g->offsets[i + 1] == g->offsets[i]) ? 1 : 0;
  }
  for (int iter = 0; iter < cfg->max_iterations; ++iter) {
    const int pick_less = cfg->pl_period > 0 && iter % cfg->pl_period == 0;
    const int check = cfg->cc_period > 0 && iter % cfg->cc_period == 0;
    if (check) memcpy(prev, labels, (size_t)n * 4);
    const int was_pl = iter > 0 && cfg->pl_period > 0 && (iter - 1) % cfg->pl_period == 0;
    if (!cfg->prune || (was_pl && !pick_less)) memset(flags, 0, n);
    uint64_t dn = 0;
    int r = cfg->exec == OR_SEQUENTIAL
                ? seq_move(g, labels, flags, pick_less, cfg->strategy, &sc, &dn)
                : sync_move(g, labels, flags, pick_less, cfg->strategy, &sc, snap, sv, sc_c, &dn);
    if (r) {
      rc = r;
      break;
    }
    if (check) {
      const uint64_t rev = or_cross_check(g, labels, prev, flags);
      st->cc_reverts += rev;
      dn -= rev;
    }
    if (st->iterations < 256) st->delta_n[st->iterations] = dn;
    st->iterations++;
    if (pick_less) st->pl_iterations++;
    if (!pick_less && (double)dn / n < cfg->tolerance) {
      st->converged = 1;
      break;
    }
  }
  scratch_free(&sc);
out:
  free(flags);
  free(prev);
  free(snap);
  free(sv);
  free(sc_c);
  return rc;
}

/* modularity, quality.cpp:21-49 (check_labels :9-17). */
double or_modularity(const or_csr* g, const uint32_t* labels) {
  const uint32_t n = g->n;
  double two_m = 0.0;
  for (uint64_t p = 0; p < g->m2; ++p) two_m += g->weights ? (double)g->weights[p] : 1.0;
  if (!(two_m > 0.0)) return NAN;
  for (uint32_t i = 0; i < n; ++i)
    if (labels[i] >= n) return NAN;
  double* sigma = (double*)calloc(n, sizeof(double));
  double* big = (double*)calloc(n, sizeof(double));
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t ci = labels[i];
    double ki = 0.0;
    for (uint64_t p = g->offsets[i]; p < g->offsets[i + 1]; ++p) {
      const double w = g->weights ? (double)g->weights[p] : 1.0;
      ki += w;
      if (labels[g->targets[p]] == ci) sigma[ci] += w;
    }
    big[ci] += ki;
  }
  double q = 0.0;
  for (uint32_t c = 0; c < n; ++c) {
    if (big[c] == 0.0 && sigma[c] == 0.0) continue;
    const double frac = big[c] / two_m;
    q += sigma[c] / two_m - frac * frac;
  }
  free(sigma);
  free(big);
  return q;
}

/* partition_by_degree, lpa.cpp:330-336. */
uint64_t or_partition_by_degree(const or_csr* g, uint32_t switch_degree, uint32_t* low,
                                uint32_t* high) {
  uint64_t nl = 0, nh = 0;
  for (uint32_t i = 0; i < g->n; ++i) {
    if (g->offsets[i + 1] - g->offsets[i] < switch_degree)
      low[nl++] = i;
    else
      high[nh++] = i;
  }
  return nl;
}
