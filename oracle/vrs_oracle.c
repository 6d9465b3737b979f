/*
 * vrs_oracle.c -- CPU brute-force ORACLE for filtered exact top-k search.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2403_15807_b200/, libvrs.so) never links, loads
 * or calls it, and this file includes no header of the product.
 *
 * What it computes (the plain definition, no blocking / fusion / reordering):
 *
 *   PAPER.md L285-L288 (Sec. 3, eq. "Brute force similarity search with
 *   relational predicate theta"):
 *       sigma_{eps,v,theta_R}(R) <=> sigma_eps(v x sigma_{theta_R}(R))
 *   i.e. (1) evaluate the relational predicate theta_R per row  -> selection,
 *        (2) evaluate the similarity eps(v, t) for every selected row t,
 *        (3) apply eps as "the k best" (top-k, "k = 64 for top-k
 *            retrieval"; SPEC.md L141-L147 result contract).
 *   Table 1: the scan path is "Exact", so the oracle is the
 *   definition itself in fp64.
 *
 * Readings:
 *   R1  metrics: L2 = squared Euclidean (ascending), IP = raw <q,x>
 *       (descending), COS = cosine SIMILARITY (descending)  [PAPER.md L305, L350, L354]
 *   R2  ties: lower global row id first                      [SPEC.md L145, L177]
 *   R3  k > N_sel: exactly min(k, N_sel) valid entries, then padding
 *       id = -1, dist = +inf (L2) / -inf (IP, COS)           [SPEC.md L145, L236]
 *   R4  predicate: AND of closed integer intervals lo <= a[i] <= hi
 *       (lo > hi selects nothing; zero clauses select all)   [PAPER.md L138, L1395; SPEC.md L48-L52]
 *   R5  COS over a corpus with a zero-norm row -> DEGENERATE [SPEC.md L95];
 *       a zero-norm COS query yields an all-padding row.
 *
 * Arithmetic: fp32 inputs widened exactly to double; every sum runs
 * sequentially over t = 0..d-1 (compiled with -ffp-contract=off).  L2 uses
 * direct differences, never the |q|^2+|x|^2-2q.x expansion.
 *
 * Parity pins: tests/test_oracle_pins.py (closed forms, SPEC worked examples,
 * brute force on tiny inputs, invariants).  The paper itself prints no result
 * values, so no pin comes from the paper's own numbers.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* status codes: numerically identical to the ABI's, defined independently */
enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ENOTFOUND = 2, ORC_EDEGENERATE = 3, ORC_ENOMEM = 4 };
enum { ORC_L2 = 0, ORC_IP = 1, ORC_COS = 2 };
enum { ORC_I32 = 0, ORC_U8 = 1 };

typedef struct {
  int32_t attr;
  int64_t lo;
  int64_t hi;
} orc_clause;

/* ---- step 1: predicate theta_R ------------------ */

static int64_t attr_value(const void *col, int32_t type, int64_t i) {
  if (type == ORC_I32) return (int64_t)((const int32_t *)col)[i];
  return (int64_t)((const uint8_t *)col)[i];
}

static int check_pred(int32_t n_attrs, const int32_t *attr_types, const orc_clause *clauses,
                      int32_t n_clauses) {
  if (n_clauses < 0) return ORC_EINVAL;
  if (n_clauses > 0 && clauses == NULL) return ORC_EINVAL;
  for (int32_t c = 0; c < n_clauses; ++c) {
    if (clauses[c].attr < 0 || clauses[c].attr >= n_attrs) return ORC_ENOTFOUND;
    int32_t t = attr_types[clauses[c].attr];
    if (t != ORC_I32 && t != ORC_U8) return ORC_EINVAL;
  }
  return ORC_OK;
}

static int row_selected(const void *const *attrs, const int32_t *attr_types, const orc_clause *clauses,
                        int32_t n_clauses, int64_t i) {
  for (int32_t c = 0; c < n_clauses; ++c) {
    int64_t a = attr_value(attrs[clauses[c].attr], attr_types[clauses[c].attr], i);
    if (!(clauses[c].lo <= a && a <= clauses[c].hi)) return 0;
  }
  return 1;
}

/* bitmap: word w bit b <-> row 32w+b, LSB first, bits past n are zero.
 * ids (optional): ascending qualifying row ids.  Returns the count. */
int orc_select(const void *const *attrs, const int32_t *attr_types, int32_t n_attrs, int64_t n,
               const orc_clause *clauses, int32_t n_clauses, uint32_t *bitmap, int64_t *count,
               int64_t *ids) {
  if (n < 1) return ORC_EINVAL;
  int st = check_pred(n_attrs, attr_types, clauses, n_clauses);
  if (st != ORC_OK) return st;
  int64_t nwords = (n + 31) / 32;
  if (bitmap) memset(bitmap, 0, (size_t)nwords * sizeof(uint32_t));
  int64_t cnt = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (row_selected(attrs, attr_types, clauses, n_clauses, i)) {
      if (bitmap) bitmap[i >> 5] |= (uint32_t)1u << (i & 31);
      if (ids) ids[cnt] = i;
      ++cnt;
    }
  }
  if (count) *count = cnt;
  return ORC_OK;
}

/* ---- step 2: similarity eps --------------------- */

static double dot64(const float *a, const float *b, int32_t d) {
  double s = 0.0;
  for (int32_t t = 0; t < d; ++t) s += (double)a[t] * (double)b[t];
  return s;
}

static double l2sq64(const float *a, const float *b, int32_t d) {
  double s = 0.0;
  for (int32_t t = 0; t < d; ++t) {
    double diff = (double)a[t] - (double)b[t];
    s += diff * diff;
  }
  return s;
}

/* eps(q, x) in fp64 for one row. */
static double score64(const float *q, const float *x, int32_t d, int32_t metric) {
  if (metric == ORC_L2) return l2sq64(q, x, d);
  if (metric == ORC_IP) return dot64(q, x, d);
  /* COS: (sum q_t x_t) / (sqrt(nq) * sqrt(nx)) */
  double nq = dot64(q, q, d), nx = dot64(x, x, d);
  return dot64(q, x, d) / (sqrt(nq) * sqrt(nx));
}

int orc_score(const float *X, int32_t d, const float *q, const int64_t *local_ids, int64_t m,
              int32_t metric, double *out) {
  if (d < 1 || m < 0) return ORC_EINVAL;
  if (metric < ORC_L2 || metric > ORC_COS) return ORC_EINVAL;
  for (int64_t j = 0; j < m; ++j) out[j] = score64(q, X + local_ids[j] * (int64_t)d, d, metric);
  return ORC_OK;
}

/* ---- step 3: order and take k -------------------- */

typedef struct {
  double s;
  int64_t id;
} orc_entry;

static int cmp_ascending(const void *pa, const void *pb) { /* L2: smaller first */
  const orc_entry *a = (const orc_entry *)pa, *b = (const orc_entry *)pb;
  if (a->s < b->s) return -1;
  if (a->s > b->s) return 1;
  return (a->id < b->id) ? -1 : (a->id > b->id);
}

static int cmp_descending(const void *pa, const void *pb) { /* IP, COS: larger first */
  const orc_entry *a = (const orc_entry *)pa, *b = (const orc_entry *)pb;
  if (a->s > b->s) return -1;
  if (a->s < b->s) return 1;
  return (a->id < b->id) ? -1 : (a->id > b->id);
}

static float pad_dist(int32_t metric) { return metric == ORC_L2 ? INFINITY : -INFINITY; }

static int all_finite(const float *v, int64_t m) {
  for (int64_t i = 0; i < m; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/*
 * Full search: predicate, fp64 scores for every qualifying row, sort, take k.
 * ids/dists: [q x k]; scores64 (optional): the fp64 scores behind dists.
 * nthreads <= 0: OpenMP default.
 */
int orc_search(const float *X, int64_t n, int32_t d, const void *const *attrs, const int32_t *attr_types,
               int32_t n_attrs, const orc_clause *clauses, int32_t n_clauses, const float *Qv, int64_t q,
               int32_t k, int32_t metric, int64_t row_offset, int64_t *ids, float *dists,
               double *scores64, int32_t nthreads) {
  if (n < 1 || d < 1 || q < 0 || k < 1) return ORC_EINVAL;
  if (metric < ORC_L2 || metric > ORC_COS) return ORC_EINVAL;
  int st = check_pred(n_attrs, attr_types, clauses, n_clauses);
  if (st != ORC_OK) return st;
  if (!all_finite(X, n * (int64_t)d) || !all_finite(Qv, q * (int64_t)d)) return ORC_EINVAL;
  if (metric == ORC_COS) {
    for (int64_t i = 0; i < n; ++i)
      if (dot64(X + i * (int64_t)d, X + i * (int64_t)d, d) == 0.0) return ORC_EDEGENERATE;
  }
  if (q == 0) return ORC_OK;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif

  /* sigma_theta(R): ascending ids of qualifying rows */
  int64_t *sel = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  if (!sel) return ORC_ENOMEM;
  int64_t nsel = 0;
  st = orc_select(attrs, attr_types, n_attrs, n, clauses, n_clauses, NULL, &nsel, sel);
  if (st != ORC_OK) {
    free(sel);
    return st;
  }
  orc_entry *ent = (orc_entry *)malloc((size_t)(nsel > 0 ? nsel : 1) * sizeof(orc_entry));
  if (!ent) {
    free(sel);
    return ORC_ENOMEM;
  }
  int (*cmp)(const void *, const void *) = (metric == ORC_L2) ? cmp_ascending : cmp_descending;

  for (int64_t j = 0; j < q; ++j) {
    const float *qv = Qv + j * (int64_t)d;
    int64_t m = nsel < k ? nsel : k;
    int zero_cos_query = (metric == ORC_COS && dot64(qv, qv, d) == 0.0);
    if (zero_cos_query) m = 0;
    if (m > 0) {
      /* eps over v x sigma_theta(R), every qualifying row */
#pragma omp parallel for schedule(static)
      for (int64_t r = 0; r < nsel; ++r) {
        ent[r].s = score64(qv, X + sel[r] * (int64_t)d, d, metric);
        ent[r].id = row_offset + sel[r];
      }
      qsort(ent, (size_t)nsel, sizeof(orc_entry), cmp);
    }
    for (int64_t r = 0; r < k; ++r) {
      int64_t o = j * (int64_t)k + r;
      if (r < m) {
        ids[o] = ent[r].id;
        dists[o] = (float)ent[r].s;
        if (scores64) scores64[o] = ent[r].s;
      } else {
        ids[o] = -1;
        dists[o] = pad_dist(metric);
        if (scores64) scores64[o] = (double)pad_dist(metric);
      }
    }
  }
  free(ent);
  free(sel);
  return ORC_OK;
}

/*
 * Multi-part merge (north_star (4); top-k is decomposable under the total
 * order (score, id)): top-k of the union of n_parts candidate lists
 * [n_parts x q x k].  Padding entries (id < 0) are dropped.  Scores are
 * the fp32 dists as given.
 */
int orc_merge(const int64_t *cand_ids, const float *cand_dists, int32_t n_parts, int64_t q, int32_t k,
              int32_t metric, int64_t *ids, float *dists) {
  if (n_parts < 1 || q < 0 || k < 1) return ORC_EINVAL;
  if (metric < ORC_L2 || metric > ORC_COS) return ORC_EINVAL;
  orc_entry *ent = (orc_entry *)malloc((size_t)n_parts * (size_t)k * sizeof(orc_entry));
  if (!ent) return ORC_ENOMEM;
  int (*cmp)(const void *, const void *) = (metric == ORC_L2) ? cmp_ascending : cmp_descending;
  for (int64_t j = 0; j < q; ++j) {
    int64_t m = 0;
    for (int32_t p = 0; p < n_parts; ++p)
      for (int32_t r = 0; r < k; ++r) {
        int64_t o = ((int64_t)p * q + j) * k + r;
        if (cand_ids[o] < 0) continue;
        ent[m].s = (double)cand_dists[o];
        ent[m].id = cand_ids[o];
        ++m;
      }
    qsort(ent, (size_t)m, sizeof(orc_entry), cmp);
    for (int32_t r = 0; r < k; ++r) {
      int64_t o = j * (int64_t)k + r;
      if (r < m) {
        ids[o] = ent[r].id;
        dists[o] = (float)ent[r].s;
      } else {
        ids[o] = -1;
        dists[o] = pad_dist(metric);
      }
    }
  }
  free(ent);
  return ORC_OK;
}

/*
 * Range (threshold) selection -- eps as "the score satisfies tau" instead of
 * "the k best":
 *   PAPER.md L354 (Sec. 5): "We use cosine similarity > 0.9 as a vector
 *   distance metric"; L1436 (Sec. 6): "range instead of top-k search";
 *   SPEC.md L129-L133 THRESHOLD mode, L144 "THRESHOLD mode: every returned score
 *   satisfies the threshold; sorted by row_id ascending", L178 ">= tau".
 * For each query every qualifying row with score >= tau (IP, COS) or squared
 * distance <= tau (L2; reading R14), ascending global id, scores in fp64 as in
 * orc_search.  A zero-norm COS query selects nothing (as its top-k row is padding).
 * offsets [q + 1] are always written; ids / dists / scores64 (optional) only
 * when capacity >= offsets[q], else ORC_ERANGE (call again with the total).
 */
enum { ORC_ERANGE = 8 };

static int range_keep(double s, double tau, int32_t metric) { return metric == ORC_L2 ? (s <= tau) : (s >= tau); }

int orc_range(const float *X, int64_t n, int32_t d, const void *const *attrs, const int32_t *attr_types,
              int32_t n_attrs, const orc_clause *clauses, int32_t n_clauses, const float *Qv, int64_t q, double tau,
              int32_t metric, int64_t row_offset, int64_t capacity, int64_t *offsets, int64_t *ids, float *dists,
              double *scores64, int32_t nthreads) {
  if (n < 1 || d < 1 || q < 0 || capacity < 0) return ORC_EINVAL;
  if (metric < ORC_L2 || metric > ORC_COS) return ORC_EINVAL;
  if (isnan(tau)) return ORC_EINVAL;
  int st = check_pred(n_attrs, attr_types, clauses, n_clauses);
  if (st != ORC_OK) return st;
  if (!all_finite(X, n * (int64_t)d) || !all_finite(Qv, q * (int64_t)d)) return ORC_EINVAL;
  if (metric == ORC_COS) {
    for (int64_t i = 0; i < n; ++i)
      if (dot64(X + i * (int64_t)d, X + i * (int64_t)d, d) == 0.0) return ORC_EDEGENERATE;
  }
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  int64_t *sel = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  double *sc = (double *)malloc((size_t)n * sizeof(double));
  if (!sel || !sc) {
    free(sel);
    free(sc);
    return ORC_ENOMEM;
  }
  int64_t nsel = 0;
  st = orc_select(attrs, attr_types, n_attrs, n, clauses, n_clauses, NULL, &nsel, sel);
  if (st != ORC_OK) {
    free(sel);
    free(sc);
    return st;
  }
  offsets[0] = 0;
  /* pass 1: how many rows each query keeps */
  for (int64_t j = 0; j < q; ++j) {
    const float *qv = Qv + j * (int64_t)d;
    int64_t m = 0;
    if (!(metric == ORC_COS && dot64(qv, qv, d) == 0.0)) {
#pragma omp parallel for schedule(static) reduction(+ : m)
      for (int64_t r = 0; r < nsel; ++r) m += range_keep(score64(qv, X + sel[r] * (int64_t)d, d, metric), tau, metric);
    }
    offsets[j + 1] = offsets[j] + m;
  }
  if (offsets[q] > capacity) {
    free(sel);
    free(sc);
    return ORC_ERANGE;
  }
  /* pass 2: the kept rows in ascending id (the selection is ascending) */
  for (int64_t j = 0; j < q; ++j) {
    const float *qv = Qv + j * (int64_t)d;
    if (offsets[j + 1] == offsets[j]) continue;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nsel; ++r) sc[r] = score64(qv, X + sel[r] * (int64_t)d, d, metric);
    int64_t o = offsets[j];
    for (int64_t r = 0; r < nsel; ++r) {
      if (!range_keep(sc[r], tau, metric)) continue;
      ids[o] = row_offset + sel[r];
      dists[o] = (float)sc[r];
      if (scores64) scores64[o] = sc[r];
      ++o;
    }
  }
  free(sel);
  free(sc);
  return ORC_OK;
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
