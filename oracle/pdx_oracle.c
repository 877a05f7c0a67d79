/*
 * pdx_oracle.c — CPU restatement of the reference PDXearch path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 product path (paper_2503_04422_b200/csrc).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  The product never links or calls it.
 *
 * It restates, function by function, the pure-Python/numpy reference
 * package `dimscan` (/root/reference/pkg/src/dimscan), which is the
 * algorithm of record for this path.  Every function cites the reference
 * file:line it follows.  Arithmetic follows numpy's per-ufunc rounding:
 * every float32 subtract / multiply / add is rounded separately (no FMA —
 * build with -ffp-contract=off), sums run in visit order, and float64
 * reductions follow numpy's association order where the reference uses one.
 *
 * Pinning: the tests/golden fixtures were produced by running the reference itself
 * (tests/golden/make_golden.py imports /root/reference); tests/test_oracle.py
 * checks this restatement against those vectors bit-for-bit.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_L2 0
#define ORC_L1 1
#define ORC_IP 2

#define ORC_PRUNER_NONE 0
#define ORC_PRUNER_ADS 1
#define ORC_PRUNER_BOND 2
#define ORC_PRUNER_BSA 3 /* this build's restatement, not in the reference */

#define ORC_SEQUENTIAL 0
#define ORC_DECREASING 1
#define ORC_DMEANS 2
#define ORC_ZONES 3

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENOMEM 2

/* A list of dimension-major blocks: mirrors list[Block] (layout.py:53-83).
 * Block b stores `d` rows of `mp[b]` floats (data[j*mp + i] = dim j of slot i)
 * at data + data_off[b]; its m[b] ids at ids + id_off[b]. */
typedef struct {
  int32_t d;
  int64_t nblocks;
  const float* data;
  const int64_t* data_off;
  const int32_t* m;
  const int32_t* mp;
  const int64_t* ids;
  const int64_t* id_off;
} orc_blocks;

/* SearchParams (search.py:61-85) + AdsPruner (pruning.py:56-65). */
typedef struct {
  int32_t k;
  int32_t metric;
  int32_t pruner;
  int32_t initial_step;
  double selection_fraction;
  int32_t ads_d;
  int32_t _pad;
  double ads_eps0;
  const float* bsa_coef; /* BSA: coef_s = 2 m c_s per schedule step */
} orc_params;

/* SearchStats (search.py:88-103).  survivors, when non-NULL, receives one
 * record per visited block: [len, v_1 .. v_len] (search.py:133, :170-172). */
typedef struct {
  int64_t values_touched;
  int64_t values_total;
  int32_t* survivors;
  int64_t survivors_cap;
  int64_t survivors_len;
  int32_t overflow;
  int32_t _pad;
} orc_stats;

/* ---------------------------------------------------------------- TopK -- */
/* TopK (search.py:27-58): keeps the k smallest (distance, id) pairs; a
 * candidate replaces the worst only if strictly better (search.py:45-51).
 * Kept as an ascending array, which yields the same member set and the same
 * threshold() as the reference's heap. */
typedef struct {
  int32_t k;
  int32_t n;
  float* dist;
  int64_t* id;
} orc_topk;

static int less_pair(float d0, int64_t i0, float d1, int64_t i1) {
  return d0 < d1 || (d0 == d1 && i0 < i1);
}

static float topk_threshold(const orc_topk* t) { /* search.py:39-42 */
  return t->n < t->k ? INFINITY : t->dist[t->n - 1];
}

static void topk_push(orc_topk* t, float d, int64_t id) { /* search.py:44-51 */
  int32_t pos;
  if (t->n < t->k) {
    pos = t->n++;
  } else if (less_pair(d, id, t->dist[t->k - 1], t->id[t->k - 1])) {
    pos = t->k - 1;
  } else {
    return;
  }
  while (pos > 0 && less_pair(d, id, t->dist[pos - 1], t->id[pos - 1])) {
    t->dist[pos] = t->dist[pos - 1];
    t->id[pos] = t->id[pos - 1];
    --pos;
  }
  t->dist[pos] = d;
  t->id[pos] = id;
}

/* ------------------------------------------------------------- kernels -- */
/* vertical_accumulate (kernels.py:41-62): every padded slot, dims
 * order[a:b] (or a..b-1), separate float32 rounding per numpy ufunc. */
static void vertical_accumulate(const float* blk, int32_t mp, const float* q, int32_t a,
                                int32_t b, int32_t metric, float* acc, const int32_t* order) {
  for (int32_t jj = a; jj < b; ++jj) {
    const int32_t j = order ? order[jj] : jj;
    const float* col = blk + (int64_t)j * mp;
    const float qj = q[j];
    if (metric == ORC_L2) {
      for (int32_t i = 0; i < mp; ++i) {
        float t = qj - col[i];
        float sq = t * t;
        acc[i] = acc[i] + sq;
      }
    } else if (metric == ORC_L1) {
      for (int32_t i = 0; i < mp; ++i) acc[i] = acc[i] + fabsf(qj - col[i]);
    } else {
      for (int32_t i = 0; i < mp; ++i) {
        float pr = qj * col[i];
        acc[i] = acc[i] + pr;
      }
    }
  }
}

/* vertical_accumulate_selected (kernels.py:65-91): only listed slots. */
static void vertical_accumulate_selected(const float* blk, int32_t mp, const float* q, int32_t a,
                                         int32_t b, int32_t metric, float* acc,
                                         const int32_t* pos, int32_t npos, const int32_t* order) {
  for (int32_t jj = a; jj < b; ++jj) {
    const int32_t j = order ? order[jj] : jj;
    const float* col = blk + (int64_t)j * mp;
    const float qj = q[j];
    for (int32_t p = 0; p < npos; ++p) {
      const int32_t i = pos[p];
      if (metric == ORC_L2) {
        float t = qj - col[i];
        float sq = t * t;
        acc[i] = acc[i] + sq;
      } else if (metric == ORC_L1) {
        acc[i] = acc[i] + fabsf(qj - col[i]);
      } else {
        float pr = qj * col[i];
        acc[i] = acc[i] + pr;
      }
    }
  }
}

/* --------------------------------------------------------------- search -- */
/* step_schedule (search.py:106-117).  Returns the number of steps; ends[s]
 * is the exclusive end of step s. */
int32_t orc_step_schedule(int32_t d, int32_t initial_step, int32_t* ends, int32_t cap) {
  int32_t n = 0;
  int64_t start = 0, width = initial_step;
  if (d < 1 || initial_step < 1) return -1;
  while (start < d) {
    int64_t end = start + width < d ? start + width : d;
    if (n < cap) ends[n] = (int32_t)end;
    ++n;
    start = end;
    width *= 2;
  }
  return n;
}

/* ads_bound (pruning.py:83-88): float64, left-to-right products. */
double orc_ads_bound(int32_t dims_seen, int32_t ads_d, double eps0, double threshold) {
  if (dims_seen >= ads_d) return threshold;
  double band = 1.0 + eps0 / sqrt((double)dims_seen);
  return threshold * ((double)dims_seen / (double)ads_d) * band * band;
}

static float merge_key(float acc, int32_t metric) { /* search.py:120-122 */
  return metric == ORC_IP ? -acc : acc;
}

static void stats_record(orc_stats* st, const int32_t* vals, int32_t n) {
  if (!st || !st->survivors) return;
  if (st->survivors_len + 1 + n > st->survivors_cap) {
    st->overflow = 1;
    return;
  }
  st->survivors[st->survivors_len++] = n;
  for (int32_t i = 0; i < n; ++i) st->survivors[st->survivors_len++] = vals[i];
}

typedef struct {
  float* acc;
  int32_t* pos;
  int32_t* ends;
  int32_t* surv;
  int32_t cap_mp;
} orc_scratch;

/* BSA residual energy sum_{j=from}^{d-1} v_j^2 of column `slot` of a
 * dimension-major array with row stride `stride` (stride 1 = a plain vector):
 * a sequential float32 sum in increasing j (pdx_bsa_residuals). */
static float residual_energy(const float* v, int32_t stride, int32_t slot, int32_t from,
                             int32_t d) {
  float r = 0.0f;
  for (int32_t j = from; j < d; ++j) {
    const float x = v[(int64_t)j * stride + slot];
    const float t = x * x;
    r = r + t;
  }
  return r;
}

/* _linear_block (search.py:125-135). */
static void linear_block(const orc_blocks* B, int64_t bi, const float* q, const orc_params* p,
                         orc_topk* tk, const int32_t* order, orc_stats* st, orc_scratch* sc) {
  const int32_t mp = B->mp[bi], m = B->m[bi], d = B->d;
  const float* blk = B->data + B->data_off[bi];
  const int64_t* ids = B->ids + B->id_off[bi];
  memset(sc->acc, 0, sizeof(float) * mp);
  vertical_accumulate(blk, mp, q, 0, d, p->metric, sc->acc, order);
  if (st) {
    st->values_touched += (int64_t)m * d;
    int32_t one = m;
    stats_record(st, &one, 1);
  }
  for (int32_t i = 0; i < m; ++i) topk_push(tk, merge_key(sc->acc[i], p->metric), ids[i]);
}

/* _search_block (search.py:138-174): WARMUP over all slots while the
 * surviving fraction stays >= selection_fraction, PRUNE over positions
 * after; a decision pass after every step against the block-start
 * threshold; survivors pushed at block end. */
static void search_block(const orc_blocks* B, int64_t bi, const float* q, const orc_params* p,
                         orc_topk* tk, const int32_t* order, orc_stats* st, orc_scratch* sc) {
  const int32_t mp = B->mp[bi], m = B->m[bi], d = B->d;
  const float* blk = B->data + B->data_off[bi];
  const int64_t* ids = B->ids + B->id_off[bi];
  const int32_t nsteps = orc_step_schedule(d, p->initial_step, sc->ends, 64);
  float* acc = sc->acc;
  int32_t* pos = sc->pos;
  int32_t npos = m;
  int warmup = 1;
  memset(acc, 0, sizeof(float) * mp);
  for (int32_t i = 0; i < m; ++i) pos[i] = i;
  int32_t a = 0;
  for (int32_t s = 0; s < nsteps; ++s) {
    const int32_t b = sc->ends[s];
    int64_t touched;
    if (warmup && ((double)npos / (double)m) >= p->selection_fraction) {
      vertical_accumulate(blk, mp, q, a, b, p->metric, acc, order);
      touched = m;
    } else {
      warmup = 0;
      vertical_accumulate_selected(blk, mp, q, a, b, p->metric, acc, pos, npos, order);
      touched = npos;
    }
    const float threshold = topk_threshold(tk);
    if (threshold != INFINITY) {
      float bound;
      if (p->pruner == ORC_PRUNER_ADS)
        bound = (float)orc_ads_bound(b, p->ads_d, p->ads_eps0, (double)threshold);
      else
        bound = threshold;
      int32_t w = 0;
      if (p->pruner == ORC_PRUNER_BSA) {
        /* BSA (this build's restatement, pdx_b200.h PDX_PRUNER_BSA): keep iff
         * ((acc + rx) + rq) - (coef * sqrt(rx)) * sqrt(rq) < T, float32 */
        const float rq = residual_energy(q, 1, 0, b, d);
        const float nq = sqrtf(rq), coef = p->bsa_coef[s];
        for (int32_t r = 0; r < npos; ++r) {
          const int32_t i = pos[r];
          const float rx = residual_energy(blk, mp, i, b, d);
          const float est = ((acc[i] + rx) + rq) - (coef * sqrtf(rx)) * nq;
          if (est < threshold) pos[w++] = i;
        }
      } else {
        for (int32_t r = 0; r < npos; ++r)
          if (acc[pos[r]] < bound) pos[w++] = pos[r];
      }
      npos = w;
    }
    if (st) st->values_touched += touched * (int64_t)(b - a);
    sc->surv[s] = npos;
    a = b;
  }
  if (st) stats_record(st, sc->surv, nsteps);
  for (int32_t r = 0; r < npos; ++r)
    topk_push(tk, merge_key(acc[pos[r]], p->metric), ids[pos[r]]);
}

static int alloc_scratch(orc_scratch* sc, int32_t cap_mp) {
  sc->cap_mp = cap_mp;
  sc->acc = (float*)malloc(sizeof(float) * (cap_mp > 0 ? cap_mp : 1));
  sc->pos = (int32_t*)malloc(sizeof(int32_t) * (cap_mp > 0 ? cap_mp : 1));
  sc->ends = (int32_t*)malloc(sizeof(int32_t) * 64);
  sc->surv = (int32_t*)malloc(sizeof(int32_t) * 64);
  return (sc->acc && sc->pos && sc->ends && sc->surv) ? ORC_OK : ORC_ENOMEM;
}

static void free_scratch(orc_scratch* sc) {
  free(sc->acc);
  free(sc->pos);
  free(sc->ends);
  free(sc->surv);
}

/* search (search.py:177-205) over B's blocks listed in block_list (NULL =
 * all blocks in stored order).  orders: NULL, or one pointer per listed
 * block (NULL entry = natural order). */
int orc_search(const orc_blocks* B, const int64_t* block_list, int64_t nlisted,
               const int32_t* const* orders, const float* q, const orc_params* p,
               float* out_dist, int64_t* out_ids, int32_t* out_count, orc_stats* st) {
  orc_topk tk = {p->k, 0, out_dist, out_ids};
  if (p->k < 1) return ORC_EINVAL;
  if (p->pruner == ORC_PRUNER_BSA && (!p->bsa_coef || p->metric != ORC_L2))
    return ORC_EINVAL; /* BSA: squared L2 ... */
  if (!block_list) nlisted = B->nblocks;
  if (p->pruner == ORC_PRUNER_BSA && orders)
    for (int64_t r = 0; r < nlisted; ++r)
      if (orders[r]) return ORC_EINVAL; /* ... in natural (principal-axis) order */
  int32_t cap = 1;
  for (int64_t r = 0; r < nlisted; ++r) {
    int64_t bi = block_list ? block_list[r] : r;
    if (B->mp[bi] > cap) cap = B->mp[bi];
  }
  orc_scratch sc;
  if (alloc_scratch(&sc, cap) != ORC_OK) {
    free_scratch(&sc);
    return ORC_ENOMEM;
  }
  if (st) {
    for (int64_t r = 0; r < nlisted; ++r) {
      int64_t bi = block_list ? block_list[r] : r;
      st->values_total += (int64_t)B->m[bi] * B->d;
    }
  }
  for (int64_t r = 0; r < nlisted; ++r) {
    int64_t bi = block_list ? block_list[r] : r;
    const int32_t* order = orders ? orders[r] : NULL;
    if (r == 0 || p->pruner == ORC_PRUNER_NONE || topk_threshold(&tk) == INFINITY)
      linear_block(B, bi, q, p, &tk, order, st, &sc);
    else
      search_block(B, bi, q, p, &tk, order, st, &sc);
  }
  *out_count = tk.n;
  free_scratch(&sc);
  return ORC_OK;
}

/* Public single-block kernels for kernel-level checks (kernels.py:41-91). */
int orc_vertical_accumulate(const float* blk, int32_t d, int32_t mp, const float* q, int32_t a,
                            int32_t b, int32_t metric, float* acc, const int32_t* order) {
  if (!(0 <= a && a <= b && b <= d)) return ORC_EINVAL;
  vertical_accumulate(blk, mp, q, a, b, metric, acc, order);
  return ORC_OK;
}

/* -------------------------------------------------------------- orders -- */
/* numpy's float64 1-D contiguous sum (pairwise with an 8-way unrolled base
 * case, block 128), which bond_dimension_order's zone scores go through
 * (pruning.py:135, `gaps[s:s+w].sum()`). */
double orc_numpy_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return orc_numpy_sum(a, n2) + orc_numpy_sum(a + n2, n - n2);
  }
}

typedef struct {
  double key;
  int32_t idx;
} orc_kv;

/* ascending key, ties to the lower index == numpy argsort(kind="stable") */
static int kv_cmp(const void* x, const void* y) {
  const orc_kv* a = (const orc_kv*)x;
  const orc_kv* b = (const orc_kv*)y;
  if (a->key < b->key) return -1;
  if (a->key > b->key) return 1;
  return (a->idx > b->idx) - (a->idx < b->idx);
}

int32_t orc_default_zone_width(int32_t d) { /* pruning.py:98-99 */
  int32_t w = d / 16 > 8 ? d / 16 : 8;
  return d < w ? d : w;
}

/* bond_dimension_order (pruning.py:107-140). zone_width <= 0 => default. */
int orc_dimension_order(const double* q, const double* means, int32_t d, int32_t criteria,
                        int32_t zone_width, int32_t* out) {
  if (criteria == ORC_SEQUENTIAL) {
    for (int32_t j = 0; j < d; ++j) out[j] = j;
    return ORC_OK;
  }
  orc_kv* kv = (orc_kv*)malloc(sizeof(orc_kv) * (d > 0 ? d : 1));
  double* gaps = (double*)malloc(sizeof(double) * (d > 0 ? d : 1));
  if (!kv || !gaps) {
    free(kv);
    free(gaps);
    return ORC_ENOMEM;
  }
  int rc = ORC_OK;
  if (criteria == ORC_DECREASING) {
    for (int32_t j = 0; j < d; ++j) kv[j].key = -q[j], kv[j].idx = j;
    qsort(kv, d, sizeof(orc_kv), kv_cmp);
    for (int32_t j = 0; j < d; ++j) out[j] = kv[j].idx;
  } else {
    for (int32_t j = 0; j < d; ++j) gaps[j] = fabs(q[j] - means[j]);
    if (criteria == ORC_DMEANS) {
      for (int32_t j = 0; j < d; ++j) kv[j].key = -gaps[j], kv[j].idx = j;
      qsort(kv, d, sizeof(orc_kv), kv_cmp);
      for (int32_t j = 0; j < d; ++j) out[j] = kv[j].idx;
    } else if (criteria == ORC_ZONES) {
      if (zone_width <= 0) zone_width = orc_default_zone_width(d);
      int32_t nz = (d + zone_width - 1) / zone_width;
      for (int32_t z = 0; z < nz; ++z) {
        int32_t s = z * zone_width;
        int32_t e = s + zone_width < d ? s + zone_width : d;
        kv[z].key = -orc_numpy_sum(gaps + s, e - s);
        kv[z].idx = z;
      }
      qsort(kv, nz, sizeof(orc_kv), kv_cmp);
      int32_t w = 0;
      for (int32_t r = 0; r < nz; ++r) {
        int32_t s = kv[r].idx * zone_width;
        int32_t e = s + zone_width < d ? s + zone_width : d;
        for (int32_t j = s; j < e; ++j) out[w++] = j;
      }
    } else {
      rc = ORC_EINVAL;
    }
  }
  free(kv);
  free(gaps);
  return rc;
}

/* --------------------------------------------------------- IVF / exact -- */
/* ivf_select_buckets (index.py:111-127): vertical kernel over the centroid
 * chain, stable argsort of the float32 distances (negated for IP). */
int orc_select_buckets(const orc_blocks* C, int32_t nlist, const float* q, int32_t metric,
                       int32_t nprobe, int32_t* out) {
  if (!(1 <= nprobe && nprobe <= nlist)) return ORC_EINVAL;
  orc_kv* kv = (orc_kv*)malloc(sizeof(orc_kv) * nlist);
  int32_t cap = 1;
  for (int64_t b = 0; b < C->nblocks; ++b)
    if (C->mp[b] > cap) cap = C->mp[b];
  float* acc = (float*)malloc(sizeof(float) * cap);
  if (!kv || !acc) {
    free(kv);
    free(acc);
    return ORC_ENOMEM;
  }
  int32_t pos = 0;
  for (int64_t b = 0; b < C->nblocks; ++b) {
    memset(acc, 0, sizeof(float) * C->mp[b]);
    vertical_accumulate(C->data + C->data_off[b], C->mp[b], q, 0, C->d, metric, acc, NULL);
    for (int32_t i = 0; i < C->m[b]; ++i, ++pos) {
      float dist = acc[i];
      kv[pos].key = metric == ORC_IP ? -(double)dist : (double)dist;
      kv[pos].idx = pos;
    }
  }
  qsort(kv, nlist, sizeof(orc_kv), kv_cmp);
  for (int32_t r = 0; r < nprobe; ++r) out[r] = kv[r].idx;
  free(kv);
  free(acc);
  return ORC_OK;
}

/* An IvfIndex (index.py:75-88): centroid chain + bucket chains stored back to
 * back in `buckets`, bucket c owning blocks [bucket_off[c], bucket_off[c+1]),
 * plus per-bucket float64 means. */
typedef struct {
  int32_t nlist;
  int32_t _pad;
  const orc_blocks* centroids;
  const orc_blocks* buckets;
  const int64_t* bucket_off;
  const double* bucket_means;
} orc_ivf;

/* Batched query outputs; per query q: dist/ids rows of k, count, stats. */
typedef struct {
  float* dist;
  int64_t* ids;
  int32_t* count;
  int64_t* touched;
  int64_t* total;
  int32_t* survivors; /* optional [nq][surv_cap] records as orc_stats */
  int64_t surv_cap;
  int64_t* surv_len;  /* optional [nq] */
  int32_t* selected;  /* optional [nq][nprobe] (IVF only) */
} orc_batch_out;

typedef struct {
  int kind; /* 0 = ivf, 1 = exact */
  const orc_ivf* ivf;
  const orc_blocks* flat;
  const double* global_means;
  const float* queries;
  int64_t nq;
  const orc_params* p;
  int32_t nprobe;
  int32_t criteria;
  int32_t zone_width;
  const orc_batch_out* out;
  int64_t next;
  pthread_mutex_t mu;
  int rc;
} orc_job;

/* ivf_search (index.py:130-156) for one query. */
static int ivf_one(const orc_job* J, int64_t qi) {
  const orc_ivf* I = J->ivf;
  const int32_t d = I->buckets->d;
  const float* q = J->queries + qi * d;
  const orc_params* p = J->p;
  int32_t* sel = (int32_t*)malloc(sizeof(int32_t) * J->nprobe);
  double* qd = (double*)malloc(sizeof(double) * d);
  if (!sel || !qd) return ORC_ENOMEM;
  int rc = orc_select_buckets(I->centroids, I->nlist, q, p->metric, J->nprobe, sel);
  if (rc) return rc;
  if (J->out->selected)
    memcpy(J->out->selected + qi * J->nprobe, sel, sizeof(int32_t) * J->nprobe);
  int64_t nb = 0;
  for (int32_t r = 0; r < J->nprobe; ++r) nb += I->bucket_off[sel[r] + 1] - I->bucket_off[sel[r]];
  int64_t* list = (int64_t*)malloc(sizeof(int64_t) * (nb > 0 ? nb : 1));
  const int32_t** ord = (const int32_t**)malloc(sizeof(int32_t*) * (nb > 0 ? nb : 1));
  int32_t* ordbuf = NULL;
  int use_orders = p->pruner == ORC_PRUNER_BOND && J->criteria != ORC_SEQUENTIAL;
  if (use_orders) ordbuf = (int32_t*)malloc(sizeof(int32_t) * d * J->nprobe);
  for (int32_t j = 0; j < d; ++j) qd[j] = (double)q[j];
  int64_t w = 0;
  for (int32_t r = 0; r < J->nprobe; ++r) {
    const int32_t c = sel[r];
    const int32_t* o = NULL;
    if (use_orders) {
      rc = orc_dimension_order(qd, I->bucket_means + (int64_t)c * d, d, J->criteria,
                               J->zone_width, ordbuf + (int64_t)r * d);
      if (rc) return rc;
      o = ordbuf + (int64_t)r * d;
    }
    for (int64_t b = I->bucket_off[c]; b < I->bucket_off[c + 1]; ++b) {
      list[w] = b;
      ord[w] = o;
      ++w;
    }
  }
  orc_stats st = {0, 0, NULL, 0, 0, 0, 0};
  if (J->out->survivors) {
    st.survivors = J->out->survivors + qi * J->out->surv_cap;
    st.survivors_cap = J->out->surv_cap;
  }
  rc = orc_search(I->buckets, list, nb, ord, q, p, J->out->dist + qi * p->k,
                  J->out->ids + qi * p->k, J->out->count + qi, &st);
  if (J->out->touched) J->out->touched[qi] = st.values_touched;
  if (J->out->total) J->out->total[qi] = st.values_total;
  if (J->out->surv_len) J->out->surv_len[qi] = st.overflow ? -1 : st.survivors_len;
  free(sel);
  free(qd);
  free(list);
  free(ord);
  free(ordbuf);
  return rc;
}

/* exact_search (index.py:182-191) for one query. */
static int exact_one(const orc_job* J, int64_t qi) {
  const orc_blocks* B = J->flat;
  const int32_t d = B->d;
  const float* q = J->queries + qi * d;
  const orc_params* p = J->p;
  int32_t* order = NULL;
  const int32_t** ord = NULL;
  int rc = ORC_OK;
  if (p->pruner == ORC_PRUNER_BOND && J->criteria != ORC_SEQUENTIAL) {
    double* qd = (double*)malloc(sizeof(double) * d);
    order = (int32_t*)malloc(sizeof(int32_t) * d);
    ord = (const int32_t**)malloc(sizeof(int32_t*) * (B->nblocks > 0 ? B->nblocks : 1));
    for (int32_t j = 0; j < d; ++j) qd[j] = (double)q[j];
    rc = orc_dimension_order(qd, J->global_means, d, J->criteria, J->zone_width, order);
    free(qd);
    if (rc) return rc;
    for (int64_t b = 0; b < B->nblocks; ++b) ord[b] = order;
  }
  orc_stats st = {0, 0, NULL, 0, 0, 0, 0};
  if (J->out->survivors) {
    st.survivors = J->out->survivors + qi * J->out->surv_cap;
    st.survivors_cap = J->out->surv_cap;
  }
  rc = orc_search(B, NULL, B->nblocks, ord, q, p, J->out->dist + qi * p->k,
                  J->out->ids + qi * p->k, J->out->count + qi, &st);
  if (J->out->touched) J->out->touched[qi] = st.values_touched;
  if (J->out->total) J->out->total[qi] = st.values_total;
  if (J->out->surv_len) J->out->surv_len[qi] = st.overflow ? -1 : st.survivors_len;
  free(order);
  free(ord);
  return rc;
}

static void* job_worker(void* arg) {
  orc_job* J = (orc_job*)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int64_t qi = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (qi >= J->nq) break;
    int rc = J->kind == 0 ? ivf_one(J, qi) : exact_one(J, qi);
    if (rc) {
      pthread_mutex_lock(&J->mu);
      J->rc = rc;
      pthread_mutex_unlock(&J->mu);
    }
  }
  return NULL;
}

static int run_job(orc_job* J, int32_t nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_mutex_init(&J->mu, NULL);
  J->next = 0;
  J->rc = ORC_OK;
  if (nthreads == 1) {
    job_worker(J);
  } else {
    pthread_t th[256];
    for (int32_t t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, job_worker, J);
    for (int32_t t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  }
  pthread_mutex_destroy(&J->mu);
  return J->rc;
}

/* IvfNearestNeighbors.kneighbors' per-query loop (estimators.py:127-131)
 * over already-rotated queries, spread over `nthreads` host threads (the
 * reference notes distinct queries may run concurrently). */
int orc_ivf_search_batch(const orc_ivf* I, const float* queries, int64_t nq, const orc_params* p,
                         int32_t nprobe, int32_t criteria, int32_t zone_width,
                         const orc_batch_out* out, int32_t nthreads) {
  if (!(1 <= nprobe && nprobe <= I->nlist) || p->k < 1) return ORC_EINVAL;
  orc_job J;
  memset(&J, 0, sizeof(J));
  J.kind = 0;
  J.ivf = I;
  J.queries = queries;
  J.nq = nq;
  J.p = p;
  J.nprobe = nprobe;
  J.criteria = criteria;
  J.zone_width = zone_width;
  J.out = out;
  return run_job(&J, nthreads);
}

/* ExactNearestNeighbors.kneighbors' per-query loop (estimators.py:71-75). */
int orc_exact_search_batch(const orc_blocks* B, const double* global_means, const float* queries,
                           int64_t nq, const orc_params* p, int32_t criteria, int32_t zone_width,
                           const orc_batch_out* out, int32_t nthreads) {
  if (p->k < 1) return ORC_EINVAL;
  orc_job J;
  memset(&J, 0, sizeof(J));
  J.kind = 1;
  J.flat = B;
  J.global_means = global_means;
  J.queries = queries;
  J.nq = nq;
  J.p = p;
  J.criteria = criteria;
  J.zone_width = zone_width;
  J.out = out;
  return run_job(&J, nthreads);
}
