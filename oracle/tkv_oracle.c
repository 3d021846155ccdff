/*
 * tkv_oracle.c — CPU restatement of the reference's top-k decode attention, in C.
 *
 * TEST INFRASTRUCTURE ONLY: used by tests/ (cross-check of the numpy oracle), by
 * bench.py's cpu_baseline / `--impl reference` legs (timed on the host cores), never by the
 * product path. Every step follows the reference (/root/reference/pkg/src/topk_kv):
 *
 *   scan    ann_kernels.py:31-47  s[i] = sum_j f64(K[i,j]) * f64(q[j]), strict left-to-right
 *   select  ann.py:154-167        k >= N: all rows by (score desc, id asc); else the k-th
 *                                 largest score t, every row with s > t plus the LOWEST-id
 *                                 rows with s == t, ordered (score desc, id asc)
 *   pinned  attention.py:152-154  ids = unique(concat(arange(min(p, N)), ids)) (ascending)
 *   attend  attention.py:158-167  s_ctx = (K[ids]·q)/sqrt(d) and s_gen = (K_gen·q)/sqrt(d)
 *                                 in f64, then _joint_attend (attention.py:107-122):
 *                                 joint softmax over [s_ctx, s_gen], or the additive form.
 * Layer batching follows decode_step's per-head loop (attention.py:213-230) with the GQA
 * mapping q head h -> kv head h / (Hq/Hkv). Parallelism: OpenMP over heads, or over rows of
 * the scan when there are fewer heads than threads.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static double dot_strict(const float* a, const float* b, int d) {
  double s = 0.0;
  for (int j = 0; j < d; ++j) s += (double)a[j] * (double)b[j];
  return s;
}

/* quickselect: value of rank r (0-based) in descending order of x[0..n) (x is permuted) */
static double kth_desc(double* x, int64_t n, int64_t r) {
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const double pivot = x[lo + (hi - lo) / 2];
    int64_t i = lo, j = hi;
    while (i <= j) {
      while (x[i] > pivot) ++i;
      while (x[j] < pivot) --j;
      if (i <= j) {
        const double t = x[i];
        x[i] = x[j];
        x[j] = t;
        ++i;
        --j;
      }
    }
    if (r <= j)
      hi = j;
    else if (r >= i)
      lo = i;
    else
      return x[r];
  }
  return x[r];
}

typedef struct {
  double s;
  int64_t id;
} scored_t;

static int cmp_desc_id_asc(const void* a, const void* b) {
  const scored_t* x = (const scored_t*)a;
  const scored_t* y = (const scored_t*)b;
  if (x->s > y->s) return -1;
  if (x->s < y->s) return 1;
  return (x->id > y->id) - (x->id < y->id);
}

static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* _flat_topk (ann.py:154-167) on precomputed scores; returns count, ids ordered. */
static int64_t flat_topk(const double* s, int64_t n, int64_t k, int64_t* ids, double* work) {
  if (k > n) k = n;
  scored_t* c = (scored_t*)malloc(sizeof(scored_t) * (size_t)(k > 0 ? k : 1));
  int64_t m = 0;
  if (k == n) {
    for (int64_t i = 0; i < n; ++i) c[m++] = (scored_t){s[i], i};
  } else {
    memcpy(work, s, sizeof(double) * (size_t)n);
    const double t = kth_desc(work, n, k - 1);
    for (int64_t i = 0; i < n; ++i)
      if (s[i] > t) c[m++] = (scored_t){s[i], i};
    for (int64_t i = 0; i < n && m < k; ++i)
      if (s[i] == t) c[m++] = (scored_t){s[i], i};
  }
  qsort(c, (size_t)m, sizeof(scored_t), cmp_desc_id_asc);
  for (int64_t i = 0; i < m; ++i) ids[i] = c[i].id;
  free(c);
  return m;
}

static void joint_attend(const double* s_ctx, const double* v_ctx, int64_t m, const double* s_gen,
                         const double* v_gen, int64_t g, int d, int combine, float* out) {
  double* acc = (double*)calloc((size_t)d, sizeof(double));
  if (combine == 0) {
    double mx = -INFINITY;
    for (int64_t i = 0; i < m; ++i) mx = s_ctx[i] > mx ? s_ctx[i] : mx;
    for (int64_t i = 0; i < g; ++i) mx = s_gen[i] > mx ? s_gen[i] : mx;
    double den = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      const double w = exp(s_ctx[i] - mx);
      den += w;
      for (int j = 0; j < d; ++j) acc[j] += w * v_ctx[i * d + j];
    }
    for (int64_t i = 0; i < g; ++i) {
      const double w = exp(s_gen[i] - mx);
      den += w;
      for (int j = 0; j < d; ++j) acc[j] += w * v_gen[i * d + j];
    }
    for (int j = 0; j < d; ++j) out[j] = (float)(acc[j] / den);
  } else {
    for (int part = 0; part < 2; ++part) {
      const double* s = part ? s_gen : s_ctx;
      const double* v = part ? v_gen : v_ctx;
      const int64_t cnt = part ? g : m;
      if (!cnt) continue;
      double mx = -INFINITY, den = 0.0;
      for (int64_t i = 0; i < cnt; ++i) mx = s[i] > mx ? s[i] : mx;
      double* num = (double*)calloc((size_t)d, sizeof(double));
      for (int64_t i = 0; i < cnt; ++i) {
        const double w = exp(s[i] - mx);
        den += w;
        for (int j = 0; j < d; ++j) num[j] += w * v[i * d + j];
      }
      for (int j = 0; j < d; ++j) acc[j] += num[j] / den;
      free(num);
    }
    for (int j = 0; j < d; ++j) out[j] = (float)acc[j];
  }
  free(acc);
}

/*
 * One head: topk_attend (attention.py:125-167) with a flat index and in-memory values.
 * ids_out must hold min(k, n) + max(0, pinned) entries; returns the number of logged ids
 * (the retrieval log, attention.py:155-156). scores_out (optional, n doubles) receives the scan.
 */
int64_t tkv_oracle_attend(const float* q, const float* keys, const float* values, int64_t n, int d,
                          const float* win_k, const float* win_v, int64_t n_gen, int64_t k,
                          int combine, int64_t pinned, int scan_threads, float* out, int64_t* ids_out,
                          double* scores_out) {
  double* s = scores_out ? scores_out : (double*)malloc(sizeof(double) * (size_t)n);
  double* work = (double*)malloc(sizeof(double) * (size_t)n);
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(scan_threads > 0 ? scan_threads : 1) if (scan_threads > 1 && n >= 65536)
#endif
  for (int64_t i = 0; i < n; ++i) s[i] = dot_strict(keys + i * d, q, d);
  if (k > n) k = n;
  int64_t m = flat_topk(s, n, k, ids_out, work);
  if (pinned > 0) {
    const int64_t p = pinned < n ? pinned : n;
    for (int64_t i = 0; i < p; ++i) ids_out[m + i] = i;
    qsort(ids_out, (size_t)(m + p), sizeof(int64_t), cmp_i64);
    int64_t u = 0;
    for (int64_t i = 0; i < m + p; ++i)
      if (u == 0 || ids_out[i] != ids_out[u - 1]) ids_out[u++] = ids_out[i];
    m = u;
  }
  const double scale = 1.0 / sqrt((double)d);
  double* s_ctx = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  double* v_ctx = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1) * d);
  for (int64_t i = 0; i < m; ++i) {
    s_ctx[i] = dot_strict(keys + ids_out[i] * d, q, d) * scale;
    for (int j = 0; j < d; ++j) v_ctx[i * d + j] = (double)values[ids_out[i] * d + j];
  }
  double* s_gen = (double*)malloc(sizeof(double) * (size_t)(n_gen > 0 ? n_gen : 1));
  double* v_gen = (double*)malloc(sizeof(double) * (size_t)(n_gen > 0 ? n_gen : 1) * d);
  for (int64_t i = 0; i < n_gen; ++i) {
    s_gen[i] = dot_strict(win_k + i * d, q, d) * scale;
    for (int j = 0; j < d; ++j) v_gen[i * d + j] = (double)win_v[i * d + j];
  }
  joint_attend(s_ctx, v_ctx, m, s_gen, v_gen, n_gen, d, combine, out);
  free(s_ctx);
  free(v_ctx);
  free(s_gen);
  free(v_gen);
  free(work);
  if (!scores_out) free(s);
  return m;
}

/*
 * One layer for a batch (decode_step's head loop, attention.py:213-230; GQA h -> h/G).
 * q [B,Hq,d], caches [B,Hkv,rows,d] f32; window rows follow the context. ids_out
 * [B*Hq*(k+pinned)], counts_out [B*Hq]. threads: total host threads to use.
 */
int tkv_oracle_layer(const float* q, const float* kc, const float* vc, int B, int Hq, int Hkv,
                     int64_t rows, int d, const int32_t* n_ctx, const int32_t* n_win, int64_t k,
                     int combine, int64_t pinned, int threads, float* out, int64_t* ids_out,
                     int64_t* counts_out) {
  const int G = Hq / Hkv;
  const int nh = B * Hq;
  const int64_t stride_ids = k + (pinned > 0 ? pinned : 0);
  if (threads < 1) threads = 1;
  const int head_par = nh >= threads;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic) num_threads(threads) if (head_par)
#endif
  for (int bh = 0; bh < nh; ++bh) {
    const int b = bh / Hq, h = bh % Hq, kv = h / G;
    const int64_t n = n_ctx[b], w = n_win ? n_win[b] : 0;
    const float* kb = kc + ((int64_t)b * Hkv + kv) * rows * d;
    const float* vb = vc + ((int64_t)b * Hkv + kv) * rows * d;
    counts_out[bh] = tkv_oracle_attend(q + (int64_t)bh * d, kb, vb, n, d, kb + n * d, vb + n * d, w, k,
                                       combine, pinned, head_par ? 1 : threads, out + (int64_t)bh * d,
                                       ids_out + (int64_t)bh * stride_ids, NULL);
  }
  return 0;
}

int tkv_oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
