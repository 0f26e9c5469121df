/*
 * so_mpchol.c — oracle restatement of proj/src/mpchol.cpp and
 * proj/tests/support/reference.cpp:10-44 (TEST INFRASTRUCTURE, see
 * sphemu_oracle.h). Tile kernels compute in double and store through the
 * tile's precision after every write (mpchol.cpp:283-316, 360-363).
 */
#define _GNU_SOURCE
#include <dlfcn.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "sphemu_oracle.h"

/* ---------------- config, precision map (mpchol.cpp:55-93) ---------------- */
int so_config_validate(const so_chol_config* c) {
  if (c->tile_size < 1) return -1;
  if (c->band_width_dp < 1) return -1;
  if (!(c->sp_fraction >= 0.0 && c->sp_fraction <= 1.0)) return -1;
  if (c->workers < 1) return -1;
  if (c->variant < 0 || c->variant > 3) return -1;
  return 0;
}

int so_assign_precisions(int nt, const so_chol_config* c, uint8_t* out) {
  if (so_config_validate(c) || nt < 1) return -1;
  const int64_t total = (int64_t)nt * (nt + 1) / 2;
  memset(out, SO_DP, (size_t)total);
  if (c->variant == SO_V_DP) return 0;
  /* Off-band tiles sorted by (distance, i, j) (mpchol.cpp:75-79): for fixed
   * distance d the tiles are (j + d, j), j ascending, which is i ascending. */
  int64_t n_off = 0;
  for (int d = c->band_width_dp; d < nt; ++d) n_off += nt - d;
  int64_t n_sp = n_off;
  if (c->variant == SO_V_DPSPHP) n_sp = (int64_t)ceil(c->sp_fraction * (double)n_off);
  else if (c->variant == SO_V_DPHP) n_sp = 0;
  int64_t t = 0;
  for (int d = c->band_width_dp; d < nt; ++d)
    for (int j = 0; j + d < nt; ++j, ++t) {
      int i = j + d;
      out[(int64_t)i * (i + 1) / 2 + j] = (uint8_t)(t < n_sp ? SO_SP : SO_HP);
    }
  return 0;
}

/* ---------------- task graph (mpchol.cpp:156-205) ---------------- */
int64_t so_task_count(int nt) {
  int64_t n = nt;
  return n + n * (n - 1) / 2 * 2 + n * (n - 1) * (n - 2) / 6;
}

typedef struct {
  int nt;
  int64_t* potrf;
  int64_t* trsm; /* [i*nt+k] */
  int64_t* syrk; /* [i*nt+k] */
  int64_t* gemm; /* [(i*nt+j)*nt+k] */
} so_ids;

int64_t so_task_graph(int nt, uint8_t* kind, int32_t* ti, int32_t* tj, int32_t* tk,
                      int64_t* succ_off, int32_t* succ, int32_t* indegree, int64_t succ_cap) {
  const int64_t count = so_task_count(nt);
  int64_t* potrf = calloc((size_t)nt, sizeof(int64_t));
  int64_t* trsm = malloc(sizeof(int64_t) * (size_t)nt * nt);
  int64_t* syrk = malloc(sizeof(int64_t) * (size_t)nt * nt);
  int64_t* gemm = malloc(sizeof(int64_t) * (size_t)nt * nt * nt);
  int64_t id = 0;
#define ADD(K, I, J, KK) (kind[id] = (K), ti[id] = (I), tj[id] = (J), tk[id] = (KK), id++)
  for (int k = 0; k < nt; ++k) {
    potrf[k] = ADD(0, k, k, k);
    for (int i = k + 1; i < nt; ++i) trsm[i * nt + k] = ADD(1, i, k, k);
    for (int i = k + 1; i < nt; ++i) syrk[i * nt + k] = ADD(2, i, i, k);
  }
  for (int k = 0; k < nt; ++k)
    for (int j = k + 1; j < nt; ++j)
      for (int i = j + 1; i < nt; ++i) gemm[((int64_t)i * nt + j) * nt + k] = ADD(3, i, j, k);
#undef ADD
  /* Two passes over the same edge list: count, then fill (CSR). */
  int64_t edges = 0;
  for (int pass = 0; pass < 2; ++pass) {
    int64_t* fill = NULL;
    if (pass == 1) {
      succ_off[0] = 0;
      for (int64_t t = 0; t < count; ++t) succ_off[t + 1] += succ_off[t];
      fill = calloc((size_t)count, sizeof(int64_t));
      if (edges > succ_cap) {
        free(fill);
        edges = -edges;
        break;
      }
    } else {
      memset(succ_off, 0, sizeof(int64_t) * (size_t)(count + 1));
      memset(indegree, 0, sizeof(int32_t) * (size_t)count);
    }
#define EDGE(F, T)                                              \
  do {                                                          \
    if (pass == 0) {                                            \
      succ_off[(F) + 1]++;                                      \
      indegree[(T)]++;                                          \
      edges++;                                                  \
    } else {                                                    \
      succ[succ_off[(F)] + fill[(F)]++] = (int32_t)(T);         \
    }                                                           \
  } while (0)
    for (int k = 0; k < nt; ++k)
      for (int i = k + 1; i < nt; ++i) {
        EDGE(potrf[k], trsm[i * nt + k]);
        EDGE(trsm[i * nt + k], syrk[i * nt + k]);
        for (int j = k + 1; j < i; ++j) EDGE(trsm[i * nt + k], gemm[((int64_t)i * nt + j) * nt + k]);
        for (int j = i + 1; j < nt; ++j) EDGE(trsm[i * nt + k], gemm[((int64_t)j * nt + i) * nt + k]);
      }
    for (int i = 1; i < nt; ++i) {
      for (int k = 0; k + 1 < i; ++k) EDGE(syrk[i * nt + k], syrk[i * nt + k + 1]);
      EDGE(syrk[i * nt + i - 1], potrf[i]);
    }
    for (int i = 0; i < nt; ++i)
      for (int j = 1; j < i; ++j) {
        for (int k = 0; k + 1 < j; ++k)
          EDGE(gemm[((int64_t)i * nt + j) * nt + k], gemm[((int64_t)i * nt + j) * nt + k + 1]);
        EDGE(gemm[((int64_t)i * nt + j) * nt + j - 1], trsm[i * nt + j]);
      }
#undef EDGE
    if (fill) free(fill);
  }
  free(potrf);
  free(trsm);
  free(syrk);
  free(gemm);
  return edges;
}

/* ---------------- quantization (mpchol.cpp:207-225) ---------------- */
void so_quantize_tile(double* t, int64_t n, int prec, int hp_format, so_counters* c) {
  if (prec == SO_DP) return;
  if (prec == SO_SP) {
    for (int64_t i = 0; i < n; ++i) t[i] = (double)(float)t[i];
    if (c) c->demotions_sp += n;
    return;
  }
  long long sat = 0;
  if (hp_format == SO_HP_BF16)
    for (int64_t i = 0; i < n; ++i) t[i] = so_quantize_bf16(t[i], &sat);
  else
    for (int64_t i = 0; i < n; ++i) t[i] = so_quantize_half(t[i], &sat);
  if (c) {
    c->demotions_hp += n;
    c->half_saturations += sat;
  }
}

/* ---------------- packed tiles (mpchol.cpp:95-154) ---------------- */
static int tile_rows(int n, int b, int i) { return (n - i * b) < b ? (n - i * b) : b; }

int64_t so_tiled_size(int n, int b) {
  int nt = (n + b - 1) / b;
  int64_t off = 0;
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j <= i; ++j) off += (int64_t)tile_rows(n, b, i) * tile_rows(n, b, j);
  return off;
}

static int64_t* tile_offsets(int n, int b) {
  int nt = (n + b - 1) / b;
  int64_t* off = malloc(sizeof(int64_t) * ((size_t)nt * (nt + 1) / 2 + 1));
  int64_t o = 0, idx = 0;
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j <= i; ++j) {
      off[idx++] = o;
      o += (int64_t)tile_rows(n, b, i) * tile_rows(n, b, j);
    }
  off[idx] = o;
  return off;
}

void so_tiled_from_dense(const double* a, int n, int b, double* tiles) {
  int nt = (n + b - 1) / b;
  int64_t* off = tile_offsets(n, b);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j <= i; ++j) {
      double* dst = tiles + off[(int64_t)i * (i + 1) / 2 + j];
      int bi = tile_rows(n, b, i), bj = tile_rows(n, b, j);
      for (int r = 0; r < bi; ++r)
        for (int c = 0; c < bj; ++c)
          dst[(int64_t)r * bj + c] = a[(int64_t)(i * b + r) * n + (j * b + c)];
    }
  free(off);
}

void so_tiled_to_dense_lower(const double* tiles, int n, int b, double* a) {
  int nt = (n + b - 1) / b;
  int64_t* off = tile_offsets(n, b);
  memset(a, 0, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j <= i; ++j) {
      const double* src = tiles + off[(int64_t)i * (i + 1) / 2 + j];
      int bi = tile_rows(n, b, i), bj = tile_rows(n, b, j);
      for (int r = 0; r < bi; ++r)
        for (int c = 0; c < bj; ++c) {
          int row = i * b + r, col = j * b + c;
          if (col <= row) a[(int64_t)row * n + col] = src[(int64_t)r * bj + c];
        }
    }
  free(off);
}

/* ---------------- tile kernels ---------------- */
/* Optional BLAS (OpenBLAS from scipy.libs) as the Eigen stand-in for timing. */
typedef void (*dgemm_fn)(int, int, int, int, int, int, double, const double*, int, const double*,
                         int, double, double*, int);
typedef void (*dtrsm_fn)(int, int, int, int, int, int, int, double, const double*, int, double*,
                         int);
static dgemm_fn g_dgemm = NULL;
static dtrsm_fn g_dtrsm = NULL;

int so_use_blas(const char* path) {
  if (!path) {
    g_dgemm = NULL;
    g_dtrsm = NULL;
    return 0;
  }
  void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!h) return -1;
  g_dgemm = (dgemm_fn)dlsym(h, "scipy_cblas_dgemm");
  g_dtrsm = (dtrsm_fn)dlsym(h, "scipy_cblas_dtrsm");
  if (!g_dgemm) g_dgemm = (dgemm_fn)dlsym(h, "cblas_dgemm");
  if (!g_dtrsm) g_dtrsm = (dtrsm_fn)dlsym(h, "cblas_dtrsm");
  typedef void (*setnt_fn)(int);
  setnt_fn snt = (setnt_fn)dlsym(h, "scipy_openblas_set_num_threads");
  if (!snt) snt = (setnt_fn)dlsym(h, "openblas_set_num_threads");
  if (snt) snt(1); /* one BLAS thread per DAG task, like Eigen inside a worker */
  return (g_dgemm && g_dtrsm) ? 0 : -1;
}

/* mpchol.cpp:230-252: unblocked Cholesky-Crout of one diagonal tile. */
static int potrf_tile(double* a, int b) {
  for (int c = 0; c < b; ++c) {
    double pivot = a[(int64_t)c * b + c];
    for (int k = 0; k < c; ++k) {
      double v = a[(int64_t)c * b + k];
      pivot -= v * v;
    }
    if (!(pivot > 0.0)) return c + 1;
    double l = sqrt(pivot);
    a[(int64_t)c * b + c] = l;
    for (int r = c + 1; r < b; ++r) {
      double v = a[(int64_t)r * b + c];
      for (int k = 0; k < c; ++k) v -= a[(int64_t)r * b + k] * a[(int64_t)c * b + k];
      a[(int64_t)r * b + c] = v / l;
    }
  }
  for (int r = 0; r < b; ++r)
    for (int c = r + 1; c < b; ++c) a[(int64_t)r * b + c] = 0.0;
  return 0;
}

/* mpchol.cpp:293-299: X <- X * L^{-T} (X is bi x bk, L is bk x bk lower). */
static void trsm_tile(double* x, const double* l, int bi, int bk) {
  if (g_dtrsm) {
    /* CblasRowMajor=101, Right=142, Lower=122, Trans=112, NonUnit=131 */
    g_dtrsm(101, 142, 122, 112, 131, bi, bk, 1.0, l, bk, x, bk);
    return;
  }
  for (int r = 0; r < bi; ++r) {
    double* xr = x + (int64_t)r * bk;
    for (int c = 0; c < bk; ++c) {
      double v = xr[c];
      const double* lc = l + (int64_t)c * bk;
      for (int t = 0; t < c; ++t) v -= xr[t] * lc[t];
      xr[c] = v / lc[c];
    }
  }
}

/* mpchol.cpp:300-314: C -= P * Q^T (C bi x bj, P bi x bk, Q bj x bk). */
static void gemm_nt_sub(double* c, const double* p, const double* q, int bi, int bj, int bk) {
  if (g_dgemm) {
    /* RowMajor, NoTrans=111, Trans=112 */
    g_dgemm(101, 111, 112, bi, bj, bk, -1.0, p, bk, q, bk, 1.0, c, bj);
    return;
  }
  double* qt = malloc(sizeof(double) * (size_t)bk * bj);
  for (int s = 0; s < bj; ++s)
    for (int t = 0; t < bk; ++t) qt[(int64_t)t * bj + s] = q[(int64_t)s * bk + t];
  double* acc = malloc(sizeof(double) * (size_t)bj);
  for (int r = 0; r < bi; ++r) {
    memset(acc, 0, sizeof(double) * (size_t)bj);
    const double* pr = p + (int64_t)r * bk;
    for (int t = 0; t < bk; ++t) {
      const double pv = pr[t];
      const double* qrow = qt + (int64_t)t * bj;
      for (int s = 0; s < bj; ++s) acc[s] += pv * qrow[s];
    }
    double* cr = c + (int64_t)r * bj;
    for (int s = 0; s < bj; ++s) cr[s] -= acc[s];
  }
  free(acc);
  free(qt);
}

/* ---------------- DAG scheduler (mpchol.cpp:254-347) ---------------- */
typedef struct {
  int32_t k, kind, i, j, id;
} heap_key;

static int key_less(const heap_key* a, const heap_key* b) {
  if (a->k != b->k) return a->k < b->k;
  if (a->kind != b->kind) return a->kind < b->kind;
  if (a->i != b->i) return a->i < b->i;
  if (a->j != b->j) return a->j < b->j;
  return a->id < b->id;
}

typedef struct {
  int n, b, nt, hp_format;
  double* tiles;
  int64_t* off;
  const uint8_t* pmap;
  int64_t count;
  uint8_t* kind;
  int32_t *ti, *tj, *tk, *indeg, *succ;
  int64_t* succ_off;
  heap_key* heap;
  int64_t heap_n;
  int64_t done;
  int abort, failed_tile;
  so_counters counters;
  pthread_mutex_t mu;
  pthread_cond_t cv;
} sched;

static void heap_push(sched* s, int32_t t) {
  heap_key key = {s->tk[t], s->kind[t], s->ti[t], s->tj[t], t};
  int64_t pos = s->heap_n++;
  while (pos > 0) {
    int64_t parent = (pos - 1) / 2;
    if (!key_less(&key, &s->heap[parent])) break;
    s->heap[pos] = s->heap[parent];
    pos = parent;
  }
  s->heap[pos] = key;
}

static heap_key heap_pop(sched* s) {
  heap_key top = s->heap[0];
  heap_key last = s->heap[--s->heap_n];
  int64_t pos = 0;
  for (;;) {
    int64_t l = 2 * pos + 1, r = l + 1, m = pos;
    const heap_key* best = &last;
    if (l < s->heap_n && key_less(&s->heap[l], best)) {
      m = l;
      best = &s->heap[l];
    }
    if (r < s->heap_n && key_less(&s->heap[r], best)) m = r;
    if (m == pos) break;
    s->heap[pos] = s->heap[m];
    pos = m;
  }
  if (s->heap_n > 0) s->heap[pos] = last;
  return top;
}

#define TILE(s, i, j) ((s)->tiles + (s)->off[(int64_t)(i) * ((i) + 1) / 2 + (j)])
#define PREC(s, i, j) ((s)->pmap[(int64_t)(i) * ((i) + 1) / 2 + (j)])

/* mpchol.cpp:283-316 */
static int run_task(sched* s, int32_t id, so_counters* local) {
  const int i = s->ti[id], j = s->tj[id], k = s->tk[id];
  const int bi = tile_rows(s->n, s->b, i), bj = tile_rows(s->n, s->b, j),
            bk = tile_rows(s->n, s->b, k);
  switch (s->kind[id]) {
    case 0:
      if (potrf_tile(TILE(s, k, k), bk)) return -1;
      so_quantize_tile(TILE(s, k, k), (int64_t)bk * bk, PREC(s, k, k), s->hp_format, local);
      break;
    case 1:
      trsm_tile(TILE(s, i, k), TILE(s, k, k), bi, bk);
      so_quantize_tile(TILE(s, i, k), (int64_t)bi * bk, PREC(s, i, k), s->hp_format, local);
      break;
    case 2:
      gemm_nt_sub(TILE(s, i, i), TILE(s, i, k), TILE(s, i, k), bi, bi, bk);
      so_quantize_tile(TILE(s, i, i), (int64_t)bi * bi, PREC(s, i, i), s->hp_format, local);
      break;
    default:
      gemm_nt_sub(TILE(s, i, j), TILE(s, i, k), TILE(s, j, k), bi, bj, bk);
      so_quantize_tile(TILE(s, i, j), (int64_t)bi * bj, PREC(s, i, j), s->hp_format, local);
      break;
  }
  return 0;
}

static void* worker(void* arg) {
  sched* s = arg;
  pthread_mutex_lock(&s->mu);
  for (;;) {
    while (!s->abort && s->heap_n == 0 && s->done != s->count) pthread_cond_wait(&s->cv, &s->mu);
    if (s->abort || s->done == s->count) break;
    heap_key key = heap_pop(s);
    pthread_mutex_unlock(&s->mu);
    so_counters local = {0, 0, 0};
    int rc = run_task(s, key.id, &local);
    pthread_mutex_lock(&s->mu);
    if (rc) {
      if (s->failed_tile < 0) s->failed_tile = s->tk[key.id];
      s->abort = 1;
      pthread_cond_broadcast(&s->cv);
      break;
    }
    s->counters.demotions_sp += local.demotions_sp;
    s->counters.demotions_hp += local.demotions_hp;
    s->counters.half_saturations += local.half_saturations;
    ++s->done;
    for (int64_t e = s->succ_off[key.id]; e < s->succ_off[key.id + 1]; ++e) {
      int32_t t = s->succ[e];
      if (--s->indeg[t] == 0) heap_push(s, t);
    }
    pthread_cond_broadcast(&s->cv);
  }
  pthread_mutex_unlock(&s->mu);
  return NULL;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* mpchol.cpp:351-410; map (optional): an explicit precision map replacing
 * assign_precisions (the tile-norm policy of the GPU path). */
static int tiled_cholesky_impl(double* tiles, int n, const so_chol_config* c, const uint8_t* map,
                               so_chol_stats* st, int* failed_tile);
int so_tiled_cholesky(double* tiles, int n, const so_chol_config* c, so_chol_stats* st,
                      int* failed_tile) {
  return tiled_cholesky_impl(tiles, n, c, NULL, st, failed_tile);
}
static int tiled_cholesky_impl(double* tiles, int n, const so_chol_config* c, const uint8_t* map,
                               so_chol_stats* st, int* failed_tile) {
  if (so_config_validate(c) || n < 1) return -1;
  const double t0 = now_s();
  sched s;
  memset(&s, 0, sizeof s);
  s.n = n;
  s.b = c->tile_size;
  s.nt = (n + s.b - 1) / s.b;
  s.hp_format = c->hp_format;
  s.tiles = tiles;
  s.off = tile_offsets(n, s.b);
  const int nt = s.nt;
  uint8_t* pmap = malloc((size_t)nt * (nt + 1) / 2);
  if (map) memcpy(pmap, map, (size_t)nt * (nt + 1) / 2);
  else so_assign_precisions(nt, c, pmap);
  s.pmap = pmap;
  s.count = so_task_count(nt);
  s.kind = malloc((size_t)s.count);
  s.ti = malloc(sizeof(int32_t) * (size_t)s.count);
  s.tj = malloc(sizeof(int32_t) * (size_t)s.count);
  s.tk = malloc(sizeof(int32_t) * (size_t)s.count);
  s.indeg = malloc(sizeof(int32_t) * (size_t)s.count);
  s.succ_off = malloc(sizeof(int64_t) * (size_t)(s.count + 1));
  int64_t cap = 4 * s.count + 16;
  s.succ = malloc(sizeof(int32_t) * (size_t)cap);
  int64_t edges = so_task_graph(nt, s.kind, s.ti, s.tj, s.tk, s.succ_off, s.succ, s.indeg, cap);
  if (edges < 0) {
    free(s.succ);
    cap = -edges;
    s.succ = malloc(sizeof(int32_t) * (size_t)cap);
    so_task_graph(nt, s.kind, s.ti, s.tj, s.tk, s.succ_off, s.succ, s.indeg, cap);
  }
  s.heap = malloc(sizeof(heap_key) * (size_t)s.count);
  s.failed_tile = -1;
  pthread_mutex_init(&s.mu, NULL);
  pthread_cond_init(&s.cv, NULL);
  for (int64_t t = 0; t < s.count; ++t)
    if (s.indeg[t] == 0) heap_push(&s, (int32_t)t);

  /* mpchol.cpp:360-363: inputs stored at their precision before arithmetic. */
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j <= i; ++j)
      so_quantize_tile(TILE(&s, i, j), (int64_t)tile_rows(n, s.b, i) * tile_rows(n, s.b, j),
                       PREC(&s, i, j), s.hp_format, &s.counters);

  if (c->workers == 1) {
    worker(&s);
  } else {
    pthread_t* th = malloc(sizeof(pthread_t) * (size_t)c->workers);
    for (int w = 0; w < c->workers; ++w) pthread_create(&th[w], NULL, worker, &s);
    for (int w = 0; w < c->workers; ++w) pthread_join(th[w], NULL);
    free(th);
  }
  int rc = 0;
  if (s.failed_tile >= 0) {
    rc = 1;
    if (failed_tile) *failed_tile = s.failed_tile;
  }
  if (st) {
    memset(st, 0, sizeof *st);
    st->n = n;
    st->tile_size = s.b;
    st->n_tiles = nt;
    st->workers = c->workers;
    st->variant = c->variant;
    int64_t N = nt;
    st->tasks_potrf = N;
    st->tasks_trsm = N * (N - 1) / 2;
    st->tasks_syrk = N * (N - 1) / 2;
    st->tasks_gemm = N * (N - 1) * (N - 2) / 6;
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j <= i; ++j) {
        int64_t e = (int64_t)tile_rows(n, s.b, i) * tile_rows(n, s.b, j);
        switch (PREC(&s, i, j)) {
          case SO_DP: st->tiles_dp++; st->bytes_dp += 8 * e; break;
          case SO_SP: st->tiles_sp++; st->bytes_sp += 4 * e; break;
          default: st->tiles_hp++; st->bytes_hp += 2 * e; break;
        }
      }
    st->conv = s.counters;
    st->wall_seconds = now_s() - t0;
  }
  pthread_mutex_destroy(&s.mu);
  pthread_cond_destroy(&s.cv);
  free(s.heap);
  free(s.succ);
  free(s.succ_off);
  free(s.indeg);
  free(s.tk);
  free(s.tj);
  free(s.ti);
  free(s.kind);
  free(pmap);
  free(s.off);
  return rc;
}

int so_tiled_cholesky_dense(const double* a, int n, const so_chol_config* c, double* factor,
                            so_chol_stats* st, int* failed_tile) {
  if (so_config_validate(c) || n < 1) return -1;
  double* tiles = malloc(sizeof(double) * (size_t)so_tiled_size(n, c->tile_size));
  so_tiled_from_dense(a, n, c->tile_size, tiles);
  int rc = so_tiled_cholesky(tiles, n, c, st, failed_tile);
  if (rc == 0) so_tiled_to_dense_lower(tiles, n, c->tile_size, factor);
  free(tiles);
  return rc;
}

int so_tiled_cholesky_dense_map(const double* a, int n, const so_chol_config* c, const uint8_t* map,
                                double* factor, so_chol_stats* st, int* failed_tile) {
  if (so_config_validate(c) || n < 1) return -1;
  double* tiles = malloc(sizeof(double) * (size_t)so_tiled_size(n, c->tile_size));
  so_tiled_from_dense(a, n, c->tile_size, tiles);
  int rc = tiled_cholesky_impl(tiles, n, c, map, st, failed_tile);
  if (rc == 0) so_tiled_to_dense_lower(tiles, n, c->tile_size, factor);
  free(tiles);
  return rc;
}

/* mpchol.cpp:419-435 */
void so_make_spd_factors(int n, uint64_t seed, double* d, double* pw) {
  so_rng r;
  so_rng_seed(&r, seed);
  for (int i = 0; i < n; ++i) d[i] = exp(0.6 * so_rng_uniform(&r) - 0.3);
  if (pw)
    for (int k = 0; k < n; ++k) pw[k] = pow(0.9, (double)k);
}

void so_make_spd(int n, uint64_t seed, double* a) {
  double* d = malloc(sizeof(double) * (size_t)n);
  double* pw = malloc(sizeof(double) * (size_t)n);
  so_make_spd_factors(n, seed, d, pw);
  for (int i = 0; i < n; ++i) {
    a[(int64_t)i * n + i] = d[i] * d[i] * 1.25;
    for (int j = 0; j < i; ++j) {
      double v = d[i] * d[j] * 0.25 * pw[i - j];
      a[(int64_t)i * n + j] = v;
      a[(int64_t)j * n + i] = v;
    }
  }
  free(pw);
  free(d);
}

/* tests/support/reference.cpp:10-30 */
int so_dense_cholesky(const double* a, int n, double* l) {
  memset(l, 0, sizeof(double) * (size_t)n * n);
  for (int j = 0; j < n; ++j) {
    double diag = a[(int64_t)j * n + j];
    for (int k = 0; k < j; ++k) {
      double v = l[(int64_t)j * n + k];
      diag -= v * v;
    }
    if (!(diag > 0.0)) return 1;
    diag = sqrt(diag);
    l[(int64_t)j * n + j] = diag;
    for (int i = j + 1; i < n; ++i) {
      double s = a[(int64_t)i * n + j];
      for (int k = 0; k < j; ++k) s -= l[(int64_t)i * n + k] * l[(int64_t)j * n + k];
      l[(int64_t)i * n + j] = s / diag;
    }
  }
  return 0;
}

/* tests/support/reference.cpp:32-44, rows split over threads (sum order per
 * row is fixed; the row partials are added in row order). */
typedef struct {
  const double *a, *l;
  int n, r0, r1;
  double *num, *den;
} resid_job;

static void* resid_rows(void* arg) {
  resid_job* jb = arg;
  const int n = jb->n;
  for (int i = jb->r0; i < jb->r1; ++i) {
    double num = 0.0, den = 0.0;
    for (int j = 0; j < n; ++j) {
      double prod = 0.0;
      int kmax = i < j ? i : j;
      for (int k = 0; k <= kmax; ++k) prod += jb->l[(int64_t)i * n + k] * jb->l[(int64_t)j * n + k];
      double aij = jb->a[(int64_t)i * n + j];
      num += (aij - prod) * (aij - prod);
      den += aij * aij;
    }
    jb->num[i] = num;
    jb->den[i] = den;
  }
  return NULL;
}

double so_relative_residual(const double* a, const double* l, int n, int threads) {
  if (threads < 1) threads = 1;
  double* num = malloc(sizeof(double) * (size_t)n);
  double* den = malloc(sizeof(double) * (size_t)n);
  pthread_t* th = malloc(sizeof(pthread_t) * (size_t)threads);
  resid_job* jobs = malloc(sizeof(resid_job) * (size_t)threads);
  for (int w = 0; w < threads; ++w) {
    jobs[w] = (resid_job){a, l, n, (int)((int64_t)n * w / threads),
                          (int)((int64_t)n * (w + 1) / threads), num, den};
    pthread_create(&th[w], NULL, resid_rows, &jobs[w]);
  }
  for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
  double sn = 0.0, sd = 0.0;
  for (int i = 0; i < n; ++i) {
    sn += num[i];
    sd += den[i];
  }
  free(jobs);
  free(th);
  free(num);
  free(den);
  return sqrt(sn) / sqrt(sd);
}
