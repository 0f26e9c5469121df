/*
 * so_sht.c — oracle restatement of proj/src/wigner.cpp, proj/src/sht.cpp and
 * the FFTW wrapper proj/src/fft.cpp (TEST INFRASTRUCTURE, see sphemu_oracle.h).
 * Expression order follows the reference so results agree to the last bit
 * with oracle/_ref (which links the same exact-DFT shim); complex products use
 * the (ac-bd, ad+bc) form that std::complex<double> multiplication produces
 * for finite operands.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "sphemu_oracle.h"

static const double kPi = 3.14159265358979323846264338327950288;
static const double kTwoPi = 2.0 * 3.14159265358979323846264338327950288;

#include "so_dft.h"

void so_dft(int n, int sign, const double* in_ri, double* out_ri) {
  cplx* tw = malloc(sizeof(cplx) * (size_t)n);
  for (int t = 0; t < n; ++t) {
    double a = kTwoPi * (double)t / (double)n;
    tw[t].re = cos(a);
    tw[t].im = sign < 0 ? -sin(a) : sin(a);
  }
  cplx* scratch = malloc(sizeof(cplx) * (size_t)n);
  cplx* out = malloc(sizeof(cplx) * (size_t)n);
  dft_rec(n, n, tw, (const cplx*)in_ri, 1, out, scratch);
  memcpy(out_ri, out, sizeof(cplx) * (size_t)n);
  free(out);
  free(scratch);
  free(tw);
}

/* ---------------- sht.cpp:30-37 ---------------- */
void so_i_integral(long long q, double* re, double* im) {
  if (q & 1) {
    *re = 0.0;
    *im = q == 1 ? kPi / 2.0 : (q == -1 ? -kPi / 2.0 : 0.0);
    return;
  }
  *re = 2.0 / (1.0 - (double)q * (double)q);
  *im = 0.0;
}

/* ---------------- wigner.cpp ---------------- */
struct so_wigner {
  int L, renorm;
  double* d;
  size_t* d_off;
  double* q;
};

static int parity(int e) { return (e & 1) ? -1 : 1; }

/* wigner.cpp:20-28 */
static double chain_seed(int m2, int m) {
  int l0 = m2 > m ? m2 : m;
  int lo = m2 < m ? m2 : m;
  long double prod = 1.0L;
  for (int k = 1; k <= l0 - lo; ++k) prod *= (long double)(l0 + lo + k) / k;
  long double v = ldexpl(1.0L, -l0) * sqrtl(prod);
  return (double)(parity(l0 - m) * v);
}

/* wigner.cpp:31-47 */
double so_wigner_brute(int l, int m2, int m) {
  if (l < 0 || abs(m2) > l || abs(m) > l) return 0.0;
#define LG(k) lgammal((long double)(k))
  long double pref = 0.5L * (LG(l + m2 + 1) + LG(l - m2 + 1) + LG(l + m + 1) + LG(l - m + 1)) -
                     l * logl(2.0L);
  int s_lo = 0 > m - m2 ? 0 : m - m2;
  int s_hi = (l + m) < (l - m2) ? (l + m) : (l - m2);
  long double sum = 0.0L;
  for (int s = s_lo; s <= s_hi; ++s) {
    long double ln_den = LG(l + m - s + 1) + LG(s + 1) + LG(m2 - m + s + 1) + LG(l - m2 - s + 1);
    sum += parity(m2 - m + s) * expl(pref - ln_den);
  }
#undef LG
  return (double)sum;
}

size_t so_wigner_bytes(int L) {
  size_t d_entries = 0;
  for (int a = 0; a < L; ++a)
    for (int b = 0; b < L; ++b) d_entries += (size_t)(L - (a > b ? a : b));
  size_t q_entries = (size_t)L * L * (L + 1) / 2;
  return (d_entries + q_entries) * sizeof(double) + ((size_t)L * L + 1) * sizeof(size_t);
}

/* wigner.cpp:136-150 */
double so_wigner_d(const so_wigner* w, int l, int m2, int m) {
  if (l < 0 || l >= w->L) return NAN;
  if (abs(m2) > l || abs(m) > l) return 0.0;
  int sign = 1;
  if (m2 < 0) {
    sign *= parity(l + m);
    m2 = -m2;
  }
  if (m < 0) {
    sign *= parity(l + m2);
    m = -m;
  }
  size_t o = w->d_off[(size_t)m2 * w->L + m];
  return sign * w->d[o + l - (m2 > m ? m2 : m)];
}

/* wigner.cpp:49-134 + build_q 152-163 */
so_wigner* so_wigner_build(int L, size_t cap) {
  if (L < 1 || so_wigner_bytes(L) > cap) return NULL;
  so_wigner* t = calloc(1, sizeof *t);
  t->L = L;
  t->d_off = malloc(sizeof(size_t) * ((size_t)L * L + 1));
  size_t off = 0;
  for (int a = 0; a < L; ++a)
    for (int b = 0; b < L; ++b) {
      t->d_off[(size_t)a * L + b] = off;
      off += (size_t)(L - (a > b ? a : b));
    }
  t->d_off[(size_t)L * L] = off;
  t->d = calloc(off, sizeof(double));
  for (int a = 0; a < L; ++a)
    for (int b = 0; b < L; ++b) {
      int l0 = a > b ? a : b;
      double* chain = t->d + t->d_off[(size_t)a * L + b];
      chain[0] = chain_seed(a, b);
      if (l0 + 1 >= L) continue;
      double prev = 0.0, cur = chain[0];
      for (int l = l0; l + 1 < L; ++l) {
        double next;
        if (l == 0) {
          next = 0.0;
        } else {
          double c1 = sqrt((double)(l + 1 + a)) * sqrt((double)(l + 1 - a)) *
                      sqrt((double)(l + 1 + b)) * sqrt((double)(l + 1 - b));
          double c0 = sqrt((double)(l + a)) * sqrt((double)(l - a)) * sqrt((double)(l + b)) *
                      sqrt((double)(l - b));
          next = (-(2.0 * l + 1.0) * a * b * cur - (l + 1.0) * c0 * prev) / (l * c1);
        }
        chain[l + 1 - l0] = next;
        prev = cur;
        cur = next;
      }
    }
  for (int l = 0; l < L; ++l)
    for (int b = 0; b <= l; ++b) {
      int bad = 0;
      double s = 0.0;
      for (int a = 0; a <= l; ++a) {
        double v = so_wigner_d(t, l, a, b);
        if (fabs(v) > 1.0 + 1e-9) bad = 1;
        s += (a == 0 ? 1.0 : 2.0) * v * v;
      }
      if (!bad) continue;
      ++t->renorm;
      double scale = 1.0 / sqrt(s);
      for (int a = 0; a <= l; ++a) {
        size_t o = t->d_off[(size_t)a * L + b];
        t->d[o + l - (a > b ? a : b)] *= scale;
      }
    }
  t->q = calloc((size_t)L * L * (L + 1) / 2, sizeof(double));
  for (int l = 0; l < L; ++l) {
    double norm = sqrt((2.0 * l + 1.0) / (4.0 * kPi));
    for (int m = 0; m <= l; ++m) {
      size_t row = ((size_t)l * (l + 1) / 2 + m) * L;
      for (int m2 = 0; m2 <= l; ++m2)
        t->q[row + m2] = norm * so_wigner_d(t, l, m2, 0) * so_wigner_d(t, l, m2, m);
    }
  }
  return t;
}

void so_wigner_free(so_wigner* w) {
  if (!w) return;
  free(w->d);
  free(w->d_off);
  free(w->q);
  free(w);
}

double so_wigner_q(const so_wigner* w, int l, int m, int m2) {
  if (l < 0 || l >= w->L || m < 0 || m > l || m2 < 0 || m2 >= w->L) return NAN;
  if (m2 > l) return 0.0;
  return w->q[((size_t)l * (l + 1) / 2 + m) * w->L + m2];
}

int so_wigner_renorm_warnings(const so_wigner* w) { return w->renorm; }
const double* so_wigner_q_table(const so_wigner* w) { return w->q; }

/* ---------------- plan (sht.cpp:111-171) ---------------- */
struct so_plan {
  int n_theta, n_phi, L, n_ext, cols;
  const so_wigner* wt;
  so_wigner* owned;
  cplx* i_mat;
  double* parity;
  dft_plan ring_a, ring_s, ext_a, ext_s;
};

int so_grid_max_band_limit(int n_theta, int n_phi) {
  int a = n_theta - 1, b = (n_phi + 1) / 2;
  return a < b ? a : b;
}

so_plan* so_plan_build(int n_theta, int n_phi, int L, const so_wigner* tables) {
  if (n_theta < 2 || n_phi < 1) return NULL;
  if (L < 1 || L > so_grid_max_band_limit(n_theta, n_phi)) return NULL;
  if (tables && tables->L < L) return NULL;
  so_plan* p = calloc(1, sizeof *p);
  p->n_theta = n_theta;
  p->n_phi = n_phi;
  p->L = L;
  p->n_ext = 2 * n_theta - 2;
  p->cols = 2 * L - 1;
  if (tables) {
    p->wt = tables;
  } else {
    p->owned = so_wigner_build(L, (size_t)1 << 62);
    p->wt = p->owned;
  }
  const int cols = p->cols;
  p->i_mat = malloc(sizeof(cplx) * (size_t)cols * cols);
  for (int c1 = 0; c1 < cols; ++c1)
    for (int c2 = 0; c2 < cols; ++c2)
      so_i_integral((long long)(c1 - (L - 1)) + (long long)(c2 - (L - 1)),
                    &p->i_mat[(size_t)c1 * cols + c2].re, &p->i_mat[(size_t)c1 * cols + c2].im);
  p->parity = malloc(sizeof(double) * (size_t)L);
  for (int m = 0; m < L; ++m) p->parity[m] = (m & 1) ? -1.0 : 1.0;
  plan_dft(&p->ring_a, n_phi, -1);
  plan_dft(&p->ring_s, n_phi, +1);
  plan_dft(&p->ext_a, p->n_ext, -1);
  plan_dft(&p->ext_s, p->n_ext, +1);
  return p;
}

void so_plan_free(so_plan* p) {
  if (!p) return;
  free(p->i_mat);
  free(p->parity);
  free(p->ring_a.tw);
  free(p->ring_s.tw);
  free(p->ext_a.tw);
  free(p->ext_s.tw);
  so_wigner_free(p->owned);
  free(p);
}

int so_plan_points(const so_plan* p) { return p->n_theta * p->n_phi; }

typedef struct {
  cplx *ring_in, *ring_out, *g, *ext, *spec1, *j, *k, *scratch;
} workspace;

static void ws_alloc(const so_plan* p, workspace* ws) {
  int big = p->n_phi > p->n_ext ? p->n_phi : p->n_ext;
  ws->ring_in = malloc(sizeof(cplx) * (size_t)p->n_phi);
  ws->ring_out = malloc(sizeof(cplx) * (size_t)p->n_phi);
  ws->g = malloc(sizeof(cplx) * (size_t)p->L * p->n_theta);
  ws->ext = malloc(sizeof(cplx) * (size_t)p->n_ext);
  ws->spec1 = malloc(sizeof(cplx) * (size_t)p->n_ext);
  ws->j = malloc(sizeof(cplx) * (size_t)p->cols);
  ws->k = malloc(sizeof(cplx) * (size_t)p->L);
  ws->scratch = malloc(sizeof(cplx) * (size_t)big);
}

static void ws_free(workspace* ws) {
  free(ws->ring_in);
  free(ws->ring_out);
  free(ws->g);
  free(ws->ext);
  free(ws->spec1);
  free(ws->j);
  free(ws->k);
  free(ws->scratch);
}

static cplx inv_i_pow(int m) {
  cplx r;
  switch (m & 3) {
    case 0: r.re = 1.0; r.im = 0.0; break;
    case 1: r.re = 0.0; r.im = -1.0; break;
    case 2: r.re = -1.0; r.im = 0.0; break;
    default: r.re = 0.0; r.im = 1.0; break;
  }
  return r;
}

/* sht.cpp:189-208 */
static void contract_row(const so_plan* p, int m, const cplx* j_row, double* out) {
  const int L = p->L, mid = L - 1;
  const double par = p->parity[m];
  const cplx phase = cscale(kTwoPi, inv_i_pow(m));
  for (int l = m; l < L; ++l) {
    cplx acc = cscale(so_wigner_q(p->wt, l, m, 0), j_row[mid]);
    for (int m2 = 1; m2 <= l; ++m2)
      acc = cadd(acc, cscale(so_wigner_q(p->wt, l, m, m2),
                             cadd(j_row[mid + m2], cscale(par, j_row[mid - m2]))));
    cplx f = cmul(phase, acc);
    if (m == 0) {
      out[(size_t)l * l] = f.re;
    } else {
      out[(size_t)l * l + 2 * m - 1] = f.re;
      out[(size_t)l * l + 2 * m] = f.im;
    }
  }
}

/* sht.cpp:211-222 */
static void ring_stage(const so_plan* p, const double* field, workspace* ws) {
  for (int i = 0; i < p->n_theta; ++i) {
    const double* row = field + (size_t)i * p->n_phi;
    for (int jj = 0; jj < p->n_phi; ++jj) {
      ws->ring_in[jj].re = row[jj];
      ws->ring_in[jj].im = 0.0;
    }
    exec_dft(&p->ring_a, ws->ring_in, ws->ring_out, ws->scratch);
    for (int m = 0; m < p->L; ++m)
      ws->g[(size_t)m * p->n_theta + i] = cdivd(ws->ring_out[m], (double)p->n_phi);
  }
}

/* sht.cpp:226-263 */
static void forward_ws(const so_plan* p, const double* field, double* coeffs, workspace* ws) {
  const int n_theta = p->n_theta, L = p->L, cols = p->cols, mid = L - 1, n_ext = p->n_ext;
  ring_stage(p, field, ws);
  for (int m = 0; m < L; ++m) {
    const cplx* g = ws->g + (size_t)m * n_theta;
    double par = p->parity[m];
    for (int i = 0; i < n_theta; ++i) ws->ext[i] = g[i];
    for (int k = 1; k <= n_theta - 2; ++k) ws->ext[n_theta - 1 + k] = cscale(par, g[n_theta - 1 - k]);
    exec_dft(&p->ext_a, ws->ext, ws->spec1, ws->scratch);
    for (int c2 = 0; c2 < cols; ++c2) {
      cplx acc = {0.0, 0.0};
      for (int c1 = 0; c1 < cols; ++c1) {
        int mp = c1 - mid;
        cplx kv = cdivd(ws->spec1[(mp % n_ext + n_ext) % n_ext], (double)n_ext);
        acc = cadd(acc, cmul(kv, p->i_mat[(size_t)c1 * cols + c2]));
      }
      ws->j[c2] = acc;
    }
    contract_row(p, m, ws->j, coeffs);
  }
}

/* sht.cpp:304-357 */
static void inverse_ws(const so_plan* p, const double* coeffs, double* field, workspace* ws) {
  const int n_theta = p->n_theta, n_phi = p->n_phi, L = p->L, n_ext = p->n_ext;
  for (int m = 0; m < L; ++m) {
    for (int mp = 0; mp < L; ++mp) {
      cplx acc = {0.0, 0.0};
      for (int l = (m > mp ? m : mp); l < L; ++l) {
        cplx z;
        if (m == 0) {
          z.re = coeffs[(size_t)l * l];
          z.im = 0.0;
        } else {
          z.re = coeffs[(size_t)l * l + 2 * m - 1];
          z.im = coeffs[(size_t)l * l + 2 * m];
        }
        acc = cadd(acc, cscale(so_wigner_q(p->wt, l, m, mp), z));
      }
      ws->k[mp] = acc;
    }
    memset(ws->spec1, 0, sizeof(cplx) * (size_t)n_ext);
    const cplx phase = inv_i_pow(m);
    const double par = p->parity[m];
    ws->spec1[0] = cmul(phase, ws->k[0]);
    for (int mp = 1; mp < L; ++mp) {
      ws->spec1[mp] = cmul(phase, ws->k[mp]);
      ws->spec1[n_ext - mp] = cmul(phase, cscale(par, ws->k[mp]));
    }
    exec_dft(&p->ext_s, ws->spec1, ws->ext, ws->scratch);
    for (int i = 0; i < n_theta; ++i) ws->g[(size_t)m * n_theta + i] = ws->ext[i];
  }
  for (int i = 0; i < n_theta; ++i) {
    memset(ws->ring_in, 0, sizeof(cplx) * (size_t)n_phi);
    ws->ring_in[0] = ws->g[i];
    for (int m = 1; m < L; ++m) {
      cplx v = ws->g[(size_t)m * n_theta + i];
      cplx vc = {v.re, -v.im};
      ws->ring_in[m] = cadd(ws->ring_in[m], v);
      ws->ring_in[n_phi - m] = cadd(ws->ring_in[n_phi - m], vc);
    }
    exec_dft(&p->ring_s, ws->ring_in, ws->ring_out, ws->scratch);
    double* row = field + (size_t)i * n_phi;
    for (int jj = 0; jj < n_phi; ++jj) row[jj] = ws->ring_out[jj].re;
  }
}

void so_forward_sht(const so_plan* p, const double* field, double* coeffs) {
  workspace ws;
  ws_alloc(p, &ws);
  forward_ws(p, field, coeffs, &ws);
  ws_free(&ws);
}

void so_inverse_sht(const so_plan* p, const double* coeffs, double* field) {
  workspace ws;
  ws_alloc(p, &ws);
  inverse_ws(p, coeffs, field, &ws);
  ws_free(&ws);
}

/* sht.cpp:374-404 with the static partition of thread_pool.hpp:17-43. */
typedef struct {
  const so_plan* p;
  const double* in;
  double* out;
  int64_t lo, hi;
  int forward;
} batch_job;

static void* batch_run(void* arg) {
  batch_job* jb = arg;
  const so_plan* p = jb->p;
  const size_t pts = (size_t)p->n_theta * p->n_phi, nc = (size_t)p->L * p->L;
  workspace ws;
  ws_alloc(p, &ws);
  for (int64_t s = jb->lo; s < jb->hi; ++s) {
    if (jb->forward)
      forward_ws(p, jb->in + (size_t)s * pts, jb->out + (size_t)s * nc, &ws);
    else
      inverse_ws(p, jb->in + (size_t)s * nc, jb->out + (size_t)s * pts, &ws);
  }
  ws_free(&ws);
  return NULL;
}

static void run_batch(const so_plan* p, const double* in, int64_t n, double* out, int threads,
                      int forward) {
  if (threads < 1) threads = 1;
  if (n <= 0) return;
  int workers = (int64_t)threads < n ? threads : (int)n;
  pthread_t* th = malloc(sizeof(pthread_t) * (size_t)workers);
  batch_job* jobs = malloc(sizeof(batch_job) * (size_t)workers);
  for (int w = 0; w < workers; ++w) {
    jobs[w] = (batch_job){p, in, out, n * w / workers, n * (w + 1) / workers, forward};
    if (workers == 1)
      batch_run(&jobs[w]);
    else
      pthread_create(&th[w], NULL, batch_run, &jobs[w]);
  }
  if (workers > 1)
    for (int w = 0; w < workers; ++w) pthread_join(th[w], NULL);
  free(jobs);
  free(th);
}

void so_forward_sht_batch(const so_plan* p, const double* fields, int64_t n, double* coeffs,
                          int threads) {
  run_batch(p, fields, n, coeffs, threads, 1);
}

void so_inverse_sht_batch(const so_plan* p, const double* coeffs, int64_t n, double* fields,
                          int threads) {
  run_batch(p, coeffs, n, fields, threads, 0);
}

/* sht.cpp:406-427 */
void so_normalized_legendre_all(int L, double theta, double* p) {
  memset(p, 0, sizeof(double) * (size_t)L * (L + 1) / 2);
  const double ct = cos(theta), st = sin(theta);
#define AT(l, m) p[(size_t)(l) * ((l) + 1) / 2 + (m)]
  AT(0, 0) = 1.0 / sqrt(4.0 * kPi);
  for (int m = 1; m < L; ++m) AT(m, m) = -sqrt((2.0 * m + 1.0) / (2.0 * m)) * st * AT(m - 1, m - 1);
  for (int m = 0; m + 1 < L; ++m) AT(m + 1, m) = sqrt(2.0 * m + 3.0) * ct * AT(m, m);
  for (int m = 0; m < L; ++m)
    for (int l = m + 2; l < L; ++l) {
      double a = sqrt((4.0 * l * l - 1.0) / ((double)l * l - m * m));
      double b = sqrt(((double)(l - 1) * (l - 1) - m * m) / (4.0 * (double)(l - 1) * (l - 1) - 1.0));
      AT(l, m) = a * (ct * AT(l - 1, m) - b * AT(l - 2, m));
    }
#undef AT
}

/* sht.cpp:435-466 */
void so_synth_bandlimited(const double* coeffs, int L, int n_theta, int n_phi, double* field) {
  double* p = malloc(sizeof(double) * (size_t)L * (L + 1) / 2);
  cplx* s_m = malloc(sizeof(cplx) * (size_t)L);
  for (int i = 0; i < n_theta; ++i) {
    so_normalized_legendre_all(L, kPi * i / (n_theta - 1), p);
    for (int m = 0; m < L; ++m) {
      cplx acc = {0.0, 0.0};
      for (int l = m; l < L; ++l) {
        cplx z;
        if (m == 0) {
          z.re = coeffs[(size_t)l * l];
          z.im = 0.0;
        } else {
          z.re = coeffs[(size_t)l * l + 2 * m - 1];
          z.im = coeffs[(size_t)l * l + 2 * m];
        }
        acc = cadd(acc, cscale(p[(size_t)l * (l + 1) / 2 + m], z));
      }
      s_m[m] = acc;
    }
    for (int j = 0; j < n_phi; ++j) {
      double ph = 2.0 * kPi * j / n_phi;
      cplx step = {cos(ph), sin(ph)};
      cplx e = {1.0, 0.0};
      double v = s_m[0].re;
      for (int m = 1; m < L; ++m) {
        e = cmul(e, step);
        v += 2.0 * cmul(s_m[m], e).re;
      }
      field[(size_t)i * n_phi + j] = v;
    }
  }
  free(s_m);
  free(p);
}

/* sht.cpp:507-518 */
void so_draw_random_coefficients(int L, uint64_t seed, double* out) {
  so_rng r;
  so_rng_seed(&r, seed);
  memset(out, 0, sizeof(double) * (size_t)L * L);
  for (int l = 0; l < L; ++l) {
    double scale = 1.0 / (l + 1);
    size_t lo = (size_t)l * l;
    for (size_t idx = lo; idx <= lo + 2 * (size_t)l; ++idx) out[idx] = scale * so_rng_normal(&r);
  }
}

/* sht.cpp:58-69 */
double so_parseval_energy(const double* v, int L) {
  double e = 0.0;
  for (int l = 0; l < L; ++l) {
    double x = v[(size_t)l * l];
    e += x * x;
    for (int m = 1; m <= l; ++m) {
      double re = v[(size_t)l * l + 2 * m - 1], im = v[(size_t)l * l + 2 * m];
      e += 2.0 * (re * re + im * im);
    }
  }
  return e;
}

/* sht.cpp:529-574 */
double so_field_energy_quadrature(const double* field, int n_theta, int n_phi) {
  const int L = so_grid_max_band_limit(n_theta, n_phi);
  const int n_ext = 2 * n_theta - 2, cols = 2 * L - 1, mid = L - 1;
  dft_plan rf, ef;
  plan_dft(&rf, n_phi, -1);
  plan_dft(&ef, n_ext, -1);
  int big = n_phi > n_ext ? n_phi : n_ext;
  cplx* in = malloc(sizeof(cplx) * (size_t)n_phi);
  cplx* out = malloc(sizeof(cplx) * (size_t)n_phi);
  cplx* scratch = malloc(sizeof(cplx) * (size_t)big);
  cplx* g = malloc(sizeof(cplx) * (size_t)cols * n_theta);
  for (int i = 0; i < n_theta; ++i) {
    for (int j = 0; j < n_phi; ++j) {
      in[j].re = field[(size_t)i * n_phi + j];
      in[j].im = 0.0;
    }
    exec_dft(&rf, in, out, scratch);
    for (int c = 0; c < cols; ++c) {
      int m = c - mid;
      g[(size_t)c * n_theta + i] = cdivd(out[(m % n_phi + n_phi) % n_phi], (double)n_phi);
    }
  }
  cplx* ext = malloc(sizeof(cplx) * (size_t)n_ext);
  cplx* spec1 = malloc(sizeof(cplx) * (size_t)n_ext);
  cplx* kappa = malloc(sizeof(cplx) * (size_t)cols);
  double energy = 0.0;
  for (int c = 0; c < cols; ++c) {
    int m = c - mid;
    double par = (m & 1) ? -1.0 : 1.0;
    const cplx* gm = g + (size_t)c * n_theta;
    for (int i = 0; i < n_theta; ++i) ext[i] = gm[i];
    for (int k = 1; k <= n_theta - 2; ++k) ext[n_theta - 1 + k] = cscale(par, gm[n_theta - 1 - k]);
    exec_dft(&ef, ext, spec1, scratch);
    for (int cc = 0; cc < cols; ++cc) {
      int mp = cc - mid;
      kappa[cc] = cdivd(spec1[(mp % n_ext + n_ext) % n_ext], (double)n_ext);
    }
    cplx contrib = {0.0, 0.0};
    for (int a = 0; a < cols; ++a)
      for (int b = 0; b < cols; ++b) {
        cplx kb = {kappa[b].re, -kappa[b].im};
        cplx ii;
        so_i_integral(a - b, &ii.re, &ii.im);
        contrib = cadd(contrib, cmul(cmul(kappa[a], kb), ii));
      }
    energy += contrib.re;
  }
  free(kappa);
  free(spec1);
  free(ext);
  free(g);
  free(scratch);
  free(out);
  free(in);
  free(rf.tw);
  free(ef.tw);
  return kTwoPi * energy;
}
