/*
 * so_dft.h — exact mixed-radix complex DFT shared by the oracle (so_sht.c) and
 * the FFTW shim of oracle/_ref (ref/fft_shim.cpp), so both compute identical
 * ring and extended-line transforms (TEST INFRASTRUCTURE). Stands in for the
 * FFTW plans of proj/src/fft.cpp:26-50.
 */
#ifndef SO_DFT_H
#define SO_DFT_H
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double re, im;
} cplx;

static inline cplx cmul(cplx a, cplx b) {
  cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}
static inline cplx cadd(cplx a, cplx b) {
  cplx r = {a.re + b.re, a.im + b.im};
  return r;
}
static inline cplx cscale(double s, cplx a) {
  cplx r = {s * a.re, s * a.im};
  return r;
}
static inline cplx cdivd(cplx a, double d) {
  cplx r = {a.re / d, a.im / d};
  return r;
}

#define SO_TWO_PI (2.0 * 3.14159265358979323846264338327950288)
static inline int smallest_factor(int n) {
  if (n % 2 == 0) return 2;
  for (int p = 3; p * p <= n; p += 2)
    if (n % p == 0) return p;
  return n;
}

/* out[k] = sum_j in[j*stride] * w^(j k), w = exp(sign 2 pi i / n), via
 * recursive decimation in time; tw[t] = exp(sign 2 pi i t / N). */
static inline void dft_rec(int n, int N, const cplx* tw, const cplx* in, int stride, cplx* out,
                    cplx* scratch) {
  if (n == 1) {
    out[0] = in[0];
    return;
  }
  const int p = smallest_factor(n);
  const int m = n / p;
  for (int r = 0; r < p; ++r) dft_rec(m, N, tw, in + (size_t)r * stride, stride * p, out + (size_t)r * m, scratch);
  const int tstep = N / n;
  cplx t[64];
  cplx* tt = p <= 64 ? t : (cplx*)malloc(sizeof(cplx) * (size_t)p);
  for (int k = 0; k < m; ++k) {
    for (int r = 0; r < p; ++r) tt[r] = cmul(out[(size_t)r * m + k], tw[((size_t)r * k * tstep) % N]);
    for (int q = 0; q < p; ++q) {
      cplx acc = tt[0];
      for (int r = 1; r < p; ++r) acc = cadd(acc, cmul(tt[r], tw[((size_t)r * q * m * tstep) % N]));
      scratch[k + (size_t)q * m] = acc;
    }
  }
  if (tt != t) free(tt);
  memcpy(out, scratch, sizeof(cplx) * (size_t)n);
}

typedef struct {
  int n, sign;
  cplx* tw;
} dft_plan;

static inline void plan_dft(dft_plan* d, int n, int sign) {
  d->n = n;
  d->sign = sign;
  d->tw = (cplx*)malloc(sizeof(cplx) * (size_t)n);
  for (int t = 0; t < n; ++t) {
    double a = SO_TWO_PI * (double)t / (double)n;
    d->tw[t].re = cos(a);
    d->tw[t].im = sign < 0 ? -sin(a) : sin(a);
  }
}

static inline void exec_dft(const dft_plan* d, const cplx* in, cplx* out, cplx* scratch) {
  dft_rec(d->n, d->n, d->tw, in, 1, out, scratch);
}

#endif
