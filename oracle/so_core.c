/*
 * so_core.c — oracle restatement of rng.hpp and half.hpp (TEST INFRASTRUCTURE,
 * see sphemu_oracle.h). Bit-exact semantics are the point of this file.
 */
#include <math.h>
#include <string.h>

#include "sphemu_oracle.h"

/* ---- std::mt19937_64 (the C++ standard fixes the sequence; rng.hpp:26) ---- */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void so_rng_seed(so_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = MT_N;
  r->spare = 0.0;
  r->has_spare = 0;
}

uint64_t so_rng_raw(so_rng* r) {
  if (r->mti >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->mti = 0;
  }
  uint64_t y = r->mt[r->mti++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:20: uniform in (0, 1], 53-bit resolution. */
double so_rng_uniform(so_rng* r) { return (double)((so_rng_raw(r) >> 11) + 1) * 0x1.0p-53; }

/* rng.hpp:22-32: explicit Box-Muller with a cached spare. */
double so_rng_normal(so_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  const double u1 = so_rng_uniform(r);
  const double u2 = so_rng_uniform(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double a = 6.283185307179586476925286766559 * u2;
  r->spare = rad * sin(a);
  r->has_spare = 1;
  return rad * cos(a);
}

void so_rng_normals(uint64_t seed, int64_t n, double* out) {
  so_rng r;
  so_rng_seed(&r, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = so_rng_normal(&r);
}

/* ---- half.hpp:13-52: float -> binary16, RNE, saturating to +-65504 ---- */
uint16_t so_half_from_float(float value, long long* saturations) {
  uint32_t f;
  memcpy(&f, &value, 4);
  const uint16_t hsign = (uint16_t)((f >> 16) & 0x8000u);
  const uint32_t fexp = (f >> 23) & 0xffu;
  uint32_t man = f & 0x7fffffu;
  if (fexp == 0xffu) {
    if (man != 0) return (uint16_t)(hsign | 0x7e00u);
    if (saturations) ++*saturations;
    return (uint16_t)(hsign | 0x7bffu);
  }
  const int32_t e = (int32_t)fexp - 127 + 15;
  if (e >= 31) {
    if (saturations) ++*saturations;
    return (uint16_t)(hsign | 0x7bffu);
  }
  if (e <= 0) {
    if (e < -10) return hsign;
    man |= 0x800000u;
    const int shift = 14 - e;
    uint32_t hman = man >> shift;
    const uint32_t rem = man & ((1u << shift) - 1u);
    const uint32_t halfway = 1u << (shift - 1);
    if (rem > halfway || (rem == halfway && (hman & 1u))) ++hman;
    return (uint16_t)(hsign | hman);
  }
  uint16_t h = (uint16_t)(hsign | ((uint32_t)e << 10) | (man >> 13));
  const uint32_t rem = man & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) {
    ++h;
    if ((h & 0x7fffu) >= 0x7c00u) {
      if (saturations) ++*saturations;
      return (uint16_t)(hsign | 0x7bffu);
    }
  }
  return h;
}

/* half.hpp:54-77 */
float so_half_to_float(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1fu;
  const uint32_t man = h & 0x3ffu;
  uint32_t f;
  if (e == 0) {
    if (man == 0) {
      f = sign;
    } else {
      uint32_t m = man;
      int sh = 0;
      while (!(m & 0x400u)) {
        m <<= 1;
        ++sh;
      }
      f = sign | ((uint32_t)(113 - sh) << 23) | ((m & 0x3ffu) << 13);
    }
  } else if (e == 31) {
    f = sign | 0x7f800000u | (man << 13);
  } else {
    f = sign | ((e + 112) << 23) | (man << 13);
  }
  float out;
  memcpy(&out, &f, 4);
  return out;
}

/* half.hpp:80-82: double -> float (RNE) -> binary16 (RNE) -> double. */
double so_quantize_half(double v, long long* saturations) {
  return (double)so_half_to_float(so_half_from_float((float)v, saturations));
}

/* half.hpp:85 */
double so_quantize_single(double v) { return (double)(float)v; }

/* BF16 storage class (extension, F2): double -> float (RNE) -> bf16 (RNE),
 * NaN kept, overflow past the largest finite bf16 saturates and is counted. */
double so_quantize_bf16(double v, long long* saturations) {
  float x = (float)v;
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) {
    if (u & 0x7fffffu) {
      u = (u | 0x00400000u) & 0xffff0000u;
      memcpy(&x, &u, 4);
      return (double)x;
    }
    if (saturations) ++*saturations;
    u = (u & 0x80000000u) | 0x7f7f0000u;
    memcpy(&x, &u, 4);
    return (double)x;
  }
  uint32_t lsb = (u >> 16) & 1u;
  uint32_t r = u + 0x7fffu + lsb;
  if ((r & 0x7f800000u) == 0x7f800000u) {
    if (saturations) ++*saturations;
    r = (u & 0x80000000u) | 0x7f7f0000u;
  }
  r &= 0xffff0000u;
  memcpy(&x, &r, 4);
  return (double)x;
}
