/* Synthetic logit rows of the benchmark and parity workloads,
 * bit-identical on the device (dsdv_synth_logits) and on the host (the
 * oracle's generator behind bench.py --impl reference): Philox integers plus
 * correctly rounded +, -, *, /, sqrt and explicit fma only — no libm
 * transcendentals, whose last bits differ between CUDA and glibc — so that
 * the CPU arm can build the same window without the GPU library.
 *
 * Families by b mod 4: Zipf target l_t[i] = -sigma ln(1 + pi(i)),
 * pi(i) = (a i + c) mod V with gcd(a, V) = 1 (sigma 1.2 / 2.5 / 3.5), or
 * Gaussian target sigma 6; draft = stored target + delta N(0, 1)
 * (delta 0.8 / 1.0 / 1.5 / 2). Row (b, j) of the target is item
 * b * (gamma + 1) + j; draft row (b, j < gamma) shares the item's noise.
 */
#ifndef DSDV_SYNTH_H_
#define DSDV_SYNTH_H_

#include <stdint.h>

#include "dsdv/philox.h"

#if defined(__CUDA_ARCH__)
#define DSDV_SY_ADD(a, b) __fadd_rn((a), (b))
#define DSDV_SY_SUB(a, b) __fsub_rn((a), (b))
#define DSDV_SY_MUL(a, b) __fmul_rn((a), (b))
#define DSDV_SY_DIV(a, b) __fdiv_rn((a), (b))
#define DSDV_SY_FMA(a, b, c) __fmaf_rn((a), (b), (c))
#define DSDV_SY_SQRT(a) __fsqrt_rn(a)
#define DSDV_SY_F2U(x) __float_as_uint(x)
#define DSDV_SY_U2F(x) __uint_as_float(x)
#else
#include <math.h>
#include <string.h>
/* host: SSE scalar float, compiled with -ffp-contract=off (oracle/Makefile) */
#define DSDV_SY_ADD(a, b) ((a) + (b))
#define DSDV_SY_SUB(a, b) ((a) - (b))
#define DSDV_SY_MUL(a, b) ((a) * (b))
#define DSDV_SY_DIV(a, b) ((a) / (b))
#define DSDV_SY_FMA(a, b, c) fmaf((a), (b), (c))
#define DSDV_SY_SQRT(a) sqrtf(a)
static inline uint32_t dsdv_sy_f2u(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  return u;
}
static inline float dsdv_sy_u2f(uint32_t u) {
  float x;
  memcpy(&x, &u, 4);
  return x;
}
#define DSDV_SY_F2U(x) dsdv_sy_f2u(x)
#define DSDV_SY_U2F(x) dsdv_sy_u2f(x)
#endif

/* (0, 1) from the top 24 bits */
DSDV_HD float dsdv_synth_u01(uint32_t x) {
  return DSDV_SY_MUL(DSDV_SY_ADD((float)(x >> 8), 0.5f), 1.0f / 16777216.0f);
}

/* ln x for finite x > 0 (normal): x = 2^e m, m in [sqrt(1/2), sqrt 2),
 * ln m = 2 atanh((m - 1) / (m + 1)) by its odd series. */
DSDV_HD float dsdv_synth_log(float x) {
  const uint32_t bits = DSDV_SY_F2U(x);
  int e = (int)((bits >> 23) & 0xffu) - 127;
  float m = DSDV_SY_U2F((bits & 0x7fffffu) | 0x3f800000u);
  if (m > 1.41421356f) {
    m = DSDV_SY_MUL(m, 0.5f);
    e += 1;
  }
  const float s = DSDV_SY_DIV(DSDV_SY_SUB(m, 1.0f), DSDV_SY_ADD(m, 1.0f));
  const float s2 = DSDV_SY_MUL(s, s);
  float q = DSDV_SY_FMA(s2, 0.11111111f, 0.14285715f);
  q = DSDV_SY_FMA(q, s2, 0.2f);
  q = DSDV_SY_FMA(q, s2, 0.33333334f);
  q = DSDV_SY_FMA(q, s2, 1.0f);
  const float lm = DSDV_SY_MUL(DSDV_SY_MUL(2.0f, s), q);
  return DSDV_SY_FMA((float)e, 0.69314718f, lm);
}

/* cos(2 pi u), sin(2 pi u) for u in [0, 1): quarter-turn reduction, then
 * Taylor polynomials on [0, pi/2]. */
DSDV_HD void dsdv_synth_cossin(float u, float *c, float *s) {
  const float q = DSDV_SY_MUL(u, 4.0f);
  const int k = (int)q;
  const float x = DSDV_SY_MUL(DSDV_SY_SUB(q, (float)k), 1.57079637f);
  const float x2 = DSDV_SY_MUL(x, x);
  float sp = DSDV_SY_FMA(x2, 1.6059044e-10f, -2.5052108e-8f);
  sp = DSDV_SY_FMA(sp, x2, 2.7557319e-6f);
  sp = DSDV_SY_FMA(sp, x2, -1.9841270e-4f);
  sp = DSDV_SY_FMA(sp, x2, 8.3333333e-3f);
  sp = DSDV_SY_FMA(sp, x2, -1.6666667e-1f);
  sp = DSDV_SY_FMA(sp, x2, 1.0f);
  const float sn = DSDV_SY_MUL(sp, x);
  float cp = DSDV_SY_FMA(x2, -1.1470746e-11f, 2.0876757e-9f);
  cp = DSDV_SY_FMA(cp, x2, -2.7557319e-7f);
  cp = DSDV_SY_FMA(cp, x2, 2.4801587e-5f);
  cp = DSDV_SY_FMA(cp, x2, -1.3888889e-3f);
  cp = DSDV_SY_FMA(cp, x2, 4.1666667e-2f);
  cp = DSDV_SY_FMA(cp, x2, -0.5f);
  const float cs = DSDV_SY_FMA(cp, x2, 1.0f);
  switch (k & 3) {
    case 0: *c = cs; *s = sn; break;
    case 1: *c = -sn; *s = cs; break;
    case 2: *c = -cs; *s = -sn; break;
    default: *c = sn; *s = -cs; break;
  }
}

DSDV_HD uint32_t dsdv_synth_gcd(uint32_t a, uint32_t b) {
  while (b) {
    const uint32_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

typedef struct {
  int fam;
  float sigma, delta;
  uint32_t a, c; /* Zipf permutation pi(i) = (a i + c) mod V */
} dsdv_synth_row;

DSDV_HD dsdv_synth_row dsdv_synth_row_params(uint64_t seed, uint32_t item, int b, int V) {
  dsdv_synth_row r;
  r.fam = b & 3;
  r.sigma = r.fam == 0 ? 1.2f : r.fam == 1 ? 2.5f : r.fam == 2 ? 3.5f : 6.0f;
  r.delta = r.fam == 0 ? 0.8f : r.fam == 1 ? 1.0f : r.fam == 2 ? 1.5f : 2.0f;
  const dsdv_philox_out rp =
      dsdv_philox4x32_10(0xffffffffu, item, 0x5eedu, 0u, (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint32_t half = (uint32_t)(V / 2 > 0 ? V / 2 : 1);
  uint32_t a = 1u + 2u * (rp.v[0] % half);
  while (dsdv_synth_gcd(a % (uint32_t)V, (uint32_t)V) != 1u) a += 2u;
  r.a = a % (uint32_t)V;
  r.c = rp.v[1] % (uint32_t)V;
  return r;
}

/* Element i of item `item`: the target logit (fp32, before storage rounding)
 * and the unit Gaussian z1 of the draft noise. */
DSDV_HD void dsdv_synth_element(uint64_t seed, uint32_t item, const dsdv_synth_row *r, int V,
                                int i, float *lt, float *z1) {
  const dsdv_philox_out o = dsdv_philox4x32_10((uint32_t)i, item, 0x10917u, 0u, (uint32_t)seed,
                                               (uint32_t)(seed >> 32));
  const float rad =
      DSDV_SY_SQRT(DSDV_SY_MUL(-2.0f, dsdv_synth_log(dsdv_synth_u01(o.v[0]))));
  float c, s;
  dsdv_synth_cossin(dsdv_synth_u01(o.v[1]), &c, &s);
  *z1 = DSDV_SY_MUL(rad, s);
  if (r->fam < 3) {
    const uint32_t pi = (uint32_t)(((uint64_t)r->a * (uint32_t)i + r->c) % (uint32_t)V);
    *lt = DSDV_SY_MUL(-r->sigma, dsdv_synth_log(DSDV_SY_ADD(1.0f, (float)pi)));
  } else {
    *lt = DSDV_SY_MUL(r->sigma, DSDV_SY_MUL(rad, c));
  }
}

/* fp32 -> bf16 bits, round to nearest even (as __float2bfloat16_rn) */
DSDV_HD uint16_t dsdv_synth_bf16_bits(float x) {
  const uint32_t u = DSDV_SY_F2U(x);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u); /* NaN */
  return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}
DSDV_HD float dsdv_synth_bf16_value(uint16_t h) { return DSDV_SY_U2F((uint32_t)h << 16); }

/* draft logit from the stored target value: round(stored + delta z1) */
DSDV_HD float dsdv_synth_draft(float stored_target, float delta, float z1) {
  return DSDV_SY_FMA(delta, z1, stored_target);
}

#endif /* DSDV_SYNTH_H_ */
