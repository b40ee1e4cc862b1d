/* CPU oracle for the DSD verifier hot path — TEST INFRASTRUCTURE ONLY.
 * See dsd_oracle.h. Every function restates the reference function cited
 * beside it (paths relative to /root/reference/proj) with the same fp64
 * operations in the same order, so results are bit-identical to the
 * reference built from its sources with the same libm (checked against
 * oracle/_ref in tests/test_oracle.py).
 */
#include "dsd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double kCertainSurprisal = 1e-12; /* verifier.cpp:30 */

/* check_entries (distribution.cpp:29-40) + from_weights (:54-63) of
 * w_i = exp(l_i - max). */
int oracle_softmax(const double *logits, int V, double *probs) {
  if (V < 2) return ORACLE_E_INVARIANT;
  double m = -INFINITY;
  for (int i = 0; i < V; ++i) {
    if (isnan(logits[i]) || logits[i] == INFINITY) return ORACLE_E_INVARIANT;
    if (logits[i] > m) m = logits[i];
  }
  if (m == -INFINITY) return ORACLE_E_INVARIANT; /* zero total mass */
  for (int i = 0; i < V; ++i) probs[i] = exp(logits[i] - m);
  double sum = 0.0;
  for (int i = 0; i < V; ++i) sum += probs[i];
  if (!(sum > 0.0)) return ORACLE_E_INVARIANT;
  for (int i = 0; i < V; ++i) probs[i] /= sum;
  return ORACLE_OK;
}

/* token_cross_entropy, verifier.cpp:112-117 */
double oracle_cross_entropy(const double *p, int V, int token) {
  if (token < 0 || token >= V) return NAN;
  const double q = p[token];
  if (q <= 0.0) return INFINITY;
  return -log(q);
}

/* top_ids, verifier.cpp:40-51: ids ordered by (p desc, id asc), first m.
 * A stable sort of all ids restated as an ascending scan that keeps the m
 * best: an equal-probability newcomer always has the larger id, so it
 * lands behind existing equals exactly as the stable sort orders them. */
static void top_ids(const double *p, int V, int m, int *out) {
  int n = 0;
  for (int i = 0; i < V; ++i) {
    const double v = p[i];
    if (n == m && !(v > p[out[m - 1]])) continue;
    int pos = n < m ? n : m - 1;
    while (pos > 0 && v > p[out[pos - 1]]) {
      out[pos] = out[pos - 1];
      --pos;
    }
    out[pos] = i;
    if (n < m) ++n;
  }
}

/* norm_match, verifier.cpp:119-134 */
double oracle_norm_match(const double *pt, const double *pd, int V, int top_m) {
  if (top_m < 1 || top_m > V) return NAN;
  int *tt = (int *)malloc(sizeof(int) * (size_t)top_m);
  int *td = (int *)malloc(sizeof(int) * (size_t)top_m);
  top_ids(pt, V, top_m, tt);
  top_ids(pd, V, top_m, td);
  int shared = 0;
  for (int a = 0; a < top_m; ++a)
    for (int b = 0; b < top_m; ++b)
      if (td[a] == tt[b]) {
        ++shared;
        break;
      }
  free(tt);
  free(td);
  return (double)shared / (double)top_m;
}

static double fmax1(double x) { return x > 1.0 ? x : 1.0; }

/* is_key, verifier.cpp:136-159 */
int oracle_is_key(const double *pt, const double *pd, int V, int token, const oracle_criteria *c,
                  double *margins) {
  const double h_draft = oracle_cross_entropy(pd, V, token);
  const double h_target = oracle_cross_entropy(pt, V, token);
  int ratio;
  double m_ratio = INFINITY;
  if (h_target < kCertainSurprisal) {
    ratio = h_draft > 0.0;
    m_ratio = h_target; /* distance into the certain branch */
  } else {
    ratio = (h_draft / h_target) > c->ratio_limit;
    if (isfinite(c->ratio_limit) && isfinite(h_draft))
      m_ratio = fabs(h_draft / h_target - c->ratio_limit) / fmax1(c->ratio_limit);
  }
  const double gap = fabs(pt[token] - pd[token]);
  const int gap_c = gap > c->gap_limit;
  const int m = c->top_m < V ? c->top_m : V;
  const int overlap = oracle_norm_match(pt, pd, V, m) < c->overlap_floor;
  if (margins) {
    margins[0] = m_ratio;
    margins[1] = fabs(gap - c->gap_limit) / fmax1(c->gap_limit);
  }
  return ratio || gap_c || overlap;
}

/* soften, verifier.cpp:161-186 */
int oracle_soften(const double *pt, const double *pd, int V, double tau, double *out) {
  if (tau == 0.0) {
    memcpy(out, pt, sizeof(double) * (size_t)V);
    return ORACLE_OK;
  }
  if (tau == 1.0) {
    memcpy(out, pd, sizeof(double) * (size_t)V);
    return ORACLE_OK;
  }
  int equal = 1;
  for (int i = 0; i < V && equal; ++i) equal = pt[i] == pd[i];
  if (equal) {
    memcpy(out, pt, sizeof(double) * (size_t)V);
    return ORACLE_OK;
  }
  double mass = 0.0;
  for (int i = 0; i < V; ++i) {
    out[i] = pow(pt[i], 1.0 - tau) * pow(pd[i], tau);
    mass += out[i];
  }
  if (mass <= 0.0) return ORACLE_E_DEGENERATE_MIXTURE;
  /* from_weights: its own sequential sum, then divide (distribution.cpp:57-61) */
  double sum = 0.0;
  for (int i = 0; i < V; ++i) sum += out[i];
  for (int i = 0; i < V; ++i) out[i] /= sum;
  return ORACLE_OK;
}

/* accept_prob, verifier.cpp:188-196 */
double oracle_accept_prob(const double *eff, const double *pd, int token, int *err) {
  const double p_draft = pd[token];
  if (p_draft <= 0.0) {
    if (err) *err = ORACLE_E_DRAFTING_CONTRACT;
    return NAN;
  }
  if (err) *err = ORACLE_OK;
  const double r = eff[token] / p_draft;
  return r < 1.0 ? r : 1.0;
}

/* residual_distribution, verifier.cpp:198-213 */
int oracle_residual(const double *eff, const double *pd, int V, double *out) {
  double mass = 0.0;
  for (int i = 0; i < V; ++i) {
    const double d = eff[i] - pd[i];
    out[i] = d > 0.0 ? d : 0.0;
    mass += out[i];
  }
  if (mass <= 0.0) return ORACLE_E_EMPTY_RESIDUAL;
  double sum = 0.0;
  for (int i = 0; i < V; ++i) sum += out[i];
  for (int i = 0; i < V; ++i) out[i] /= sum;
  return ORACLE_OK;
}

/* sample_with_uniform, distribution.cpp:103-114 */
int oracle_sample_with_uniform(const double *p, int V, double u, double *margin) {
  double cum = 0.0;
  int last_supported = -1;
  for (int i = 0; i < V; ++i) {
    if (p[i] > 0.0) last_supported = i;
    const double prev = cum;
    cum += p[i];
    if (u < cum) {
      if (margin) {
        const double a = u - prev, b = cum - u;
        *margin = a < b ? a : b;
      }
      return i;
    }
  }
  if (margin) *margin = 0.0;
  return last_supported;
}

/* ---- uniform sources ---- */
double oracle_slot_next(void *state) {
  oracle_slot_stream *s = (oracle_slot_stream *)state;
  return s->u[s->cursor++];
}

/* std::mt19937_64 (the engine of SeededStream, rng.hpp:34-44). */
void oracle_mt64_seed(oracle_mt64 *s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_raw(oracle_mt64 *s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

double oracle_mt64_next(void *state) {
  return (double)(mt64_raw((oracle_mt64 *)state) >> 11) * 0x1.0p-53; /* rng.hpp:39 */
}

/* The per-position loop of verify_round (verifier.cpp:223-256). Rows are
 * evaluated lazily: an invalid row only fails once the loop reaches it. */
int oracle_verify_window(const oracle_window *w, oracle_result *out) {
  const int V = w->V, G = w->gamma;
  double *eff = (double *)malloc(sizeof(double) * (size_t)V);
  double *res = (double *)malloc(sizeof(double) * (size_t)V);
  int st = ORACLE_OK;
  out->accepted_count = 0;
  out->extra_token = -1;
  out->extra_source = 0;
  out->key_count = 0;
  out->evaluated = 0;
  out->margin_extra = INFINITY;
  for (int j = 0; j < G; ++j) {
    const double *pt = w->pt + (size_t)j * V;
    const double *pd = w->pd + (size_t)j * V;
    const int y = w->tokens[j];
    if (w->row_err && (w->row_err[G + j] || w->row_err[j])) {
      st = ORACLE_E_INVARIANT;
      break;
    }
    if (y < 0 || y >= V) {
      st = ORACLE_E_INVARIANT; /* check_token_in_vocab, verifier.cpp:32-37 */
      break;
    }
    double km[2];
    const int key = oracle_is_key(pt, pd, V, y, &w->crit, km);
    if (key) {
      memcpy(eff, pt, sizeof(double) * (size_t)V);
    } else if ((st = oracle_soften(pt, pd, V, w->tau, eff)) != ORACLE_OK) {
      break;
    }
    int err = 0;
    const double a = oracle_accept_prob(eff, pd, y, &err);
    if (err) {
      st = err;
      break;
    }
    const double u = w->next_uniform(w->rng);
    const int accepted = u < a; /* verifier.cpp:237 */
    out->evaluated = j + 1;
    out->key_count += key;
    if (out->key) out->key[j] = (uint8_t)key;
    if (out->accepted) out->accepted[j] = (uint8_t)accepted;
    if (out->accept_prob) out->accept_prob[j] = a;
    if (out->h_target) out->h_target[j] = oracle_cross_entropy(pt, V, y);
    if (out->h_draft) out->h_draft[j] = oracle_cross_entropy(pd, V, y);
    if (out->p_target_y) out->p_target_y[j] = pt[y];
    if (out->p_draft_y) out->p_draft_y[j] = pd[y];
    if (out->norm_match) {
      const int m = w->crit.top_m < V ? w->crit.top_m : V;
      out->norm_match[j] = oracle_norm_match(pt, pd, V, m);
    }
    if (out->p_eff_y) out->p_eff_y[j] = eff[y];
    if (out->uniform) out->uniform[j] = u;
    if (out->margin_u) out->margin_u[j] = fabs(u - a);
    if (out->margin_key) out->margin_key[j] = km[0] < km[1] ? km[0] : km[1];
    if (accepted) {
      out->accepted_count += 1;
      continue;
    }
    out->extra_source = 1; /* ResidualResample */
    if ((st = oracle_residual(eff, pd, V, res)) != ORACLE_OK) break;
    out->extra_token =
        oracle_sample_with_uniform(res, V, w->next_uniform(w->rng), &out->margin_extra);
    goto done;
  }
  if (st == ORACLE_OK) {
    /* whole window accepted: bonus from target row gamma (verifier.cpp:253-256) */
    out->extra_source = 0;
    if (w->row_err && w->row_err[G + G])
      st = ORACLE_E_INVARIANT;
    else
      out->extra_token = oracle_sample_with_uniform(w->pt + (size_t)G * V, V,
                                                    w->next_uniform(w->rng), &out->margin_extra);
  }
done:
  out->status = st;
  free(eff);
  free(res);
  return st;
}

int oracle_verify_window_logits(int gamma, int V, const double *draft_logits,
                                const double *target_logits, const int32_t *tokens, double tau,
                                const oracle_criteria *crit, const double *uniforms,
                                oracle_result *out) {
  double *pd = (double *)malloc(sizeof(double) * (size_t)gamma * V);
  double *pt = (double *)malloc(sizeof(double) * (size_t)(gamma + 1) * V);
  int *row_err = (int *)calloc((size_t)(2 * gamma + 1), sizeof(int));
  for (int j = 0; j < gamma; ++j)
    row_err[j] = oracle_softmax(draft_logits + (size_t)j * V, V, pd + (size_t)j * V);
  for (int j = 0; j <= gamma; ++j)
    row_err[gamma + j] = oracle_softmax(target_logits + (size_t)j * V, V, pt + (size_t)j * V);
  oracle_slot_stream ss = {uniforms, gamma};
  oracle_window w = {gamma, V, pd, pt, row_err, tokens, tau, *crit, oracle_slot_next, &ss};
  const int st = oracle_verify_window(&w, out);
  free(pd);
  free(pt);
  free(row_err);
  return st;
}

int oracle_draft_tokens(const double *draft_logits, int gamma, int V, const double *uniforms,
                        int32_t *tokens, double *margins) {
  double *p = (double *)malloc(sizeof(double) * (size_t)V);
  int st = ORACLE_OK;
  for (int j = 0; j < gamma && st == ORACLE_OK; ++j) {
    st = oracle_softmax(draft_logits + (size_t)j * V, V, p);
    if (st == ORACLE_OK)
      tokens[j] = oracle_sample_with_uniform(p, V, uniforms[j], margins ? &margins[j] : NULL);
  }
  free(p);
  return st;
}

/* generate (verifier.cpp:259-282) over categorical-iid models. */
int oracle_generate_iid(const double *pd, const double *pt, int V, int gamma, double tau,
                        const oracle_criteria *crit, int max_new, uint64_t seed, int *ks,
                        int max_rounds) {
  oracle_mt64 rng;
  oracle_mt64_seed(&rng, seed);
  double *pdr = (double *)malloc(sizeof(double) * (size_t)gamma * V);
  double *ptr = (double *)malloc(sizeof(double) * (size_t)(gamma + 1) * V);
  int32_t *tok = (int32_t *)malloc(sizeof(int32_t) * (size_t)gamma);
  for (int j = 0; j < gamma; ++j) memcpy(pdr + (size_t)j * V, pd, sizeof(double) * (size_t)V);
  for (int j = 0; j <= gamma; ++j) memcpy(ptr + (size_t)j * V, pt, sizeof(double) * (size_t)V);
  int committed = 0, rounds = 0, st = ORACLE_OK;
  while (committed < max_new) {
    for (int j = 0; j < gamma; ++j) /* draft_window: one draw per position */
      tok[j] = oracle_sample_with_uniform(pd, V, oracle_mt64_next(&rng), NULL);
    oracle_window w = {gamma, V, pdr, ptr, NULL, tok, tau, *crit, oracle_mt64_next, &rng};
    oracle_result r;
    memset(&r, 0, sizeof(r));
    st = oracle_verify_window(&w, &r);
    if (st != ORACLE_OK) break;
    if (rounds < max_rounds) ks[rounds] = r.accepted_count;
    ++rounds;
    committed += r.accepted_count + 1;
  }
  free(pdr);
  free(ptr);
  free(tok);
  return st == ORACLE_OK ? rounds : -st;
}

/* ---- CPU baseline: B windows on nthreads POSIX threads ---- */
#include <pthread.h>

typedef struct {
  int B, gamma, V, stride, nthreads, tid;
  const float *draft, *target;
  const int32_t *tokens;
  double tau;
  const oracle_criteria *crit;
  const double *uniforms;
  int32_t *k_out, *extra_out, *status_out;
} batch_job;

static void *batch_worker(void *arg) {
  batch_job *j = (batch_job *)arg;
  const int G = j->gamma, V = j->V;
  double *dl = (double *)malloc(sizeof(double) * (size_t)G * V);
  double *tl = (double *)malloc(sizeof(double) * (size_t)(G + 1) * V);
  for (int b = j->tid; b < j->B; b += j->nthreads) {
    for (int r = 0; r < G; ++r)
      for (int i = 0; i < V; ++i)
        dl[(size_t)r * V + i] = j->draft[((size_t)b * G + r) * j->stride + i];
    for (int r = 0; r <= G; ++r)
      for (int i = 0; i < V; ++i)
        tl[(size_t)r * V + i] = j->target[((size_t)b * (G + 1) + r) * j->stride + i];
    oracle_result res;
    memset(&res, 0, sizeof(res));
    oracle_verify_window_logits(G, V, dl, tl, j->tokens + (size_t)b * G, j->tau, j->crit,
                                j->uniforms + (size_t)b * (2 * G + 1), &res);
    j->k_out[b] = res.accepted_count;
    j->extra_out[b] = res.extra_token;
    j->status_out[b] = res.status;
  }
  free(dl);
  free(tl);
  return NULL;
}

int oracle_verify_batch_f32(int B, int gamma, int V, int stride, const float *draft,
                            const float *target, const int32_t *tokens, double tau,
                            const oracle_criteria *crit, const double *uniforms, int nthreads,
                            int32_t *k_out, int32_t *extra_out, int32_t *status_out) {
  if (nthreads < 1) nthreads = 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  batch_job *jobs = (batch_job *)malloc(sizeof(batch_job) * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) {
    batch_job j = {B, gamma, V, stride, nthreads, t, draft, target, tokens, tau, crit,
                   uniforms, k_out, extra_out, status_out};
    jobs[t] = j;
    pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}

/* ---- parity checker: B windows x ncfg (tau, criteria) configurations ---- */

static double bf16_to_double(uint16_t h) {
  union {
    uint32_t u;
    float f;
  } v;
  v.u = (uint32_t)h << 16;
  return (double)v.f;
}

static void row_to_f64(const void *base, int dtype, size_t row, int stride, int V, double *out) {
  if (dtype == 1) {
    const uint16_t *r = (const uint16_t *)base + row * (size_t)stride;
    for (int i = 0; i < V; ++i) out[i] = bf16_to_double(r[i]);
  } else {
    const float *r = (const float *)base + row * (size_t)stride;
    for (int i = 0; i < V; ++i) out[i] = (double)r[i];
  }
}

typedef struct {
  int B, gamma, V, stride, dtype, ncfg, all_positions, nthreads, tid;
  const void *draft, *target;
  const int32_t *tokens;
  const double *taus;
  const oracle_criteria *crits;
  const double *uniforms;
  oracle_batch_out *outs;
} full_job;

/* Per-position quantities of verify_round (verifier.cpp:223-236) without the
 * draw: for positions after the first rejection, which the reference never
 * evaluates but the device computes (numerics only). */
static void position_numerics(const double *pt, const double *pd, int V, int y, double tau,
                              const oracle_criteria *c, double *eff, oracle_batch_out *o,
                              size_t pos) {
  if (y < 0 || y >= V) return;
  double km[2];
  const int key = oracle_is_key(pt, pd, V, y, c, km);
  if (key)
    memcpy(eff, pt, sizeof(double) * (size_t)V);
  else if (oracle_soften(pt, pd, V, tau, eff) != ORACLE_OK)
    return;
  int err = 0;
  const double a = oracle_accept_prob(eff, pd, y, &err);
  const int m = c->top_m < V ? c->top_m : V;
  o->key[pos] = (uint8_t)key;
  o->accept_prob[pos] = err ? NAN : a;
  o->h_target[pos] = oracle_cross_entropy(pt, V, y);
  o->h_draft[pos] = oracle_cross_entropy(pd, V, y);
  o->p_target_y[pos] = pt[y];
  o->p_draft_y[pos] = pd[y];
  o->norm_match[pos] = oracle_norm_match(pt, pd, V, m);
  o->p_eff_y[pos] = eff[y];
  o->margin_key[pos] = km[0] < km[1] ? km[0] : km[1];
}

static void *full_worker(void *arg) {
  full_job *j = (full_job *)arg;
  const int G = j->gamma, V = j->V;
  double *raw = (double *)malloc(sizeof(double) * (size_t)V);
  double *pd = (double *)malloc(sizeof(double) * (size_t)G * V);
  double *pt = (double *)malloc(sizeof(double) * (size_t)(G + 1) * V);
  double *eff = (double *)malloc(sizeof(double) * (size_t)V);
  int *row_err = (int *)malloc(sizeof(int) * (size_t)(2 * G + 1));
  for (int b = j->tid; b < j->B; b += j->nthreads) {
    for (int r = 0; r < G; ++r) {
      row_to_f64(j->draft, j->dtype, (size_t)b * G + r, j->stride, V, raw);
      row_err[r] = oracle_softmax(raw, V, pd + (size_t)r * V);
    }
    for (int r = 0; r <= G; ++r) {
      row_to_f64(j->target, j->dtype, (size_t)b * (G + 1) + r, j->stride, V, raw);
      row_err[G + r] = oracle_softmax(raw, V, pt + (size_t)r * V);
    }
    const int32_t *tok = j->tokens + (size_t)b * G;
    for (int c = 0; c < j->ncfg; ++c) {
      oracle_batch_out *o = &j->outs[c];
      const size_t p0 = (size_t)b * G;
      oracle_result r;
      memset(&r, 0, sizeof(r));
      r.key = o->key + p0;
      r.accepted = o->accepted + p0;
      r.accept_prob = o->accept_prob + p0;
      r.h_target = o->h_target + p0;
      r.h_draft = o->h_draft + p0;
      r.p_target_y = o->p_target_y + p0;
      r.p_draft_y = o->p_draft_y + p0;
      r.norm_match = o->norm_match + p0;
      r.p_eff_y = o->p_eff_y + p0;
      r.margin_u = o->margin_u + p0;
      r.margin_key = o->margin_key + p0;
      oracle_slot_stream ss = {j->uniforms + (size_t)b * (2 * G + 1), G};
      oracle_window w = {G,   V,         pd,   pt, row_err, tok, j->taus[c], j->crits[c],
                         oracle_slot_next, &ss};
      oracle_verify_window(&w, &r);
      o->k[b] = r.accepted_count;
      o->extra_token[b] = r.extra_token;
      o->extra_source[b] = r.extra_source;
      o->key_count[b] = r.key_count;
      o->status[b] = r.status;
      o->evaluated[b] = r.evaluated;
      o->margin_extra[b] = r.margin_extra;
      if (j->all_positions)
        for (int q = r.evaluated; q < G; ++q)
          if (!row_err[q] && !row_err[G + q])
            position_numerics(pt + (size_t)q * V, pd + (size_t)q * V, V, tok[q], j->taus[c],
                              &j->crits[c], eff, o, p0 + (size_t)q);
    }
  }
  free(raw);
  free(pd);
  free(pt);
  free(eff);
  free(row_err);
  return NULL;
}

int oracle_verify_batch(int B, int gamma, int V, int stride, int dtype, const void *draft,
                        const void *target, const int32_t *tokens, int ncfg, const double *taus,
                        const oracle_criteria *crits, const double *uniforms, int all_positions,
                        int nthreads, oracle_batch_out *outs) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > B) nthreads = B;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  full_job *jobs = (full_job *)malloc(sizeof(full_job) * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) {
    full_job j = {B,      gamma,  V,        stride, dtype, ncfg, all_positions, nthreads, t,
                  draft,  target, tokens,   taus,   crits, uniforms, outs};
    jobs[t] = j;
    pthread_create(&th[t], NULL, full_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}

/* ---- host generator of the synthetic windows (include/dsdv/synth.h) ---- */
#include "dsdv/synth.h"

typedef struct {
  int B, gamma, V, stride, dtype, nthreads, tid;
  uint64_t seed;
  void *draft, *target;
} synth_job;

static void *synth_worker(void *arg) {
  synth_job *j = (synth_job *)arg;
  const int G1 = j->gamma + 1;
  for (int item = j->tid; item < j->B * G1; item += j->nthreads) {
    const int b = item / G1, r = item - b * G1;
    const dsdv_synth_row rp = dsdv_synth_row_params(j->seed, (uint32_t)item, b, j->V);
    const size_t t0 = (size_t)item * j->stride;
    const size_t d0 = ((size_t)b * j->gamma + r) * j->stride;
    for (int i = 0; i < j->stride; ++i) {
      float lt = -INFINITY, ld = -INFINITY, z1 = 0.0f;
      if (i < j->V) {
        dsdv_synth_element(j->seed, (uint32_t)item, &rp, j->V, i, &lt, &z1);
      }
      if (j->dtype == 1) {
        const uint16_t tb = dsdv_synth_bf16_bits(lt);
        ((uint16_t *)j->target)[t0 + i] = tb;
        if (r < j->gamma) {
          if (i < j->V) ld = dsdv_synth_draft(dsdv_synth_bf16_value(tb), rp.delta, z1);
          ((uint16_t *)j->draft)[d0 + i] = dsdv_synth_bf16_bits(ld);
        }
      } else {
        ((float *)j->target)[t0 + i] = lt;
        if (r < j->gamma) {
          if (i < j->V) ld = dsdv_synth_draft(lt, rp.delta, z1);
          ((float *)j->draft)[d0 + i] = ld;
        }
      }
    }
  }
  return NULL;
}

int oracle_synth_logits(int B, int gamma, int V, int stride, uint64_t seed, int dtype,
                        void *draft, void *target, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  synth_job *jobs = (synth_job *)malloc(sizeof(synth_job) * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) {
    synth_job j = {B, gamma, V, stride, dtype, nthreads, t, seed, draft, target};
    jobs[t] = j;
    pthread_create(&th[t], NULL, synth_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}
