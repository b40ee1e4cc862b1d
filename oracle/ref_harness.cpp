// Harness around the REFERENCE's own verifier sources — TEST INFRASTRUCTURE ONLY.
//
// Compiled together with /root/reference/proj/src/{distribution,token_model,
// verifier,enumerate}.cpp (unmodified, read in place) into oracle/_ref/libdsdref.so
// by oracle/Makefile. It exposes a C interface so the Python tests and the
// bench's reference arm can drive the reference implementation directly:
//   * the primitives (is_key, soften, accept_prob, residual_distribution,
//     sample_with_uniform, norm_match, token_cross_entropy) on probability rows;
//   * "Oracle-A": dsd::verify_round unchanged, with categorical models and a
//     Philox UniformStream that hands out consecutive counter slots
//     (include/dsdv/philox.h) — exactly the reference's consumption order;
//   * "Oracle-B": per-position rows (logits -> Distribution::from_weights),
//     the loop of verify_round (verifier.cpp:223-256) calling only reference
//     primitives; multi-threaded over sequences for the CPU baseline;
//   * dsd::generate with SeededStream (acceptance criterion 6).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <thread>
#include <vector>

#include "dsd/distribution.hpp"
#include "dsd/enumerate.hpp"
#include "dsd/error.hpp"
#include "dsd/rng.hpp"
#include "dsd/token_model.hpp"
#include "dsd/calibrate.hpp"
#include "dsd/verifier.hpp"
#include "../include/dsdv/philox.h"

namespace {

enum { kOk = 0, kInvariant = 1, kDegenerate = 2, kDrafting = 3, kEmptyResidual = 4, kOther = 9 };

int code_of(const std::exception_ptr &ep) {
  try {
    std::rethrow_exception(ep);
  } catch (const dsd::DegenerateMixtureError &) {
    return kDegenerate;
  } catch (const dsd::DraftingContractError &) {
    return kDrafting;
  } catch (const dsd::EmptyResidualError &) {
    return kEmptyResidual;
  } catch (const dsd::InvariantError &) {
    return kInvariant;
  } catch (const dsd::InvalidContextError &) {
    return kInvariant;
  } catch (...) {
    return kOther;
  }
}

dsd::Distribution dist(const double *p, int V) {
  return dsd::Distribution(std::vector<double>(p, p + V));
}

dsd::Distribution from_logits(const double *l, int V) {
  double m = -INFINITY;
  for (int i = 0; i < V; ++i) m = l[i] > m ? l[i] : m;
  std::vector<double> w((size_t)V);
  for (int i = 0; i < V; ++i) w[(size_t)i] = std::exp(l[i] - m);
  return dsd::Distribution::from_weights(std::move(w));
}

// Consecutive Philox counter slots: replays the reference's draw order.
class PhiloxStream final : public dsd::UniformStream {
 public:
  PhiloxStream(uint64_t seed, uint64_t window, uint32_t seq, uint32_t first_slot = 0)
      : seed_(seed), window_(window), seq_(seq), slot_(first_slot) {}
  double next_uniform() override { return dsdv_philox_uniform(seed_, window_, seq_, slot_++); }
  uint32_t slot() const { return slot_; }

 private:
  uint64_t seed_, window_;
  uint32_t seq_, slot_;
};

dsd::KeyCriteria crit_of(double r, double g, double o, int m) { return dsd::KeyCriteria{r, g, o, m}; }

struct WindowOut {
  int32_t k, extra, source, key_count, status, evaluated;
};

// Oracle-B over one window of logit rows.
WindowOut oracle_b(int G, int V, const double *dl, const double *tl, const int32_t *tok, double tau,
                   const dsd::KeyCriteria &c, dsd::UniformStream &rng, uint8_t *key,
                   uint8_t *acc, double *aprob) {
  WindowOut o{0, -1, 0, 0, 0, 0};
  try {
    for (int j = 0; j < G; ++j) {
      const dsd::Distribution pt = from_logits(tl + (size_t)j * V, V);
      const dsd::Distribution pd = from_logits(dl + (size_t)j * V, V);
      const int y = tok[j];
      const bool is_key = dsd::is_key(pt, pd, y, c);
      const dsd::Distribution eff = is_key ? pt : dsd::soften(pt, pd, tau);
      const double a = dsd::accept_prob(eff, pd, y);
      const double u = rng.next_uniform();
      const bool accepted = u < a;
      o.evaluated = j + 1;
      o.key_count += is_key ? 1 : 0;
      if (key) key[j] = is_key;
      if (acc) acc[j] = accepted;
      if (aprob) aprob[j] = a;
      if (accepted) {
        ++o.k;
        continue;
      }
      o.source = 1;
      o.extra = dsd::sample(dsd::residual_distribution(eff, pd), rng);
      return o;
    }
    o.source = 0;
    o.extra = dsd::sample(from_logits(tl + (size_t)G * V, V), rng);
  } catch (...) {
    o.status = code_of(std::current_exception());
  }
  return o;
}

}  // namespace

extern "C" {

// ---- primitives on probability rows ----
int ref_cross_entropy(const double *p, int V, int token, double *out) {
  try {
    *out = dsd::token_cross_entropy(dist(p, V), token);
    return kOk;
  } catch (...) {
    return code_of(std::current_exception());
  }
}
int ref_norm_match(const double *pt, const double *pd, int V, int m, double *out) {
  try {
    *out = dsd::norm_match(dist(pt, V), dist(pd, V), m);
    return kOk;
  } catch (...) {
    return code_of(std::current_exception());
  }
}
int ref_is_key(const double *pt, const double *pd, int V, int token, double r, double g, double o,
               int m, int *out) {
  try {
    *out = dsd::is_key(dist(pt, V), dist(pd, V), token, crit_of(r, g, o, m)) ? 1 : 0;
    return kOk;
  } catch (...) {
    return code_of(std::current_exception());
  }
}
int ref_soften(const double *pt, const double *pd, int V, double tau, double *out) {
  try {
    const dsd::Distribution s = dsd::soften(dist(pt, V), dist(pd, V), tau);
    std::memcpy(out, s.probs().data(), sizeof(double) * (size_t)V);
    return kOk;
  } catch (...) {
    return code_of(std::current_exception());
  }
}
int ref_accept_prob(const double *eff, const double *pd, int V, int token, double *out) {
  try {
    *out = dsd::accept_prob(dist(eff, V), dist(pd, V), token);
    return kOk;
  } catch (...) {
    return code_of(std::current_exception());
  }
}
int ref_residual(const double *eff, const double *pd, int V, double *out) {
  try {
    const dsd::Distribution r = dsd::residual_distribution(dist(eff, V), dist(pd, V));
    std::memcpy(out, r.probs().data(), sizeof(double) * (size_t)V);
    return kOk;
  } catch (...) {
    return code_of(std::current_exception());
  }
}
int ref_sample_with_uniform(const double *p, int V, double u, int *out) {
  try {
    *out = dsd::sample_with_uniform(dist(p, V), u);
    return kOk;
  } catch (...) {
    return code_of(std::current_exception());
  }
}
int ref_softmax(const double *logits, int V, double *out) {
  try {
    const dsd::Distribution d = from_logits(logits, V);
    std::memcpy(out, d.probs().data(), sizeof(double) * (size_t)V);
    return kOk;
  } catch (...) {
    return code_of(std::current_exception());
  }
}
double ref_seeded_uniform(uint64_t seed, int index) {
  dsd::SeededStream s(seed);
  double u = 0.0;
  for (int i = 0; i <= index; ++i) u = s.next_uniform();
  return u;
}

// ---- Oracle-A: verify_round unchanged, categorical models, Philox stream ----
// Writes draft tokens [gamma], key/accepted/accept_prob [gamma] (valid up to
// the number of decisions, returned in *n_decisions).
int ref_verify_round_iid(const double *pd, const double *pt, int V, int gamma, double tau,
                         double r, double g, double o, int m, uint64_t seed, uint64_t window,
                         uint32_t seq, int32_t *tokens, uint8_t *key, uint8_t *accepted,
                         double *aprob, int32_t *res /* k, extra, source, key_count, n_dec */) {
  try {
    const dsd::TokenModel draft = dsd::TokenModel::categorical(dist(pd, V));
    const dsd::TokenModel target = dsd::TokenModel::categorical(dist(pt, V));
    PhiloxStream rng(seed, window, seq, 0);
    const dsd::VerificationResult vr = dsd::verify_round(
        draft, target, dsd::Context{}, dsd::VerifyParams{gamma, tau, crit_of(r, g, o, m)}, rng);
    // draft tokens are the decisions' tokens, plus the unevaluated tail, which
    // we recover by replaying the draft draws (slots 0..gamma-1).
    const std::vector<double> pdv(pd, pd + V);
    for (int j = 0; j < gamma; ++j)
      tokens[j] = dsd::sample_with_uniform(dist(pd, V), dsdv_philox_uniform(seed, window, seq, j));
    for (size_t j = 0; j < vr.decisions.size(); ++j) {
      key[j] = vr.decisions[j].is_key;
      accepted[j] = vr.decisions[j].accepted;
      aprob[j] = vr.decisions[j].accept_prob;
    }
    res[0] = vr.accepted_count;
    res[1] = vr.extra_token;
    res[2] = vr.extra_source == dsd::ExtraSource::ResidualResample ? 1 : 0;
    res[3] = vr.key_count();
    res[4] = (int32_t)vr.decisions.size();
    return kOk;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// ---- Oracle-B on one window of fp64 logit rows, Philox slot uniforms ----
int ref_verify_window_logits(int gamma, int V, const double *draft_logits,
                             const double *target_logits, const int32_t *tokens, double tau,
                             double r, double g, double o, int m, const double *uniforms,
                             uint8_t *key, uint8_t *accepted, double *aprob,
                             int32_t *res /* k, extra, source, key_count, status, evaluated */) {
  struct Slots final : dsd::UniformStream {
    const double *u;
    int cur;
    double next_uniform() override { return u[cur++]; }
  } s;
  s.u = uniforms;
  s.cur = gamma;
  const WindowOut w = oracle_b(gamma, V, draft_logits, target_logits, tokens, tau,
                               crit_of(r, g, o, m), s, key, accepted, aprob);
  res[0] = w.k;
  res[1] = w.extra;
  res[2] = w.source;
  res[3] = w.key_count;
  res[4] = w.status;
  res[5] = w.evaluated;
  return w.status;
}

// ---- Oracle-B batch over fp32 logits: the CPU baseline (all host threads) ----
int ref_verify_batch_f32(int B, int gamma, int V, int stride, const float *draft,
                         const float *target, const int32_t *tokens, double tau, double r,
                         double g, double o, int m, const double *uniforms /*[B][2g+1]*/,
                         int nthreads, int32_t *k_out, int32_t *extra_out, int32_t *status_out) {
  if (nthreads < 1) nthreads = 1;
  const dsd::KeyCriteria c = crit_of(r, g, o, m);
  auto work = [&](int t) {
    std::vector<double> dl((size_t)gamma * V), tl((size_t)(gamma + 1) * V);
    for (int b = t; b < B; b += nthreads) {
      for (int rr = 0; rr < gamma; ++rr)
        for (int i = 0; i < V; ++i)
          dl[(size_t)rr * V + i] = draft[((size_t)b * gamma + rr) * stride + i];
      for (int rr = 0; rr <= gamma; ++rr)
        for (int i = 0; i < V; ++i)
          tl[(size_t)rr * V + i] = target[((size_t)b * (gamma + 1) + rr) * stride + i];
      struct Slots final : dsd::UniformStream {
        const double *u;
        int cur;
        double next_uniform() override { return u[cur++]; }
      } s;
      s.u = uniforms + (size_t)b * (2 * gamma + 1);
      s.cur = gamma;
      const WindowOut w = oracle_b(gamma, V, dl.data(), tl.data(), tokens + (size_t)b * gamma,
                                   tau, c, s, nullptr, nullptr, nullptr);
      k_out[b] = w.k;
      extra_out[b] = w.extra;
      status_out[b] = w.status;
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nthreads; ++t) th.emplace_back(work, t);
  work(0);
  for (auto &x : th) x.join();
  return 0;
}

// ---- generate with SeededStream (acceptance criterion 6) ----
int ref_generate_iid(const double *pd, const double *pt, int V, int gamma, double tau, double r,
                     double g, double o, int m, int max_new, uint64_t seed, int32_t *ks,
                     int max_rounds) {
  try {
    const dsd::TokenModel draft = dsd::TokenModel::categorical(dist(pd, V));
    const dsd::TokenModel target = dsd::TokenModel::categorical(dist(pt, V));
    dsd::SeededStream rng(seed);
    const dsd::GenerationResult gen = dsd::generate(
        draft, target, dsd::Context{}, max_new, dsd::VerifyParams{gamma, tau, crit_of(r, g, o, m)},
        rng);
    const int n = (int)gen.rounds.size();
    for (int i = 0; i < n && i < max_rounds; ++i) ks[i] = gen.rounds[(size_t)i].accepted_count;
    return n;
  } catch (...) {
    return -code_of(std::current_exception());
  }
}

// ---- temperature_scale (distribution.cpp:65-97) ----
int ref_temperature_scale(const double *p, int V, double T, double *out) {
  try {
    const dsd::Distribution d = dsd::temperature_scale(dist(p, V), T);
    std::memcpy(out, d.probs().data(), sizeof(double) * (size_t)V);
    return 0;
  } catch (...) {
    return -code_of(std::current_exception());
  }
}

// ---- exact enumeration (enumerate.cpp) for the GPU statistical checks ----
// Distribution of the first committed token and E[accepted] of one round,
// categorical-iid models.
int ref_enumerate_first(const double *pd, const double *pt, int V, int gamma, double tau,
                        double r, double g, double o, int m, double *out, double *expected_k) {
  try {
    const dsd::TokenModel draft = dsd::TokenModel::categorical(dist(pd, V));
    const dsd::TokenModel target = dsd::TokenModel::categorical(dist(pt, V));
    const dsd::VerifyParams params{gamma, tau, crit_of(r, g, o, m)};
    const dsd::SequenceDistribution d =
        dsd::enumerate_output_distribution(draft, target, dsd::Context{}, 1, params);
    for (int i = 0; i < V; ++i) out[i] = 0.0;
    for (const auto &kv : d) out[kv.first.at(0)] += kv.second;
    *expected_k = dsd::expected_accepted_count(draft, target, dsd::Context{}, params);
    return 0;
  } catch (...) {
    return -code_of(std::current_exception());
  }
}

// acceptance criterion 8 (acceptance.cpp:345-398) through the reference's own
// calibrate_thresholds: the winner (len, divergence, ratio, gap, overlap) and the
// grid log [64][6] (ratio, gap, overlap, len, divergence, feasible)
int ref_calibrate_c8(double budget, double *best, double *log, int cap) {
  try {
    using namespace dsd;
    const std::vector<ValidationItem> items = {
        ValidationItem{Context{}, TokenModel::categorical(Distribution({0.5, 0.5})),
                       TokenModel::categorical(Distribution({0.9, 0.1})), 2},
        ValidationItem{Context{},
                       TokenModel::categorical(Distribution({0.15, 0.2, 0.25, 0.2, 0.1, 0.1})),
                       TokenModel::categorical(Distribution({0.45, 0.3, 0.1, 0.08, 0.04, 0.03})),
                       2},
        ValidationItem{Context({0}),
                       TokenModel::markov({Distribution({0.6, 0.2, 0.2}),
                                           Distribution({0.25, 0.5, 0.25}),
                                           Distribution({0.2, 0.3, 0.5})},
                                          Distribution({0.4, 0.3, 0.3})),
                       TokenModel::markov({Distribution({0.8, 0.1, 0.1}),
                                           Distribution({0.1, 0.8, 0.1}),
                                           Distribution({0.05, 0.15, 0.8})},
                                          Distribution({0.5, 0.3, 0.2})),
                       2},
        ValidationItem{Context{}, TokenModel::categorical(Distribution({0.3, 0.3, 0.2, 0.2})),
                       TokenModel::categorical(Distribution({0.55, 0.25, 0.15, 0.05})), 2},
        ValidationItem{Context{}, TokenModel::categorical(Distribution({0.6, 0.25, 0.15})),
                       TokenModel::categorical(Distribution({0.6, 0.25, 0.15})), 2},
    };
    const CalibrationResult r =
        calibrate_thresholds(items, 0.5, budget, ThresholdGrid::defaults(), 3, 6);
    best[0] = r.avg_accepted_len;
    best[1] = r.divergence;
    best[2] = r.criteria.ratio_limit;
    best[3] = r.criteria.gap_limit;
    best[4] = r.criteria.overlap_floor;
    int n = 0;
    for (const GridPointEval &e : r.grid_log) {
      if (n >= cap) break;
      double *row = log + 6 * n++;
      row[0] = e.criteria.ratio_limit;
      row[1] = e.criteria.gap_limit;
      row[2] = e.criteria.overlap_floor;
      row[3] = e.avg_accepted_len;
      row[4] = e.divergence;
      row[5] = e.feasible ? 1.0 : 0.0;
    }
    return n;
  } catch (...) {
    return -1;
  }
}

}  // extern "C"
