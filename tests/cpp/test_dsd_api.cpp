// C++ tests of the drop-in dsd:: API (include/dsd/) running on the GPU.
//
//   test_dsd_api kat        known answers and properties of the reference's
//                           proj/tests/test_verifier.cpp, acceptance criterion 6
//                           (acceptance.cpp:257-288, test_output.txt:50) and the
//                           SURVEY.md §8(c) survey-time goldens
//   test_dsd_api gen G TAU SEED MAX_NEW RATIO GAP OVERLAP TOP_M
//                           prints the accepted count of every round of
//                           generate() on the default divergent pair
//                           (compared with oracle/_ref by tests/test_cpp_api.py)
//   test_dsd_api calib B   acceptance criterion 8's calibration (acceptance.cpp:345-398)
//                           at budget B on the device: the winner, then the grid log
//   test_dsd_api rows FILE  one (draft, target) probability-row pair at any
//                           vocabulary and top_m: prints norm_match, is_key and
//                           the accepted counts of generate() with categorical
//                           models, then the mean ms per round
//                           (tests/test_cpp_api.py, scripts/dropin_timing.py)
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <limits>
#include <string>
#include <vector>

#include "dsd/calibrate.hpp"
#include "dsd/error.hpp"
#include "dsd/verifier.hpp"

using namespace dsd;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                         \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(c)) {                                                          \
      ++g_fail;                                                          \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #c); \
    }                                                                    \
  } while (0)
template <class E>
static bool throws_as(const std::function<void()> &f) {
  try {
    f();
  } catch (const E &) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}
#define CHECK_THROWS_AS(expr, E) CHECK(throws_as<E>([&] { (void)(expr); }))

static const double kInf = std::numeric_limits<double>::infinity();
// default divergent pair (support/generators.hpp:77-85)
static TokenModel divergent_draft() {
  return TokenModel::categorical(Distribution({0.15, 0.2, 0.25, 0.2, 0.1, 0.1}));
}
static TokenModel divergent_target() {
  return TokenModel::categorical(Distribution({0.45, 0.3, 0.1, 0.08, 0.04, 0.03}));
}
static TokenModel chain(int V) {  // token i -> (i + 1) mod V
  std::vector<Distribution> rows;
  for (int i = 0; i < V; ++i) {
    std::vector<double> r(V, 0.0);
    r[(i + 1) % V] = 1.0;
    rows.emplace_back(r);
  }
  std::vector<double> init(V, 0.0);
  init[0] = 1.0;
  return TokenModel::markov(rows, Distribution(init));
}
static Distribution random_dist(SeededStream &s, int V) {
  std::vector<double> w(V);
  for (double &x : w) x = 0.05 + s.next_uniform();
  return Distribution::from_weights(w);
}
static TokenModel random_markov(SeededStream &s, int V) {
  std::vector<Distribution> rows;
  for (int i = 0; i < V; ++i) rows.push_back(random_dist(s, V));
  return TokenModel::markov(rows, random_dist(s, V));
}
struct Scripted : UniformStream {
  std::vector<double> u;
  size_t i = 0;
  explicit Scripted(std::vector<double> v) : u(std::move(v)) {}
  double next_uniform() override { return u.at(i++); }
};

static void kat_primitives() {
  // token_cross_entropy (test_verifier.cpp:80-87)
  CHECK(token_cross_entropy(Distribution({1.0, 0.0}), 0) == 0.0);
  const double e = std::exp(-1.0);
  CHECK(std::abs(token_cross_entropy(Distribution({e, 1 - e}), 0) - 1.0) <= 1e-12);
  CHECK(std::isinf(token_cross_entropy(Distribution({1.0, 0.0}), 1)));
  CHECK_THROWS_AS(token_cross_entropy(Distribution({1.0, 0.0}), 2), InvariantError);
  // norm_match on the device (:89-103)
  const Distribution p({0.5, 0.3, 0.1, 0.1});
  CHECK(norm_match(p, p, 2) == 1.0);
  CHECK(norm_match(p, p, 4) == 1.0);
  CHECK(norm_match(Distribution({0.4, 0.4, 0.1, 0.1}), Distribution({0.1, 0.1, 0.4, 0.4}), 2) == 0.0);
  CHECK(norm_match(Distribution({0.5, 0.3, 0.1, 0.1}), Distribution({0.05, 0.5, 0.4, 0.05}), 2) == 0.5);
  CHECK(norm_match(Distribution({0.25, 0.25, 0.25, 0.25}), Distribution({0.25, 0.25, 0.25, 0.25}), 2) == 1.0);
  CHECK_THROWS_AS(norm_match(p, p, 5), InvariantError);
  // is_key clauses on the device (:105-137)
  const Distribution q({0.7, 0.3});
  CHECK(!is_key(q, q, 0, KeyCriteria{1.0, 0.5, 0.5, 2}));
  CHECK(is_key(q, q, 0, KeyCriteria{0.99, 1.0, 0.0, 2}));
  CHECK(is_key(Distribution({0.9, 0.1}), Distribution({0.3, 0.7}), 0, KeyCriteria{kInf, 0.5, 0.0, 2}));
  CHECK(!is_key(Distribution({0.9, 0.1}), Distribution({0.3, 0.7}), 0, KeyCriteria{kInf, 0.65, 0.0, 2}));
  CHECK(is_key(Distribution({0.9, 0.1}), Distribution({0.5, 0.5}), 0, KeyCriteria{2.0, 1.0, 0.0, 2}));
  CHECK(is_key(Distribution({0.9, 0.1}), Distribution({0.1, 0.9}), 1, KeyCriteria{kInf, 1.0, 0.5, 1}));
  CHECK(!is_key(q, q, 0, KeyCriteria{kInf, 1.0, 0.0, 1}));
  CHECK(is_key(Distribution({1.0, 0.0}), Distribution({0.9, 0.1}), 0, KeyCriteria{kInf, 1.0, 0.0, 2}));
  CHECK(!is_key(Distribution({1.0, 0.0}), Distribution({1.0, 0.0}), 0, KeyCriteria{kInf, 1.0, 0.0, 2}));
  CHECK_THROWS_AS(is_key(q, q, 0, KeyCriteria{0.0, 0.5, 0.5, 2}), InvariantError);
  // soften (:170-191): endpoints bit for bit, geometric interior on the device
  const Distribution t({0.9, 0.1}), d({0.5, 0.5});
  CHECK(soften(t, d, 0.0) == t);
  CHECK(soften(t, d, 1.0) == d);
  const Distribution m = soften(t, d, 0.5);
  CHECK(std::abs(m[0] - 0.75) <= 1e-12 && std::abs(m[1] - 0.25) <= 1e-12);
  CHECK_THROWS_AS(soften(Distribution({1.0, 0.0}), Distribution({0.0, 1.0}), 0.5),
                  DegenerateMixtureError);
  CHECK(soften(Distribution({1.0, 0.0}), Distribution({0.0, 1.0}), 0.0) == Distribution({1.0, 0.0}));
  // log of the softened ratio is affine in tau (:193-208)
  {
    const Distribution a({0.6, 0.3, 0.1}), b({0.2, 0.3, 0.5});
    for (double tau : {0.1, 0.4, 0.7}) {
      const Distribution s = soften(a, b, tau);
      const double lhs = std::log(s[0] / s[2]);
      const double rhs = (1 - tau) * std::log(a[0] / a[2]) + tau * std::log(b[0] / b[2]);
      CHECK(std::abs(lhs - rhs) <= 1e-9);
    }
  }
  // accept_prob and residual (:210-231)
  CHECK(accept_prob(Distribution({0.9, 0.1}), d, 0) == 1.0);
  CHECK(std::abs(accept_prob(Distribution({0.1, 0.9}), d, 0) - 0.2) <= 1e-12);
  CHECK(accept_prob(d, d, 1) == 1.0);
  CHECK_THROWS_AS(accept_prob(d, Distribution({1.0, 0.0}), 1), DraftingContractError);
  CHECK(residual_distribution(Distribution({0.9, 0.1}), d).probs() == std::vector<double>({1.0, 0.0}));
  CHECK(residual_distribution(Distribution({0.2, 0.3, 0.5}), Distribution({0.5, 0.3, 0.2})).probs() ==
        std::vector<double>({0.0, 0.0, 1.0}));
  CHECK(residual_distribution(Distribution({1.0, 0.0}), d).probs() == std::vector<double>({1.0, 0.0}));
  CHECK_THROWS_AS(residual_distribution(d, d), EmptyResidualError);
  // inverse CDF boundary goes up (test_distribution.cpp:96-109)
  CHECK(sample_with_uniform(d, 0.3) == 0);
  CHECK(sample_with_uniform(d, 0.5) == 1);
  CHECK(sample_with_uniform(Distribution({0.0, 1.0, 0.0}), 0.7) == 1);
}

static void kat_rounds() {
  // draft_window (:50-63)
  {
    SeededStream rng(1);
    CHECK(draft_window(chain(8), Context({0}), 3, rng).tokens == std::vector<int>({1, 2, 3}));
    Scripted s({0.3, 0.7});
    CHECK(draft_window(TokenModel::categorical(Distribution({0.5, 0.5})), Context{}, 2, s).tokens ==
          std::vector<int>({0, 1}));
    CHECK(s.i == 2);
  }
  // identical models accept the whole window (:233-243)
  {
    SeededStream meta(3);
    for (int trial = 0; trial < 10; ++trial) {
      const TokenModel m = random_markov(meta, 4);
      SeededStream rng(50 + trial);
      const VerificationResult r = verify_round(m, m, Context{}, VerifyParams{3, 0.0, KeyCriteria::none()}, rng);
      CHECK(r.accepted_count == 3);
      CHECK(r.extra_source == ExtraSource::BonusFromTarget);
    }
  }
  // tau = 1 with no key tokens accepts everything (:245-254)
  {
    SeededStream rng(77);
    for (int trial = 0; trial < 100; ++trial)
      CHECK(verify_round(divergent_draft(), divergent_target(), Context{},
                         VerifyParams{4, 1.0, KeyCriteria::none()}, rng)
                .accepted_count == 4);
  }
  // P(first committed token = 0) = 0.9 (:256-272), 20000 rounds
  {
    const TokenModel dr = TokenModel::categorical(Distribution({0.5, 0.5}));
    const TokenModel tg = TokenModel::categorical(Distribution({0.9, 0.1}));
    SeededStream rng(2718);
    const int n = 20000;
    int zeros = 0;
    for (int i = 0; i < n; ++i) {
      const VerificationResult r = verify_round(dr, tg, Context{}, VerifyParams{1, 0.0, KeyCriteria::none()}, rng);
      zeros += (r.accepted_count > 0 ? r.decisions.front().token : r.extra_token) == 0;
    }
    CHECK(std::abs((double)zeros / n - 0.9) <= 0.9 * 0.011);
  }
  // every round commits between 1 and gamma + 1 tokens (:274-304)
  {
    SeededStream meta(23);
    for (int trial = 0; trial < 50; ++trial) {
      const int V = 2 + trial % 4;
      const TokenModel dr = random_markov(meta, V), tg = random_markov(meta, V);
      const int gamma = 1 + trial % 4;
      SeededStream rng(900 + trial);
      const VerificationResult r = verify_round(dr, tg, Context{}, VerifyParams{gamma, (trial % 5) * 0.25, KeyCriteria{}}, rng);
      CHECK(r.tokens_committed() >= 1 && r.tokens_committed() <= gamma + 1);
      int acc = 0;
      bool rej = false;
      for (const TokenDecision &x : r.decisions) {
        CHECK(!rej);
        if (x.accepted) {
          ++acc;
          CHECK(!x.replacement.has_value());
        } else {
          rej = true;
          CHECK(x.replacement.has_value());
        }
        if (x.is_key) CHECK(x.tau_used == 0.0);
      }
      CHECK(acc == r.accepted_count);
      CHECK(rej == (r.extra_source == ExtraSource::ResidualResample));
    }
  }
  // generate on a deterministic chain, and truncation (:326-347)
  {
    SeededStream rng(1);
    const GenerationResult g = generate(chain(8), chain(8), Context({0}), 5, VerifyParams{2, 0.0, KeyCriteria::none()}, rng);
    CHECK(g.tokens == std::vector<int>({1, 2, 3, 4, 5}));
    CHECK(g.rounds.size() == 2);
    SeededStream r2(88);
    const GenerationResult h = generate(divergent_draft(), divergent_target(), Context{}, 17, VerifyParams{1, 0.0, KeyCriteria{}}, r2);
    CHECK(h.tokens.size() == 17);
  }
  // validation (:349-360)
  {
    const TokenModel m = TokenModel::categorical(Distribution({0.5, 0.5}));
    SeededStream rng(4);
    CHECK_THROWS_AS(verify_round(m, m, Context{}, VerifyParams{0, 0.0, KeyCriteria{}}, rng), InvariantError);
    CHECK_THROWS_AS(verify_round(m, m, Context{}, VerifyParams{2, 1.5, KeyCriteria{}}, rng), InvariantError);
    CHECK_THROWS_AS(generate(m, m, Context{}, 0, VerifyParams{}, rng), InvariantError);
  }
  // survey-time goldens: gamma 4, tau 0.2, criteria {2, 0.2, 0.5, 6}
  {
    SeededStream rng(1);
    const VerifyParams vp{4, 0.2, KeyCriteria{2.0, 0.2, 0.5, 6}};
    const int want[5][4] = {{4, 1, 0, 3}, {4, 2, 0, 1}, {4, 0, 0, 0}, {1, 0, 1, 1}, {2, 0, 1, 0}};
    for (int i = 0; i < 5; ++i) {
      const VerificationResult r = verify_round(divergent_draft(), divergent_target(), Context{}, vp, rng);
      CHECK(r.accepted_count == want[i][0]);
      CHECK(r.extra_token == want[i][1]);
      CHECK((r.extra_source == ExtraSource::ResidualResample) == (want[i][2] == 1));
      CHECK(r.key_count() == want[i][3]);
    }
  }
}

// acceptance criterion 6: mean committed length per tau over seeds 1..12
static void criterion6() {
  const double want[5] = {2.50364, 3.02053, 3.81058, 5.06016, 6.77729};
  const double taus[5] = {0.0, 0.2, 0.4, 0.6, 0.8};
  for (int i = 0; i < 5; ++i) {
    long total = 0, rounds = 0;
    for (int seed = 1; seed <= 12; ++seed) {
      SeededStream rng(seed);
      const GenerationResult g = generate(divergent_draft(), divergent_target(), Context{}, 256,
                                          VerifyParams{8, taus[i], KeyCriteria{2.0, 0.2, 0.5, 6}}, rng);
      for (const VerificationResult &r : g.rounds) total += r.tokens_committed();
      rounds += (long)g.rounds.size();
    }
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.6g", (double)total / rounds);
    std::printf("criterion6 tau=%.1f mean=%s want=%.6g\n", taus[i], buf, want[i]);
    CHECK(std::strtod(buf, nullptr) == want[i]);
  }
}

int main(int argc, char **argv) {
  const std::string mode = argc > 1 ? argv[1] : "kat";
  try {
    if (mode == "gen" && argc == 10) {
      SeededStream rng(std::strtoull(argv[4], nullptr, 10));
      const VerifyParams vp{std::atoi(argv[2]), std::atof(argv[3]),
                            KeyCriteria{std::atof(argv[6]), std::atof(argv[7]), std::atof(argv[8]),
                                        std::atoi(argv[9])}};
      const GenerationResult g = generate(divergent_draft(), divergent_target(), Context{},
                                          std::atoi(argv[5]), vp, rng);
      for (const VerificationResult &r : g.rounds) std::printf("%d ", r.accepted_count);
      std::printf("\n");
      return 0;
    }
    if (mode == "calib" && argc == 3) {
      // the 5-item set of acceptance.cpp:346-368
      const std::vector<ValidationItem> items = {
          ValidationItem{Context{}, TokenModel::categorical(Distribution({0.5, 0.5})),
                         TokenModel::categorical(Distribution({0.9, 0.1})), 2},
          ValidationItem{Context{}, divergent_draft(), divergent_target(), 2},
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
          calibrate_thresholds(items, 0.5, std::atof(argv[2]), ThresholdGrid::defaults(), 3, 6);
      std::printf("%.17g %.17g %.17g %.17g %.17g\n", r.avg_accepted_len, r.divergence,
                  r.criteria.ratio_limit, r.criteria.gap_limit, r.criteria.overlap_floor);
      for (const GridPointEval &e : r.grid_log)
        std::printf("%.17g %.17g %.17g %.17g %.17g %d\n", e.criteria.ratio_limit,
                    e.criteria.gap_limit, e.criteria.overlap_floor, e.avg_accepted_len,
                    e.divergence, e.feasible ? 1 : 0);
      return 0;
    }
    if (mode == "rows" && argc == 3) {
      FILE *f = std::fopen(argv[2], "rb");
      if (!f) return 3;
      int32_t V, gamma, top_m, max_new, y;
      double tau, ratio, gap, overlap;
      uint64_t seed;
      bool ok = std::fread(&V, 4, 1, f) == 1 && std::fread(&gamma, 4, 1, f) == 1 &&
                std::fread(&tau, 8, 1, f) == 1 && std::fread(&ratio, 8, 1, f) == 1 &&
                std::fread(&gap, 8, 1, f) == 1 && std::fread(&overlap, 8, 1, f) == 1 &&
                std::fread(&top_m, 4, 1, f) == 1 && std::fread(&seed, 8, 1, f) == 1 &&
                std::fread(&max_new, 4, 1, f) == 1 && std::fread(&y, 4, 1, f) == 1;
      std::vector<double> pd(V), pt(V);
      ok = ok && std::fread(pd.data(), 8, V, f) == (size_t)V &&
           std::fread(pt.data(), 8, V, f) == (size_t)V;
      std::fclose(f);
      if (!ok) return 3;
      const Distribution dd(pd), dt(pt);
      const KeyCriteria c{ratio, gap, overlap, top_m};
      std::printf("%.17g\n", norm_match(dt, dd, std::min<int>(top_m, V)));
      std::printf("%d\n", is_key(dt, dd, y, c) ? 1 : 0);
      const VerifyParams vp{gamma, tau, c};
      {  // warm-up: device context, arenas, pinned staging
        SeededStream warm(seed + 1);
        (void)generate(TokenModel::categorical(dd), TokenModel::categorical(dt), Context{}, 1, vp,
                       warm);
      }
      SeededStream rng(seed);
      const auto t0 = std::chrono::steady_clock::now();
      const GenerationResult g = generate(TokenModel::categorical(dd), TokenModel::categorical(dt),
                                          Context{}, max_new, vp, rng);
      const auto t1 = std::chrono::steady_clock::now();
      for (const VerificationResult &r : g.rounds) std::printf("%d ", r.accepted_count);
      std::printf("\n%.6f\n",
                  std::chrono::duration<double, std::milli>(t1 - t0).count() / g.rounds.size());
      return 0;
    }
    kat_primitives();
    kat_rounds();
    criterion6();
  } catch (const std::exception &e) {
    std::fprintf(stderr, "uncaught: %s\n", e.what());
    return 2;
  }
  std::printf("%d checks, %d failed, %llu launches\n", g_checks, g_fail, gpu::launch_count());
  return g_fail ? 1 : 0;
}
