// Drop-in verifier API (reference: proj/include/dsd/verifier.hpp:32-146).
//
// Same types, functions and error behaviour as the reference's dsd::
// verifier; the work runs on the B200 through the dsdv C-ABI
// (include/dsdv/dsdv.h):
//   * verify_round / generate: one dsdv_window_stats launch per round computes
//     every position's key flag and accept probability (fp64 rows); the host
//     walks the window with the caller's UniformStream in the reference's
//     consumption order (draft draws, then one accept draw per evaluated
//     position, then the extra draw) and the extra token comes from
//     dsdv_sample_extra (residual or bonus inverse CDF on the device);
//   * norm_match / is_key / soften / residual_distribution: device kernels
//     (the O(V log V) top-m sort and the O(V) mixtures of the reference);
//   * token_cross_entropy / accept_prob: O(1) reads of one entry.
// The device is the current CUDA device of the calling thread (dsd::gpu).
#pragma once

#include <optional>
#include <vector>

#include "dsd/distribution.hpp"
#include "dsd/rng.hpp"
#include "dsd/token_model.hpp"

namespace dsd {

struct KeyCriteria {
  double ratio_limit = 2.0;    // > 0, may be +inf
  double gap_limit = 0.2;      // [0, 1]
  double overlap_floor = 0.5;  // [0, 1]
  int top_m = 10;              // >= 1, clamped to the vocabulary at use
  void validate() const;
  static KeyCriteria none();   // nothing is key
};

struct DraftWindow {
  std::vector<int> tokens;
  std::vector<Distribution> draft_dists;
  std::size_t size() const { return tokens.size(); }
};

struct TokenDecision {
  int token = 0;
  bool is_key = false;
  double tau_used = 0.0;
  double accept_prob = 0.0;
  bool accepted = false;
  std::optional<int> replacement;  // set iff rejected
};

enum class ExtraSource { BonusFromTarget, ResidualResample };

struct VerificationResult {
  std::vector<TokenDecision> decisions;  // up to and including the first rejection
  int accepted_count = 0;
  int extra_token = 0;
  ExtraSource extra_source = ExtraSource::BonusFromTarget;
  int key_count() const;
  int tokens_committed() const { return accepted_count + 1; }
};

struct VerifyParams {
  int gamma = 8;
  double tau = 0.2;
  KeyCriteria criteria = {};
  void validate() const;
};

struct GenerationResult {
  std::vector<int> tokens;
  std::vector<VerificationResult> rounds;
};

DraftWindow draft_window(const TokenModel& draft, const Context& ctx, int gamma,
                         UniformStream& rng);
double token_cross_entropy(const Distribution& d, int token);
double norm_match(const Distribution& target, const Distribution& draft, int top_m);
bool is_key(const Distribution& target, const Distribution& draft, int token,
            const KeyCriteria& criteria);
Distribution soften(const Distribution& target, const Distribution& draft, double tau);
double accept_prob(const Distribution& effective, const Distribution& draft, int token);
Distribution residual_distribution(const Distribution& effective, const Distribution& draft);
VerificationResult verify_round(const TokenModel& draft, const TokenModel& target,
                                const Context& ctx, const VerifyParams& params,
                                UniformStream& rng);
GenerationResult generate(const TokenModel& draft, const TokenModel& target,
                          const Context& prompt, int max_new, const VerifyParams& params,
                          UniformStream& rng);

namespace gpu {
// CUDA device used by the calling thread's verifier engine (default: the
// thread's current device). Each host thread owns its own dsdv context and
// stream, so concurrent calls on distinct UniformStreams are safe, as in the
// reference (commands.cpp:175-203).
void set_device(int device);
// Kernel launches issued by the calling thread's engine (evidence for tests).
unsigned long long launch_count();
}  // namespace gpu

}  // namespace dsd
