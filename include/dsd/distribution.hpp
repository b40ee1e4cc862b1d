// Probability vectors of the drop-in API (reference:
// proj/include/dsd/distribution.hpp:28-68). fp64 entries, validated once at
// construction: size >= 2, finite, non-negative, sum within 1e-9 of one.
#pragma once

#include <cstddef>
#include <vector>

#include "dsd/rng.hpp"

namespace dsd {

class Distribution {
 public:
  static constexpr double kSumTolerance = 1e-9;
  explicit Distribution(std::vector<double> probs);  // throws InvariantError
  // Renormalised non-negative weights (throws InvariantError on zero mass).
  static Distribution from_weights(std::vector<double> weights);

  std::size_t size() const { return p_.size(); }
  double operator[](std::size_t i) const { return p_[i]; }
  const std::vector<double>& probs() const { return p_; }
  bool operator==(const Distribution& o) const { return p_ == o.p_; }

 private:
  struct Trusted {};
  Distribution(std::vector<double> p, Trusted) : p_(std::move(p)) {}
  std::vector<double> p_;
};

// T = 1 identity, T = 0 one-hot argmax (lowest id on ties), else p^(1/T)
// renormalised in log space (distribution.cpp:65-97).
Distribution temperature_scale(const Distribution& d, double temperature);
// Inverse CDF over ascending ids, one uniform (distribution.cpp:99-114).
int sample(const Distribution& d, UniformStream& rng);
int sample_with_uniform(const Distribution& d, double u);
double total_variation(const Distribution& a, const Distribution& b);

}  // namespace dsd
