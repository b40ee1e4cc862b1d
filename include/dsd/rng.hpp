// Uniform-draw sources of the drop-in API (reference: proj/include/dsd/rng.hpp:25-57).
// Every stochastic step pulls from a caller-owned UniformStream, in the
// reference's consumption order, so scripted and seeded streams replay the
// reference's rounds draw for draw.
#pragma once

#include <cstdint>
#include <random>

namespace dsd {

class UniformStream {
 public:
  virtual ~UniformStream() = default;
  virtual double next_uniform() = 0;  // in [0, 1)
};

// std::mt19937_64 with the 53-bit mapping (x >> 11) * 2^-53 (rng.hpp:39).
class SeededStream final : public UniformStream {
 public:
  explicit SeededStream(std::uint64_t seed) : seed_(seed), engine_(seed) {}
  double next_uniform() override {
    const std::uint64_t x = engine_();
    return static_cast<double>(x >> 11) * (1.0 / 9007199254740992.0);
  }
  std::uint64_t seed() const { return seed_; }
  // Independent stream for a named purpose: SplitMix64 finaliser over
  // seed + golden-ratio * (tag + 1) (rng.hpp:46-52).
  SeededStream fork(std::uint64_t tag) const {
    std::uint64_t z = seed_ + 0x9e3779b97f4a7c15ULL * (tag + 1);
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return SeededStream(z);
  }

 private:
  std::uint64_t seed_;
  std::mt19937_64 engine_;
};

}  // namespace dsd
