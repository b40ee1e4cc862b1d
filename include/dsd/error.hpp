// Error taxonomy of the drop-in verifier API. Same class names and
// hierarchy as the reference's dsd::Error family (proj/include/dsd/error.hpp:24-71),
// so callers' catch clauses keep working; C-ABI status codes (dsdv.h) map
// onto them in dsd_api.cpp (throw_status).
#pragma once

#include <stdexcept>
#include <string>

namespace dsd {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// bad parameter, token id out of range, non-stochastic vector
struct InvariantError : Error {
  using Error::Error;
};
// context token outside a model's vocabulary
struct InvalidContextError : Error {
  using Error::Error;
};
// soften(): disjoint supports at an interior tau
struct DegenerateMixtureError : Error {
  using Error::Error;
};
// accept_prob(): the drafted token has no draft probability
struct DraftingContractError : Error {
  using Error::Error;
};
// residual_distribution(): max(0, p_eff - p_d) has no mass
struct EmptyResidualError : Error {
  using Error::Error;
};
// exact enumeration beyond the tractability guard (enumerate.cpp:35)
struct EnumerationTooLargeError : Error {
  using Error::Error;
};
// two simulation reports over different token counts (netsim.cpp:206)
struct IncomparableReportsError : Error {
  using Error::Error;
};
// a CSV / report file could not be written (metrics.cpp:150)
struct WriteError : Error {
  using Error::Error;
};
// the GPU runtime failed (no counterpart in the reference: its path is host-only)
struct DeviceError : Error {
  using Error::Error;
};

}  // namespace dsd
