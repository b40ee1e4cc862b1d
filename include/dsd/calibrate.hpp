// Training-free threshold calibration of the drop-in API (reference:
// proj/include/dsd/calibrate.hpp): the same types and entry point, with every
// grid point's exact evaluation (evaluate_point, calibrate.cpp:51-76) run on
// the device (dsdv_calibrate); the selection and the errors follow
// calibrate.cpp:78-147.
#pragma once

#include <string>
#include <utility>
#include <vector>

#if __has_include("dsd/enumerate.hpp")
#include "dsd/enumerate.hpp"  // the reference's enumerators, when on the include path
#endif
#include "dsd/error.hpp"
#include "dsd/token_model.hpp"
#include "dsd/verifier.hpp"

namespace dsd {

struct ValidationItem {
  Context prompt;
  TokenModel draft;
  TokenModel target;
  int horizon = 2;
};

struct ThresholdGrid {
  std::vector<double> ratio_limits;
  std::vector<double> gap_limits;
  std::vector<double> overlap_floors;
  static ThresholdGrid defaults();
  void validate() const;
  KeyCriteria strictest(int top_m) const;
};

struct GridPointEval {
  KeyCriteria criteria;
  double avg_accepted_len = 0.0;
  double divergence = 0.0;
  bool feasible = false;
};

struct CalibrationResult {
  KeyCriteria criteria;
  double avg_accepted_len = 0.0;
  double divergence = 0.0;
  std::vector<GridPointEval> grid_log;
};

struct InfeasibleBudgetError : Error {
  InfeasibleBudgetError(const std::string& message, GridPointEval strictest_point)
      : Error(message), strictest(std::move(strictest_point)) {}
  GridPointEval strictest;
};

CalibrationResult calibrate_thresholds(const std::vector<ValidationItem>& items, double tau,
                                       double budget, const ThresholdGrid& grid, int gamma,
                                       int top_m = 10);

}  // namespace dsd
