// dsd::calibrate_thresholds of the drop-in API (include/dsd/calibrate.hpp):
// calibrate.cpp:25-147 with every grid point evaluated on the device
// (dsdv_calibrate: exact enumerations per (point, item), fp64, the
// reference's operation order). Grid walk, validation messages, selection and
// InfeasibleBudgetError follow the reference.
#include <algorithm>
#include <string>
#include <tuple>
#include <vector>

#include "dsd/calibrate.hpp"
#include "dsdv/dsdv.h"

namespace dsd {

namespace gpu {
dsdv_ctx *context();  // the calling thread's engine (dsd_api.cpp)
}

ThresholdGrid ThresholdGrid::defaults() {
  ThresholdGrid g;
  g.ratio_limits = {1.2, 1.5, 2.0, 3.0};
  g.gap_limits = {0.05, 0.1, 0.2, 0.4};
  g.overlap_floors = {0.1, 0.3, 0.5, 0.8};
  return g;
}

void ThresholdGrid::validate() const {
  if (ratio_limits.empty() || gap_limits.empty() || overlap_floors.empty())
    throw InvariantError("threshold grid must be nonempty on every axis");
}

KeyCriteria ThresholdGrid::strictest(int top_m) const {
  validate();
  KeyCriteria c;
  c.ratio_limit = *std::min_element(ratio_limits.begin(), ratio_limits.end());
  c.gap_limit = *std::min_element(gap_limits.begin(), gap_limits.end());
  c.overlap_floor = *std::max_element(overlap_floors.begin(), overlap_floors.end());
  c.top_m = top_m;
  return c;
}

namespace {

// EnumerationGuard (enumerate.hpp:30-34, enumerate.cpp:29-42)
void check_guard(const TokenModel &draft, const TokenModel &target, int horizon, int gamma) {
  if (draft.vocab_size() != target.vocab_size())
    throw InvariantError("draft and target models must share a vocabulary");
  if (draft.vocab_size() > 8 || horizon < 1 || horizon > 4 || gamma > 4)
    throw EnumerationTooLargeError(
        "enumeration guard exceeded: need vocab <= 8, 1 <= horizon <= 4, gamma <= 4");
}

void append_rows(std::vector<double> &rows, const TokenModel &m, const Context &prompt) {
  const int V = static_cast<int>(m.vocab_size());
  for (int s = 0; s <= V; ++s) {
    const Distribution d = s < V ? next_distribution(m, Context({s})) : next_distribution(m, prompt);
    rows.insert(rows.end(), d.probs().begin(), d.probs().end());
  }
}

}  // namespace

CalibrationResult calibrate_thresholds(const std::vector<ValidationItem> &items, double tau,
                                       double budget, const ThresholdGrid &grid, int gamma,
                                       int top_m) {
  if (items.empty()) throw InvariantError("calibration needs at least one validation item");
  if (!(budget > 0.0 && budget < 1.0))
    throw InvariantError("calibration budget must lie in (0, 1), got " + std::to_string(budget));
  grid.validate();
  std::vector<double> ratios = grid.ratio_limits, gaps = grid.gap_limits,
                      overlaps = grid.overlap_floors;
  std::sort(ratios.begin(), ratios.end());
  std::sort(gaps.begin(), gaps.end());
  std::sort(overlaps.begin(), overlaps.end());
  std::vector<KeyCriteria> crit;
  for (double ratio : ratios)
    for (double gap : gaps)
      for (double overlap : overlaps) {
        KeyCriteria c{ratio, gap, overlap, top_m};
        c.validate();
        crit.push_back(c);
      }
  // evaluate_point's parameter checks (VerifyParams::validate, check_guard)
  VerifyParams{gamma, tau, crit.front()}.validate();
  std::vector<dsdv_calib_item> citems;
  std::vector<double> rows;
  for (const ValidationItem &it : items) {
    check_guard(it.draft, it.target, it.horizon, gamma);
    for (int id : it.prompt.tokens)
      if (id < 0 || static_cast<size_t>(id) >= it.draft.vocab_size())
        throw InvalidContextError("context token id " + std::to_string(id) +
                                  " outside vocabulary of size " +
                                  std::to_string(it.draft.vocab_size()));
    dsdv_calib_item ci;
    ci.vocab = static_cast<int32_t>(it.draft.vocab_size());
    ci.horizon = it.horizon;
    ci.rows_offset = static_cast<int64_t>(rows.size());
    append_rows(rows, it.draft, it.prompt);
    append_rows(rows, it.target, it.prompt);
    citems.push_back(ci);
  }
  std::vector<dsdv_key_criteria> pts;
  for (const KeyCriteria &c : crit)
    pts.push_back(dsdv_key_criteria{c.ratio_limit, c.gap_limit, c.overlap_floor, c.top_m});
  std::vector<dsdv_grid_eval> ev(pts.size());
  dsdv_ctx *ctx = gpu::context();
  if (dsdv_calibrate(ctx, citems.data(), static_cast<int32_t>(citems.size()), rows.data(),
                     static_cast<int64_t>(rows.size()), pts.data(),
                     static_cast<int32_t>(pts.size()), tau, gamma, budget, ev.data()) != DSDV_OK)
    throw DeviceError(std::string("dsdv: ") + dsdv_last_error(ctx));

  CalibrationResult result;
  for (size_t i = 0; i < ev.size(); ++i) {
    if (ev[i].status == DSDV_E_DEGENERATE_MIXTURE)
      throw DegenerateMixtureError(
          "softened distribution has zero mass: target and draft supports are disjoint");
    if (ev[i].status == DSDV_E_EMPTY_RESIDUAL)
      throw EmptyResidualError("residual is empty: effective and draft distributions match");
    GridPointEval g;
    g.criteria = crit[i];
    g.avg_accepted_len = ev[i].avg_accepted_len;
    g.divergence = ev[i].divergence;
    g.feasible = ev[i].feasible != 0;
    result.grid_log.push_back(g);
  }
  const GridPointEval *best = nullptr;
  const auto key = [](const GridPointEval &e) {
    return std::make_tuple(-e.avg_accepted_len, e.divergence, e.criteria.ratio_limit,
                           e.criteria.gap_limit, e.criteria.overlap_floor);
  };
  for (const GridPointEval &e : result.grid_log) {
    if (!e.feasible) continue;
    if (best == nullptr || key(e) < key(*best)) best = &e;
  }
  if (best == nullptr) {
    const KeyCriteria s = grid.strictest(top_m);
    GridPointEval se;
    for (const GridPointEval &e : result.grid_log)
      if (e.criteria.ratio_limit == s.ratio_limit && e.criteria.gap_limit == s.gap_limit &&
          e.criteria.overlap_floor == s.overlap_floor) {
        se = e;
        break;
      }
    throw InfeasibleBudgetError("no grid point meets the divergence budget " +
                                    std::to_string(budget) +
                                    "; strictest point diverges by " +
                                    std::to_string(se.divergence),
                                se);
  }
  result.criteria = best->criteria;
  result.avg_accepted_len = best->avg_accepted_len;
  result.divergence = best->divergence;
  return result;
}

}  // namespace dsd
