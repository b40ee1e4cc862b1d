// Training-free threshold calibration on the device (calibrate.cpp:51-148):
// every (grid point, validation item) pair is one thread that evaluates the
// item exactly — expected_accepted_count (enumerate.cpp:154-181) and the total
// variation between the adaptive and the strict (tau = 0) output distributions
// over the item's horizon (enumerate_output_distribution :54-119,
// total_variation :183-203) — in fp64, with the reference's operation order:
// the forward dynamic program keeps one dense level of (committed sequence,
// window position) states and visits them in std::map order (sequences of
// one length compare lexicographically = numerically in base V, then the
// position), so every state accumulates its inflows in the reference's order.
// A second pass reduces each grid point over the items in item order.
//
// Model rows come from the host (next_distribution applied per context, so
// temperature and the model kind are already resolved): for an item of
// vocabulary V, rows[s] for s < V is the distribution after last token s and
// rows[V] the one after the prompt; the draft rows, then the target rows.
#include <cuda_runtime.h>

#include <cmath>

#include "dsdv/dsdv.h"

namespace dsdv {

namespace {

constexpr int kMaxV = 8;  // EnumerationGuard::kMaxVocab (enumerate.hpp:31)
constexpr double kCertain = 1e-12;

struct Row {
  double p[kMaxV];
};

__device__ double cross_entropy(const Row &d, int y) {  // verifier.cpp:112-117
  const double q = d.p[y];
  return q > 0.0 ? -log(q) : INFINITY;
}

// top_ids (verifier.cpp:40-51) as an ascending scan keeping the m best
__device__ void top_ids(const Row &d, int V, int m, int *out) {
  int n = 0;
  for (int i = 0; i < V; ++i) {
    const double v = d.p[i];
    if (n == m && !(v > d.p[out[m - 1]])) continue;
    int pos = n < m ? n : m - 1;
    while (pos > 0 && v > d.p[out[pos - 1]]) {
      out[pos] = out[pos - 1];
      --pos;
    }
    out[pos] = i;
    if (n < m) ++n;
  }
}

__device__ double norm_match(const Row &t, const Row &d, int V, int m) {  // :119-134
  int tt[kMaxV], td[kMaxV];
  top_ids(t, V, m, tt);
  top_ids(d, V, m, td);
  int shared = 0;
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b)
      if (td[a] == tt[b]) {
        ++shared;
        break;
      }
  return (double)shared / (double)m;
}

__device__ bool is_key(const Row &t, const Row &d, int V, int y, const dsdv_key_criteria &c) {
  const double h_draft = cross_entropy(d, y);  // verifier.cpp:136-159
  const double h_target = cross_entropy(t, y);
  const bool ratio = h_target < kCertain ? h_draft > 0.0 : (h_draft / h_target) > c.ratio_limit;
  const bool gap = fabs(t.p[y] - d.p[y]) > c.gap_limit;
  const int m = c.top_m < V ? c.top_m : V;
  const bool overlap = norm_match(t, d, V, m) < c.overlap_floor;
  return ratio || gap || overlap;
}

// soften (verifier.cpp:161-186); returns false on zero mass
__device__ bool soften(const Row &t, const Row &d, int V, double tau, Row &out) {
  if (tau == 0.0) {
    out = t;
    return true;
  }
  if (tau == 1.0) {
    out = d;
    return true;
  }
  bool equal = true;
  for (int i = 0; i < V && equal; ++i) equal = t.p[i] == d.p[i];
  if (equal) {
    out = t;
    return true;
  }
  double mass = 0.0;
  for (int i = 0; i < V; ++i) {
    out.p[i] = pow(t.p[i], 1.0 - tau) * pow(d.p[i], tau);
    mass += out.p[i];
  }
  if (mass <= 0.0) return false;
  double sum = 0.0;  // from_weights: its own sum, then divide (distribution.cpp:57-61)
  for (int i = 0; i < V; ++i) sum += out.p[i];
  for (int i = 0; i < V; ++i) out.p[i] /= sum;
  return true;
}

__device__ bool residual(const Row &eff, const Row &d, int V, Row &out) {  // :198-213
  double mass = 0.0;
  for (int i = 0; i < V; ++i) {
    const double x = eff.p[i] - d.p[i];
    out.p[i] = x > 0.0 ? x : 0.0;
    mass += out.p[i];
  }
  if (mass <= 0.0) return false;
  double sum = 0.0;
  for (int i = 0; i < V; ++i) sum += out.p[i];
  for (int i = 0; i < V; ++i) out.p[i] /= sum;
  return true;
}

// effective distribution and accept probability of drafted token y in context s
struct Step {
  bool ok;
  Row eff;
  double accept;
};

__device__ Step step_of(const Row &pd, const Row &pt, int V, int y, double tau,
                        const dsdv_key_criteria &c) {
  Step st;
  st.ok = true;
  const bool key = is_key(pt, pd, V, y, c);
  if (key)
    st.eff = pt;
  else
    st.ok = soften(pt, pd, V, tau, st.eff);
  st.accept = 0.0;
  if (!st.ok) return st;
  const double r = st.eff.p[y] / pd.p[y];  // accept_prob :188-196 (p_d(y) > 0 here)
  st.accept = r < 1.0 ? r : 1.0;
  if (st.accept > 1.0 - 1e-12) st.accept = 1.0;  // enumerate.cpp:92-95
  return st;
}

__device__ int ipow(int b, int e) {
  int r = 1;
  while (e-- > 0) r *= b;
  return r;
}

// forward DP of enumerate_output_distribution; fills dist[V^H] (sequences in
// lexicographic order). level/next: scratch of V^H * (gamma + 1) doubles each.
// Returns the DegenerateMixture / EmptyResidual status the reference would throw.
__device__ int enumerate(const Row *rd, const Row *rt, int V, int H, int gamma, double tau,
                          const dsdv_key_criteria &c, double *level, double *next, double *dist) {
  const int G1 = gamma + 1;
  int nseq = 1;  // sequences of the current length
  level[0] = 1.0;
  for (int i = 1; i < G1; ++i) level[i] = 0.0;
  for (int step = 0; step < H; ++step) {
    const int nnext = nseq * V;
    for (int i = 0; i < nnext * G1; ++i) next[i] = 0.0;
    for (int sq = 0; sq < nseq; ++sq) {
      const int s = step == 0 ? V : sq % V;  // context: the prompt, or the last token
      const Row &pd = rd[s];
      const Row &pt = rt[s];
      for (int pos = 0; pos < G1; ++pos) {
        const double prob = level[sq * G1 + pos];
        if (!(prob > 0.0)) continue;  // absent states (inflows are positive)
        if (pos == gamma) {
          for (int z = 0; z < V; ++z) {
            if (pt.p[z] <= 0.0) continue;
            next[(sq * V + z) * G1 + 0] += prob * pt.p[z];
          }
          continue;
        }
        for (int y = 0; y < V; ++y) {
          const double draft_mass = pd.p[y];
          if (draft_mass <= 0.0) continue;
          const Step st = step_of(pd, pt, V, y, tau, c);
          if (!st.ok) return DSDV_E_DEGENERATE_MIXTURE;
          if (st.accept > 0.0) next[(sq * V + y) * G1 + pos + 1] += prob * draft_mass * st.accept;
          if (st.accept < 1.0) {
            const double reject_mass = prob * draft_mass * (1.0 - st.accept);
            Row res;
            if (!residual(st.eff, pd, V, res)) return DSDV_E_EMPTY_RESIDUAL;
            for (int z = 0; z < V; ++z) {
              if (res.p[z] <= 0.0) continue;
              next[(sq * V + z) * G1 + 0] += reject_mass * res.p[z];
            }
          }
        }
      }
    }
    double *t = level;
    level = next;
    next = t;
    nseq = nnext;
  }
  for (int sq = 0; sq < nseq; ++sq) {
    double acc = 0.0;
    for (int pos = 0; pos < G1; ++pos) acc += level[sq * G1 + pos];
    dist[sq] = acc;
  }
  return DSDV_OK;
}

// expected_accepted_count (enumerate.cpp:154-181) with the sub-results of a
// context memoised: E depends on the prefix only through its last token
__device__ bool expected_count(const Row *rd, const Row *rt, int V, int gamma, double tau,
                               const dsdv_key_criteria &c, double *out) {
  double E[5][kMaxV + 1];  // [pos][context], gamma <= 4
  for (int s = 0; s <= V; ++s) E[gamma][s] = 0.0;
  for (int pos = gamma - 1; pos >= 0; --pos) {
    for (int s = 0; s <= V; ++s) {
      const Row &pd = rd[s];
      const Row &pt = rt[s];
      double expected = 0.0;
      for (int y = 0; y < V; ++y) {
        const double draft_mass = pd.p[y];
        if (draft_mass <= 0.0) continue;
        const Step st = step_of(pd, pt, V, y, tau, c);
        if (!st.ok) return false;
        if (st.accept <= 0.0) continue;
        expected += draft_mass * st.accept * (1.0 + E[pos + 1][y]);
      }
      E[pos][s] = expected;
    }
  }
  *out = E[0][V];
  return true;
}

__global__ void calib_kernel(const dsdv_calib_item *items, int n_items, const double *rows,
                             const dsdv_key_criteria *points, int n_points, double tau, int gamma,
                             double *scratch, size_t scratch_per_thread, double *len_out,
                             double *tv_out, int32_t *status) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_points * n_items) return;
  const int pi = t / n_items, ii = t - pi * n_items;
  const dsdv_calib_item it = items[ii];
  const int V = it.vocab;
  Row rd[kMaxV + 1], rt[kMaxV + 1];
  for (int s = 0; s <= V; ++s)
    for (int i = 0; i < V; ++i) {
      rd[s].p[i] = rows[it.rows_offset + (size_t)s * V + i];
      rt[s].p[i] = rows[it.rows_offset + (size_t)(V + 1 + s) * V + i];
    }
  const dsdv_key_criteria c = points[pi];
  double len = 0.0;
  int32_t st = DSDV_OK;
  if (!expected_count(rd, rt, V, gamma, tau, c, &len)) st = DSDV_E_DEGENERATE_MIXTURE;
  const int nseq = ipow(V, it.horizon);
  const size_t lvl = (size_t)nseq * (gamma + 1);
  double *base = scratch + (size_t)t * scratch_per_thread;
  double *a = base + 2 * lvl, *b = a + nseq;
  if (st == DSDV_OK) st = enumerate(rd, rt, V, it.horizon, gamma, tau, c, base, base + lvl, a);
  if (st == DSDV_OK) st = enumerate(rd, rt, V, it.horizon, gamma, 0.0, c, base, base + lvl, b);
  double l1 = 0.0;  // total_variation over the union of sequences, in order
  if (st == DSDV_OK)
    for (int q = 0; q < nseq; ++q) l1 += fabs(a[q] - b[q]);
  len_out[t] = len + 1.0;
  tv_out[t] = 0.5 * l1;
  status[t] = st;
}

// evaluate_point's means (calibrate.cpp:57-75): one thread per grid point,
// the items in order
__global__ void calib_reduce(const double *len, const double *tv, const int32_t *status,
                             int n_points, int n_items, double budget, dsdv_grid_eval *out) {
  const int pi = blockIdx.x * blockDim.x + threadIdx.x;
  if (pi >= n_points) return;
  double ls = 0.0, ts = 0.0;
  int32_t st = DSDV_OK;
  for (int i = 0; i < n_items; ++i) {
    ls += len[pi * n_items + i];
    ts += tv[pi * n_items + i];
    if (status[pi * n_items + i] != DSDV_OK && st == DSDV_OK) st = status[pi * n_items + i];
  }
  out[pi].avg_accepted_len = ls / (double)n_items;
  out[pi].divergence = ts / (double)n_items;
  out[pi].feasible = out[pi].divergence <= budget ? 1 : 0;
  out[pi].status = st;
}

}  // namespace

size_t calib_scratch_doubles(int max_vocab, int max_horizon, int gamma) {
  size_t nseq = 1;
  for (int h = 0; h < max_horizon; ++h) nseq *= (size_t)max_vocab;
  return 2 * nseq * (gamma + 1) + 2 * nseq;
}

cudaError_t launch_calibrate(const dsdv_calib_item *items, int n_items, const double *rows,
                             const dsdv_key_criteria *points, int n_points, double tau, int gamma,
                             double budget, double *scratch, size_t scratch_per_thread,
                             double *len, double *tv, int32_t *status, dsdv_grid_eval *out,
                             cudaStream_t stream) {
  const int n = n_points * n_items;
  calib_kernel<<<(n + 127) / 128, 128, 0, stream>>>(items, n_items, rows, points, n_points, tau,
                                                    gamma, scratch, scratch_per_thread, len, tv,
                                                    status);
  calib_reduce<<<(n_points + 127) / 128, 128, 0, stream>>>(len, tv, status, n_points, n_items,
                                                           budget, out);
  return cudaGetLastError();
}

}  // namespace dsdv
