// Drop-in dsd:: verifier API over the dsdv C-ABI (include/dsd/*.hpp).
//
// Host side of the reference-facing boundary: the reference's callers
// (generate <- execute_run, commands.cpp:51-53; the enumerators and the sweep
// workers) link this library instead of proj/src/verifier.cpp and keep their
// types, call order, uniform consumption and exception classes. Every
// O(V)-and-up step of a round runs on the device:
//   round  = host draft_window (caller's stream) -> dsdv_window_stats (all
//            positions: key flags, accept probabilities, fp64 rows) -> host
//            walk with the caller's stream -> dsdv_sample_extra (residual or
//            bonus inverse CDF);
//   norm_match / is_key -> dsdv_window_stats on a one-position window;
//   soften / residual_distribution -> dsdv_mix_rows.
// There is no host fallback: without a usable device every call throws
// dsd::DeviceError.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "dsd/error.hpp"
#include "dsd/verifier.hpp"
#include "dsdv/dsdv.h"

namespace dsd {

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr int kRecWords = DSDV_RECORD_WORDS;
constexpr int kRecFlagsWord = 5;  // kind | error << 8 | key << 16 (csrc/common.cuh)

std::string num(double v) { return std::to_string(v); }
std::string num(long long v) { return std::to_string(v); }

// ---- per-thread device engine -------------------------------------------
struct Engine {
  dsdv_ctx *ctx = nullptr;
  cudaStream_t stream = nullptr;
  int device = -1;
  int wanted = -1;  // gpu::set_device
  // device arena (grown on demand) and pinned staging
  void *dbuf = nullptr;
  size_t dcap = 0;
  void *hbuf = nullptr;
  size_t hcap = 0;

  ~Engine() {
    if (ctx) dsdv_destroy(ctx);
    if (stream) cudaStreamDestroy(stream);
    if (dbuf) cudaFree(dbuf);
    if (hbuf) cudaFreeHost(hbuf);
  }

  [[noreturn]] void cuda_fail(cudaError_t e, const char *what) {
    throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
  }

  void ready() {
    int dev = wanted;
    if (dev < 0) {
      cudaError_t e = cudaGetDevice(&dev);
      if (e != cudaSuccess) cuda_fail(e, "dsd::gpu: no CUDA device");
    }
    if (ctx && dev == device) return;
    if (ctx) {
      dsdv_destroy(ctx);
      ctx = nullptr;
      cudaStreamDestroy(stream);
      cudaFree(dbuf);
      dbuf = nullptr;
      dcap = 0;
    }
    cudaError_t e = cudaSetDevice(dev);
    if (e != cudaSuccess) cuda_fail(e, "dsd::gpu: cudaSetDevice");
    if (dsdv_create(dev, &ctx) != DSDV_OK) {
      const std::string m = dsdv_last_error(ctx);
      ctx = nullptr;
      throw DeviceError("dsd::gpu: " + m);
    }
    e = cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) cuda_fail(e, "dsd::gpu: cudaStreamCreate");
    device = dev;
  }

  void *dev_arena(size_t bytes) {
    if (bytes > dcap) {
      if (dbuf) cudaFree(dbuf);
      dbuf = nullptr;
      const size_t cap = std::max(bytes, dcap * 2);
      cudaError_t e = cudaMalloc(&dbuf, cap);
      if (e != cudaSuccess) cuda_fail(e, "dsd::gpu: cudaMalloc");
      dcap = cap;
    }
    return dbuf;
  }
  void *host_arena(size_t bytes) {
    if (bytes > hcap) {
      if (hbuf) cudaFreeHost(hbuf);
      hbuf = nullptr;
      const size_t cap = std::max(bytes, hcap * 2);
      cudaError_t e = cudaMallocHost(&hbuf, cap);
      if (e != cudaSuccess) cuda_fail(e, "dsd::gpu: cudaMallocHost");
      hcap = cap;
    }
    return hbuf;
  }
  void check(dsdv_status st) {
    if (st != DSDV_OK) throw DeviceError(std::string("dsdv: ") + dsdv_last_error(ctx));
  }
  void sync() {
    cudaError_t e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) cuda_fail(e, "dsd::gpu: stream");
  }
};

Engine &raw_engine() {
  thread_local Engine eng;
  return eng;
}
Engine &engine() {
  Engine &eng = raw_engine();
  eng.ready();
  return eng;
}

// Bump allocator over one arena.
struct Carve {
  char *base;
  size_t off = 0;
  explicit Carve(void *b) : base(static_cast<char *>(b)) {}
  template <class T>
  T *take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T *p = reinterpret_cast<T *>(base + off);
    off += n * sizeof(T);
    return p;
  }
};
template <class T>
size_t carve_size(size_t n) {
  return ((n * sizeof(T)) + 255) & ~size_t(255);
}

void check_token(const Distribution &d, int token, const char *what) {
  if (token < 0 || static_cast<size_t>(token) >= d.size())
    throw InvariantError(std::string(what) + ": token id " + std::to_string(token) +
                         " outside vocabulary of size " + std::to_string(d.size()));
}


// ---- one window on the device ------------------------------------------
// rows: gamma draft rows, gamma + 1 target rows, all of one vocabulary.
struct WindowStats {
  int gamma = 0;
  std::vector<uint8_t> key;
  std::vector<double> accept;
  std::vector<double> norm_match;
  std::vector<int> err;   // per position dsdv_status the reference would raise there
  std::vector<int> kind;  // dsdv_effective_kind
};

struct DeviceWindow {
  Engine &eng;
  dsdv_params prm{};
  int V = 0, stride = 0, gamma = 0;
  double *d_draft = nullptr, *d_target = nullptr;
  int32_t *d_tokens = nullptr;
  dsdv_outputs out{};
  double *d_records = nullptr;
  int32_t *d_position = nullptr, *d_token = nullptr, *d_status = nullptr;
  double *d_u = nullptr;
  // top_m beyond the fused kernel's warp selection (32): NormMatch from an
  // exact device sort of the probability rows (dsdv_norm_match_rows)
  int m = 1;
  bool big_m = false;
  double *d_pd = nullptr, *d_pt = nullptr, *d_nm = nullptr;
  void *d_scratch = nullptr;
  size_t scratch_bytes = 0;

  DeviceWindow(Engine &e, const std::vector<const Distribution *> &draft,
               const std::vector<const Distribution *> &target, const std::vector<int> &tokens,
               double tau, const KeyCriteria &c)
      : eng(e) {
    gamma = static_cast<int>(draft.size());
    V = static_cast<int>(target[0]->size());
    stride = (V + 1) & ~1;  // 16-byte rows of fp64
    const int G1 = gamma + 1;
    const size_t rows_draft = (size_t)gamma * stride, rows_target = (size_t)G1 * stride;
    m = c.top_m < V ? c.top_m : V;  // verifier.cpp:155
    big_m = m > 32;
    if (big_m) scratch_bytes = dsdv_norm_match_scratch_bytes(gamma, V, stride);
    const size_t bytes = carve_size<double>(rows_draft) + carve_size<double>(rows_target) +
                         carve_size<int32_t>(gamma) + 6 * carve_size<int32_t>(1) +
                         2 * carve_size<uint8_t>(gamma) + 8 * carve_size<double>(gamma) +
                         carve_size<double>((size_t)G1 * kRecWords) + 3 * carve_size<int32_t>(1) +
                         carve_size<double>(1) + carve_size<uint8_t>(1) +
                         (big_m ? 2 * carve_size<double>(rows_draft) + carve_size<double>(gamma) +
                                      carve_size<char>(scratch_bytes)
                                : 0);
    Carve dv(eng.dev_arena(bytes));
    d_draft = dv.take<double>(rows_draft);
    d_target = dv.take<double>(rows_target);
    d_tokens = dv.take<int32_t>(gamma);
    out.accepted_count = dv.take<int32_t>(1);
    out.extra_token = dv.take<int32_t>(1);
    out.extra_source = dv.take<uint8_t>(1);
    out.key_count = dv.take<int32_t>(1);
    out.status = dv.take<int32_t>(1);
    out.near_threshold = dv.take<int32_t>(1);
    out.key_mask = dv.take<uint8_t>(gamma);
    out.accepted = dv.take<uint8_t>(gamma);
    out.accept_prob = dv.take<double>(gamma);
    out.h_target = dv.take<double>(gamma);
    out.h_draft = dv.take<double>(gamma);
    out.p_target_y = dv.take<double>(gamma);
    out.p_draft_y = dv.take<double>(gamma);
    out.norm_match = dv.take<double>(gamma);
    out.p_effective_y = dv.take<double>(gamma);
    out.uniform = dv.take<double>(gamma);
    d_records = dv.take<double>((size_t)G1 * kRecWords);
    out.records = d_records;
    d_position = dv.take<int32_t>(1);
    d_token = dv.take<int32_t>(1);
    d_status = dv.take<int32_t>(1);
    d_u = dv.take<double>(1);
    if (big_m) {
      d_pd = dv.take<double>(rows_draft);
      d_pt = dv.take<double>(rows_draft);
      d_nm = dv.take<double>(gamma);
      d_scratch = dv.take<char>(scratch_bytes);
    }

    // stage the rows in pinned memory, one copy
    // stage the probability rows as they are (pinned, one copy per region); the
    // device takes their logs (dsdv_log_rows) — no O(V) host transcendentals
    const size_t hbytes = (rows_draft + rows_target) * sizeof(double) + gamma * sizeof(int32_t);
    char *h = static_cast<char *>(eng.host_arena(hbytes));
    double *hd = reinterpret_cast<double *>(h);
    double *ht = hd + rows_draft;
    int32_t *htok = reinterpret_cast<int32_t *>(ht + rows_target);
    auto put_row = [&](double *dst, const Distribution &d) {
      std::memcpy(dst, d.probs().data(), V * sizeof(double));
      for (int i = V; i < stride; ++i) dst[i] = 0.0;
    };
    for (int j = 0; j < gamma; ++j) put_row(hd + (size_t)j * stride, *draft[j]);
    for (int j = 0; j < G1; ++j) put_row(ht + (size_t)j * stride, *target[j]);
    for (int j = 0; j < gamma; ++j) htok[j] = tokens[j];
    cudaMemcpyAsync(d_draft, hd, rows_draft * sizeof(double), cudaMemcpyHostToDevice, eng.stream);
    cudaMemcpyAsync(d_target, ht, rows_target * sizeof(double), cudaMemcpyHostToDevice,
                    eng.stream);
    cudaMemcpyAsync(d_tokens, htok, gamma * sizeof(int32_t), cudaMemcpyHostToDevice, eng.stream);
    if (big_m) {
      // top_ids orders by p (verifier.cpp:40-51): keep the probabilities
      cudaMemcpyAsync(d_pd, d_draft, rows_draft * sizeof(double), cudaMemcpyDeviceToDevice,
                      eng.stream);
      cudaMemcpyAsync(d_pt, d_target, rows_draft * sizeof(double), cudaMemcpyDeviceToDevice,
                      eng.stream);
    }
    eng.check(dsdv_log_rows(eng.ctx, d_draft, rows_draft, eng.stream));
    eng.check(dsdv_log_rows(eng.ctx, d_target, rows_target, eng.stream));

    prm.batch = 1;
    prm.gamma = gamma;
    prm.vocab = V;
    prm.row_stride = stride;
    prm.dtype = DSDV_DTYPE_F64;
    prm.top_m = big_m ? 1 : c.top_m;  // big_m: the overlap clause comes from d_nm
    prm.tau = tau;
    prm.ratio_limit = c.ratio_limit;
    prm.gap_limit = c.gap_limit;
    prm.overlap_floor = c.overlap_floor;
    prm.seed = 0;
    prm.window = 0;
    prm.sequence_offset = 0;
    prm.vocab_offset = 0;
    prm.vocab_local = V;
    prm.eps_u = 1e-12;
    prm.eps_lambda = 1e-12;
  }

  WindowStats stats() {
    if (big_m) {
      eng.check(dsdv_norm_match_rows(eng.ctx, d_pd, d_pt, gamma, V, stride, m, d_scratch,
                                     scratch_bytes, d_nm, eng.stream));
      eng.check(dsdv_window_stats_nm(eng.ctx, &prm, d_draft, d_target, d_tokens, d_nm, &out,
                                     eng.stream));
    } else {
      eng.check(dsdv_window_stats(eng.ctx, &prm, d_draft, d_target, d_tokens, &out, eng.stream));
    }
    WindowStats ws;
    ws.gamma = gamma;
    ws.key.resize(gamma);
    ws.accept.resize(gamma);
    ws.norm_match.resize(gamma);
    std::vector<double> rec((size_t)(gamma + 1) * kRecWords);
    cudaMemcpyAsync(ws.key.data(), out.key_mask, gamma, cudaMemcpyDeviceToHost, eng.stream);
    cudaMemcpyAsync(ws.accept.data(), out.accept_prob, gamma * sizeof(double),
                    cudaMemcpyDeviceToHost, eng.stream);
    cudaMemcpyAsync(ws.norm_match.data(), out.norm_match, gamma * sizeof(double),
                    cudaMemcpyDeviceToHost, eng.stream);
    cudaMemcpyAsync(rec.data(), d_records, rec.size() * sizeof(double), cudaMemcpyDeviceToHost,
                    eng.stream);
    eng.sync();
    ws.err.resize(gamma + 1);
    ws.kind.resize(gamma + 1);
    for (int j = 0; j <= gamma; ++j) {
      const int f = static_cast<int>(rec[(size_t)j * kRecWords + kRecFlagsWord]);
      ws.kind[j] = f & 0xff;
      ws.err[j] = (f >> 8) & 0xff;
    }
    return ws;
  }

  // extra token at `position` (< gamma: residual, == gamma: bonus) for uniform u
  int extra(int position, double u, int *status) {
    const int32_t pos = position;
    cudaMemcpyAsync(d_position, &pos, sizeof(pos), cudaMemcpyHostToDevice, eng.stream);
    cudaMemcpyAsync(d_u, &u, sizeof(u), cudaMemcpyHostToDevice, eng.stream);
    eng.check(dsdv_sample_extra(eng.ctx, &prm, d_draft, d_target, d_records, d_position, d_u,
                                d_token, d_status, eng.stream));
    int32_t tok = -1, st = 0;
    cudaMemcpyAsync(&tok, d_token, sizeof(tok), cudaMemcpyDeviceToHost, eng.stream);
    cudaMemcpyAsync(&st, d_status, sizeof(st), cudaMemcpyDeviceToHost, eng.stream);
    eng.sync();
    *status = st;
    return tok;
  }
};

[[noreturn]] void throw_position_error(int err, int token, const Distribution &draft) {
  switch (err) {
    case DSDV_E_DEGENERATE_MIXTURE:
      throw DegenerateMixtureError(
          "softened distribution has zero mass: target and draft supports are disjoint");
    case DSDV_E_DRAFTING_CONTRACT:
      throw DraftingContractError("token " + std::to_string(token) +
                                  " has zero draft probability; it cannot have been drafted");
    case DSDV_E_EMPTY_RESIDUAL:
      throw EmptyResidualError("residual is empty: effective and draft distributions match");
    default:
      check_token(draft, token, "is_key");
      throw InvariantError("verifier: invalid distribution row at this position");
  }
}

void check_entries(const std::vector<double> &v) {
  if (v.size() < 2)
    throw InvariantError("distribution needs a vocabulary of at least 2 tokens, got " +
                         std::to_string(v.size()));
  for (size_t i = 0; i < v.size(); ++i)
    if (!(std::isfinite(v[i]) && v[i] >= 0.0))
      throw InvariantError("distribution entry " + std::to_string(i) +
                           " is negative or non-finite: " + num(v[i]));
}

double left_sum(const std::vector<double> &v) {
  double s = 0.0;
  for (double x : v) s += x;
  return s;
}

Distribution mix_on_device(int kind, const Distribution &a, const Distribution &b, double tau) {
  Engine &eng = engine();
  const size_t V = a.size();
  Carve dv(eng.dev_arena(3 * carve_size<double>(V) + carve_size<int32_t>(1)));
  double *da = dv.take<double>(V), *db = dv.take<double>(V), *dout = dv.take<double>(V);
  int32_t *dst = dv.take<int32_t>(1);
  cudaMemcpyAsync(da, a.probs().data(), V * sizeof(double), cudaMemcpyHostToDevice, eng.stream);
  cudaMemcpyAsync(db, b.probs().data(), V * sizeof(double), cudaMemcpyHostToDevice, eng.stream);
  eng.check(dsdv_mix_rows(eng.ctx, kind, static_cast<int32_t>(V), da, db, tau, dout, dst,
                          eng.stream));
  std::vector<double> w(V);
  int32_t st = 0;
  cudaMemcpyAsync(w.data(), dout, V * sizeof(double), cudaMemcpyDeviceToHost, eng.stream);
  cudaMemcpyAsync(&st, dst, sizeof(st), cudaMemcpyDeviceToHost, eng.stream);
  eng.sync();
  if (st == DSDV_E_DEGENERATE_MIXTURE)
    throw DegenerateMixtureError(
        "softened distribution has zero mass: target and draft supports are disjoint");
  if (st == DSDV_E_EMPTY_RESIDUAL)
    throw EmptyResidualError("residual is empty: effective and draft distributions match");
  return Distribution(std::move(w));
}

// One-position window (norm_match / is_key): draft row, target row twice.
WindowStats single_position(const Distribution &target, const Distribution &draft, int token,
                            const KeyCriteria &c) {
  Engine &eng = engine();
  DeviceWindow w(eng, {&draft}, {&target, &target}, {token}, 0.0, c);
  return w.stats();
}

}  // namespace

// ---- Distribution (distribution.cpp:29-125) ------------------------------
Distribution::Distribution(std::vector<double> probs) : p_(std::move(probs)) {
  check_entries(p_);
  const double s = left_sum(p_);
  if (std::abs(s - 1.0) > kSumTolerance)
    throw InvariantError("distribution entries sum to " + num(s) + ", expected 1 within 1e-9");
}

Distribution Distribution::from_weights(std::vector<double> w) {
  check_entries(w);
  const double s = left_sum(w);
  if (s <= 0.0) throw InvariantError("cannot normalize weights with zero total mass");
  for (double &x : w) x /= s;
  return Distribution(std::move(w), Trusted{});
}

Distribution temperature_scale(const Distribution &d, double t) {
  if (!(std::isfinite(t) && t >= 0.0))
    throw InvariantError("temperature must be a finite non-negative real, got " + num(t));
  if (t == 1.0) return d;
  const size_t n = d.size();
  if (t == 0.0) {
    // one-hot at the first maximum
    const size_t best = static_cast<size_t>(
        std::max_element(d.probs().begin(), d.probs().end()) - d.probs().begin());
    std::vector<double> oh(n, 0.0);
    oh[best] = 1.0;
    return Distribution(std::move(oh));
  }
  const double k = 1.0 / t;
  std::vector<double> lw(n);
  double top = -kInf;
  for (size_t i = 0; i < n; ++i) {
    lw[i] = d[i] > 0.0 ? k * std::log(d[i]) : -kInf;
    top = std::max(top, lw[i]);
  }
  for (size_t i = 0; i < n; ++i) lw[i] = std::isinf(lw[i]) ? 0.0 : std::exp(lw[i] - top);
  return Distribution::from_weights(std::move(lw));
}

int sample_with_uniform(const Distribution &d, double u) {
  double acc = 0.0;
  int last = -1;
  const int n = static_cast<int>(d.size());
  for (int i = 0; i < n; ++i) {
    const double p = d[static_cast<size_t>(i)];
    last = p > 0.0 ? i : last;
    acc += p;
    if (u < acc) return i;
  }
  return last;  // u in the rounding gap: the last supported id
}

int sample(const Distribution &d, UniformStream &rng) { return sample_with_uniform(d, rng.next_uniform()); }

double total_variation(const Distribution &a, const Distribution &b) {
  if (a.size() != b.size()) throw InvariantError("total variation requires equal vocabulary sizes");
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += std::abs(a[i] - b[i]);
  return 0.5 * s;
}

// ---- TokenModel (token_model.cpp) ----------------------------------------
namespace {
void check_model_temperature(double t) {
  if (!(std::isfinite(t) && t >= 0.0))
    throw InvariantError("model temperature must be finite and >= 0, got " + num(t));
}
}  // namespace

TokenModel TokenModel::categorical(Distribution next, double temperature) {
  check_model_temperature(temperature);
  TokenModel m(Kind::CategoricalIid, next.size(), temperature);
  m.rows_.push_back(std::move(next));
  return m;
}

TokenModel TokenModel::markov(std::vector<Distribution> rows, Distribution initial,
                              double temperature) {
  check_model_temperature(temperature);
  const size_t V = initial.size();
  if (rows.size() != V)
    throw InvariantError("markov transition table must have one row per token: " +
                         std::to_string(rows.size()) + " rows for vocab " + std::to_string(V));
  for (size_t i = 0; i < rows.size(); ++i)
    if (rows[i].size() != V)
      throw InvariantError("markov row " + std::to_string(i) + " has length " +
                           std::to_string(rows[i].size()) + ", expected " + std::to_string(V));
  TokenModel m(Kind::MarkovOrder1, V, temperature);
  m.rows_ = std::move(rows);
  m.init_.push_back(std::move(initial));
  return m;
}

Distribution next_distribution(const TokenModel &model, const Context &ctx) {
  for (int id : ctx.tokens)
    if (id < 0 || static_cast<size_t>(id) >= model.vocab_size())
      throw InvalidContextError("context token id " + std::to_string(id) +
                                " outside vocabulary of size " +
                                std::to_string(model.vocab_size()));
  const Distribution &row =
      model.kind() == TokenModel::Kind::CategoricalIid
          ? model.rows_.front()
          : (ctx.tokens.empty() ? model.init_.front()
                                : model.rows_[static_cast<size_t>(ctx.tokens.back())]);
  return temperature_scale(row, model.temperature());
}

// ---- verifier parameters (verifier.cpp:55-91) ----------------------------
void KeyCriteria::validate() const {
  if (std::isnan(ratio_limit) || !(ratio_limit > 0.0))
    throw InvariantError("criteria.ratio_limit must be > 0, got " + num(ratio_limit));
  if (!(std::isfinite(gap_limit) && gap_limit >= 0.0 && gap_limit <= 1.0))
    throw InvariantError("criteria.gap_limit must lie in [0, 1], got " + num(gap_limit));
  if (!(std::isfinite(overlap_floor) && overlap_floor >= 0.0 && overlap_floor <= 1.0))
    throw InvariantError("criteria.overlap_floor must lie in [0, 1], got " + num(overlap_floor));
  if (top_m < 1) throw InvariantError("criteria.top_m must be >= 1, got " + std::to_string(top_m));
}

KeyCriteria KeyCriteria::none() { return KeyCriteria{kInf, 1.0, 0.0, 1}; }

int VerificationResult::key_count() const {
  return static_cast<int>(std::count_if(decisions.begin(), decisions.end(),
                                         [](const TokenDecision &d) { return d.is_key; }));
}

void VerifyParams::validate() const {
  if (gamma < 1) throw InvariantError("gamma must be >= 1, got " + std::to_string(gamma));
  if (!(std::isfinite(tau) && tau >= 0.0 && tau <= 1.0))
    throw InvariantError("tau must lie in [0, 1], got " + num(tau));
  criteria.validate();
}

// ---- primitives ----------------------------------------------------------
DraftWindow draft_window(const TokenModel &draft, const Context &ctx, int gamma,
                         UniformStream &rng) {
  if (gamma < 1)
    throw InvariantError("draft window length must be >= 1, got " + std::to_string(gamma));
  DraftWindow w;
  Context cur = ctx;
  for (int j = 0; j < gamma; ++j) {
    Distribution d = next_distribution(draft, cur);
    const int tok = sample(d, rng);
    cur.tokens.push_back(tok);
    w.tokens.push_back(tok);
    w.draft_dists.push_back(std::move(d));
  }
  return w;
}

double token_cross_entropy(const Distribution &d, int token) {
  check_token(d, token, "token_cross_entropy");
  const double p = d[static_cast<size_t>(token)];
  return p > 0.0 ? -std::log(p) : kInf;
}

double accept_prob(const Distribution &effective, const Distribution &draft, int token) {
  check_token(draft, token, "accept_prob");
  const double pd = draft[static_cast<size_t>(token)];
  if (!(pd > 0.0))
    throw DraftingContractError("token " + std::to_string(token) +
                                " has zero draft probability; it cannot have been drafted");
  return std::min(1.0, effective[static_cast<size_t>(token)] / pd);
}

double norm_match(const Distribution &target, const Distribution &draft, int top_m) {
  if (target.size() != draft.size())
    throw InvariantError("norm_match requires equal vocabulary sizes");
  if (top_m < 1 || static_cast<size_t>(top_m) > target.size())
    throw InvariantError("norm_match top_m must lie in [1, vocab], got " + std::to_string(top_m));
  KeyCriteria c;
  c.top_m = top_m;
  return single_position(target, draft, 0, c).norm_match[0];
}

bool is_key(const Distribution &target, const Distribution &draft, int token,
            const KeyCriteria &criteria) {
  criteria.validate();
  check_token(target, token, "is_key");
  check_token(draft, token, "token_cross_entropy");
  if (target.size() != draft.size())
    throw InvariantError("norm_match requires equal vocabulary sizes");
  return single_position(target, draft, token, criteria).key[0] != 0;
}

Distribution soften(const Distribution &target, const Distribution &draft, double tau) {
  if (!(std::isfinite(tau) && tau >= 0.0 && tau <= 1.0))
    throw InvariantError("soften tau must lie in [0, 1], got " + num(tau));
  if (target.size() != draft.size()) throw InvariantError("soften requires equal vocabulary sizes");
  // exact endpoints (verifier.cpp:170-172)
  if (tau == 0.0) return target;
  if (tau == 1.0) return draft;
  if (target == draft) return target;
  return mix_on_device(DSDV_MIX_SOFTEN, target, draft, tau);
}

Distribution residual_distribution(const Distribution &effective, const Distribution &draft) {
  if (effective.size() != draft.size())
    throw InvariantError("residual requires equal vocabulary sizes");
  return mix_on_device(DSDV_MIX_RESIDUAL, effective, draft, 0.0);
}

// ---- the round (verifier.cpp:215-257) -------------------------------------
VerificationResult verify_round(const TokenModel &draft, const TokenModel &target,
                                const Context &ctx, const VerifyParams &params,
                                UniformStream &rng) {
  params.validate();
  const DraftWindow win = draft_window(draft, ctx, params.gamma, rng);
  const int G = params.gamma;
  // target rows: position j sees the context plus drafts 0..j-1 (all accepted
  // if position j is ever reached); row G feeds the bonus draw
  std::vector<Distribution> trows;
  trows.reserve(G + 1);
  Context prefix = ctx;
  for (int j = 0; j <= G; ++j) {
    trows.push_back(next_distribution(target, prefix));
    if (j < G) prefix.tokens.push_back(win.tokens[j]);
  }
  if (trows[0].size() != win.draft_dists[0].size()) {
    check_token(trows[0], win.tokens[0], "is_key");
    check_token(win.draft_dists[0], win.tokens[0], "token_cross_entropy");
    throw InvariantError("norm_match requires equal vocabulary sizes");
  }
  std::vector<const Distribution *> dp, tp;
  for (const auto &d : win.draft_dists) dp.push_back(&d);
  for (const auto &t : trows) tp.push_back(&t);
  Engine &eng = engine();
  DeviceWindow dw(eng, dp, tp, win.tokens, params.tau, params.criteria);
  const WindowStats ws = dw.stats();

  VerificationResult res;
  for (int j = 0; j < G; ++j) {
    const int tok = win.tokens[j];
    if (ws.err[j] != DSDV_OK) throw_position_error(ws.err[j], tok, win.draft_dists[j]);
    TokenDecision dec;
    dec.token = tok;
    dec.is_key = ws.key[j] != 0;
    dec.tau_used = dec.is_key ? 0.0 : params.tau;
    dec.accept_prob = ws.accept[j];
    const double u = rng.next_uniform();
    dec.accepted = u < dec.accept_prob;
    if (dec.accepted) {
      res.decisions.push_back(dec);
      ++res.accepted_count;
      continue;
    }
    // residual of the effective distribution (verifier.cpp:245): the reference
    // builds it (and may throw) before drawing, so probe emptiness first
    int st = 0;
    if (ws.kind[j] == DSDV_EFF_DRAFT)
      throw EmptyResidualError("residual is empty: effective and draft distributions match");
    dw.extra(j, 0.0, &st);
    if (st != DSDV_OK) throw_position_error(st, tok, win.draft_dists[j]);
    const double u2 = rng.next_uniform();
    const int x = dw.extra(j, u2, &st);
    dec.replacement = x;
    res.extra_token = x;
    res.extra_source = ExtraSource::ResidualResample;
    res.decisions.push_back(dec);
    return res;
  }
  if (ws.err[G] != DSDV_OK) throw InvariantError("verifier: invalid bonus row");
  int st = 0;
  res.extra_token = dw.extra(G, rng.next_uniform(), &st);
  res.extra_source = ExtraSource::BonusFromTarget;
  return res;
}

GenerationResult generate(const TokenModel &draft, const TokenModel &target, const Context &prompt,
                          int max_new, const VerifyParams &params, UniformStream &rng) {
  params.validate();
  if (max_new < 1) throw InvariantError("max_new must be >= 1, got " + std::to_string(max_new));
  GenerationResult g;
  Context ctx = prompt;
  while (static_cast<int>(g.tokens.size()) < max_new) {
    VerificationResult r = verify_round(draft, target, ctx, params, rng);
    for (const TokenDecision &d : r.decisions)
      if (d.accepted) {
        g.tokens.push_back(d.token);
        ctx.tokens.push_back(d.token);
      }
    g.tokens.push_back(r.extra_token);
    ctx.tokens.push_back(r.extra_token);
    g.rounds.push_back(std::move(r));
  }
  g.tokens.resize(static_cast<size_t>(max_new));
  return g;
}

namespace gpu {
void set_device(int device) {
  Engine &eng = raw_engine();
  eng.wanted = device;
  eng.ready();
}
unsigned long long launch_count() { return dsdv_launch_count(engine().ctx); }
dsdv_ctx *context() { return engine().ctx; }
}  // namespace gpu

}  // namespace dsd
