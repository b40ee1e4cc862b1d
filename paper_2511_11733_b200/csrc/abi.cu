// C-ABI entry points (include/dsdv/dsdv.h): validation with the reference's
// messages, scratch management, dtype dispatch and error mapping.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace dsdv {
int fused_max_vocab(int esize, int top_m);
size_t norm_match_scratch_bytes(int gamma, int V, int stride);
size_t calib_scratch_doubles(int max_vocab, int max_horizon, int gamma);
cudaError_t launch_calibrate(const dsdv_calib_item *items, int n_items, const double *rows,
                             const dsdv_key_criteria *points, int n_points, double tau, int gamma,
                             double budget, double *scratch, size_t scratch_per_thread,
                             double *len, double *tv, int32_t *status, dsdv_grid_eval *out,
                             cudaStream_t stream);
cudaError_t launch_norm_match(const double *draft, const double *target, int gamma, int V,
                              int stride, int M, void *scratch, double *nm_out,
                              cudaStream_t stream);
template <class In>
cudaError_t launch_fused(const DevParams &, const void *, const void *, const int32_t *,
                         const DevOut &, const DevScratch &, cudaStream_t, int *);
template <class In>
cudaError_t launch_sample_extra(const DevParams &, const void *, const void *, const double *,
                                const int32_t *, const double *, int32_t *, int32_t *,
                                cudaStream_t);
template <class In>
cudaError_t launch_draft_sample(const DevParams &, const void *, int32_t *, double,
                                cudaStream_t);
template <class In>
cudaError_t launch_shard_merge(const DevParams &p, const double *rec, const double *topv,
                               const int32_t *topi, int P, size_t rank_bytes, const void *draft,
                               const void *target, const int32_t *tokens, const DevOut &o,
                               int32_t *position, double *uniform, double *mass_out,
                               double *tiles, cudaStream_t stream,
                               const long long *mass_delta = nullptr, int n_delta = 0);
template <class In>
cudaError_t launch_shard_sample(const DevParams &p, int mode, int rank, int nranks,
                                const void *draft, const void *target, const double *records,
                                const int32_t *position, const double *uniform,
                                const double *masses, double *mass_out, int32_t *token_out,
                                int32_t *status, const double *tiles, cudaStream_t stream,
                                const long long *tok_delta = nullptr, int n_delta = 0,
                                size_t mstride = 0);
cudaError_t launch_tokens_max(const int32_t *tok, size_t stride_elems, int nranks, int B,
                              int32_t *out, cudaStream_t stream);
cudaError_t launch_mix_rows(int kind, int V, const double *a, const double *b, double tau,
                            double *out, int32_t *status, cudaStream_t stream);
cudaError_t launch_spin(unsigned long long ns, cudaStream_t stream);
cudaError_t launch_peer_signal(char *const *bases, int nranks, int rank, unsigned long long stride,
                               unsigned long long epoch, cudaStream_t stream);
cudaError_t launch_peer_wait(const unsigned long long *flags, int nranks, unsigned long long epoch,
                             unsigned long long timeout_ns, int *status, cudaStream_t stream);
cudaError_t launch_peer_round(char *const *bases, int nranks, int rank, unsigned long long stride,
                              unsigned long long epoch, const unsigned long long *flags,
                              unsigned long long timeout_ns, int *status, int reset,
                              cudaStream_t stream);
cudaError_t launch_tokens_fold(const int32_t *tok, size_t stride, int nranks, int B, int32_t *out,
                               const int32_t *peer_status, int32_t *status, cudaStream_t stream);
cudaError_t launch_log_rows(double *x, size_t n, cudaStream_t stream);
cudaError_t launch_hop_send(unsigned long long t1_ns, int32_t *dst_payload, const int32_t *payload,
                            unsigned long long *dst_flag, unsigned long long value,
                            cudaStream_t stream);
cudaError_t launch_hop_recv(const unsigned long long *flag, unsigned long long value,
                            unsigned long long timeout_ns, int *status, const int32_t *slot,
                            int32_t *payload, cudaStream_t stream);
cudaError_t launch_synth(int dtype, int B, int gamma, int V, int stride, uint64_t seed,
                         void *draft, void *target, cudaStream_t stream);
}  // namespace dsdv

struct dsdv_ctx {
  int device = 0;
  std::string last_error;
  unsigned int *counters = nullptr;  // [0] ticket, [1] exit count
  unsigned int *flags = nullptr;  // [positions]
  int2 *slots = nullptr;          // [positions]
  unsigned int *done = nullptr;   // [sequences]
  unsigned long long *stop = nullptr;      // [sequences] early-exit stop keys
  // dsdv_shard_verify_peers: extra-draw position, uniform, tile sums, peer status
  void *shard_scratch = nullptr;
  size_t shard_scratch_cap = 0;
  unsigned long long *streamed = nullptr;  // logit bytes copied by the fused kernel
  unsigned long long *trace = nullptr;  // DSDV_TRACE builds: [grid][kTraceWords]
  size_t flags_cap = 0;
  size_t done_cap = 0;
  uint32_t epoch = 0;
  uint64_t launches = 0;
  int last_grid = 0;
};

namespace {

using dsdv::DevOut;
using dsdv::DevParams;
using dsdv::DevScratch;

// Messages of calls made without a context (host-only validation).
thread_local std::string g_host_error;

dsdv_status fail(dsdv_ctx *ctx, dsdv_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  (ctx ? ctx->last_error : g_host_error) = buf;
  return st;
}

// std::to_string(double) formatting, as the reference messages use it.
std::string dstr(double x) {
  char b[64];
  snprintf(b, sizeof(b), "%f", x);
  return b;
}

dsdv_status cuda_fail(dsdv_ctx *ctx, cudaError_t e, const char *what) {
  return fail(ctx, DSDV_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

int esize(int dtype) {
  return dtype == DSDV_DTYPE_BF16 ? 2 : (dtype == DSDV_DTYPE_F32 ? 4 : 8);
}

dsdv_status ensure_scratch(dsdv_ctx *ctx, size_t n_positions, size_t n_sequences) {
  cudaError_t e;
  if (!ctx->counters) {
    e = cudaMalloc(&ctx->counters, 2 * sizeof(unsigned int));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(counters)");
    e = cudaMemset(ctx->counters, 0, 2 * sizeof(unsigned int));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemset(counters)");
    e = cudaMalloc(&ctx->streamed, sizeof(unsigned long long));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(streamed)");
    e = cudaMemset(ctx->streamed, 0, sizeof(unsigned long long));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemset(streamed)");
  }
  if (n_positions > ctx->flags_cap) {
    if (ctx->flags) cudaFree(ctx->flags);
    e = cudaMalloc(&ctx->flags, n_positions * sizeof(unsigned int));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(flags)");
    e = cudaMemset(ctx->flags, 0, n_positions * sizeof(unsigned int));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemset(flags)");
    if (ctx->slots) cudaFree(ctx->slots);
    e = cudaMalloc(&ctx->slots, n_positions * sizeof(int2));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(slots)");
    ctx->flags_cap = n_positions;  // zeroed words carry epoch 0, never a live one
  }
  if (n_sequences > ctx->done_cap) {
    if (ctx->done) cudaFree(ctx->done);
    e = cudaMalloc(&ctx->done, n_sequences * sizeof(unsigned int));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(done)");
    e = cudaMemset(ctx->done, 0, n_sequences * sizeof(unsigned int));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemset(done)");
    if (ctx->stop) cudaFree(ctx->stop);
    e = cudaMalloc(&ctx->stop, n_sequences * sizeof(unsigned long long));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(stop)");
    e = cudaMemset(ctx->stop, 0, n_sequences * sizeof(unsigned long long));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemset(stop)");
    ctx->done_cap = n_sequences;
  }
  return DSDV_OK;
}

dsdv_status build_params(dsdv_ctx *ctx, const dsdv_params *pp, DevParams &d) {
  dsdv_status st = dsdv_validate(ctx, pp);
  if (st != DSDV_OK) return st;
  const dsdv_params &p = *pp;
  std::memset(&d, 0, sizeof(d));
  d.B = p.batch;
  d.gamma = p.gamma;
  d.V = p.vocab;
  d.stride = p.row_stride;
  d.top_m = p.top_m < p.vocab ? p.top_m : p.vocab;  // clamp, verifier.cpp:155
  d.vocab_offset = p.vocab_offset;
  d.vocab_local = p.vocab_local;
  const int chunk_elems = dsdv::kChunkBytes / esize(p.dtype);
  d.n_chunks = (p.vocab_local + chunk_elems - 1) / chunk_elems;
  d.n_items = p.batch * (p.gamma + 1);
  d.stats_only = 0;
  d.need_z = (p.tau > 0.0 && p.tau < 1.0) ? 1 : 0;
  d.tau_f = (float)p.tau;
  d.omt_f = (float)(1.0 - p.tau);
  d.tau = p.tau;
  d.ratio_limit = p.ratio_limit;
  d.gap_limit = p.gap_limit;
  d.overlap_floor = p.overlap_floor;
  d.eps_u = p.eps_u;
  d.eps_lambda = p.eps_lambda;
  d.seed = p.seed;
  d.window = p.window;
  d.seq_offset = p.sequence_offset;
  return DSDV_OK;
}

DevOut to_dev(const dsdv_outputs *o) {
  DevOut d;
  std::memset(&d, 0, sizeof(d));
  if (!o) return d;
  d.accepted_count = o->accepted_count;
  d.extra_token = o->extra_token;
  d.key_count = o->key_count;
  d.status = o->status;
  d.near_threshold = o->near_threshold;
  d.extra_source = o->extra_source;
  d.key_mask = o->key_mask;
  d.accepted = o->accepted;
  d.accept_prob = o->accept_prob;
  d.h_target = o->h_target;
  d.h_draft = o->h_draft;
  d.p_target_y = o->p_target_y;
  d.p_draft_y = o->p_draft_y;
  d.norm_match = o->norm_match;
  d.p_effective_y = o->p_effective_y;
  d.uniform = o->uniform;
  d.records = o->records;
  return d;
}

bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

dsdv_status run_fused(dsdv_ctx *ctx, const dsdv_params *params, const void *draft,
                      const void *target, const int32_t *tokens, const dsdv_outputs *out,
                      void *stream, bool stats_only, double *topv = nullptr,
                      int32_t *topi = nullptr, int npeer = 0,
                      const long long *peer_delta = nullptr, bool early_exit = false,
                      const double *nm_in = nullptr) {
  const bool partial = topv != nullptr;
  if (!ctx) return DSDV_E_INVARIANT;
  DevParams d;
  dsdv_status st = build_params(ctx, params, d);
  if (st != DSDV_OK) return st;
  d.stats_only = stats_only ? 1 : 0;
  d.partial = partial ? 1 : 0;
  d.early_exit = early_exit ? 1 : 0;
  d.nm_in = nm_in;
  if (partial && !topi)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_shard_stats: top lists are required");
  if (!draft || !target || !tokens || !out)
    return fail(ctx, DSDV_E_INVARIANT, "logits, draft tokens and outputs must be non-null");
  if (!aligned16(draft) || !aligned16(target))
    return fail(ctx, DSDV_E_UNSUPPORTED, "logit base pointers must be 16-byte aligned");
  if (!stats_only && (!out->accepted_count || !out->extra_token || !out->extra_source ||
                      !out->key_count || !out->status || !out->near_threshold))
    return fail(ctx, DSDV_E_INVARIANT,
                "dsdv_verify: the per-sequence outputs (accepted_count, extra_token, "
                "extra_source, key_count, status, near_threshold) are required");
  if (stats_only && !out->records)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_window_stats: records output is required");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  st = ensure_scratch(ctx, (size_t)d.n_items, (size_t)d.B);
  if (st != DSDV_OK) return st;
  ctx->epoch = (ctx->epoch + 1) & 0x0fffffffu;
  if (ctx->epoch == 0) {
    // wrap-around: no word may still carry a recycled epoch
    cudaMemsetAsync(ctx->flags, 0, ctx->flags_cap * sizeof(unsigned int), (cudaStream_t)stream);
    cudaMemsetAsync(ctx->stop, 0, ctx->done_cap * sizeof(unsigned long long),
                    (cudaStream_t)stream);
    ctx->epoch = 1;
  }
  d.epoch = ctx->epoch;
  DevScratch s;
  s.ticket = ctx->counters;
  s.exit_count = ctx->counters + 1;
  s.flags = ctx->flags;
  s.slots = ctx->slots;
  s.done = ctx->done;
  s.stop = ctx->stop;
  s.streamed = ctx->streamed;
  s.trace = nullptr;
#if defined(DSDV_TRACE) || defined(DSDV_TRACE_LOCAL)
  if (!ctx->trace) {
    cudaMalloc(&ctx->trace, 1024 * dsdv::kTraceWords * sizeof(unsigned long long));
    cudaMemset(ctx->trace, 0, 1024 * dsdv::kTraceWords * sizeof(unsigned long long));
  }
  s.trace = ctx->trace;
#endif
  DevOut o = to_dev(out);
  o.topv = topv;
  o.topi = topi;
  o.npeer = npeer;
  for (int q = 0; q < npeer; ++q) o.peer_delta[q] = peer_delta[q];
  switch (params->dtype) {
    case DSDV_DTYPE_BF16:
      e = dsdv::launch_fused<__nv_bfloat16>(d, draft, target, tokens, o, s, (cudaStream_t)stream,
                                            &ctx->last_grid);
      break;
    case DSDV_DTYPE_F32:
      e = dsdv::launch_fused<float>(d, draft, target, tokens, o, s, (cudaStream_t)stream,
                                    &ctx->last_grid);
      break;
    default:
      e = dsdv::launch_fused<double>(d, draft, target, tokens, o, s, (cudaStream_t)stream,
                                     &ctx->last_grid);
      break;
  }
  if (e != cudaSuccess) return cuda_fail(ctx, e, "fused verifier launch");
  ctx->launches += 1;
  return DSDV_OK;
}

}  // namespace

extern "C" {

int dsdv_abi_version(void) { return DSDV_ABI_VERSION; }

dsdv_status dsdv_create(int device, dsdv_ctx **out) {
  if (!out) return DSDV_E_INVARIANT;
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0 || device < 0 || device >= n) return DSDV_E_CUDA;
  dsdv_ctx *ctx = new dsdv_ctx();
  ctx->device = device;
  e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete ctx;
    return DSDV_E_CUDA;
  }
  if (ensure_scratch(ctx, 1, 1) != DSDV_OK) {
    delete ctx;
    return DSDV_E_CUDA;
  }
  *out = ctx;
  return DSDV_OK;
}

dsdv_status dsdv_destroy(dsdv_ctx *ctx) {
  if (!ctx) return DSDV_OK;
  cudaSetDevice(ctx->device);
  if (ctx->counters) cudaFree(ctx->counters);
  if (ctx->flags) cudaFree(ctx->flags);
  if (ctx->slots) cudaFree(ctx->slots);
  if (ctx->done) cudaFree(ctx->done);
  if (ctx->stop) cudaFree(ctx->stop);
  if (ctx->streamed) cudaFree(ctx->streamed);
  if (ctx->shard_scratch) cudaFree(ctx->shard_scratch);
  if (ctx->trace) cudaFree(ctx->trace);
  delete ctx;
  return DSDV_OK;
}

const char *dsdv_last_error(const dsdv_ctx *ctx) {
  return ctx ? ctx->last_error.c_str() : g_host_error.c_str();
}

uint64_t dsdv_launch_count(const dsdv_ctx *ctx) { return ctx ? ctx->launches : 0; }

// Development aid (not part of the ABI header): copies and clears the per-CTA
// cycle counters of a DSDV_TRACE build. Returns the number of CTAs, 0 if the
// library was built without tracing.
int dsdv_debug_trace(dsdv_ctx *ctx, unsigned long long *host, int max_ctas) {
#if defined(DSDV_TRACE) || defined(DSDV_TRACE_LOCAL)
  if (!ctx || !ctx->trace) return 0;
  const int n = max_ctas < 1024 ? max_ctas : 1024;
  cudaDeviceSynchronize();
  cudaMemcpy(host, ctx->trace, (size_t)n * dsdv::kTraceWords * 8, cudaMemcpyDeviceToHost);
  cudaMemset(ctx->trace, 0, 1024 * dsdv::kTraceWords * 8);
  return ctx->last_grid;
#else
  (void)ctx; (void)host; (void)max_ctas;
  return 0;
#endif
}

double dsdv_uniform(uint64_t seed, uint64_t window, uint32_t sequence, uint32_t slot) {
  return dsdv_philox_uniform(seed, window, sequence, slot);
}

// VerifyParams::validate + KeyCriteria::validate (verifier.cpp:55-91), same
// messages, then the layout rules of this ABI.
dsdv_status dsdv_validate(dsdv_ctx *ctx, const dsdv_params *pp) {
  if (!pp) return fail(ctx, DSDV_E_INVARIANT, "null parameters");
  const dsdv_params &p = *pp;
  if (p.gamma < 1)
    return fail(ctx, DSDV_E_INVARIANT, "gamma must be >= 1, got %d", p.gamma);
  if (!std::isfinite(p.tau) || p.tau < 0.0 || p.tau > 1.0)
    return fail(ctx, DSDV_E_INVARIANT, "tau must lie in [0, 1], got %s", dstr(p.tau).c_str());
  if (std::isnan(p.ratio_limit) || p.ratio_limit <= 0.0)
    return fail(ctx, DSDV_E_INVARIANT, "criteria.ratio_limit must be > 0, got %s",
                dstr(p.ratio_limit).c_str());
  if (!std::isfinite(p.gap_limit) || p.gap_limit < 0.0 || p.gap_limit > 1.0)
    return fail(ctx, DSDV_E_INVARIANT, "criteria.gap_limit must lie in [0, 1], got %s",
                dstr(p.gap_limit).c_str());
  if (!std::isfinite(p.overlap_floor) || p.overlap_floor < 0.0 || p.overlap_floor > 1.0)
    return fail(ctx, DSDV_E_INVARIANT, "criteria.overlap_floor must lie in [0, 1], got %s",
                dstr(p.overlap_floor).c_str());
  if (p.top_m < 1)
    return fail(ctx, DSDV_E_INVARIANT, "criteria.top_m must be >= 1, got %d", p.top_m);
  if (p.batch < 1) return fail(ctx, DSDV_E_INVARIANT, "batch must be >= 1, got %d", p.batch);
  if (p.vocab < 2)
    return fail(ctx, DSDV_E_INVARIANT,
                "distribution needs a vocabulary of at least 2 tokens, got %d", p.vocab);
  if (p.dtype != DSDV_DTYPE_F32 && p.dtype != DSDV_DTYPE_BF16 && p.dtype != DSDV_DTYPE_F64)
    return fail(ctx, DSDV_E_UNSUPPORTED, "unknown logits dtype %d", p.dtype);
  if (p.vocab_local < 1 || p.vocab_offset < 0 || p.vocab_offset + p.vocab_local > p.vocab)
    return fail(ctx, DSDV_E_INVARIANT, "vocab slice [%d, %d) outside vocabulary of size %d",
                p.vocab_offset, p.vocab_offset + p.vocab_local, p.vocab);
  const int es = esize(p.dtype), vec = 16 / es;
  const int need = (p.vocab_local + vec - 1) / vec * vec;
  if (p.row_stride < need || ((size_t)p.row_stride * es) % 16 != 0)
    return fail(ctx, DSDV_E_UNSUPPORTED,
                "row_stride %d must be >= %d and a multiple of %d elements (16-byte rows)",
                p.row_stride, need, vec);
  const int m = p.top_m < p.vocab ? p.top_m : p.vocab;
  if (p.vocab_local > dsdv::fused_max_vocab(es, m))
    return fail(ctx, DSDV_E_UNSUPPORTED,
                "vocab slice %d exceeds the fused kernel limit %d for this dtype and top_m",
                p.vocab_local, dsdv::fused_max_vocab(es, m));
  if (m > dsdv::kMaxTopM)
    return fail(ctx, DSDV_E_UNSUPPORTED, "top_m %d exceeds the kernel limit %d", m,
                dsdv::kMaxTopM);
  if (!(p.eps_u >= 0.0) || !(p.eps_lambda >= 0.0))
    return fail(ctx, DSDV_E_INVARIANT, "eps bands must be >= 0");
  return DSDV_OK;
}

dsdv_status dsdv_verify(dsdv_ctx *ctx, const dsdv_params *params, const void *draft_logits,
                        const void *target_logits, const int32_t *draft_tokens,
                        const dsdv_outputs *out, void *stream) {
  return run_fused(ctx, params, draft_logits, target_logits, draft_tokens, out, stream, false);
}

dsdv_status dsdv_verify_early_exit(dsdv_ctx *ctx, const dsdv_params *params,
                                   const void *draft_logits, const void *target_logits,
                                   const int32_t *draft_tokens, const dsdv_outputs *out,
                                   void *stream) {
  return run_fused(ctx, params, draft_logits, target_logits, draft_tokens, out, stream, false,
                   nullptr, nullptr, 0, nullptr, true);
}

dsdv_status dsdv_window_stats_nm(dsdv_ctx *ctx, const dsdv_params *params,
                                 const void *draft_logits, const void *target_logits,
                                 const int32_t *draft_tokens, const double *norm_match_in,
                                 const dsdv_outputs *out, void *stream) {
  if (!ctx || !params) return DSDV_E_INVARIANT;
  if (!norm_match_in)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_window_stats_nm: norm_match_in is required");
  if (params->top_m < 1)
    return fail(ctx, DSDV_E_INVARIANT, "criteria.top_m must be >= 1, got %d", params->top_m);
  // the overlap clause comes from the caller; the kernel's own selection is
  // reduced to one id per row (its NormMatch output is the caller's value)
  dsdv_params q = *params;
  q.top_m = 1;
  return run_fused(ctx, &q, draft_logits, target_logits, draft_tokens, out, stream, true,
                   nullptr, nullptr, 0, nullptr, false, norm_match_in);
}

size_t dsdv_norm_match_scratch_bytes(int32_t gamma, int32_t vocab, int32_t row_stride) {
  return dsdv::norm_match_scratch_bytes(gamma, vocab, row_stride);
}

dsdv_status dsdv_norm_match_rows(dsdv_ctx *ctx, const double *draft_probs,
                                 const double *target_probs, int32_t gamma, int32_t vocab,
                                 int32_t row_stride, int32_t top_m, void *scratch,
                                 size_t scratch_bytes, double *norm_match_out, void *stream) {
  if (!ctx) return DSDV_E_INVARIANT;
  if (!draft_probs || !target_probs || !scratch || !norm_match_out || gamma < 1 || vocab < 1 ||
      row_stride < vocab)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_norm_match_rows: bad argument");
  if (top_m < 1 || top_m > vocab)
    return fail(ctx, DSDV_E_INVARIANT, "top_m %d outside [1, %d]", top_m, vocab);
  if (scratch_bytes < dsdv::norm_match_scratch_bytes(gamma, vocab, row_stride))
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_norm_match_rows: scratch too small");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  e = dsdv::launch_norm_match(draft_probs, target_probs, gamma, vocab, row_stride, top_m, scratch,
                              norm_match_out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "norm_match launch");
  ctx->launches += 1;
  return DSDV_OK;
}

dsdv_status dsdv_calibrate(dsdv_ctx *ctx, const dsdv_calib_item *items, int32_t n_items,
                           const double *rows, int64_t n_row_doubles,
                           const dsdv_key_criteria *points, int32_t n_points, double tau,
                           int32_t gamma, double budget, dsdv_grid_eval *out) {
  if (!ctx) return DSDV_E_INVARIANT;
  if (!items || n_items < 1 || !rows || !points || n_points < 1 || !out)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_calibrate: bad argument");
  if (gamma < 1 || gamma > 4)
    return fail(ctx, DSDV_E_UNSUPPORTED, "enumeration guard exceeded: need gamma <= 4");
  int maxV = 2, maxH = 1;
  for (int i = 0; i < n_items; ++i) {
    const dsdv_calib_item &it = items[i];
    if (it.vocab < 2 || it.vocab > 8 || it.horizon < 1 || it.horizon > 4)
      return fail(ctx, DSDV_E_UNSUPPORTED,
                  "enumeration guard exceeded: need vocab <= 8, 1 <= horizon <= 4");
    if (it.rows_offset < 0 ||
        it.rows_offset + (int64_t)2 * (it.vocab + 1) * it.vocab > n_row_doubles)
      return fail(ctx, DSDV_E_INVARIANT, "dsdv_calibrate: item %d rows out of range", i);
    maxV = it.vocab > maxV ? it.vocab : maxV;
    maxH = it.horizon > maxH ? it.horizon : maxH;
  }
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  const size_t per = dsdv::calib_scratch_doubles(maxV, maxH, gamma);
  const size_t nt = (size_t)n_points * n_items;
  const size_t bytes = n_items * sizeof(dsdv_calib_item) + n_row_doubles * sizeof(double) +
                       n_points * sizeof(dsdv_key_criteria) + nt * per * sizeof(double) +
                       2 * nt * sizeof(double) + nt * sizeof(int32_t) +
                       n_points * sizeof(dsdv_grid_eval) + 8 * 256;
  char *d = nullptr;
  e = cudaMalloc(&d, bytes);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(calibrate)");
  size_t off = 0;
  auto take = [&](size_t n) {
    char *p = d + off;
    off = (off + n + 255) & ~size_t(255);
    return p;
  };
  auto *d_items = reinterpret_cast<dsdv_calib_item *>(take(n_items * sizeof(dsdv_calib_item)));
  auto *d_rows = reinterpret_cast<double *>(take(n_row_doubles * sizeof(double)));
  auto *d_points = reinterpret_cast<dsdv_key_criteria *>(take(n_points * sizeof(dsdv_key_criteria)));
  auto *d_scratch = reinterpret_cast<double *>(take(nt * per * sizeof(double)));
  auto *d_len = reinterpret_cast<double *>(take(nt * sizeof(double)));
  auto *d_tv = reinterpret_cast<double *>(take(nt * sizeof(double)));
  auto *d_st = reinterpret_cast<int32_t *>(take(nt * sizeof(int32_t)));
  auto *d_out = reinterpret_cast<dsdv_grid_eval *>(take(n_points * sizeof(dsdv_grid_eval)));
  cudaMemcpy(d_items, items, n_items * sizeof(dsdv_calib_item), cudaMemcpyHostToDevice);
  cudaMemcpy(d_rows, rows, n_row_doubles * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(d_points, points, n_points * sizeof(dsdv_key_criteria), cudaMemcpyHostToDevice);
  e = dsdv::launch_calibrate(d_items, n_items, d_rows, d_points, n_points, tau, gamma, budget,
                             d_scratch, per, d_len, d_tv, d_st, d_out, nullptr);
  if (e == cudaSuccess)
    e = cudaMemcpy(out, d_out, n_points * sizeof(dsdv_grid_eval), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "calibrate");
  ctx->launches += 2;
  return DSDV_OK;
}

dsdv_status dsdv_streamed_bytes(dsdv_ctx *ctx, int reset, uint64_t *bytes) {
  if (!ctx || !bytes) return DSDV_E_INVARIANT;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  unsigned long long v = 0;
  e = cudaMemcpy(&v, ctx->streamed, sizeof(v), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "dsdv_streamed_bytes");
  *bytes = (uint64_t)v;
  if (reset) {
    e = cudaMemset(ctx->streamed, 0, sizeof(unsigned long long));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "dsdv_streamed_bytes reset");
  }
  return DSDV_OK;
}

dsdv_status dsdv_window_stats(dsdv_ctx *ctx, const dsdv_params *params, const void *draft_logits,
                              const void *target_logits, const int32_t *draft_tokens,
                              const dsdv_outputs *out, void *stream) {
  return run_fused(ctx, params, draft_logits, target_logits, draft_tokens, out, stream, true);
}

dsdv_status dsdv_sample_extra(dsdv_ctx *ctx, const dsdv_params *params, const void *draft_logits,
                              const void *target_logits, const double *records,
                              const int32_t *position, const double *uniform, int32_t *token_out,
                              int32_t *status, void *stream) {
  if (!ctx) return DSDV_E_INVARIANT;
  DevParams d;
  dsdv_status st = build_params(ctx, params, d);
  if (st != DSDV_OK) return st;
  if (!draft_logits || !target_logits || !records || !position || !uniform || !token_out || !status)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_sample_extra: null argument");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  switch (params->dtype) {
    case DSDV_DTYPE_BF16:
      e = dsdv::launch_sample_extra<__nv_bfloat16>(d, draft_logits, target_logits, records,
                                                   position, uniform, token_out, status,
                                                   (cudaStream_t)stream);
      break;
    case DSDV_DTYPE_F32:
      e = dsdv::launch_sample_extra<float>(d, draft_logits, target_logits, records, position,
                                           uniform, token_out, status, (cudaStream_t)stream);
      break;
    default:
      e = dsdv::launch_sample_extra<double>(d, draft_logits, target_logits, records, position,
                                            uniform, token_out, status, (cudaStream_t)stream);
      break;
  }
  if (e != cudaSuccess) return cuda_fail(ctx, e, "sample_extra launch");
  ctx->launches += 1;
  return DSDV_OK;
}

dsdv_status dsdv_shard_stats(dsdv_ctx *ctx, const dsdv_params *params, const void *draft_logits,
                             const void *target_logits, const int32_t *draft_tokens,
                             double *records, double *top_values, int32_t *top_ids,
                             void *stream) {
  if (!records || !top_values || !top_ids)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_shard_stats: records and top lists are required");
  dsdv_outputs out;
  std::memset(&out, 0, sizeof(out));
  out.records = records;
  return run_fused(ctx, params, draft_logits, target_logits, draft_tokens, &out, stream, true,
                   top_values, top_ids);
}

dsdv_status dsdv_dev_alloc(dsdv_ctx *ctx, uint64_t bytes, void **dev_ptr) {
  if (!ctx || !dev_ptr || !bytes) return DSDV_E_INVARIANT;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess) e = cudaMalloc(dev_ptr, bytes);
  if (e == cudaSuccess) e = cudaMemset(*dev_ptr, 0, bytes);
  return e == cudaSuccess ? DSDV_OK : cuda_fail(ctx, e, "dsdv_dev_alloc");
}

dsdv_status dsdv_dev_free(dsdv_ctx *ctx, void *dev_ptr) {
  if (!ctx) return DSDV_E_INVARIANT;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess) e = cudaFree(dev_ptr);
  return e == cudaSuccess ? DSDV_OK : cuda_fail(ctx, e, "dsdv_dev_free");
}

dsdv_status dsdv_ipc_handle(dsdv_ctx *ctx, void *dev_ptr, uint8_t handle[64]) {
  if (!ctx || !dev_ptr || !handle) return DSDV_E_INVARIANT;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, dev_ptr);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaIpcGetMemHandle");
  std::memcpy(handle, &h, 64);
  return DSDV_OK;
}

dsdv_status dsdv_ipc_open(dsdv_ctx *ctx, const uint8_t handle[64], void **dev_ptr) {
  if (!ctx || !dev_ptr || !handle) return DSDV_E_INVARIANT;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess) e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? DSDV_OK : cuda_fail(ctx, e, "cudaIpcOpenMemHandle");
}

dsdv_status dsdv_ipc_close(dsdv_ctx *ctx, void *dev_ptr) {
  if (!ctx) return DSDV_E_INVARIANT;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess) e = cudaIpcCloseMemHandle(dev_ptr);
  return e == cudaSuccess ? DSDV_OK : cuda_fail(ctx, e, "cudaIpcCloseMemHandle");
}

dsdv_status dsdv_shard_stats_peers(dsdv_ctx *ctx, const dsdv_params *params,
                                   const void *draft_logits, const void *target_logits,
                                   const int32_t *draft_tokens, int32_t nranks, int32_t rank,
                                   void *const *rank_bases, uint64_t rank_stride_bytes,
                                   uint64_t off_records, uint64_t off_top_values,
                                   uint64_t off_top_ids, void *stream) {
  if (!ctx) return DSDV_E_INVARIANT;
  if (nranks < 1 || nranks > DSDV_MAX_PEERS || rank < 0 || rank >= nranks || !rank_bases)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_shard_stats_peers: bad rank set (nranks <= %d)",
                DSDV_MAX_PEERS);
  if (off_records % 8 || off_top_values % 8 || off_top_ids % 4 || rank_stride_bytes % 8)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_shard_stats_peers: misaligned layout");
  for (int q = 0; q < nranks; ++q)
    if (!rank_bases[q]) return fail(ctx, DSDV_E_INVARIANT, "dsdv_shard_stats_peers: null base");
  char *own = (char *)rank_bases[rank] + (size_t)rank * rank_stride_bytes;
  long long delta[DSDV_MAX_PEERS];
  int np = 0;
  for (int q = 0; q < nranks; ++q)
    if (q != rank)
      delta[np++] = (long long)(((char *)rank_bases[q] + (size_t)rank * rank_stride_bytes) - own);
  dsdv_outputs out;
  std::memset(&out, 0, sizeof(out));
  out.records = (double *)(own + off_records);
  return run_fused(ctx, params, draft_logits, target_logits, draft_tokens, &out, stream, true,
                   (double *)(own + off_top_values), (int32_t *)(own + off_top_ids), np, delta);
}

dsdv_status dsdv_peer_signal(dsdv_ctx *ctx, int32_t nranks, int32_t rank,
                             void *const *rank_bases, uint64_t rank_stride_bytes, uint64_t epoch,
                             void *stream) {
  if (!ctx || nranks < 1 || nranks > DSDV_MAX_PEERS || rank < 0 || rank >= nranks || !rank_bases)
    return DSDV_E_INVARIANT;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess)
    e = dsdv::launch_peer_signal((char *const *)rank_bases, nranks, rank,
                                 (unsigned long long)rank_stride_bytes, (unsigned long long)epoch,
                                 (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "peer signal launch");
  ctx->launches += 1;
  return DSDV_OK;
}

dsdv_status dsdv_peer_wait(dsdv_ctx *ctx, int32_t nranks, void *local_base,
                           uint64_t rank_stride_bytes, uint64_t epoch, uint64_t timeout_ns,
                           int32_t *status, void *stream) {
  if (!ctx || nranks < 1 || nranks > DSDV_MAX_PEERS || !local_base) return DSDV_E_INVARIANT;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess)
    e = dsdv::launch_peer_wait(
        (const unsigned long long *)((char *)local_base + (size_t)nranks * rank_stride_bytes),
        nranks, (unsigned long long)epoch, (unsigned long long)timeout_ns, status,
        (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "peer wait launch");
  ctx->launches += 1;
  return DSDV_OK;
}

static dsdv_status shard_merge_impl(dsdv_ctx *ctx, const dsdv_params *params, int32_t nranks,
                                    const double *records_all, const double *top_values_all,
                                    const int32_t *top_ids_all, uint64_t rank_stride_bytes,
                                    const void *draft_logits, const void *target_logits,
                                    const int32_t *draft_tokens, const dsdv_outputs *out,
                                    int32_t *position, double *uniform, double *mass_out,
                                    double *tile_scratch, void *stream,
                                    const long long *mass_delta, int n_delta) {
  if (!ctx) return DSDV_E_INVARIANT;
  DevParams d;
  dsdv_status st = build_params(ctx, params, d);
  if (st != DSDV_OK) return st;
  if (!records_all || !top_values_all || !top_ids_all || !draft_tokens || !out || !position ||
      !uniform || !mass_out || !draft_logits || !target_logits || !out->records ||
      !out->accepted_count || !out->extra_token ||
      !out->extra_source || !out->key_count || !out->status || !out->near_threshold)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_shard_merge: null argument");
  if (nranks < 1 || nranks > 64)
    return fail(ctx, DSDV_E_UNSUPPORTED, "dsdv_shard_merge: 1..64 ranks, got %d", nranks);
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  const DevOut o = to_dev(out);
  switch (params->dtype) {
    case DSDV_DTYPE_BF16:
      e = dsdv::launch_shard_merge<__nv_bfloat16>(d, records_all, top_values_all, top_ids_all,
                                                  nranks, (size_t)rank_stride_bytes, draft_logits,
                                                  target_logits, draft_tokens, o, position,
                                                  uniform, mass_out, tile_scratch, (cudaStream_t)stream,
                                                  mass_delta, n_delta);
      break;
    case DSDV_DTYPE_F32:
      e = dsdv::launch_shard_merge<float>(d, records_all, top_values_all, top_ids_all, nranks,
                                          (size_t)rank_stride_bytes, draft_logits, target_logits,
                                          draft_tokens, o, position, uniform, mass_out,
                                          tile_scratch, (cudaStream_t)stream, mass_delta, n_delta);
      break;
    default:
      e = dsdv::launch_shard_merge<double>(d, records_all, top_values_all, top_ids_all, nranks,
                                           (size_t)rank_stride_bytes, draft_logits, target_logits,
                                           draft_tokens, o, position, uniform, mass_out,
                                           tile_scratch, (cudaStream_t)stream, mass_delta,
                                           n_delta);
      break;
  }
  if (e != cudaSuccess) return cuda_fail(ctx, e, "shard_merge launch");
  ctx->launches += 1;
  return DSDV_OK;
}

dsdv_status dsdv_shard_merge(dsdv_ctx *ctx, const dsdv_params *params, int32_t nranks,
                             const double *records_all, const double *top_values_all,
                             const int32_t *top_ids_all, uint64_t rank_stride_bytes,
                             const void *draft_logits, const void *target_logits,
                             const int32_t *draft_tokens, const dsdv_outputs *out,
                             int32_t *position, double *uniform, double *mass_out,
                             double *tile_scratch, void *stream) {
  return shard_merge_impl(ctx, params, nranks, records_all, top_values_all, top_ids_all,
                          rank_stride_bytes, draft_logits, target_logits, draft_tokens, out,
                          position, uniform, mass_out, tile_scratch, stream, nullptr, 0);
}

static dsdv_status shard_sample_impl(dsdv_ctx *ctx, const dsdv_params *params, int32_t mode,
                                     int32_t rank, int32_t nranks, const void *draft_logits,
                                     const void *target_logits, const double *records,
                                     const int32_t *position, const double *uniform,
                                     const double *masses_all, double *mass_out,
                                     int32_t *token_out, int32_t *status,
                                     const double *tile_scratch, void *stream,
                                     const long long *tok_delta, int n_delta, size_t mstride) {
  if (!ctx) return DSDV_E_INVARIANT;
  DevParams d;
  dsdv_status st = build_params(ctx, params, d);
  if (st != DSDV_OK) return st;
  if (mode != DSDV_SHARD_MASS && mode != DSDV_SHARD_RESOLVE)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_shard_sample: unknown mode %d", mode);
  if (!draft_logits || !target_logits || !records || !position || !uniform ||
      (mode == DSDV_SHARD_MASS && !mass_out) ||
      (mode == DSDV_SHARD_RESOLVE && (!masses_all || !token_out || !status)))
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_shard_sample: null argument");
  if (rank < 0 || rank >= nranks)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_shard_sample: rank %d of %d", rank, nranks);
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  switch (params->dtype) {
    case DSDV_DTYPE_BF16:
      e = dsdv::launch_shard_sample<__nv_bfloat16>(d, mode, rank, nranks, draft_logits,
                                                   target_logits, records, position, uniform,
                                                   masses_all, mass_out, token_out, status,
                                                   tile_scratch, (cudaStream_t)stream, tok_delta,
                                                   n_delta, mstride);
      break;
    case DSDV_DTYPE_F32:
      e = dsdv::launch_shard_sample<float>(d, mode, rank, nranks, draft_logits, target_logits,
                                           records, position, uniform, masses_all, mass_out,
                                           token_out, status, tile_scratch, (cudaStream_t)stream,
                                           tok_delta, n_delta, mstride);
      break;
    default:
      e = dsdv::launch_shard_sample<double>(d, mode, rank, nranks, draft_logits, target_logits,
                                            records, position, uniform, masses_all, mass_out,
                                            token_out, status, tile_scratch, (cudaStream_t)stream,
                                            tok_delta, n_delta, mstride);
      break;
  }
  if (e != cudaSuccess) return cuda_fail(ctx, e, "shard_sample launch");
  ctx->launches += 1;
  return DSDV_OK;
}

dsdv_status dsdv_shard_sample(dsdv_ctx *ctx, const dsdv_params *params, int32_t mode, int32_t rank,
                              int32_t nranks, const void *draft_logits, const void *target_logits,
                              const double *records, const int32_t *position,
                              const double *uniform, const double *masses_all, double *mass_out,
                              int32_t *token_out, int32_t *status, const double *tile_scratch,
                              void *stream) {
  return shard_sample_impl(ctx, params, mode, rank, nranks, draft_logits, target_logits, records,
                           position, uniform, masses_all, mass_out, token_out, status,
                           tile_scratch, stream, nullptr, 0, 0);
}

// slot `rank` of every rank's exchange buffer, relative to this rank's own slot
static int peer_deltas(void *const *rank_bases, int nranks, int rank, uint64_t stride,
                       long long *delta) {
  const char *own = (const char *)rank_bases[rank] + (size_t)rank * stride;
  int np = 0;
  for (int q = 0; q < nranks; ++q)
    if (q != rank) delta[np++] = (long long)(((const char *)rank_bases[q] + (size_t)rank * stride) - own);
  return np;
}

dsdv_status dsdv_shard_merge_peers(dsdv_ctx *ctx, const dsdv_params *params, int32_t nranks,
                                   int32_t rank, void *const *rank_bases,
                                   uint64_t rank_stride_bytes, uint64_t off_records,
                                   uint64_t off_top_values, uint64_t off_top_ids,
                                   uint64_t off_mass, const void *draft_logits,
                                   const void *target_logits, const int32_t *draft_tokens,
                                   const dsdv_outputs *out, int32_t *position, double *uniform,
                                   double *tile_scratch, void *stream) {
  if (!ctx) return DSDV_E_INVARIANT;
  if (nranks < 1 || nranks > DSDV_MAX_PEERS || rank < 0 || rank >= nranks || !rank_bases ||
      off_mass % 8 || rank_stride_bytes % 8)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_shard_merge_peers: bad rank set or layout");
  const char *local = (const char *)rank_bases[rank];
  long long delta[DSDV_MAX_PEERS];
  const int np = peer_deltas(rank_bases, nranks, rank, rank_stride_bytes, delta);
  double *mass_own = (double *)(local + (size_t)rank * rank_stride_bytes + off_mass);
  return shard_merge_impl(ctx, params, nranks, (const double *)(local + off_records),
                          (const double *)(local + off_top_values),
                          (const int32_t *)(local + off_top_ids), rank_stride_bytes, draft_logits,
                          target_logits, draft_tokens, out, position, uniform, mass_own,
                          tile_scratch, stream, delta, np);
}

dsdv_status dsdv_shard_resolve_peers(dsdv_ctx *ctx, const dsdv_params *params, int32_t nranks,
                                     int32_t rank, void *const *rank_bases,
                                     uint64_t rank_stride_bytes, uint64_t off_mass,
                                     uint64_t off_tokens, const void *draft_logits,
                                     const void *target_logits, const double *records,
                                     const int32_t *position, const double *uniform,
                                     int32_t *status, const double *tile_scratch, void *stream) {
  if (!ctx) return DSDV_E_INVARIANT;
  if (nranks < 1 || nranks > DSDV_MAX_PEERS || rank < 0 || rank >= nranks || !rank_bases ||
      off_mass % 8 || off_tokens % 4 || rank_stride_bytes % 8)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_shard_resolve_peers: bad rank set or layout");
  const char *local = (const char *)rank_bases[rank];
  long long delta[DSDV_MAX_PEERS];
  const int np = peer_deltas(rank_bases, nranks, rank, rank_stride_bytes, delta);
  int32_t *tok_own = (int32_t *)(local + (size_t)rank * rank_stride_bytes + off_tokens);
  return shard_sample_impl(ctx, params, DSDV_SHARD_RESOLVE, rank, nranks, draft_logits,
                           target_logits, records, position, uniform,
                           (const double *)(local + off_mass), nullptr, tok_own, status,
                           tile_scratch, stream, delta, np, (size_t)(rank_stride_bytes / 8));
}

dsdv_status dsdv_peer_tokens_max(dsdv_ctx *ctx, int32_t nranks, void *local_base,
                                 uint64_t rank_stride_bytes, uint64_t off_tokens, int32_t batch,
                                 int32_t *token_out, void *stream) {
  if (!ctx || nranks < 1 || nranks > DSDV_MAX_PEERS || !local_base || !token_out || batch < 1 ||
      off_tokens % 4 || rank_stride_bytes % 4)
    return DSDV_E_INVARIANT;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess)
    e = dsdv::launch_tokens_max((const int32_t *)((const char *)local_base + off_tokens),
                                (size_t)(rank_stride_bytes / 4), nranks, batch, token_out,
                                (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "tokens max launch");
  ctx->launches += 1;
  return DSDV_OK;
}

// Exchange layout of one rank's slot (paper_2511_11733_b200/sharded.py
// ShardedVerifier.exchange_layout): packed records, top values, top ids, then
// [B] slice masses and [B] RESOLVE tokens.
static void exchange_layout(int B, int G, int M, uint64_t *o_rec, uint64_t *o_tv, uint64_t *o_ti,
                            uint64_t *o_mass, uint64_t *o_tok, uint64_t *size) {
  const uint64_t n_rec = (uint64_t)B * (G + 1) * DSDV_RECORD_WORDS * 8;
  const uint64_t n_tv = (uint64_t)B * G * 2 * M * 8;
  const uint64_t n_ti = (uint64_t)B * G * 2 * M * 4;
  *o_rec = 0;
  *o_tv = n_rec;
  *o_ti = n_rec + n_tv;
  const uint64_t packed = (n_rec + n_tv + n_ti + 7) / 8 * 8;
  *o_mass = (packed + 7) / 8 * 8;
  *o_tok = *o_mass + 8ull * B;
  *size = *o_tok + 4ull * B;
}

uint64_t dsdv_shard_exchange_bytes(int32_t batch, int32_t gamma, int32_t top_m) {
  uint64_t a, b, c, d, e, size;
  exchange_layout(batch, gamma, top_m, &a, &b, &c, &d, &e, &size);
  return size;
}

dsdv_status dsdv_shard_verify_peers(dsdv_ctx *ctx, const dsdv_params *params,
                                    const void *draft_logits, const void *target_logits,
                                    const int32_t *draft_tokens, int32_t nranks, int32_t rank,
                                    void *const *buffer_bases, uint64_t rank_stride_bytes,
                                    uint64_t window_epoch, uint64_t timeout_ns,
                                    const dsdv_outputs *out, void *stream) {
  if (!ctx || !params) return DSDV_E_INVARIANT;
  if (nranks < 1 || nranks > DSDV_MAX_PEERS || rank < 0 || rank >= nranks || !buffer_bases ||
      window_epoch < 1 || !out || !out->records || !out->status || !out->extra_token)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_shard_verify_peers: bad argument");
  const int B = params->batch, G = params->gamma;
  const int M = params->top_m < params->vocab ? params->top_m : params->vocab;
  uint64_t o_rec, o_tv, o_ti, o_mass, o_tok, size;
  exchange_layout(B, G, M, &o_rec, &o_tv, &o_ti, &o_mass, &o_tok, &size);
  if (rank_stride_bytes < size || rank_stride_bytes % 256)
    return fail(ctx, DSDV_E_INVARIANT,
                "dsdv_shard_verify_peers: rank stride %llu below the exchange size %llu",
                (unsigned long long)rank_stride_bytes, (unsigned long long)size);
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  // scratch: position [B] i32, u [B] f64, tiles [B][TILE_WORDS] f64, peer status i32
  const size_t need = 256 + (size_t)B * 4 + 256 + (size_t)B * 8 + 256 +
                      (size_t)B * DSDV_SHARD_TILE_WORDS * 8 + 256 + 4;
  if (need > ctx->shard_scratch_cap) {
    if (ctx->shard_scratch) cudaFree(ctx->shard_scratch);
    ctx->shard_scratch = nullptr;
    e = cudaMalloc(&ctx->shard_scratch, need);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(shard scratch)");
    ctx->shard_scratch_cap = need;
  }
  char *sp = (char *)ctx->shard_scratch;
  auto take = [&](size_t n) {
    char *q = sp;
    sp += (n + 255) & ~size_t(255);
    return q;
  };
  int32_t *position = (int32_t *)take((size_t)B * 4);
  double *u = (double *)take((size_t)B * 8);
  double *tiles = (double *)take((size_t)B * DSDV_SHARD_TILE_WORDS * 8);
  int32_t *peer_status = (int32_t *)take(4);
  const uint64_t set_bytes = (uint64_t)nranks * rank_stride_bytes;
  void *sets[DSDV_MAX_PEERS];
  for (int q = 0; q < nranks; ++q) sets[q] = (char *)buffer_bases[q] + (window_epoch & 1) * set_bytes;
  // the arrival flags: nranks * stride past the second set of each buffer
  // (where dsdv_peer_signal / dsdv_peer_wait find them too)
  char *flag_bases[DSDV_MAX_PEERS];
  for (int q = 0; q < nranks; ++q) flag_bases[q] = (char *)buffer_bases[q] + set_bytes;
  const unsigned long long *own_flags =
      (const unsigned long long *)((char *)buffer_bases[rank] + 2 * set_bytes);
  const uint64_t f = 3 * window_epoch;
  cudaStream_t cs = (cudaStream_t)stream;
  // one launch per flag round: signal, then wait (the first round of the
  // window also clears the timeout status)
  auto round = [&](uint64_t epoch, int reset) -> dsdv_status {
    cudaError_t re = dsdv::launch_peer_round(flag_bases, nranks, rank,
                                             (unsigned long long)rank_stride_bytes, epoch,
                                             own_flags, timeout_ns, peer_status, reset, cs);
    if (re != cudaSuccess) return cuda_fail(ctx, re, "peer round launch");
    ctx->launches += 1;
    return DSDV_OK;
  };
  // 1. stats pass: the records land in every rank's set as items complete
  dsdv_status st = dsdv_shard_stats_peers(ctx, params, draft_logits, target_logits, draft_tokens,
                                          nranks, rank, sets, rank_stride_bytes, o_rec, o_tv,
                                          o_ti, stream);
  if (st == DSDV_OK) st = round(f, 1);
  // 2. merge (identical on every rank) + this slice's extra-draw masses
  if (st == DSDV_OK)
    st = dsdv_shard_merge_peers(ctx, params, nranks, rank, sets, rank_stride_bytes, o_rec, o_tv,
                                o_ti, o_mass, draft_logits, target_logits, draft_tokens, out,
                                position, u, tiles, stream);
  if (st == DSDV_OK) st = round(f + 1, 0);
  // 3. the owning slice resolves the extra token; tokens max over the ranks
  if (st == DSDV_OK)
    st = dsdv_shard_resolve_peers(ctx, params, nranks, rank, sets, rank_stride_bytes, o_mass,
                                  o_tok, draft_logits, target_logits, out->records, position, u,
                                  out->status, tiles, stream);
  if (st == DSDV_OK) st = round(f + 2, 0);
  if (st != DSDV_OK) return st;
  // 4. tokens max, and a timed-out flag round fails every sequence
  e = dsdv::launch_tokens_fold((const int32_t *)((const char *)sets[rank] + o_tok),
                               (size_t)(rank_stride_bytes / 4), nranks, B, out->extra_token,
                               peer_status, out->status, cs);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "tokens fold launch");
  ctx->launches += 1;
  return DSDV_OK;
}

dsdv_status dsdv_pipeline_run(dsdv_ctx *ctx, int32_t n_stages, int32_t nranks, int32_t rank,
                              void *const *buffer_bases, uint64_t rank_stride_bytes,
                              const uint64_t *compute_ns, int32_t n_units, uint64_t t1_ns,
                              uint64_t run_index, uint64_t timeout_ns, int32_t *status,
                              void *stream) {
  if (!ctx || n_stages < 1 || nranks < 1 || nranks > DSDV_MAX_PEERS || rank < 0 ||
      rank >= nranks || !compute_ns || n_units < 0 || run_index < 1 || run_index >= (1ull << 31) ||
      (nranks > 1 && (!buffer_bases || rank_stride_bytes < 64 || rank_stride_bytes % 8)))
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_pipeline_run: bad argument");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  cudaStream_t st = (cudaStream_t)stream;
  // this rank's own committed-token payload: slot `rank` of its set 0 (never a
  // peer's destination)
  int32_t *payload =
      nranks > 1 ? (int32_t *)((char *)buffer_bases[rank] + (size_t)rank * rank_stride_bytes)
                 : nullptr;
  const uint64_t flags_off = 2ull * nranks * rank_stride_bytes;
  uint32_t sent[DSDV_MAX_PEERS] = {0}, recvd[DSDV_MAX_PEERS] = {0};
  const uint64_t base = run_index << 32;
  auto owner = [&](int s) { return s % nranks; };
  auto send = [&](int dst, uint64_t t1) -> cudaError_t {
    ++sent[dst];
    int32_t *dst_slot = (int32_t *)((char *)buffer_bases[dst] + (size_t)rank * rank_stride_bytes);
    unsigned long long *dst_flag =
        (unsigned long long *)((char *)buffer_bases[dst] + flags_off) + rank;
    return dsdv::launch_hop_send(t1, dst_slot, payload, dst_flag, base | sent[dst], st);
  };
  auto recv = [&](int src) -> cudaError_t {
    ++recvd[src];
    const unsigned long long *flag =
        (const unsigned long long *)((char *)buffer_bases[rank] + flags_off) + src;
    const int32_t *slot = (const int32_t *)((char *)buffer_bases[rank] + (size_t)src * rank_stride_bytes);
    return dsdv::launch_hop_recv(flag, base | recvd[src], timeout_ns, status, slot, payload, st);
  };
  size_t launches = 0;
  for (int u = 0; u < n_units && e == cudaSuccess; ++u) {
    for (int s = 0; s < n_stages && e == cudaSuccess; ++s) {
      if (owner(s) != rank) continue;
      if (s == 0) {
        if (compute_ns[u]) {
          e = dsdv::launch_spin(compute_ns[u], st);  // the unit's compute (k t0 or t0)
          ++launches;
        }
      } else if (owner(s - 1) != rank) {
        e = recv(owner(s - 1));
        ++launches;
      }
      if (e != cudaSuccess || s == n_stages - 1) continue;
      if (owner(s + 1) != rank) {
        e = send(owner(s + 1), t1_ns);  // t1 spin, then the NVLink store
      } else if (t1_ns) {
        e = dsdv::launch_spin(t1_ns, st);  // next stage on this GPU: the latency only
      }
      ++launches;
    }
    // back edge: the committed tokens return to stage 0 for the next unit
    if (e == cudaSuccess && owner(n_stages - 1) != owner(0)) {
      if (rank == owner(n_stages - 1)) {
        e = send(owner(0), 0);
        ++launches;
      } else if (rank == owner(0)) {
        e = recv(owner(n_stages - 1));
        ++launches;
      }
    }
  }
  if (e != cudaSuccess) return cuda_fail(ctx, e, "pipeline hop launch");
  ctx->launches += launches;
  return DSDV_OK;
}

dsdv_status dsdv_enable_peer_access(dsdv_ctx *ctx, int32_t peer_device) {
  if (!ctx) return DSDV_E_INVARIANT;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  int ok = 0;
  e = cudaDeviceCanAccessPeer(&ok, ctx->device, peer_device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaDeviceCanAccessPeer");
  if (!ok) return fail(ctx, DSDV_E_UNSUPPORTED, "device %d cannot access device %d", ctx->device,
                       peer_device);
  e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    e = cudaSuccess;
  }
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaDeviceEnablePeerAccess");
  return DSDV_OK;
}

dsdv_status dsdv_log_rows(dsdv_ctx *ctx, double *values, uint64_t count, void *stream) {
  if (!ctx || (!values && count)) return DSDV_E_INVARIANT;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess) e = dsdv::launch_log_rows(values, (size_t)count, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "log rows launch");
  ctx->launches += 1;
  return DSDV_OK;
}

dsdv_status dsdv_spin(dsdv_ctx *ctx, uint64_t nanoseconds, void *stream) {
  if (!ctx) return DSDV_E_INVARIANT;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  e = dsdv::launch_spin((unsigned long long)nanoseconds, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "spin launch");
  ctx->launches += 1;
  return DSDV_OK;
}

dsdv_status dsdv_mix_rows(dsdv_ctx *ctx, int32_t kind, int32_t vocab, const double *a,
                          const double *b, double tau, double *out, int32_t *status,
                          void *stream) {
  if (!ctx) return DSDV_E_INVARIANT;
  if (kind != DSDV_MIX_SOFTEN && kind != DSDV_MIX_RESIDUAL)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_mix_rows: unknown kind %d", kind);
  if (vocab < 1 || !a || !b || !out || !status)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_mix_rows: bad argument");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  e = dsdv::launch_mix_rows(kind, vocab, a, b, tau, out, status, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "mix_rows launch");
  ctx->launches += 1;
  return DSDV_OK;
}

dsdv_status dsdv_draft_sample(dsdv_ctx *ctx, const dsdv_params *params, const void *draft_logits,
                              int32_t *draft_tokens, void *stream) {
  return dsdv_draft_sample_temperature(ctx, params, 1.0, draft_logits, draft_tokens, stream);
}

dsdv_status dsdv_draft_sample_temperature(dsdv_ctx *ctx, const dsdv_params *params,
                                          double temperature, const void *draft_logits,
                                          int32_t *draft_tokens, void *stream) {
  if (!ctx) return DSDV_E_INVARIANT;
  if (!(std::isfinite(temperature) && temperature >= 0.0))
    return fail(ctx, DSDV_E_INVARIANT, "temperature must be a finite non-negative real, got %s",
                std::to_string(temperature).c_str());
  DevParams d;
  dsdv_status st = build_params(ctx, params, d);
  if (st != DSDV_OK) return st;
  if (params->vocab_local != params->vocab || params->vocab_offset != 0)
    return fail(ctx, DSDV_E_UNSUPPORTED, "dsdv_draft_sample needs the whole vocabulary");
  if (!draft_logits || !draft_tokens)
    return fail(ctx, DSDV_E_INVARIANT, "dsdv_draft_sample: null argument");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  switch (params->dtype) {
    case DSDV_DTYPE_BF16:
      e = dsdv::launch_draft_sample<__nv_bfloat16>(d, draft_logits, draft_tokens, temperature,
                                                   (cudaStream_t)stream);
      break;
    case DSDV_DTYPE_F32:
      e = dsdv::launch_draft_sample<float>(d, draft_logits, draft_tokens, temperature,
                                           (cudaStream_t)stream);
      break;
    default:
      e = dsdv::launch_draft_sample<double>(d, draft_logits, draft_tokens, temperature,
                                            (cudaStream_t)stream);
      break;
  }
  if (e != cudaSuccess) return cuda_fail(ctx, e, "draft_sample launch");
  ctx->launches += 1;
  return DSDV_OK;
}

dsdv_status dsdv_synth_logits(dsdv_ctx *ctx, const dsdv_params *params, uint64_t logits_seed,
                              void *draft_logits, void *target_logits, void *stream) {
  if (!ctx) return DSDV_E_INVARIANT;
  dsdv_status st = dsdv_validate(ctx, params);
  if (st != DSDV_OK) return st;
  if (params->dtype == DSDV_DTYPE_F64)
    return fail(ctx, DSDV_E_UNSUPPORTED, "synthetic logits are f32 or bf16");
  if (params->vocab_local != params->vocab)
    return fail(ctx, DSDV_E_UNSUPPORTED, "synthetic logits cover the whole vocabulary");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  e = dsdv::launch_synth(params->dtype, params->batch, params->gamma, params->vocab,
                         params->row_stride, logits_seed, draft_logits, target_logits,
                         (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "synth launch");
  ctx->launches += 1;
  return DSDV_OK;
}

dsdv_status dsdv_sync(dsdv_ctx *ctx, const dsdv_params *params, const int32_t *status,
                      void *stream) {
  if (!ctx) return DSDV_E_INVARIANT;
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamSynchronize");
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel");
  if (!status || !params) return DSDV_OK;
  std::vector<int32_t> h((size_t)params->batch);
  e = cudaMemcpy(h.data(), status, h.size() * sizeof(int32_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemcpy(status)");
  for (size_t b = 0; b < h.size(); ++b) {
    switch (h[b]) {
      case DSDV_OK:
        continue;
      case DSDV_E_INVARIANT:
        return fail(ctx, DSDV_E_INVARIANT,
                    "sequence %zu: a logit row has no finite mass or a draft token lies outside "
                    "the vocabulary of size %d",
                    b, params->vocab);
      case DSDV_E_DEGENERATE_MIXTURE:
        return fail(ctx, DSDV_E_DEGENERATE_MIXTURE,
                    "softened distribution has zero mass: target and draft supports are "
                    "disjoint (sequence %zu)",
                    b);
      case DSDV_E_DRAFTING_CONTRACT:
        return fail(ctx, DSDV_E_DRAFTING_CONTRACT,
                    "drafted token has zero draft probability; it cannot have been drafted "
                    "(sequence %zu)",
                    b);
      case DSDV_E_EMPTY_RESIDUAL:
        return fail(ctx, DSDV_E_EMPTY_RESIDUAL,
                    "residual is empty: effective and draft distributions match (sequence %zu)",
                    b);
      default:
        return fail(ctx, (dsdv_status)h[b], "sequence %zu failed with status %d", b, h[b]);
    }
  }
  return DSDV_OK;
}

}  // extern "C"
