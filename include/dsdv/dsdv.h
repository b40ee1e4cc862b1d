/* dsdv — C-ABI of the B200 adaptive speculative verifier (DSD, arXiv 2511.11733).
 *
 * This is the drop-in boundary between host code (the C++ `dsd::` API in
 * include/dsd/, Python ctypes, or any FFI) and the sm_100a kernels in
 * paper_2511_11733_b200/csrc/. No C++ or torch types cross it: plain pointers,
 * sizes and POD structs only. All device pointers are caller-owned.
 *
 * Reference interfaces replaced (paths relative to /root/reference):
 *   dsdv_verify          <- dsd::verify_round        proj/src/verifier.cpp:215-257
 *                           (whole window: is_key :136-159, soften :161-186,
 *                            accept_prob :188-196, first-rejection break :223-250,
 *                            residual_distribution :198-213, bonus draw :253-256)
 *   dsdv_window_stats    <- the per-position front half of the same loop
 *                           (token_cross_entropy :112-117, norm_match :119-134,
 *                            is_key, soften's normaliser, accept_prob) for callers
 *                            that own their UniformStream (proj/include/dsd/rng.hpp:25-29)
 *   dsdv_sample_extra    <- residual_distribution + sample (verifier.cpp:245-246)
 *                           and the bonus draw (verifier.cpp:253-256) with
 *                           sample_with_uniform semantics (distribution.cpp:103-114)
 *   dsdv_draft_sample    <- draft_window's per-position inverse-CDF draw
 *                           (verifier.cpp:93-110 -> distribution.cpp:99-114)
 *   dsdv_status codes    <- dsd::Error tree (proj/include/dsd/error.hpp:24-71)
 *   dsdv_uniform         <- UniformStream::next_uniform (rng.hpp:25-40), counter form
 *
 * Data layout in HBM (row-major, vocabulary contiguous):
 *   draft_logits [batch][gamma    ][row_stride]
 *   target_logits[batch][gamma + 1][row_stride]   (row gamma feeds the bonus draw)
 *   draft_tokens [batch][gamma] int32
 * Only the first vocab_local entries of a row are read as logits; the kernels
 * stream rows with 1-D bulk (TMA) copies, so row_stride * sizeof(dtype) must be a
 * multiple of 16 bytes and the base pointers 16-byte aligned.
 *
 * Inputs are logits (natural-log scale, -inf allowed for unsupported tokens).
 * The reference works on probability vectors; P = softmax(logits) is the
 * front end it lacks (its Distribution::from_weights, distribution.cpp:54-63).
 */
#ifndef DSDV_DSDV_H_
#define DSDV_DSDV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSDV_ABI_VERSION 1

typedef struct dsdv_ctx dsdv_ctx; /* one per host thread / stream; no globals */

typedef enum {
  DSDV_OK = 0,
  DSDV_E_INVARIANT = 1,          /* dsd::InvariantError          error.hpp:30 */
  DSDV_E_DEGENERATE_MIXTURE = 2, /* dsd::DegenerateMixtureError  error.hpp:41 */
  DSDV_E_DRAFTING_CONTRACT = 3,  /* dsd::DraftingContractError   error.hpp:47 */
  DSDV_E_EMPTY_RESIDUAL = 4,     /* dsd::EmptyResidualError      error.hpp:53 */
  DSDV_E_CUDA = 5,               /* device / driver failure (no reference analogue) */
  DSDV_E_NCCL = 6,               /* collective failure (sharded verifier) */
  DSDV_E_UNSUPPORTED = 7         /* shape outside what the kernels accept */
} dsdv_status;

typedef enum { DSDV_DTYPE_F32 = 0, DSDV_DTYPE_BF16 = 1, DSDV_DTYPE_F64 = 2 } dsdv_dtype;

/* Order of dsd::ExtraSource (verifier.hpp:65-68). */
typedef enum { DSDV_EXTRA_BONUS = 0, DSDV_EXTRA_RESIDUAL = 1 } dsdv_extra_source;

/* Kind of effective distribution used at a position (verifier.cpp:231-233,
 * soften's short-circuits :170-172). */
typedef enum {
  DSDV_EFF_TARGET = 0,   /* key token, tau == 0, or target row == draft row */
  DSDV_EFF_DRAFT = 1,    /* non-key, tau == 1 */
  DSDV_EFF_SOFTENED = 2  /* non-key, 0 < tau < 1: softmax((1-tau) l_t + tau l_d) */
} dsdv_effective_kind;

typedef struct {
  int32_t batch;        /* B >= 1 */
  int32_t gamma;        /* draft window length >= 1           (VerifyParams::gamma) */
  int32_t vocab;        /* V >= 2, global vocabulary size */
  int32_t row_stride;   /* elements between consecutive rows */
  int32_t dtype;        /* dsdv_dtype of the logits; F64 computes in fp64 */
  int32_t top_m;        /* >= 1, clamped to V at use           (KeyCriteria::top_m) */
  double tau;           /* [0, 1]                              (VerifyParams::tau) */
  double ratio_limit;   /* > 0, may be +inf                    (KeyCriteria) */
  double gap_limit;     /* [0, 1] */
  double overlap_floor; /* [0, 1] */
  uint64_t seed;        /* Philox key (include/dsdv/philox.h) */
  uint64_t window;      /* Philox counter words 2-3: verification window index */
  uint32_t sequence_offset; /* Philox counter word 1 = sequence_offset + b */
  int32_t vocab_offset; /* sharded verifier: first global id of this slice (0 when unsharded) */
  int32_t vocab_local;  /* sharded verifier: ids in this slice (== vocab when unsharded) */
  double eps_u;         /* near-threshold band for |u - a| (counted, reported) */
  double eps_lambda;    /* relative band for |clause - lambda| */
} dsdv_params;

/* Per-position record kept between dsdv_window_stats and dsdv_sample_extra
 * (natural-log normalisers of P_t, P_d and the softened mix, and the kind of
 * effective distribution). Layout: double[batch][gamma + 1][DSDV_RECORD_WORDS]. */
#define DSDV_RECORD_WORDS 8

typedef struct {
  /* per sequence, [batch] (required by dsdv_verify, ignored by window_stats) */
  int32_t *accepted_count;   /* k (VerificationResult::accepted_count) */
  int32_t *extra_token;      /* VerificationResult::extra_token */
  uint8_t *extra_source;     /* dsdv_extra_source */
  int32_t *key_count;        /* key tokens among the evaluated positions */
  int32_t *status;           /* dsdv_status of the sequence (0 = ok) */
  int32_t *near_threshold;   /* evaluated draws/clauses inside the eps bands */
  /* per position, [batch][gamma], optional (NULL skips). Positions past the
   * first rejection are computed too but are not part of the round. */
  uint8_t *key_mask;         /* TokenDecision::is_key */
  uint8_t *accepted;         /* TokenDecision::accepted (u < accept_prob) */
  double *accept_prob;       /* TokenDecision::accept_prob */
  double *h_target;          /* -ln P_t(y)   (token_cross_entropy) */
  double *h_draft;           /* -ln P_d(y) */
  double *p_target_y;        /* P_t(y) */
  double *p_draft_y;         /* P_d(y) */
  double *norm_match;        /* top-m overlap, multiple of 1/m */
  double *p_effective_y;     /* P_eff(y): P_t for key tokens, softened otherwise */
  double *uniform;           /* the accept draw u at this position */
  /* [batch][gamma + 1][DSDV_RECORD_WORDS], optional for dsdv_verify,
   * required by dsdv_window_stats -> dsdv_sample_extra */
  double *records;
} dsdv_outputs;

/* ---- lifetime ---------------------------------------------------------- */
dsdv_status dsdv_create(int device, dsdv_ctx **out);
dsdv_status dsdv_destroy(dsdv_ctx *ctx);
/* Message of the last failing call on ctx; with ctx == NULL, of the last
 * context-free call (dsdv_validate(NULL, ...)) on this host thread. */
const char *dsdv_last_error(const dsdv_ctx *ctx);
int dsdv_abi_version(void);

/* Host-side validation only (VerifyParams::validate, verifier.cpp:55-91, plus
 * layout checks). Every entry point below runs it before launching. ctx may
 * be NULL (no device needed). */
dsdv_status dsdv_validate(dsdv_ctx *ctx, const dsdv_params *params);

/* ---- the hot path ------------------------------------------------------ */
/* One verification window for all B sequences in ONE fused persistent kernel:
 * softmax statistics, surprisals, gap, NormMatch, key flags, softened
 * normaliser, accept test with Philox draws, first-rejection scan and the
 * residual / bonus draw. Asynchronous on `stream` (a cudaStream_t). */
dsdv_status dsdv_verify(dsdv_ctx *ctx, const dsdv_params *params, const void *draft_logits,
                        const void *target_logits, const int32_t *draft_tokens,
                        const dsdv_outputs *out, void *stream);

/* dsdv_verify with early exit (verifier.cpp:250): a sequence's
 * positions past its first rejection are never evaluated by the reference, so
 * their rows are not streamed once the rejection is known (items not yet
 * started are skipped, items in flight stop at their next chunk), nor is
 * target row gamma unless every position was accepted. Same per-sequence
 * results (k, extra token, key count, status) as dsdv_verify; per-position
 * outputs are defined up to and including the first rejection only. */
dsdv_status dsdv_verify_early_exit(dsdv_ctx *ctx, const dsdv_params *params,
                                   const void *draft_logits, const void *target_logits,
                                   const int32_t *draft_tokens, const dsdv_outputs *out,
                                   void *stream);

/* dsdv_window_stats with the overlap clause decided by the caller's NormMatch
 * (norm_match_in[B][gamma], device), so any 1 <= top_m <= V works: the C++
 * drop-in computes it with dsdv_norm_match_rows when top_m exceeds the fused
 * kernel's warp selection (32). */
dsdv_status dsdv_window_stats_nm(dsdv_ctx *ctx, const dsdv_params *params,
                                 const void *draft_logits, const void *target_logits,
                                 const int32_t *draft_tokens, const double *norm_match_in,
                                 const dsdv_outputs *out, void *stream);

/* NormMatch (norm_match, verifier.cpp:119-134) of gamma positions for any
 * top_m: the top_m ids of each fp64 probability row by (p desc, id asc)
 * (top_ids, :40-51: a stable segmented radix sort on the device), then
 * |T cap D| / top_m per position. Rows are [gamma][row_stride]; scratch is
 * device memory of dsdv_norm_match_scratch_bytes(). Asynchronous. */
size_t dsdv_norm_match_scratch_bytes(int32_t gamma, int32_t vocab, int32_t row_stride);
dsdv_status dsdv_norm_match_rows(dsdv_ctx *ctx, const double *draft_probs,
                                 const double *target_probs, int32_t gamma, int32_t vocab,
                                 int32_t row_stride, int32_t top_m, void *scratch,
                                 size_t scratch_bytes, double *norm_match_out, void *stream);

/* One whole vocabulary-sharded window on this rank in one call, with no
 * collective: the exchange of dsdv_shard_stats_peers (records stored into every
 * rank's buffer as items complete), the merge and its slice masses, RESOLVE and
 * the tokens maximum, each followed by a flag round (dsdv_peer_signal /
 * dsdv_peer_wait), then the peer-wait status folded into out->status (a timed-out
 * round fails every sequence with DSDV_E_NCCL). buffer_bases[q] is rank q's
 * exchange buffer (CUDA-IPC mapped): two sets of [nranks][rank_stride_bytes]
 * (set = window_epoch & 1) followed by nranks uint64 arrival flags; rank_stride
 * >= dsdv_shard_exchange_bytes(), a multiple of 256. window_epoch >= 1 grows by
 * one per window (flag values 3e, 3e+1, 3e+2). out needs records, status and
 * extra_token. Asynchronous on stream. */
uint64_t dsdv_shard_exchange_bytes(int32_t batch, int32_t gamma, int32_t top_m);
dsdv_status dsdv_shard_verify_peers(dsdv_ctx *ctx, const dsdv_params *params,
                                    const void *draft_logits, const void *target_logits,
                                    const int32_t *draft_tokens, int32_t nranks, int32_t rank,
                                    void *const *buffer_bases, uint64_t rank_stride_bytes,
                                    uint64_t window_epoch, uint64_t timeout_ns,
                                    const dsdv_outputs *out, void *stream);

/* Pipeline-sharded decoding emulation (the reference's
 * run_pipeline, netsim.cpp:110-172): N logical stages, stage s on rank s mod
 * nranks. For each unit u (compute_ns[u]: t0 per token for standard decoding,
 * k t0 per window for DSD) the owner of stage 0 spins the compute, every link
 * s -> s+1 spins t1_ns and, across GPUs, stores the committed-token payload
 * into the next rank's buffer over NVLink and releases a per-source counter
 * the receiver waits on; the last stage returns the commit to stage 0. The
 * whole loop is enqueued here, in C++, on `stream` (one call per run).
 * buffer_bases as for dsdv_shard_verify_peers (set 0 slot q receives rank q's
 * payload, the nranks uint64 flags count its messages); run_index >= 1 grows
 * per call. status (device int32) gets DSDV_E_NCCL if a wait times out. */
dsdv_status dsdv_pipeline_run(dsdv_ctx *ctx, int32_t n_stages, int32_t nranks, int32_t rank,
                              void *const *buffer_bases, uint64_t rank_stride_bytes,
                              const uint64_t *compute_ns, int32_t n_units, uint64_t t1_ns,
                              uint64_t run_index, uint64_t timeout_ns, int32_t *status,
                              void *stream);

/* In place, on the device: values[i] = ln(values[i]), -inf for zero. The C++
 * drop-in uploads its fp64 probability rows as they are and turns them into
 * the logit rows the fused kernel folds (softmax(ln p) = p). Asynchronous. */
dsdv_status dsdv_log_rows(dsdv_ctx *ctx, double *values, uint64_t count, void *stream);

/* One process driving several GPUs (no IPC): let ctx's device store into
 * peer_device's memory over NVLink (cudaDeviceEnablePeerAccess). */
dsdv_status dsdv_enable_peer_access(dsdv_ctx *ctx, int32_t peer_device);

/* ---- threshold calibration (calibrate.cpp:51-148) ------------------------ */
typedef struct {
  double ratio_limit, gap_limit, overlap_floor; /* KeyCriteria (verifier.hpp:32-43) */
  int32_t top_m;
} dsdv_key_criteria;

typedef struct {
  int32_t vocab;       /* 2 <= V <= 8 (EnumerationGuard, enumerate.hpp:31) */
  int32_t horizon;     /* 1..4 */
  int64_t rows_offset; /* into the rows array: (V + 1) draft rows, then (V + 1) target rows of
                          V doubles; row s < V follows last token s, row V the prompt */
} dsdv_calib_item;

typedef struct {
  double avg_accepted_len; /* mean over items of E[accepted] + 1 */
  double divergence;       /* mean TV(adaptive, strict tau = 0) over the horizon */
  int32_t feasible;        /* divergence <= budget */
  int32_t status;          /* DSDV_OK, or the error an item's enumeration would raise */
} dsdv_grid_eval;

/* evaluate_point (calibrate.cpp:51-76) for every grid point, on the device: one
 * thread per (point, item) runs the exact enumerations in fp64 with the
 * reference's operation order. Host arrays in and out; synchronous. */
dsdv_status dsdv_calibrate(dsdv_ctx *ctx, const dsdv_calib_item *items, int32_t n_items,
                           const double *rows, int64_t n_row_doubles,
                           const dsdv_key_criteria *points, int32_t n_points, double tau,
                           int32_t gamma, double budget, dsdv_grid_eval *out);

/* Logit bytes the fused verifier's producers copied from global memory since
 * the last reset (accumulated over launches on this context). Synchronous:
 * waits for the device. reset != 0 clears the counter after reading. */
dsdv_status dsdv_streamed_bytes(dsdv_ctx *ctx, int reset, uint64_t *bytes);

/* Statistics and accept probabilities for every position, no draws. Fills the
 * per-position outputs, records, and status[B] (first error position, as the
 * reference would raise it walking left to right with all positions evaluated). */
dsdv_status dsdv_window_stats(dsdv_ctx *ctx, const dsdv_params *params,
                              const void *draft_logits, const void *target_logits,
                              const int32_t *draft_tokens, const dsdv_outputs *out,
                              void *stream);

/* Extra token per sequence from the records of dsdv_window_stats:
 * position[b] < gamma -> residual of that position's effective distribution
 * against P_d; position[b] == gamma -> bonus draw from target row gamma.
 * uniform[b] is the caller's draw. status[b] gets DSDV_E_EMPTY_RESIDUAL when
 * the residual has no mass. */
dsdv_status dsdv_sample_extra(dsdv_ctx *ctx, const dsdv_params *params,
                              const void *draft_logits, const void *target_logits,
                              const double *records, const int32_t *position,
                              const double *uniform, int32_t *token_out, int32_t *status,
                              void *stream);

/* Draft-side step: tokens[b][j] = inverse-CDF draw from softmax(draft row j)
 * with the Philox draft slot j (philox.h). */
dsdv_status dsdv_draft_sample(dsdv_ctx *ctx, const dsdv_params *params,
                              const void *draft_logits, int32_t *draft_tokens, void *stream);
/* The same under a sampling temperature (temperature_scale,
 * distribution.cpp:65-97): T = 1 identity, T = 0 the argmax with the lowest id
 * on ties, else softmax(l / T). */
dsdv_status dsdv_draft_sample_temperature(dsdv_ctx *ctx, const dsdv_params *params,
                                          double temperature, const void *draft_logits,
                                          int32_t *draft_tokens, void *stream);

/* Whole-row mixtures of two fp64 probability vectors of length vocab (the
 * drop-in API's soften and residual_distribution, verifier.cpp:161-186 and
 * :198-213): DSDV_MIX_SOFTEN w = a^(1-tau) b^tau, DSDV_MIX_RESIDUAL
 * w = max(0, a - b); out = w / sum(w). *status (device) becomes
 * DSDV_E_DEGENERATE_MIXTURE / DSDV_E_EMPTY_RESIDUAL when sum(w) <= 0. The
 * reference's endpoint short-circuits (tau 0 / 1 / equal rows) are the
 * caller's (they return an input unchanged). */
enum { DSDV_MIX_SOFTEN = 0, DSDV_MIX_RESIDUAL = 1 };
dsdv_status dsdv_mix_rows(dsdv_ctx *ctx, int32_t kind, int32_t vocab, const double *a,
                          const double *b, double tau, double *out, int32_t *status,
                          void *stream);

/* Waits for `stream`, then reports the first failing sequence's status with a
 * reference-style message in dsdv_last_error (status may be NULL to only sync). */
dsdv_status dsdv_sync(dsdv_ctx *ctx, const dsdv_params *params, const int32_t *status,
                      void *stream);

/* ---- vocabulary-sharded verification --------
 * Rank p of P holds ids [vocab_offset, vocab_offset + vocab_local) of every
 * row (params->vocab = global V; row_stride and pointers refer to the slice).
 * Per window, with the caller's collectives in between (csrc/shard.cu):
 *   dsdv_shard_stats   -> all-gather records [P][B][gamma+1][DSDV_RECORD_WORDS]
 *                         and top lists [P][B][gamma][2][m] (m = min(top_m, V))
 *   dsdv_shard_merge   (identical on every rank: k, key flags, accept draws;
 *                       this slice's mass of the extra row) -> all-gather [B] masses
 *   dsdv_shard_sample(DSDV_SHARD_RESOLVE) -> all-reduce(max) the [B] tokens
 * Decisions equal the unsharded verifier's except inside the eps bands (the
 * merged fp32 sums are re-associated). */
dsdv_status dsdv_shard_stats(dsdv_ctx *ctx, const dsdv_params *params, const void *draft_logits,
                             const void *target_logits, const int32_t *draft_tokens,
                             double *records, double *top_values, int32_t *top_ids,
                             void *stream);
/* rank_stride_bytes: 0 when the three gathered arrays are each [nranks][...]
 * contiguous; else the byte distance between consecutive ranks' copies of
 * all three (one packed exchange buffer per rank, one all-gather).
 * out: per-sequence outputs (extra_token is set to -1 until the resolve step),
 * optional per-position outputs, and out->records (required) receives the
 * merged global records. position[b] = the row of the extra draw (k for a
 * residual, gamma for the bonus, -1 when the sequence stopped on an error);
 * uniform[b] = its Philox draw; mass_out[b] = this slice's weight total of
 * that row (the MASS step, fused; gamma <= 31). tile_scratch (optional,
 * [B][DSDV_SHARD_TILE_WORDS] doubles) keeps the row's tile sums so that the
 * RESOLVE step of the owning rank re-reads one tile instead of the slice. */
#define DSDV_SHARD_TILE_WORDS 514
dsdv_status dsdv_shard_merge(dsdv_ctx *ctx, const dsdv_params *params, int32_t nranks,
                             const double *records_all, const double *top_values_all,
                             const int32_t *top_ids_all, uint64_t rank_stride_bytes,
                             const void *draft_logits, const void *target_logits,
                             const int32_t *draft_tokens, const dsdv_outputs *out,
                             int32_t *position, double *uniform, double *mass_out,
                             double *tile_scratch, void *stream);
enum { DSDV_SHARD_MASS = 0, DSDV_SHARD_RESOLVE = 1 };

/* ---- peer exchange over NVLink (one process per GPU) ---------------------
 * Replaces the record all-gather: every rank maps every rank's exchange
 * buffer (CUDA IPC) and the stats kernel stores its partial records straight
 * into all of them, item by item, while it streams (fused compute + exchange).
 * Exchange buffer of rank q: [nranks][rank_stride_bytes] packed records (the
 * dsdv_shard_stats layout at off_records / off_top_values / off_top_ids inside
 * each rank's slot), then nranks uint64 arrival flags at nranks * stride. */
#define DSDV_MAX_PEERS 8
dsdv_status dsdv_dev_alloc(dsdv_ctx *ctx, uint64_t bytes, void **dev_ptr); /* zeroed */
dsdv_status dsdv_dev_free(dsdv_ctx *ctx, void *dev_ptr);
dsdv_status dsdv_ipc_handle(dsdv_ctx *ctx, void *dev_ptr, uint8_t handle[64]);
dsdv_status dsdv_ipc_open(dsdv_ctx *ctx, const uint8_t handle[64], void **dev_ptr);
dsdv_status dsdv_ipc_close(dsdv_ctx *ctx, void *dev_ptr);
/* rank_bases[q]: rank q's exchange buffer as mapped in this process (q ==
 * rank: the local one). The records of this rank land in slot `rank` of all. */
dsdv_status dsdv_shard_stats_peers(dsdv_ctx *ctx, const dsdv_params *params,
                                   const void *draft_logits, const void *target_logits,
                                   const int32_t *draft_tokens, int32_t nranks, int32_t rank,
                                   void *const *rank_bases, uint64_t rank_stride_bytes,
                                   uint64_t off_records, uint64_t off_top_values,
                                   uint64_t off_top_ids, void *stream);
/* After the stats pass on `stream`: flag `rank` in every rank's buffer = epoch
 * (system-scope release). */
dsdv_status dsdv_peer_signal(dsdv_ctx *ctx, int32_t nranks, int32_t rank,
                             void *const *rank_bases, uint64_t rank_stride_bytes, uint64_t epoch,
                             void *stream);
/* The merge and the RESOLVE step over the same buffers: the merge reads the
 * records from the local buffer (every rank's slot) and stores this slice's
 * [B] masses at off_mass of slot `rank` in every buffer; RESOLVE reads the
 * masses from the local buffer and stores its [B] tokens (-1 where this rank
 * is not the owner) at off_tokens of slot `rank` in every buffer;
 * dsdv_peer_tokens_max folds the P token arrays of the local buffer. With
 * dsdv_peer_signal / dsdv_peer_wait between the steps, a window needs no
 * collective call. */
dsdv_status dsdv_shard_merge_peers(dsdv_ctx *ctx, const dsdv_params *params, int32_t nranks,
                                   int32_t rank, void *const *rank_bases,
                                   uint64_t rank_stride_bytes, uint64_t off_records,
                                   uint64_t off_top_values, uint64_t off_top_ids,
                                   uint64_t off_mass, const void *draft_logits,
                                   const void *target_logits, const int32_t *draft_tokens,
                                   const dsdv_outputs *out, int32_t *position, double *uniform,
                                   double *tile_scratch, void *stream);
dsdv_status dsdv_shard_resolve_peers(dsdv_ctx *ctx, const dsdv_params *params, int32_t nranks,
                                     int32_t rank, void *const *rank_bases,
                                     uint64_t rank_stride_bytes, uint64_t off_mass,
                                     uint64_t off_tokens, const void *draft_logits,
                                     const void *target_logits, const double *records,
                                     const int32_t *position, const double *uniform,
                                     int32_t *status, const double *tile_scratch, void *stream);
dsdv_status dsdv_peer_tokens_max(dsdv_ctx *ctx, int32_t nranks, void *local_base,
                                 uint64_t rank_stride_bytes, uint64_t off_tokens, int32_t batch,
                                 int32_t *token_out, void *stream);
/* Holds `stream` until every flag of the local buffer reached epoch (acquire);
 * after timeout_ns, *status (device) = DSDV_E_NCCL and the stream continues. */
dsdv_status dsdv_peer_wait(dsdv_ctx *ctx, int32_t nranks, void *local_base,
                           uint64_t rank_stride_bytes, uint64_t epoch, uint64_t timeout_ns,
                           int32_t *status, void *stream);
/* MASS: mass_out[b] = this slice's weight total of row position[b].
 * RESOLVE: masses_all = the gathered [nranks][B] totals; token_out[b] = the
 * global id on the owning rank, -1 elsewhere; status[b] = DSDV_E_EMPTY_RESIDUAL
 * when the row has no mass. */
dsdv_status dsdv_shard_sample(dsdv_ctx *ctx, const dsdv_params *params, int32_t mode, int32_t rank,
                              int32_t nranks, const void *draft_logits, const void *target_logits,
                              const double *records, const int32_t *position,
                              const double *uniform, const double *masses_all, double *mass_out,
                              int32_t *token_out, int32_t *status, const double *tile_scratch,
                              void *stream);

/* ---- pipeline emulation -------------------
 * Holds `stream` for `nanoseconds` of device time (%globaltimer): the compute
 * step t0 of a stage or the injected latency t1 of a link, replacing the
 * reference's simulated delays (netsim.cpp:110-172) with device time. */
dsdv_status dsdv_spin(dsdv_ctx *ctx, uint64_t nanoseconds, void *stream);

/* ---- helpers ----------------------------------------------------------- */
/* The accept / extra / draft uniform the kernels use (philox.h), on the host. */
double dsdv_uniform(uint64_t seed, uint64_t window, uint32_t sequence, uint32_t slot);

/* Benchmark / test inputs: seeded synthetic logits of the four row families
 * of SURVEY.md §8(d) (b mod 4: Zipf sigma 1.2/2.5/3.5 and Gaussian sigma 6;
 * draft = target + delta * N(0,1)). Writes draft [B][gamma] and target
 * [B][gamma+1] rows (dtype F32 or BF16). Not part of the verifier. */
dsdv_status dsdv_synth_logits(dsdv_ctx *ctx, const dsdv_params *params, uint64_t logits_seed,
                              void *draft_logits, void *target_logits, void *stream);

/* Number of kernel launches issued by this context so far (bench evidence). */
uint64_t dsdv_launch_count(const dsdv_ctx *ctx);

#ifdef __cplusplus
}
#endif

#endif /* DSDV_DSDV_H_ */
