/* CPU oracle for the DSD verifier hot path — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, fp64 restatement of the reference algorithm (paths relative to
 * /root/reference/proj). It is the checker the parity tests, smoke() and the
 * bench's cpu_baseline leg compare the CUDA path against; nothing in the
 * product (paper_2511_11733_b200/, include/) may link or call it.
 *
 * Pinned against: the reference's own known-answer tests (tests/test_verifier.cpp,
 * tests/test_distribution.cpp) and acceptance criterion 6 (tests/acceptance.cpp:257-288,
 * recorded in test_output.txt:50), replayed in tests/test_oracle.py, and
 * bit-for-bit against the reference sources compiled into oracle/_ref/
 * (oracle/Makefile + oracle/ref_harness.cpp) on random windows.
 *
 * The core works on fp64 probability rows like the reference; the logits front
 * end builds them as Distribution::from_weights(exp(l - max)) would
 * (distribution.cpp:54-63).
 */
#ifndef DSD_ORACLE_H_
#define DSD_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORACLE_OK = 0,
  ORACLE_E_INVARIANT = 1,
  ORACLE_E_DEGENERATE_MIXTURE = 2,
  ORACLE_E_DRAFTING_CONTRACT = 3,
  ORACLE_E_EMPTY_RESIDUAL = 4
};

typedef struct {
  double ratio_limit, gap_limit, overlap_floor;
  int top_m;
} oracle_criteria;

/* ---- primitives (probability rows) ---- */
int oracle_softmax(const double *logits, int V, double *probs);           /* distribution.cpp:54-63 */
double oracle_cross_entropy(const double *p, int V, int token);           /* verifier.cpp:112-117 */
double oracle_norm_match(const double *pt, const double *pd, int V, int top_m); /* :40-51, :119-134 */
int oracle_is_key(const double *pt, const double *pd, int V, int token, const oracle_criteria *c,
                  double *margins);                                       /* :136-159 */
int oracle_soften(const double *pt, const double *pd, int V, double tau, double *out); /* :161-186 */
double oracle_accept_prob(const double *eff, const double *pd, int token, int *err);  /* :188-196 */
int oracle_residual(const double *eff, const double *pd, int V, double *out);        /* :198-213 */
int oracle_sample_with_uniform(const double *p, int V, double u, double *margin); /* distribution.cpp:103-114 */

/* ---- uniform sources (UniformStream, rng.hpp:25-57) ---- */
typedef double (*oracle_next_uniform)(void *state);
typedef struct {
  const double *u; /* slot-indexed draws (include/dsdv/philox.h slot map) */
  int cursor;
} oracle_slot_stream;
double oracle_slot_next(void *state);
typedef struct {
  uint64_t mt[312];
  int idx;
} oracle_mt64; /* std::mt19937_64 + the 53-bit mapping of rng.hpp:38-40 */
void oracle_mt64_seed(oracle_mt64 *s, uint64_t seed);
double oracle_mt64_next(void *state);

/* ---- one window (the loop of verify_round, verifier.cpp:223-256) ---- */
typedef struct {
  int gamma, V;
  const double *pd;      /* [gamma][V] draft probability rows */
  const double *pt;      /* [gamma + 1][V] target probability rows */
  const int *row_err;    /* optional [2*gamma+1]: invalid-row codes, draft rows then target rows */
  const int32_t *tokens; /* [gamma] */
  double tau;
  oracle_criteria crit;
  oracle_next_uniform next_uniform;
  void *rng;
} oracle_window;

typedef struct {
  int accepted_count, extra_token, extra_source, key_count, status;
  int evaluated; /* positions with a decision */
  /* per position, [gamma], optional; entries past `evaluated` untouched */
  uint8_t *key, *accepted;
  double *accept_prob, *h_target, *h_draft, *p_target_y, *p_draft_y, *norm_match, *p_eff_y,
      *uniform;
  double *margin_u;    /* |u - a| */
  double *margin_key;  /* min(ratio, gap) clause distance to its lambda */
  double margin_extra; /* CDF margin of the extra draw */
} oracle_result;

int oracle_verify_window(const oracle_window *w, oracle_result *out);

/* Logits front end: softmax every row, then the window with Philox-slot
 * uniforms uniforms[2*gamma+1] (accept/extra cursor starts at slot gamma). */
int oracle_verify_window_logits(int gamma, int V, const double *draft_logits,
                                const double *target_logits, const int32_t *tokens, double tau,
                                const oracle_criteria *crit, const double *uniforms,
                                oracle_result *out);

/* Draft-side step: tokens[j] = sample_with_uniform(softmax(row j), uniforms[j]). */
int oracle_draft_tokens(const double *draft_logits, int gamma, int V, const double *uniforms,
                        int32_t *tokens, double *margins);

/* generate (verifier.cpp:259-282) for categorical-iid models with a
 * SeededStream: per round, gamma draft draws (draft_window :93-110), then the
 * window. Writes rounds' accepted counts into ks (capacity max_rounds) and
 * returns the number of rounds, or -status on error. */
int oracle_generate_iid(const double *pd, const double *pt, int V, int gamma, double tau,
                        const oracle_criteria *crit, int max_new, uint64_t seed, int *ks,
                        int max_rounds);

/* Batch of B windows over logits (the CPU baseline), nthreads POSIX threads.
 * Logits are fp32 rows: draft [B][gamma][stride], target [B][gamma+1][stride]. */
int oracle_verify_batch_f32(int B, int gamma, int V, int stride, const float *draft,
                            const float *target, const int32_t *tokens, double tau,
                            const oracle_criteria *crit, const double *uniforms /*[B][2g+1]*/,
                            int nthreads, int32_t *k_out, int32_t *extra_out, int32_t *status_out);

/* Parity checker: B windows over raw logits (dtype 0 = fp32, 1 = bf16 bits)
 * for ncfg (tau, criteria) configurations, nthreads POSIX threads; rows are
 * softmaxed once per sequence and shared by the configurations. Every output
 * array is caller-owned: per sequence [B], per position [B][gamma]. Positions
 * after the first rejection get the numerics (no draw) when all_positions. */
typedef struct {
  int32_t *k, *extra_token, *extra_source, *key_count, *status, *evaluated;
  double *margin_extra;
  uint8_t *key, *accepted;
  double *accept_prob, *h_target, *h_draft, *p_target_y, *p_draft_y, *norm_match, *p_eff_y,
      *margin_u, *margin_key;
} oracle_batch_out;

int oracle_verify_batch(int B, int gamma, int V, int stride, int dtype, const void *draft,
                        const void *target, const int32_t *tokens, int ncfg, const double *taus,
                        const oracle_criteria *crits, const double *uniforms /*[B][2g+1]*/,
                        int all_positions, int nthreads, oracle_batch_out *outs /*[ncfg]*/);

/* The synthetic windows of SURVEY.md §8(d) on the host, bit-identical to the
 * device's dsdv_synth_logits (shared arithmetic: include/dsdv/synth.h):
 * dtype 0 = fp32, 1 = bf16 bits; rows padded to stride with -inf. */
int oracle_synth_logits(int B, int gamma, int V, int stride, uint64_t seed, int dtype,
                        void *draft, void *target, int nthreads);

#ifdef __cplusplus
}
#endif

#endif
