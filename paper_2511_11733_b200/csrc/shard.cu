// Vocabulary-sharded verification.
//
// Every rank holds a contiguous slice [vocab_offset, vocab_offset + vocab_local)
// of every draft / target row (the natural layout of a tensor-parallel LM
// head). One window is:
//   1. dsdv_shard_stats  (fused kernel, partial mode, verify.cu write_partial):
//      per position the slice's (max, log-sum-exp) of l_t, l_d and of the
//      softened mix, l_t(y) / l_d(y) when y lies in the slice, and the slice's
//      top-m (value, global id) lists of both rows;
//   2. all-gather of those records (the caller's collective: NCCL / gloo);
//   3. dsdv_shard_merge  (this file): every rank merges the P records in shard
//      order — identical inputs, identical arithmetic, identical decisions on
//      all ranks — evaluates is_key / soften / accept_prob
//      (verifier.cpp:136-196), draws the Philox accept uniforms, finds the first
//      rejection (:223-250) and writes global records for the extra draw;
//   4. dsdv_shard_sample(MASS): the slice's residual / bonus weight total;
//   5. all-gather of the [B] totals;
//   6. dsdv_shard_sample(RESOLVE): the rank whose id range holds u * W scans
//      its slice (sample_with_uniform, distribution.cpp:103-114); the others
//      write -1;
//   7. all-reduce(max) of the [B] tokens.
// Contiguous slices in shard order keep the reference's global orders: top-m
// by (value desc, id asc) and the ascending-id inverse CDF.
#include <cuda_runtime.h>

#include "common.cuh"
#include "sample.cuh"

namespace dsdv {

constexpr int kMaxShards = 64;

struct MergeIn {
  const double *rec;   // [P][B][G1][kRecordWords] partial records
  const double *topv;  // [P][B][G][2][M]
  const int32_t *topi;
  int P;
};

__device__ __forceinline__ void lse_add(double &m, double &s, double x) {
  // running log-sum-exp as (max, sum of exp(x - max))
  if (x == -INFINITY) return;
  if (x > m) {
    s = (m == -INFINITY ? 0.0 : s * exp(m - x)) + 1.0;
    m = x;
  } else {
    s += exp(x - m);
  }
}

// P-way merge of the slices' sorted top-M lists of one row into the global
// top M ids (value desc, id asc; padding entries have id -1).
__device__ __forceinline__ void merge_top(const MergeIn &in, size_t list_off, size_t stride_p,
                                          int M, int *out) {
  int ptr[kMaxShards];
  for (int q = 0; q < in.P; ++q) ptr[q] = 0;
  for (int r = 0; r < M; ++r) {
    int best = -1;
    double bv = 0.0;
    int bid = 0;
    for (int q = 0; q < in.P; ++q) {
      if (ptr[q] >= M) continue;
      const size_t at = q * stride_p + list_off + ptr[q];
      const int id = in.topi[at];
      if (id < 0) continue;
      const double v = in.topv[at];
      if (best < 0 || v > bv || (v == bv && id < bid)) {
        best = q;
        bv = v;
        bid = id;
      }
    }
    out[r] = best < 0 ? -1 : bid;
    if (best >= 0) ++ptr[best];
  }
}

// One warp per sequence; lane j evaluates position j (and the bonus row).
__global__ void __launch_bounds__(128)
    shard_merge_kernel(const __grid_constant__ DevParams p, const MergeIn in,
                       const int32_t *__restrict__ tokens, const DevOut o,
                       int32_t *__restrict__ position, double *__restrict__ uniform) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= p.B) return;
  const int b = warp;
  const int G = p.gamma, G1 = G + 1, M = p.top_m;
  const double omt = (double)p.omt_f, tau = (double)p.tau_f;
  const size_t rec_stride_p = (size_t)p.B * G1 * kRecordWords;
  const size_t top_stride_p = (size_t)p.B * G * 2 * M;
  // sequence-level scan state
  int k = G, keys = 0, nears = 0, stop_err = 0, stop_kind = 0;
  for (int j0 = 0; j0 < G1; j0 += 32) {
    const int j = j0 + lane;
    const bool active = j < G1;
    const bool pair = j < G;
    int err = 0, key = 0, kind = DSDV_EFF_TARGET, near = 0, accepted = 0;
    if (active) {
      // ---- merge the slices' normalisers ----
      double mt = -INFINITY, md = -INFINITY, lt_m = -INFINITY, lt_s = 0.0, ld_m = -INFINITY,
             ld_s = 0.0, lz_m = -INFINITY, lz_s = 0.0, lt_y = NAN, ld_y = NAN;
      int diff = 0, own = 0;
      for (int q = 0; q < in.P; ++q) {
        const double *r = in.rec + q * rec_stride_p + ((size_t)b * G1 + j) * kRecordWords;
        const double lt = r[0] + r[1];
        lse_add(lt_m, lt_s, lt);
        if (lt > -INFINITY) mt = fmax(mt, r[0]);
        if (pair) {
          const double ld = r[2] + r[3];
          lse_add(ld_m, ld_s, ld);
          if (ld > -INFINITY) md = fmax(md, r[2]);
          lse_add(lz_m, lz_s, omt * r[0] + tau * r[2] + r[4]);
          const int f = (int)r[7];
          diff |= f & 1;
          if (f & 2) {
            own = 1;
            lt_y = r[5];
            ld_y = r[6];
          }
        }
      }
      const double lse_t = lt_m == -INFINITY ? -INFINITY : lt_m + log(lt_s);
      const double lse_d = ld_m == -INFINITY ? -INFINITY : ld_m + log(ld_s);
      const double lse_z = lz_m == -INFINITY ? -INFINITY : lz_m + log(lz_s);
      PosEval ev;
      ev.mt = mt;
      ev.lst = lse_t - mt;
      ev.md = pair ? md : 0.0;
      ev.lsd = pair ? lse_d - md : 0.0;
      ev.lsz = 0.0;
      ev.h_t = ev.h_d = ev.p_t_y = ev.p_d_y = ev.nm = ev.p_eff = ev.a = ev.u = 0.0;
      // distribution invariants: every row has mass
      if (!(lse_t > -INFINITY && isfinite(lse_t))) err = DSDV_E_INVARIANT;
      if (pair) {
        if (!(lse_d > -INFINITY && isfinite(lse_d)) && !err) err = DSDV_E_INVARIANT;
        const int y = tokens[(size_t)b * G + j];
        if (!(own && y >= 0 && y < p.V) && !err) err = DSDV_E_INVARIANT;  // check_token_in_vocab
        if (!own) lt_y = ld_y = -INFINITY;
        // ---- top-m overlap (norm_match, verifier.cpp:119-134) ----
        int tt[kMaxTopM], td[kMaxTopM];
        const size_t lo = ((size_t)b * G + j) * 2 * M;
        merge_top(in, lo, top_stride_p, M, tt);
        merge_top(in, lo + M, top_stride_p, M, td);
        int shared = 0;
        for (int x = 0; x < M; ++x) {
          if (td[x] < 0) continue;
          for (int w = 0; w < M; ++w) shared += (tt[w] == td[x]) ? 1 : 0;
        }
        ev.nm = (double)shared / (double)M;
        // ---- is_key (verifier.cpp:136-159) ----
        ev.h_t = (lt_y == -INFINITY) ? INFINITY : lse_t - lt_y;
        ev.h_d = (ld_y == -INFINITY) ? INFINITY : lse_d - ld_y;
        ev.p_t_y = exp(lt_y - lse_t);
        ev.p_d_y = exp(ld_y - lse_d);
        const bool certain = ev.h_t < kCertainSurprisal;
        const bool ratio_cert = ev.h_d > 0.0;
        const bool ratio_rel = ev.h_d / ev.h_t > p.ratio_limit;
        const bool ratio = certain ? ratio_cert : ratio_rel;
        const double gap = fabs(ev.p_t_y - ev.p_d_y);
        key = (ratio || gap > p.gap_limit || ev.nm < p.overlap_floor) ? 1 : 0;
        const double el = p.eps_lambda;
        if (ev.h_t < 1e-6 && (ratio_cert != ratio_rel || ev.h_d < 1e-6)) near = 1;
        if (isfinite(p.ratio_limit) && ev.h_t >= 1e-6 && isfinite(ev.h_d) &&
            fabs(ev.h_d / ev.h_t - p.ratio_limit) < el * fmax(1.0, p.ratio_limit))
          near = 1;
        if (fabs(gap - p.gap_limit) < el * fmax(1.0, p.gap_limit)) near = 1;
        // ---- effective distribution and accept_prob (:188-196, :231-237) ----
        if (key || p.tau == 0.0 || diff == 0)
          kind = DSDV_EFF_TARGET;
        else if (p.tau == 1.0)
          kind = DSDV_EFF_DRAFT;
        else
          kind = DSDV_EFF_SOFTENED;
        double p_eff = ev.p_t_y;
        if (kind == DSDV_EFF_DRAFT) p_eff = ev.p_d_y;
        if (kind == DSDV_EFF_SOFTENED && !err) {
          if (lse_z == -INFINITY) {
            err = DSDV_E_DEGENERATE_MIXTURE;  // disjoint supports (verifier.cpp:181-184)
          } else {
            ev.lsz = lse_z - (omt * ev.mt + tau * ev.md);
            p_eff = exp((1.0 - p.tau) * lt_y + p.tau * ld_y - lse_z);
          }
        }
        if (!err && !(ev.p_d_y > 0.0)) err = DSDV_E_DRAFTING_CONTRACT;
        ev.p_eff = p_eff;
        ev.a = err ? 0.0 : fmin(1.0, p_eff / ev.p_d_y);
        ev.u = dsdv_philox_uniform(p.seed, p.window, p.seq_offset + (uint32_t)b,
                                   (uint32_t)(G + j));
        accepted = (!err && ev.u < ev.a) ? 1 : 0;
        if (!err && fabs(ev.u - ev.a) < p.eps_u) near = 1;
        const size_t pos = (size_t)b * G + j;
        if (o.key_mask) o.key_mask[pos] = (uint8_t)key;
        if (o.accepted) o.accepted[pos] = (uint8_t)accepted;
        if (o.accept_prob) o.accept_prob[pos] = ev.a;
        if (o.h_target) o.h_target[pos] = ev.h_t;
        if (o.h_draft) o.h_draft[pos] = ev.h_d;
        if (o.p_target_y) o.p_target_y[pos] = ev.p_t_y;
        if (o.p_draft_y) o.p_draft_y[pos] = ev.p_d_y;
        if (o.norm_match) o.norm_match[pos] = ev.nm;
        if (o.p_effective_y) o.p_effective_y[pos] = ev.p_eff;
        if (o.uniform) o.uniform[pos] = ev.u;
      }
      // global record of this row for the extra draw (dsdv_shard_sample)
      double *r = o.records + ((size_t)b * G1 + j) * kRecordWords;
      r[kRecMt] = ev.mt;
      r[kRecLst] = ev.lst;
      r[kRecMd] = ev.md;
      r[kRecLsd] = ev.lsd;
      r[kRecLsz] = ev.lsz;
      r[kRecFlags] = (double)(kind | (err << 8) | (key << 16));
    }
    // ---- first rejection or error, left to right (verifier.cpp:223-250) ----
    const unsigned stop = __ballot_sync(0xffffffffu, active && j < G && (err || !accepted));
    const unsigned upto = stop ? ((__ffs(stop) - 1) < 31 ? (1u << (__ffs(stop))) - 1u : 0xffffffffu)
                               : 0xffffffffu;  // evaluated lanes: up to and incl. the stop
    if (k == G) {
      keys += __popc(__ballot_sync(0xffffffffu, active && j < G && key) & upto);
      nears += __popc(__ballot_sync(0xffffffffu, active && j < G && near) & upto);
      if (stop) {
        const int src = __ffs(stop) - 1;
        k = j0 + src;
        stop_err = __shfl_sync(0xffffffffu, err, src);
        stop_kind = __shfl_sync(0xffffffffu, kind, src);
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    int st = DSDV_OK, pos = -1;
    double u = 0.0;
    if (k < G) {
      if (stop_err) {
        st = stop_err;
      } else if (stop_kind == DSDV_EFF_DRAFT) {
        st = DSDV_E_EMPTY_RESIDUAL;  // residual of P_d against itself (verifier.cpp:209-211)
      } else {
        pos = k;
        u = dsdv_philox_uniform(p.seed, p.window, p.seq_offset + (uint32_t)b, (uint32_t)(G + k + 1));
      }
    } else {
      const double *rb = o.records + ((size_t)b * G1 + G) * kRecordWords;
      const int berr = ((int)rb[kRecFlags] >> 8) & 0xff;
      if (berr) {
        st = berr;
      } else {
        pos = G;
        u = dsdv_philox_uniform(p.seed, p.window, p.seq_offset + (uint32_t)b, (uint32_t)(2 * G));
      }
    }
    o.accepted_count[b] = k;
    o.key_count[b] = keys;
    o.extra_source[b] = (k < G) ? DSDV_EXTRA_RESIDUAL : DSDV_EXTRA_BONUS;
    o.extra_token[b] = -1;
    o.status[b] = st;
    o.near_threshold[b] = nears;
    position[b] = pos;
    uniform[b] = u;
  }
}

// Extra draw over a sharded row. MASS: the slice's weight total. RESOLVE: the
// rank whose id range holds T = u * W (W summed over slices in shard order)
// scans its slice; other ranks write -1.
template <class In>
__global__ void __launch_bounds__(kConsumerThreads)
    shard_sample_kernel(const __grid_constant__ DevParams p, int mode, int rank, int nranks,
                        const In *__restrict__ draft, const In *__restrict__ target,
                        const double *__restrict__ records, const int32_t *__restrict__ position,
                        const double *__restrict__ uniform, const double *__restrict__ masses,
                        double *__restrict__ mass_out, int32_t *__restrict__ token_out,
                        int32_t *__restrict__ status) {
  using Acc = typename InTraits<In>::Acc;
  __shared__ SampleShared samp;
  __shared__ Weigher<Acc> wf;
  __shared__ double t_local;
  __shared__ int skip;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int G = p.gamma, G1 = G + 1;
  const int j = position[b];
  if (tid == 0) {
    skip = 0;
    t_local = -1.0;
    if (j < 0 || j > G) {
      skip = 1;
      if (mode == 0) mass_out[b] = 0.0;
      else token_out[b] = -1;
    } else {
      const double *r = records + ((size_t)b * G1 + j) * kRecordWords;
      const int kind = (int)r[kRecFlags] & 0xff;
      PosEval ev;
      ev.mt = r[kRecMt];
      ev.lst = r[kRecLst];
      ev.md = r[kRecMd];
      ev.lsd = r[kRecLsd];
      ev.lsz = r[kRecLsz];
      set_weigher(wf, j == G ? kWeightPlain
                             : (kind == DSDV_EFF_SOFTENED ? kWeightResSoft : kWeightResTarget),
                  ev, (double)p.omt_f, (double)p.tau_f);
      if (mode == 1) {
        // owner of T = u W: the first slice whose cumulative mass passes T
        double W = 0.0;
        for (int q = 0; q < nranks; ++q) W += masses[(size_t)q * p.B + b];
        const double T = uniform[b] * W;
        int owner = -1, last = -1;
        double cum = 0.0, base = 0.0;
        for (int q = 0; q < nranks; ++q) {
          const double w = masses[(size_t)q * p.B + b];
          if (w > 0.0) {
            last = q;
            if (owner < 0 && cum + w > T) {
              owner = q;
              base = cum;
            }
          }
          cum += w;
        }
        if (!(W > 0.0)) {
          skip = 1;
          token_out[b] = -1;
          status[b] = DSDV_E_EMPTY_RESIDUAL;
        } else {
          if (owner < 0) {  // rounding gap above the total: the last supported slice
            owner = last;
            base = cum - masses[(size_t)last * p.B + b];
          }
          if (owner != rank) {
            skip = 1;
            token_out[b] = -1;
          } else {
            t_local = fmax(0.0, T - base);
          }
        }
      }
    }
  }
  __syncthreads();
  if (skip) return;
  const In *rt = target + ((size_t)b * G1 + j) * (size_t)p.stride;
  const In *rd = draft + ((size_t)b * G + (j < G ? j : 0)) * (size_t)p.stride;
  int near = 0;
  const int idx = cdf_sample<In, Acc>(rt, rd, wf, p.vocab_local, 0.0, p.eps_u, &samp, tid, &near,
                                      mode == 1 ? t_local : -1.0);
  if (tid == 0) {
    if (mode == 0)
      mass_out[b] = samp.W;
    else
      token_out[b] = idx < 0 ? -1 : p.vocab_offset + idx;
  }
}

cudaError_t launch_shard_merge(const DevParams &p, const double *rec, const double *topv,
                               const int32_t *topi, int P, const int32_t *tokens, const DevOut &o,
                               int32_t *position, double *uniform, cudaStream_t stream) {
  if (P < 1 || P > kMaxShards) return cudaErrorInvalidValue;
  MergeIn in{rec, topv, topi, P};
  const int warps_per_block = 4;
  const int grid = (p.B + warps_per_block - 1) / warps_per_block;
  shard_merge_kernel<<<grid, 32 * warps_per_block, 0, stream>>>(p, in, tokens, o, position,
                                                                  uniform);
  return cudaGetLastError();
}

template <class In>
cudaError_t launch_shard_sample(const DevParams &p, int mode, int rank, int nranks,
                                const void *draft, const void *target, const double *records,
                                const int32_t *position, const double *uniform,
                                const double *masses, double *mass_out, int32_t *token_out,
                                int32_t *status, cudaStream_t stream) {
  shard_sample_kernel<In><<<p.B, kConsumerThreads, 0, stream>>>(
      p, mode, rank, nranks, (const In *)draft, (const In *)target, records, position, uniform,
      masses, mass_out, token_out, status);
  return cudaGetLastError();
}

template cudaError_t launch_shard_sample<__nv_bfloat16>(const DevParams &, int, int, int,
                                                        const void *, const void *, const double *,
                                                        const int32_t *, const double *,
                                                        const double *, double *, int32_t *,
                                                        int32_t *, cudaStream_t);
template cudaError_t launch_shard_sample<float>(const DevParams &, int, int, int, const void *,
                                                const void *, const double *, const int32_t *,
                                                const double *, const double *, double *,
                                                int32_t *, int32_t *, cudaStream_t);
template cudaError_t launch_shard_sample<double>(const DevParams &, int, int, int, const void *,
                                                 const void *, const double *, const int32_t *,
                                                 const double *, const double *, double *,
                                                 int32_t *, int32_t *, cudaStream_t);

}  // namespace dsdv
