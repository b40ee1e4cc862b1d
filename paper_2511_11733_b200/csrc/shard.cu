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
constexpr int kStageCand = 128;  // staged slice candidates per row (P * top_m)
constexpr int kStageWarps = 16;  // positions staged (gamma + 1 <= 16)

struct MergeIn {
  const double *rec;   // rank 0's [B][G1][kRecordWords] partial records
  const double *topv;  // rank 0's [B][G][2][M]
  const int32_t *topi;
  int P;
  // elements between consecutive ranks' copies (packed exchange buffers put
  // all three arrays of one rank side by side)
  size_t rec_stride, topv_stride, topi_stride;
};

// One CTA per sequence, one warp per position (max(256, 32 (gamma+1))
// threads): each warp merges its position's P slice records with warp
// reductions and the top-m overlap with a warp-parallel ranking, lane 0 runs
// the fp64 decision; warp 0 then finds the first rejection (verifier.cpp:
// 223-250), and the CTA's first 256 threads compute this slice's mass of the
// extra-draw row (the MASS step of dsdv_shard_sample, fused).
struct PosSummary {
  int err, key, kind, near, accepted;
};

// Peer exchange of the [B]-sized results: every store is repeated at
// address + d[q] (the same slot of rank q's mapped exchange buffer).
struct PeerDelta {
  long long d[8];
  int n;
};
template <class T>
__device__ __forceinline__ void put_peers(T *a, T v, const PeerDelta &pd) {
  *a = v;
  for (int q = 0; q < pd.n; ++q) *reinterpret_cast<T *>(reinterpret_cast<char *>(a) + pd.d[q]) = v;
}

// MAXT: the block size bound the registers are sized for (gamma + 1 <= 10
// position warps fit 320 threads and four CTAs per SM; larger gamma uses 1024)
template <class In, int MAXT = 1024, int MINB = 1>
__global__ void __launch_bounds__(MAXT, MINB)
    shard_merge_kernel(const __grid_constant__ DevParams p, const MergeIn in,
                       const In *__restrict__ draft, const In *__restrict__ target,
                       const int32_t *__restrict__ tokens, const DevOut o,
                       int32_t *__restrict__ position, double *__restrict__ uniform,
                       double *__restrict__ mass_out, double *__restrict__ tiles,
                       const PeerDelta mpd) {
  using Acc = typename InTraits<In>::Acc;
  __shared__ PosSummary summ[32];
  __shared__ int tset[32][kMaxTopM];
  // one row's P slice lists staged per warp (P * M <= kStageCand)
  __shared__ double cand_v[kStageWarps][kStageCand];
  __shared__ int cand_i[kStageWarps][kStageCand];
  __shared__ SampleShared samp;
  __shared__ Weigher<Acc> wf;
  __shared__ int s_pos;
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = p.gamma, G1 = G + 1, M = p.top_m;
  const double omt = (double)p.omt_f, tau = (double)p.tau_f;
  if (warp < G1) {
    const int j = warp;
    const bool pair = j < G;
    // ---- normalisers: lanes over slices, log-sum-exp by warp reduction ----
    double lt = -INFINITY, ld = -INFINITY, lz = -INFINITY, mtq = -INFINITY, mdq = -INFINITY;
    double lty = NAN, ldy = NAN;
    int f = 0;
    for (int q = lane; q < in.P; q += 32) {
      const double *r = in.rec + q * in.rec_stride + ((size_t)b * G1 + j) * kRecordWords;
      // running log-sum-exp over this lane's slices (the first one is exact:
      // log(0 + e^0) = 0, so it is taken as is, without the transcendentals)
      auto lse2 = [](double acc, double a) -> double {
        if (acc == -INFINITY) return a;
        const double m = fmax(acc, a);
        return m == -INFINITY ? -(double)INFINITY : m + log(exp(acc - m) + exp(a - m));
      };
      const double a_t = r[0] + r[1];
      if (a_t > -INFINITY) mtq = fmax(mtq, r[0]);
      lt = lse2(lt, a_t);
      if (pair) {
        const double a_d = r[2] + r[3];
        if (a_d > -INFINITY) mdq = fmax(mdq, r[2]);
        ld = lse2(ld, a_d);
        const double a_z = omt * r[0] + tau * r[2] + r[4];
        lz = lse2(lz, a_z);
        const int fl = (int)r[7];
        f |= fl;
        if (fl & 2) {
          lty = r[5];
          ldy = r[6];
        }
      }
    }
    auto warp_lse = [&](double x) -> double {
      double m = x;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (m == -INFINITY) return -(double)INFINITY;
      double e = (x == -INFINITY) ? 0.0 : exp(x - m);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
      return m + log(e);
    };
    auto warp_max = [&](double x) -> double {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
      return x;
    };
    const double lse_t = warp_lse(lt), lse_d = warp_lse(ld), lse_z = warp_lse(lz);
    const double mt = warp_max(mtq), md = warp_max(mdq);
    const unsigned diffq = __ballot_sync(0xffffffffu, (f & 1) != 0);
    const unsigned ownq = __ballot_sync(0xffffffffu, (f & 2) != 0);
    const int owner = ownq ? __ffs(ownq) - 1 : 0;
    const double lt_y0 = __shfl_sync(0xffffffffu, lty, owner);
    const double ld_y0 = __shfl_sync(0xffffffffu, ldy, owner);
    // ---- top-m overlap: rank every slice candidate against all others ----
    int shared = 0;
    if (pair) {
      const int nc = in.P * M;
      const size_t lo = ((size_t)b * G + j) * 2 * M;
      const bool staged = nc <= kStageCand && warp < kStageWarps;
      if (staged && in.P <= 32) {
        // P-way merge of the sorted slice lists: lane q holds the head of
        // list q, M warp arg-max steps (value desc, id asc) give the top M
        for (int r = 0; r < 2; ++r) {
          for (int c = lane; c < nc; c += 32) {
            const int q = c / M, i = c - q * M;
            const int id = in.topi[q * in.topi_stride + lo + r * M + i];
            cand_i[warp][c] = id;
            cand_v[warp][c] = id >= 0 ? in.topv[q * in.topv_stride + lo + r * M + i] : 0.0;
          }
          if (r == 0 && lane < M) tset[warp][lane] = -1;
          __syncwarp();
          int head = 0;
          for (int k = 0; k < M; ++k) {
            int bid = -1, bl = 32;
            if (sizeof(Acc) == 4) {
              // fp32 logits: (value desc, id asc) as one 64-bit key, a
              // branch-free warp max (0 = empty, below every real key)
              unsigned long long key = 0ull;
              if (lane < in.P && head < M) {
                const int id = cand_i[warp][lane * M + head];
                if (id >= 0) {
                  const unsigned fb = __float_as_uint((float)cand_v[warp][lane * M + head]);
                  const unsigned ord = (fb & 0x80000000u) ? ~fb : (fb | 0x80000000u);
                  key = ((unsigned long long)ord << 32) | (unsigned)(~id);
                }
              }
              unsigned long long best = key;
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
                best = other > best ? other : best;
              }
              if (best != 0ull) {
                bid = (int)~(unsigned)best;
                const unsigned who = __ballot_sync(0xffffffffu, key == best);
                bl = __ffs(who) - 1;
              }
            } else {
              double bv = -INFINITY;
              if (lane < in.P && head < M) {
                const int id = cand_i[warp][lane * M + head];
                if (id >= 0) {
                  bv = cand_v[warp][lane * M + head];
                  bid = id;
                  bl = lane;
                }
              }
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oid = __shfl_xor_sync(0xffffffffu, bid, o);
                const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
                if (ol < 32 && (bl == 32 || ov > bv || (ov == bv && oid < bid))) {
                  bv = ov;
                  bid = oid;
                  bl = ol;
                }
              }
            }
            if (bl == 32) break;  // every list exhausted (slices shorter than M)
            if (lane == bl) ++head;
            if (r == 0) {
              if (lane == 0) tset[warp][k] = bid;
            } else {
              __syncwarp();
              shared += __ballot_sync(0xffffffffu, lane < M && tset[warp][lane] == bid) ? 1 : 0;
            }
          }
          __syncwarp();
        }
      } else
      for (int r = 0; r < 2; ++r) {  // 0: target, 1: draft
        if (staged) {
          // the P sorted lists of this row into shared memory (one coalesced
          // pass), so the ranking below reads no global memory
          for (int c = lane; c < nc; c += 32) {
            const int q = c / M, i = c - q * M;
            const int id = in.topi[q * in.topi_stride + lo + r * M + i];
            cand_i[warp][c] = id;
            cand_v[warp][c] = id >= 0 ? in.topv[q * in.topv_stride + lo + r * M + i] : 0.0;
          }
          __syncwarp();
        }
        for (int c = lane; c < ((nc + 31) & ~31); c += 32) {
          const bool val = c < nc;
          const int q = val ? c / M : 0, i = val ? c - (c / M) * M : 0;
          int id;
          double v;
          if (staged) {
            id = val ? cand_i[warp][c] : -1;
            v = val && id >= 0 ? cand_v[warp][c] : 0.0;
          } else {
            id = val ? in.topi[q * in.topi_stride + lo + r * M + i] : -1;
            v = val && id >= 0 ? in.topv[q * in.topv_stride + lo + r * M + i] : 0.0;
          }
          int rank = 0;
          if (id >= 0) {
            for (int qq = 0; qq < in.P; ++qq) {
              if (qq == q) {
                rank += i;  // own list is sorted: its first i entries beat it
                continue;
              }
              for (int ii = 0; ii < M; ++ii) {
                int id2;
                double v2;
                if (staged) {
                  id2 = cand_i[warp][qq * M + ii];
                  if (id2 < 0) break;
                  v2 = cand_v[warp][qq * M + ii];
                } else {
                  id2 = in.topi[qq * in.topi_stride + lo + r * M + ii];
                  if (id2 < 0) break;
                  v2 = in.topv[qq * in.topv_stride + lo + r * M + ii];
                }
                if (!(v2 > v || (v2 == v && id2 < id))) break;  // sorted: no later entry beats it
                ++rank;
              }
            }
          }
          const bool top = id >= 0 && rank < M;
          if (r == 0) {
            if (top) tset[warp][rank] = id;
          } else {
            __syncwarp();
            bool hit = false;
            if (top)
              for (int k = 0; k < M; ++k) hit |= tset[warp][k] == id;
            shared += __popc(__ballot_sync(0xffffffffu, hit));
          }
        }
        __syncwarp();  // the staged lists are overwritten by the next row
        if (r == 0) {
          // fewer than M valid candidates: the rest of the set stays unmatched
          __syncwarp();
        }
      }
    }
    if (lane == 0) {
      int err = 0, key = 0, kind = DSDV_EFF_TARGET, near = 0, accepted = 0;
      double lt_y = lt_y0, ld_y = ld_y0;
      PosEval ev;
      ev.mt = mt;
      ev.lst = lse_t - mt;
      ev.md = pair ? md : 0.0;
      ev.lsd = pair ? lse_d - md : 0.0;
      ev.lsz = 0.0;
      ev.h_t = ev.h_d = ev.p_t_y = ev.p_d_y = ev.nm = ev.p_eff = ev.a = ev.u = 0.0;
      if (!(lse_t > -INFINITY && isfinite(lse_t))) err = DSDV_E_INVARIANT;
      if (pair) {
        if (!(lse_d > -INFINITY && isfinite(lse_d)) && !err) err = DSDV_E_INVARIANT;
        const int y = tokens[(size_t)b * G + j];
        if (!(ownq && y >= 0 && y < p.V) && !err) err = DSDV_E_INVARIANT;  // check_token_in_vocab
        if (!ownq) lt_y = ld_y = -INFINITY;
        ev.nm = (double)shared / (double)M;
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
        if (key || p.tau == 0.0 || diffq == 0)
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
      double *rr = o.records + ((size_t)b * G1 + j) * kRecordWords;
      rr[kRecMt] = ev.mt;
      rr[kRecLst] = ev.lst;
      rr[kRecMd] = ev.md;
      rr[kRecLsd] = ev.lsd;
      rr[kRecLsz] = ev.lsz;
      rr[kRecFlags] = (double)(kind | (err << 8) | (key << 16));
      summ[j] = PosSummary{err, key, kind, near, accepted};
    }
  }
  __syncthreads();
  // ---- first rejection or error, left to right (verifier.cpp:223-250) ----
  if (warp == 0) {
    const bool act = lane < G;
    const PosSummary sj = act ? summ[lane] : PosSummary{0, 0, 0, 0, 1};
    const unsigned stop = __ballot_sync(0xffffffffu, act && (sj.err || !sj.accepted));
    const int k = stop ? __ffs(stop) - 1 : G;
    const unsigned upto = (k >= 31) ? 0xffffffffu : ((1u << (k + 1)) - 1u);
    const int keys = __popc(__ballot_sync(0xffffffffu, act && sj.key) & upto);
    const int nears = __popc(__ballot_sync(0xffffffffu, act && sj.near) & upto);
    if (lane == 0) {
      int st = DSDV_OK, pos = -1;
      double u = 0.0;
      if (k < G) {
        if (summ[k].err) {
          st = summ[k].err;
        } else if (summ[k].kind == DSDV_EFF_DRAFT) {
          st = DSDV_E_EMPTY_RESIDUAL;  // residual of P_d against itself (verifier.cpp:209-211)
        } else {
          pos = k;
          u = dsdv_philox_uniform(p.seed, p.window, p.seq_offset + (uint32_t)b,
                                  (uint32_t)(G + k + 1));
        }
      } else if (summ[G].err) {
        st = summ[G].err;
      } else {
        pos = G;
        u = dsdv_philox_uniform(p.seed, p.window, p.seq_offset + (uint32_t)b, (uint32_t)(2 * G));
      }
      o.accepted_count[b] = k;
      o.key_count[b] = keys;
      o.extra_source[b] = (k < G) ? DSDV_EXTRA_RESIDUAL : DSDV_EXTRA_BONUS;
      o.extra_token[b] = -1;
      o.status[b] = st;
      o.near_threshold[b] = nears;
      position[b] = pos;
      uniform[b] = u;
      s_pos = pos;
      if (pos >= 0) {
        const double *r = o.records + ((size_t)b * G1 + pos) * kRecordWords;
        const int kind = (int)r[kRecFlags] & 0xff;
        PosEval ev;
        ev.mt = r[kRecMt];
        ev.lst = r[kRecLst];
        ev.md = r[kRecMd];
        ev.lsd = r[kRecLsd];
        ev.lsz = r[kRecLsz];
        set_weigher(wf, pos == G ? kWeightPlain
                                 : (kind == DSDV_EFF_SOFTENED ? kWeightResSoft : kWeightResTarget),
                    ev, omt, tau);
      }
    }
  }
  __syncthreads();
  // ---- this slice's mass of the extra-draw row (fused MASS step) ----
  const int pos = s_pos;
  if (pos < 0) {
    if (threadIdx.x == 0) {
      put_peers(mass_out + b, 0.0, mpd);
      if (mpd.n) __threadfence_system();
    }
    return;
  }
  if (threadIdx.x >= kConsumerThreads) return;
  const In *rt = target + ((size_t)b * G1 + pos) * (size_t)p.stride;
  const In *rd = draft + ((size_t)b * G + (pos < G ? pos : 0)) * (size_t)p.stride;
  int near = 0;
  cdf_sample<In, Acc>(rt, rd, wf, p.vocab_local, 0.0, p.eps_u, &samp, threadIdx.x, &near, -1.0,
                      tiles ? tiles + (size_t)b * (kMaxTiles + 2) : nullptr);
  if (threadIdx.x == 0) {
    put_peers(mass_out + b, samp.W, mpd);
    if (mpd.n) __threadfence_system();
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
                        int32_t *__restrict__ status, const double *__restrict__ tiles,
                        const PeerDelta tpd, size_t mstride) {
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
      else put_peers(token_out + b, -1, tpd);
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
        for (int q = 0; q < nranks; ++q) W += masses[(size_t)q * mstride + b];
        const double T = uniform[b] * W;
        int owner = -1, last = -1;
        double cum = 0.0, base = 0.0;
        for (int q = 0; q < nranks; ++q) {
          const double w = masses[(size_t)q * mstride + b];
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
          put_peers(token_out + b, -1, tpd);
          status[b] = DSDV_E_EMPTY_RESIDUAL;
        } else {
          if (owner < 0) {  // rounding gap above the total: the last supported slice
            owner = last;
            base = cum - masses[(size_t)last * mstride + b];
          }
          if (owner != rank) {
            skip = 1;
            put_peers(token_out + b, -1, tpd);
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
  const int idx = cdf_sample<In, Acc>(
      rt, rd, wf, p.vocab_local, 0.0, p.eps_u, &samp, tid, &near, mode == 1 ? t_local : -1.0,
      nullptr, (mode == 1 && tiles) ? tiles + (size_t)b * (kMaxTiles + 2) : nullptr);
  if (tid == 0) {
    if (mode == 0)
      mass_out[b] = samp.W;
    else
      put_peers(token_out + b, idx < 0 ? -1 : p.vocab_offset + idx, tpd);
  }
}

template <class In>
cudaError_t launch_shard_merge(const DevParams &p, const double *rec, const double *topv,
                               const int32_t *topi, int P, size_t rank_bytes, const void *draft,
                               const void *target, const int32_t *tokens, const DevOut &o,
                               int32_t *position, double *uniform, double *mass_out,
                               double *tiles, cudaStream_t stream, const long long *mass_delta,
                               int n_delta) {
  if (P < 1 || P > kMaxShards || p.gamma > 31 || n_delta > 8) return cudaErrorInvalidValue;
  PeerDelta mpd{};
  mpd.n = n_delta;
  for (int q = 0; q < n_delta; ++q) mpd.d[q] = mass_delta[q];
  const int G1 = p.gamma + 1;
  MergeIn in{rec, topv, topi, P, (size_t)p.B * G1 * kRecordWords,
             (size_t)p.B * p.gamma * 2 * p.top_m, (size_t)p.B * p.gamma * 2 * p.top_m};
  if (rank_bytes) {
    if (rank_bytes % 8) return cudaErrorInvalidValue;
    in.rec_stride = in.topv_stride = rank_bytes / 8;
    in.topi_stride = rank_bytes / 4;
  }
  const int threads = 32 * G1 > kConsumerThreads ? 32 * G1 : kConsumerThreads;
  if (threads <= 320)
    shard_merge_kernel<In, 320, 4><<<p.B, threads, 0, stream>>>(p, in, (const In *)draft,
                                                               (const In *)target, tokens, o,
                                                               position, uniform, mass_out, tiles,
                                                               mpd);
  else
    shard_merge_kernel<In><<<p.B, threads, 0, stream>>>(p, in, (const In *)draft,
                                                      (const In *)target, tokens, o, position,
                                                      uniform, mass_out, tiles, mpd);
  return cudaGetLastError();
}

template <class In>
cudaError_t launch_shard_sample(const DevParams &p, int mode, int rank, int nranks,
                                const void *draft, const void *target, const double *records,
                                const int32_t *position, const double *uniform,
                                const double *masses, double *mass_out, int32_t *token_out,
                                int32_t *status, const double *tiles, cudaStream_t stream,
                                const long long *tok_delta, int n_delta, size_t mstride) {
  if (n_delta > 8) return cudaErrorInvalidValue;
  PeerDelta tpd{};
  tpd.n = n_delta;
  for (int q = 0; q < n_delta; ++q) tpd.d[q] = tok_delta[q];
  shard_sample_kernel<In><<<p.B, kConsumerThreads, 0, stream>>>(
      p, mode, rank, nranks, (const In *)draft, (const In *)target, records, position, uniform,
      masses, mass_out, token_out, status, tiles, tpd, mstride ? mstride : (size_t)p.B);
  return cudaGetLastError();
}

#define DSDV_MERGE_INST(T)                                                                   \
  template cudaError_t launch_shard_merge<T>(const DevParams &, const double *, const double *,  \
                                             const int32_t *, int, size_t, const void *,        \
                                             const void *, const int32_t *, const DevOut &,     \
                                             int32_t *, double *, double *, double *, cudaStream_t, \
                                             const long long *, int);
DSDV_MERGE_INST(__nv_bfloat16)
DSDV_MERGE_INST(float)
DSDV_MERGE_INST(double)
#undef DSDV_MERGE_INST

template cudaError_t launch_shard_sample<__nv_bfloat16>(const DevParams &, int, int, int,
                                                        const void *, const void *, const double *,
                                                        const int32_t *, const double *,
                                                        const double *, double *, int32_t *,
                                                        int32_t *, const double *, cudaStream_t,
                                                        const long long *, int, size_t);
template cudaError_t launch_shard_sample<float>(const DevParams &, int, int, int, const void *,
                                                const void *, const double *, const int32_t *,
                                                const double *, const double *, double *,
                                                int32_t *, int32_t *, const double *, cudaStream_t,
                                                const long long *, int, size_t);
template cudaError_t launch_shard_sample<double>(const DevParams &, int, int, int, const void *,
                                                 const void *, const double *, const int32_t *,
                                                 const double *, const double *, double *,
                                                 int32_t *, int32_t *, const double *,
                                                 cudaStream_t, const long long *, int, size_t);

// ------------------------------------------------------------------ peer exchange
struct PeerBases {
  char *base[8];
};

// Flag `rank` of every rank's exchange buffer = epoch (after the stats pass
// on this stream: its peer stores were fenced at system scope per item).
__global__ void peer_signal_kernel(PeerBases pb, int nranks, int rank, unsigned long long stride,
                                   unsigned long long epoch) {
  const int q = threadIdx.x;
  if (q >= nranks) return;
  __threadfence_system();
  unsigned long long *f =
      reinterpret_cast<unsigned long long *>(pb.base[q] + (size_t)nranks * stride) + rank;
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(epoch) : "memory");
}

// Hold the stream until every rank's flag reached epoch, at most timeout_ns.
__global__ void peer_wait_kernel(const unsigned long long *flags, int nranks,
                                 unsigned long long epoch, unsigned long long timeout_ns,
                                 int *status) {
  const int q = threadIdx.x;
  if (q < nranks) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + q) : "memory");
      if (v >= epoch) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        if (status) atomicExch(status, DSDV_E_NCCL);
        break;
      }
      __nanosleep(200);
    }
  }
  __syncthreads();
  __threadfence_system();
}

cudaError_t launch_peer_signal(char *const *bases, int nranks, int rank, unsigned long long stride,
                               unsigned long long epoch, cudaStream_t stream) {
  PeerBases pb{};
  for (int q = 0; q < nranks; ++q) pb.base[q] = bases[q];
  peer_signal_kernel<<<1, 32, 0, stream>>>(pb, nranks, rank, stride, epoch);
  return cudaGetLastError();
}

cudaError_t launch_peer_wait(const unsigned long long *flags, int nranks, unsigned long long epoch,
                             unsigned long long timeout_ns, int *status, cudaStream_t stream) {
  peer_wait_kernel<<<1, 32, 0, stream>>>(flags, nranks, epoch, timeout_ns, status);
  return cudaGetLastError();
}

// token[b] = max over ranks of their RESOLVE outputs (-1 where not the owner)
__global__ void tokens_max_kernel(const int32_t *tok, size_t stride, int nranks, int B,
                                  int32_t *out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int32_t m = -1;
  for (int q = 0; q < nranks; ++q) m = max(m, tok[(size_t)q * stride + b]);
  out[b] = m;
}

cudaError_t launch_tokens_max(const int32_t *tok, size_t stride, int nranks, int B, int32_t *out,
                              cudaStream_t stream) {
  tokens_max_kernel<<<(B + 255) / 256, 256, 0, stream>>>(tok, stride, nranks, B, out);
  return cudaGetLastError();
}

// a timed-out flag round (dsdv_peer_wait status) fails every sequence
__global__ void status_fold_kernel(const int32_t *peer_status, int32_t *status, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B && *peer_status != 0) status[b] = DSDV_E_NCCL;
}

cudaError_t launch_status_fold(const int32_t *peer_status, int32_t *status, int batch,
                               cudaStream_t stream) {
  status_fold_kernel<<<(batch + 255) / 256, 256, 0, stream>>>(peer_status, status, batch);
  return cudaGetLastError();
}

// ---- pipeline emulation hops ----
// One link of the pipeline: the injected latency t1 (a device spin), then the
// committed-token payload stored into the next stage's GPU (NVLink peer store
// into its CUDA-IPC-mapped buffer) and a release of the per-source counter.
__global__ void hop_send_kernel(unsigned long long t1_ns, int32_t *dst_payload,
                                const int32_t *payload, unsigned long long *dst_flag,
                                unsigned long long value) {
  if (threadIdx.x == 0 && t1_ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < t1_ns);
  }
  __syncwarp();
  if (threadIdx.x < 16) dst_payload[threadIdx.x] = payload[threadIdx.x];
  __syncwarp();
  if (threadIdx.x == 0) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst_flag), "l"(value) : "memory");
  }
}

// The receiving stage: wait for the source's counter, take the payload.
__global__ void hop_recv_kernel(const unsigned long long *flag, unsigned long long value,
                                unsigned long long timeout_ns, int *status, const int32_t *slot,
                                int32_t *payload) {
  if (threadIdx.x == 0) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
      if (v >= value) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        if (status) atomicExch(status, DSDV_E_NCCL);
        break;
      }
      __nanosleep(100);
    }
  }
  __syncwarp();
  if (threadIdx.x < 16) payload[threadIdx.x] = *(volatile const int32_t *)(slot + threadIdx.x);
}

cudaError_t launch_hop_send(unsigned long long t1_ns, int32_t *dst_payload, const int32_t *payload,
                            unsigned long long *dst_flag, unsigned long long value,
                            cudaStream_t stream) {
  hop_send_kernel<<<1, 32, 0, stream>>>(t1_ns, dst_payload, payload, dst_flag, value);
  return cudaGetLastError();
}

cudaError_t launch_hop_recv(const unsigned long long *flag, unsigned long long value,
                            unsigned long long timeout_ns, int *status, const int32_t *slot,
                            int32_t *payload, cudaStream_t stream) {
  hop_recv_kernel<<<1, 32, 0, stream>>>(flag, value, timeout_ns, status, slot, payload);
  return cudaGetLastError();
}

}  // namespace dsdv
