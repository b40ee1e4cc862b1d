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
  const double *rec;   // rank 0's [B][G1][kRecordWords] partial records
  const double *topv;  // rank 0's [B][G][2][M]
  const int32_t *topi;
  int P;
  // elements between consecutive ranks' copies (packed exchange buffers put
  // all three arrays of one rank side by side)
  size_t rec_stride, topv_stride, topi_stride;
};

// One warp per sequence, one lane per position j in [0, gamma] (the decide
// step of the merge): lane j combines its position's P slice records in shard
// order (log-sum-exp of the slice normalisers), merges the P sorted slice
// top-m lists of both rows (a P-way merge by (value desc, id asc), the order of
// top_ids), evaluates is_key / soften / accept_prob (verifier.cpp:136-196) in
// fp64 and draws its Philox accept uniform; the warp then finds the first
// rejection (:223-250) with one ballot. Identical inputs give identical
// decisions on every rank. The extra-draw mass (MASS) is a separate streaming
// pass (shard_sample_kernel, mode 0).
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

constexpr int kDecideWarps = 4;  // sequences per CTA
constexpr size_t kDecideStageMax = 160 * 1024;  // dynamic shared memory for staged lists
constexpr int kSliceTileSubs = 4;  // MASS / RESOLVE tiles: >= 4 sub-tiles (1-2K ids)

// One row's P sorted slice lists: entry h of slice q at v[q * qs + h] (values)
// and id[q * qs + h] (ids); shared memory when the warp staged them, else the
// exchange buffer itself.
struct SliceLists {
  const double *v;
  const int32_t *id;
  size_t qs_v, qs_i;
};

// Lane-local P-way merge of one row's sorted slice lists (P <= PMAX; with
// PMAX = 8 the list heads stay in registers): calls emit(k, id) for the top M
// in order (slices shorter than M leave id -1 entries, which end a list).
template <int PMAX, class Emit>
__device__ __forceinline__ void merge_slice_lists(const SliceLists &L, int P, int M, Emit emit) {
  int heads[PMAX], hid[PMAX];
  double hv[PMAX];
#pragma unroll
  for (int q = 0; q < PMAX; ++q) {
    heads[q] = 0;
    hid[q] = (q < P && M > 0) ? L.id[q * L.qs_i] : -1;
    hv[q] = hid[q] >= 0 ? L.v[q * L.qs_v] : 0.0;
  }
  for (int n = 0; n < M; ++n) {
    int bq = -1, bid = 0;
    double bv = 0.0;
#pragma unroll
    for (int q = 0; q < PMAX; ++q) {
      const int id = hid[q];
      if (id >= 0 && (bq < 0 || hv[q] > bv || (hv[q] == bv && id < bid))) {
        bq = q;
        bv = hv[q];
        bid = id;
      }
    }
    if (bq < 0) break;  // every list exhausted
    emit(n, bid);
    // advance list bq: predicated selects, one load pair at a computed address
    int h = 0;
#pragma unroll
    for (int q = 0; q < PMAX; ++q) {
      heads[q] += (q == bq) ? 1 : 0;
      h = (q == bq) ? heads[q] : h;
    }
    const int nid = h < M ? L.id[bq * L.qs_i + h] : -1;
    const double nv = nid >= 0 ? L.v[bq * L.qs_v + h] : 0.0;
#pragma unroll
    for (int q = 0; q < PMAX; ++q) {
      hid[q] = (q == bq) ? nid : hid[q];
      hv[q] = (q == bq) ? nv : hv[q];
    }
  }
}

template <int PMAX>
__global__ void __launch_bounds__(kDecideWarps * 32)
    shard_decide_kernel(const __grid_constant__ DevParams p, const MergeIn in,
                        const int32_t *__restrict__ tokens, const DevOut o,
                        int32_t *__restrict__ position, double *__restrict__ uniform,
                        size_t stage_bytes) {
  __shared__ int tsel_s[kDecideWarps][kMaxTopM][32];  // target top-M ids per lane
  // staged slice lists of the warp's sequence ([P][gamma][2][M] values, then ids)
  extern __shared__ __align__(16) unsigned char stage_dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * kDecideWarps + warp;
  if (b >= p.B) return;  // warp-uniform
  const int G = p.gamma, G1 = G + 1, M = p.top_m;
  const int GM2 = G * 2 * M;
  double *sv = reinterpret_cast<double *>(stage_dsm + (size_t)warp * stage_bytes);
  int32_t *si = reinterpret_cast<int32_t *>(sv + (size_t)in.P * GM2);
  if (stage_bytes) {
    // one coalesced pass over this sequence's lists in every slice (the
    // merges below then read shared memory, not dependent global loads)
    // (eight loads per lane in flight: loads first, then the stores)
    const int total = in.P * GM2;
    for (int t0 = 0; t0 < total; t0 += 8 * 32) {
      double v[8];
      int32_t id[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int t = t0 + k * 32 + lane;
        if (t < total) {
          const int q = t / GM2, e = t - q * GM2;
          v[k] = __ldg(in.topv + q * in.topv_stride + (size_t)b * GM2 + e);
          id[k] = __ldg(in.topi + q * in.topi_stride + (size_t)b * GM2 + e);
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int t = t0 + k * 32 + lane;
        if (t < total) {
          sv[t] = v[k];
          si[t] = id[k];
        }
      }
    }
    __syncwarp();
  }
  const double omt = (double)p.omt_f, tau = (double)p.tau_f;
  // gamma + 1 <= 16: two lanes per position, lane j (target side and the
  // decision) and lane j + 16 (draft side), so the two P-way merges and the
  // normalisers of the two rows run side by side; otherwise one lane does both
  const bool split = G1 <= 16;
  const int j = split ? (lane & 15) : lane;
  const bool tside = !split || lane < 16, dside = !split || lane >= 16;
  const bool pair = j < G;
  const double *r0 = in.rec + ((size_t)b * G1 + (j < G1 ? j : 0)) * kRecordWords;
  int(*tsel)[32] = tsel_s[warp];
  SliceLists L{};
  if (pair) {
    if (stage_bytes) {
      L = SliceLists{sv + (size_t)j * 2 * M, si + (size_t)j * 2 * M, (size_t)GM2, (size_t)GM2};
    } else {
      const size_t lo = ((size_t)b * G + j) * 2 * M;
      L = SliceLists{in.topv + lo, in.topi + lo, in.topv_stride, in.topi_stride};
    }
  }
  // ---- target side: LSE_t in shard order, the owner of y, target top-M ----
  double mt = -INFINITY, lse_t = -INFINITY, lt_y = NAN, ld_y = NAN;
  int f = 0, owner = -1, nt = 0;
  if (j < G1 && tside) {
    double xt = -INFINITY;
#pragma unroll(PMAX <= 8 ? PMAX : 1)
    for (int q = 0; q < PMAX; ++q) {
      if (q >= in.P) break;
      const double *r = r0 + q * in.rec_stride;
      const double a_t = r[0] + r[1];
      if (a_t > -INFINITY) mt = fmax(mt, r[0]);
      xt = fmax(xt, a_t);
      if (pair) {
        const int fl = (int)r[7];
        f |= fl;
        if ((fl & 2) && owner < 0) owner = q;
      }
    }
    double et = 0.0;
    for (int q = 0; q < in.P; ++q) {
      const double a_t = r0[q * in.rec_stride] + r0[q * in.rec_stride + 1];
      if (a_t > -INFINITY) et += exp(a_t - xt);
    }
    lse_t = xt == -INFINITY ? -(double)INFINITY : xt + log(et);
    if (owner >= 0) {
      lt_y = r0[owner * in.rec_stride + 5];
      ld_y = r0[owner * in.rec_stride + 6];
    }
    if (pair)
      merge_slice_lists<PMAX>(L, in.P, M, [&](int k, int id) {
        tsel[k][lane] = id;
        nt = k + 1;
      });
  }
  // ---- draft side: LSE_d, LSE_z in shard order, draft top-M ----
  double md = -INFINITY, lse_d = -INFINITY, lse_z = -INFINITY;
  int nd = 0, shared = 0;
  if (pair && dside) {
    double xd = -INFINITY, xz = -INFINITY;
#pragma unroll(PMAX <= 8 ? PMAX : 1)
    for (int q = 0; q < PMAX; ++q) {
      if (q >= in.P) break;
      const double *r = r0 + q * in.rec_stride;
      const double a_d = r[2] + r[3];
      if (a_d > -INFINITY) md = fmax(md, r[2]);
      xd = fmax(xd, a_d);
      xz = fmax(xz, omt * r[0] + tau * r[2] + r[4]);
    }
    double ed = 0.0, ez = 0.0;
    for (int q = 0; q < in.P; ++q) {
      const double *r = r0 + q * in.rec_stride;
      const double a_d = r[2] + r[3];
      if (a_d > -INFINITY) ed += exp(a_d - xd);
      const double a_z = omt * r[0] + tau * r[2] + r[4];
      if (a_z > -INFINITY) ez += exp(a_z - xz);
    }
    lse_d = xd == -INFINITY ? -(double)INFINITY : xd + log(ed);
    lse_z = xz == -INFINITY ? -(double)INFINITY : xz + log(ez);
    L.v += M;
    L.id += M;
    if (split) {
      merge_slice_lists<PMAX>(L, in.P, M, [&](int k, int id) {
        tsel[k][lane] = id;  // column j + 16
        nd = k + 1;
      });
    } else {
      merge_slice_lists<PMAX>(L, in.P, M, [&](int, int id) {
        bool hit = false;
        for (int i = 0; i < nt; ++i) hit |= tsel[i][lane] == id;
        shared += hit ? 1 : 0;
      });
    }
  }
  __syncwarp();
  if (split) {
    const int src = (lane & 15) + 16;
    md = __shfl_sync(0xffffffffu, md, src);
    lse_d = __shfl_sync(0xffffffffu, lse_d, src);
    lse_z = __shfl_sync(0xffffffffu, lse_z, src);
    nd = __shfl_sync(0xffffffffu, nd, src);
    if (pair && tside)
      for (int k = 0; k < nd; ++k) {
        const int id = tsel[k][lane + 16];
        bool hit = false;
        for (int i = 0; i < nt; ++i) hit |= tsel[i][lane] == id;
        shared += hit ? 1 : 0;
      }
  }
  PosSummary sj{0, 0, DSDV_EFF_TARGET, 0, 1};
  if (j < G1 && tside) {
    // ---- decision (fp64) ----
    int err = 0, key = 0, kind = DSDV_EFF_TARGET, near = 0, accepted = 0;
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
      const bool own = owner >= 0;
      if (!(own && y >= 0 && y < p.V) && !err) err = DSDV_E_INVARIANT;  // check_token_in_vocab
      if (!own) lt_y = ld_y = -INFINITY;
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
      if (key || p.tau == 0.0 || (f & 1) == 0)
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
      ev.u = dsdv_philox_uniform(p.seed, p.window, p.seq_offset + (uint32_t)b, (uint32_t)(G + j));
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
    sj = PosSummary{err, key, kind, near, accepted};
  }
  // ---- first rejection or error, left to right (verifier.cpp:223-250) ----
  const bool act = lane < G;
  const unsigned stop = __ballot_sync(0xffffffffu, act && (sj.err || !sj.accepted));
  const int k = stop ? __ffs(stop) - 1 : G;
  const unsigned upto = (k >= 31) ? 0xffffffffu : ((1u << (k + 1)) - 1u);
  const int keys = __popc(__ballot_sync(0xffffffffu, act && sj.key) & upto);
  const int nears = __popc(__ballot_sync(0xffffffffu, act && sj.near) & upto);
  const int err_k = __shfl_sync(0xffffffffu, sj.err, k & 31);
  const int kind_k = __shfl_sync(0xffffffffu, sj.kind, k & 31);
  const int err_g = __shfl_sync(0xffffffffu, sj.err, G & 31);
  if (lane == 0) {
    int st = DSDV_OK, pos = -1;
    double u = 0.0;
    if (k < G) {
      if (err_k) {
        st = err_k;
      } else if (kind_k == DSDV_EFF_DRAFT) {
        st = DSDV_E_EMPTY_RESIDUAL;  // residual of P_d against itself (verifier.cpp:209-211)
      } else {
        pos = k;
        u = dsdv_philox_uniform(p.seed, p.window, p.seq_offset + (uint32_t)b,
                                (uint32_t)(G + k + 1));
      }
    } else if (err_g) {
      st = err_g;
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
  }
}

// Extra draw over a sharded row. MASS: the slice's weight total. RESOLVE: the
// rank whose id range holds T = u * W (W summed over slices in shard order)
// scans its slice; other ranks write -1.
template <class In>
__global__ void __launch_bounds__(kConsumerThreads, 4)
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
      if (mode == 0) {
        put_peers(mass_out + b, 0.0, tpd);
        if (tpd.n) __threadfence_system();
      } else {
        put_peers(token_out + b, -1, tpd);
      }
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
  // MASS keeps the tile sums (tiles_out) for this slice's RESOLVE scan
  double *tiles_b = tiles ? const_cast<double *>(tiles) + (size_t)b * (kMaxTiles + 2) : nullptr;
  const int idx = cdf_sample<In, Acc>(rt, rd, wf, p.vocab_local, 0.0, p.eps_u, &samp, tid, &near,
                                      mode == 1 ? t_local : -1.0, mode == 0 ? tiles_b : nullptr,
                                      mode == 1 ? tiles_b : nullptr, mode == 0, kSliceTileSubs);
  if (tid == 0) {
    if (mode == 0) {
      put_peers(mass_out + b, samp.W, tpd);
      if (tpd.n) __threadfence_system();
    } else {
      put_peers(token_out + b, idx < 0 ? -1 : p.vocab_offset + idx, tpd);
    }
  }
}

template <class In>
cudaError_t launch_shard_sample(const DevParams &p, int mode, int rank, int nranks,
                                const void *draft, const void *target, const double *records,
                                const int32_t *position, const double *uniform,
                                const double *masses, double *mass_out, int32_t *token_out,
                                int32_t *status, const double *tiles, cudaStream_t stream,
                                const long long *tok_delta, int n_delta, size_t mstride);

template <class In>
cudaError_t launch_shard_merge(const DevParams &p, const double *rec, const double *topv,
                               const int32_t *topi, int P, size_t rank_bytes, const void *draft,
                               const void *target, const int32_t *tokens, const DevOut &o,
                               int32_t *position, double *uniform, double *mass_out,
                               double *tiles, cudaStream_t stream, const long long *mass_delta,
                               int n_delta) {
  if (P < 1 || P > kMaxShards || p.gamma > 31 || p.top_m > kMaxTopM || n_delta > 8)
    return cudaErrorInvalidValue;
  const int G1 = p.gamma + 1;
  MergeIn in{rec, topv, topi, P, (size_t)p.B * G1 * kRecordWords,
             (size_t)p.B * p.gamma * 2 * p.top_m, (size_t)p.B * p.gamma * 2 * p.top_m};
  if (rank_bytes) {
    if (rank_bytes % 8) return cudaErrorInvalidValue;
    in.rec_stride = in.topv_stride = rank_bytes / 8;
    in.topi_stride = rank_bytes / 4;
  }
  const int grid = (p.B + kDecideWarps - 1) / kDecideWarps;
  // stage the lists in shared memory while they fit (C4: 7.7 KB per sequence at P=4)
  size_t stage = ((size_t)P * p.gamma * 2 * p.top_m * 12 + 15) & ~size_t(15);
  if (stage * kDecideWarps > kDecideStageMax) stage = 0;
  const size_t dsm = stage * kDecideWarps;
  cudaError_t e;
  // (the attribute is per device: set on every launch, a cheap host call)
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t r =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDecideStageMax);
    if (r != cudaSuccess) return r;
    kern<<<grid, kDecideWarps * 32, dsm, stream>>>(p, in, tokens, o, position, uniform, stage);
    return cudaSuccess;
  };
  if (P <= 2)
    e = go(shard_decide_kernel<2>);
  else if (P <= 4)
    e = go(shard_decide_kernel<4>);
  else if (P <= 8)
    e = go(shard_decide_kernel<8>);
  else
    e = go(shard_decide_kernel<kMaxShards>);
  if (e != cudaSuccess) return e;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // this slice's mass of the extra-draw row (MASS), tile sums kept for RESOLVE
  return launch_shard_sample<In>(p, 0, 0, 1, draft, target, o.records, position, uniform, nullptr,
                                 mass_out, nullptr, nullptr, tiles, stream, mass_delta, n_delta, 0);
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

// One flag round in one launch (dsdv_shard_verify_peers): flag `rank` of every
// rank's buffer = epoch (release, system scope), then hold the stream until
// every rank's flag in this buffer reached epoch (acquire; a timeout sets
// *status). reset: the window's first round clears *status first.
__global__ void peer_round_kernel(PeerBases pb, int nranks, int rank, unsigned long long stride,
                                  unsigned long long epoch, const unsigned long long *flags,
                                  unsigned long long timeout_ns, int *status, int reset) {
  const int q = threadIdx.x;
  if (reset && q == 0) *status = 0;
  if (q < nranks) {
    __threadfence_system();
    unsigned long long *f =
        reinterpret_cast<unsigned long long *>(pb.base[q] + (size_t)nranks * stride) + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(epoch) : "memory");
  }
  __syncwarp();
  if (q < nranks) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + q) : "memory");
      if (v >= epoch) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicExch(status, DSDV_E_NCCL);
        break;
      }
      __nanosleep(100);
    }
  }
  __syncwarp();
  __threadfence_system();
}

cudaError_t launch_peer_round(char *const *bases, int nranks, int rank, unsigned long long stride,
                              unsigned long long epoch, const unsigned long long *flags,
                              unsigned long long timeout_ns, int *status, int reset,
                              cudaStream_t stream) {
  PeerBases pb{};
  for (int q = 0; q < nranks; ++q) pb.base[q] = bases[q];
  peer_round_kernel<<<1, 32, 0, stream>>>(pb, nranks, rank, stride, epoch, flags, timeout_ns,
                                          status, reset);
  return cudaGetLastError();
}

// The window's last step (dsdv_shard_verify_peers): token[b] = max over the
// ranks' RESOLVE outputs, and a timed-out flag round fails every sequence.
__global__ void tokens_fold_kernel(const int32_t *tok, size_t stride, int nranks, int B,
                                   int32_t *out, const int32_t *peer_status, int32_t *status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int32_t m = -1;
  for (int q = 0; q < nranks; ++q) m = max(m, tok[(size_t)q * stride + b]);
  out[b] = m;
  if (*peer_status != 0) status[b] = DSDV_E_NCCL;
}

cudaError_t launch_tokens_fold(const int32_t *tok, size_t stride, int nranks, int B, int32_t *out,
                               const int32_t *peer_status, int32_t *status, cudaStream_t stream) {
  tokens_fold_kernel<<<(B + 255) / 256, 256, 0, stream>>>(tok, stride, nranks, B, out,
                                                          peer_status, status);
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
