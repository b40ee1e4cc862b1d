// Inverse-CDF draw over one softmax-derived row (or row pair), done by the 256
// consumer threads of a CTA.
//
// Semantics follow sample_with_uniform (proj/src/distribution.cpp:103-114):
// the first id (ascending) whose cumulative mass exceeds u, where the mass is
// the normalised weight vector; if u lands in the rounding gap above the total,
// the last supported id wins. Unnormalised weights w are scanned against
// T = u * sum(w), which is the same boundary.
//
// Weights (the `kind` of the row):
//   bonus / draft draw  w_i = P(i)                         (verifier.cpp:253-256, :93-110)
//   residual            w_i = max(0, P_eff(i) - P_d(i))    (verifier.cpp:198-213)
// with P_eff = P_t (key / tau 0 / equal rows) or the softened mix (soften,
// verifier.cpp:161-186, as softmax((1-tau) l_t + tau l_d)).
//
// One streaming pass: warps own contiguous spans of tiles (32 lanes x VEC
// elements x G), every tile's fp64 sum goes to shared memory; one warp scans the
// tile sums for T, and only the crossing tile is re-read to resolve the lane
// and the element.
#pragma once

#include "common.cuh"

namespace dsdv {

enum WeightKind : int { kWeightPlain = 0, kWeightResTarget = 1, kWeightResSoft = 2 };

// Per-row constants of the weight function. Exponents are formed as
// (l - m) - c_hi - c_lo with m a row reference point so that fp32 rounding
// stays relative to the (small) exponent, not to the logit magnitude.
// Correctly rounded scalar ops that the compiler never contracts, so the same
// weight evaluates bit-identically at every call site (the streaming pass and
// the resolver re-read must agree).
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

template <class Acc>
struct Weigher {
  int kind;
  Acc mt, ct_hi, ct_lo;  // P_t(i)  = exp((t_i - mt) - ct)
  Acc md, cd_hi, cd_lo;  // P_d(i)  = exp((d_i - md) - cd)
  Acc omt, tau;          // softened: exp(omt (t_i - mt) + tau (d_i - md) - cz)
  Acc cz_hi, cz_lo;
  // fp32 packed path (weigh_vec): exponents in log2 units, constants split
  // hi/lo so that they stay exact relative to the (small) exponent
  float kt_hi, kt_lo, kd_hi, kd_lo, kz_hi, kz_lo, omtL, tauL;
  // plain (bonus / draft) rows under a temperature: P(i) ~ exp((t_i - mt) / T)
  // (temperature_scale, distribution.cpp:65-97); itemp = 1 / T, 1 otherwise
  Acc itemp;
  float itL;

  __device__ __forceinline__ Acc p_t(Acc t) const {
    return fast_exp2(
        mul_rn(sub_rn(sub_rn(mul_rn(sub_rn(t, mt), itemp), ct_hi), ct_lo), log2e<Acc>()));
  }
  __device__ __forceinline__ Acc operator()(Acc t, Acc d) const {
    if (kind == kWeightPlain) return p_t(t);
    const Acc pd = fast_exp2(mul_rn(sub_rn(sub_rn(sub_rn(d, md), cd_hi), cd_lo), log2e<Acc>()));
    Acc pe;
    if (kind == kWeightResTarget) {
      pe = p_t(t);
    } else {
      const Acc x = add_rn(mul_rn(omt, sub_rn(t, mt)), mul_rn(tau, sub_rn(d, md)));
      pe = fast_exp2(mul_rn(sub_rn(sub_rn(x, cz_hi), cz_lo), log2e<Acc>()));
    }
    const Acc w = sub_rn(pe, pd);
    return w > Acc(0) ? w : Acc(0);
  }
};

// Weights of one 16-byte vector of each row. fp32: packed f32x2 arithmetic,
// one FFMA2 + FADD2 per exponent pair (a = t - mt is exact for bf16 / fp32
// rows near the maximum); every call site (streaming pass, crossing-tile
// re-read) evaluates the identical instruction sequence, so tile sums and the
// resolve agree bit for bit. fp64: the scalar correctly rounded form.
template <int VEC>
__device__ __forceinline__ void weigh_vec(const Weigher<float> &wf, const float (&vt)[VEC],
                                          const float (&vd)[VEC], float (&w)[VEC]) {
  const f32x2 L2 = pk2(kLog2eF, kLog2eF);
  const f32x2 mt2 = pk2(wf.mt, wf.mt), kth = pk2(wf.kt_hi, wf.kt_hi), ktl = pk2(wf.kt_lo, wf.kt_lo);
#pragma unroll
  for (int e = 0; e < VEC; e += 2) {
    const f32x2 a2 = sub2(pk2(vt[e], vt[e + 1]), mt2);
    f32x2 r;
    if (wf.kind == kWeightPlain) {
      const f32x2 xt = add2(fma2(a2, pk2(wf.itL, wf.itL), kth), ktl);
      r = pk2(fast_exp2(lo2(xt)), fast_exp2(hi2(xt)));
    } else {
      const f32x2 b2 = sub2(pk2(vd[e], vd[e + 1]), pk2(wf.md, wf.md));
      const f32x2 xd = add2(fma2(b2, L2, pk2(wf.kd_hi, wf.kd_hi)), pk2(wf.kd_lo, wf.kd_lo));
      const f32x2 pd = pk2(fast_exp2(lo2(xd)), fast_exp2(hi2(xd)));
      f32x2 xe;
      if (wf.kind == kWeightResTarget)
        xe = add2(fma2(a2, L2, kth), ktl);
      else
        xe = add2(fma2(pk2(wf.omtL, wf.omtL), a2,
                       fma2(pk2(wf.tauL, wf.tauL), b2, pk2(wf.kz_hi, wf.kz_hi))),
                  pk2(wf.kz_lo, wf.kz_lo));
      const f32x2 pe = pk2(fast_exp2(lo2(xe)), fast_exp2(hi2(xe)));
      r = sub2(pe, pd);
      r = pk2(fmaxf(lo2(r), 0.f), fmaxf(hi2(r), 0.f));
    }
    w[e] = lo2(r);
    w[e + 1] = hi2(r);
  }
}
template <int VEC>
__device__ __forceinline__ void weigh_vec(const Weigher<double> &wf, const double (&vt)[VEC],
                                          const double (&vd)[VEC], double (&w)[VEC]) {
#pragma unroll
  for (int e = 0; e < VEC; ++e) w[e] = wf(vt[e], vd[e]);
}

template <class Acc>
__device__ __forceinline__ void split_hi_lo(double c, Acc &hi, Acc &lo) {
  hi = (Acc)c;
  lo = (Acc)(c - (double)hi);
}

// Everything the deciding thread derives for one position (or bonus row).
struct PosEval {
  double mt, lst, md, lsd, lsz;  // record words: LSE_t = mt + lst, LSE_d = md + lsd,
                                 // LSE_z = (1-tau) mt + tau md + lsz
  double h_t, h_d, p_t_y, p_d_y, nm, lt_y, ld_y, p_eff, a, u;
  int key, kind, err, near, need_exact, accepted;
};

template <class Acc>
__device__ __forceinline__ void set_weigher(Weigher<Acc> &wf, int kind, const PosEval &ev,
                                            double omt, double tau) {
  wf.kind = kind;
  wf.mt = (Acc)ev.mt;
  split_hi_lo(ev.lst + (ev.mt - (double)wf.mt), wf.ct_hi, wf.ct_lo);
  wf.md = (Acc)ev.md;
  split_hi_lo(ev.lsd + (ev.md - (double)wf.md), wf.cd_hi, wf.cd_lo);
  wf.omt = (Acc)omt;
  wf.tau = (Acc)tau;
  // LSE_z relative to the rounded reference points
  const double lz = omt * (ev.mt - (double)wf.mt) + tau * (ev.md - (double)wf.md) + ev.lsz;
  split_hi_lo(lz, wf.cz_hi, wf.cz_lo);
  // packed fp32 constants (log2 units, relative to the rounded maxima)
  split_hi_lo(-(ev.lst + (ev.mt - (double)wf.mt)) * kLog2e, wf.kt_hi, wf.kt_lo);
  split_hi_lo(-(ev.lsd + (ev.md - (double)wf.md)) * kLog2e, wf.kd_hi, wf.kd_lo);
  split_hi_lo(-lz * kLog2e, wf.kz_hi, wf.kz_lo);
  wf.omtL = (float)(omt * kLog2e);
  wf.tauL = (float)(tau * kLog2e);
  wf.itemp = Acc(1);
  wf.itL = kLog2eF;
}

constexpr int kMaxTiles = 512;

struct SampleShared {
  double tile[kMaxTiles];
  double warp_total[kConsumerWarps];
  int warp_last[kConsumerWarps];
  double base, T, W;
  int crossing_tile;
  int result;
  int near;
};

__device__ __forceinline__ double warp_sum_f64(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Weights of the VEC elements at `base` for this lane (MASK: zero the ids at or
// past n; a vector wholly inside the row skips it).
template <class In, class Acc, bool MASK = true>
__device__ __forceinline__ void vec_weights(const uint4 &rt, const uint4 &rd, int base, int n,
                                            const Weigher<Acc> &wf, Acc (&w)[InTraits<In>::kVec]) {
  constexpr int VEC = InTraits<In>::kVec;
  Acc vt[VEC], vd[VEC];
  unpack(rt, vt, (In *)nullptr);
  unpack(rd, vd, (In *)nullptr);
  weigh_vec<VEC>(wf, vt, vd, w);
  if (MASK) {
#pragma unroll
    for (int e = 0; e < VEC; ++e)
      if (base + e >= n) w[e] = Acc(0);
  }
}

// Called by all kConsumerThreads threads (thread index `tid` in [0, 256)).
// Returns the sampled local index, or -1 when the weights have no mass; the
// total weight stays in sh->W until the next call.
template <class In, class Acc>
__device__ __noinline__ int cdf_sample(const In *row_t, const In *row_d, const Weigher<Acc> &wf_s,
                                       int n, double u, double eps, SampleShared *sh, int tid,
                                       int *near_out, double t_override = -1.0,
                                       double *tiles_out = nullptr,
                                       const double *tiles_in = nullptr,
                                       bool mass_only = false, int min_g = 1) {
  constexpr int VEC = InTraits<In>::kVec;
  constexpr int U = 4;  // tiles in flight per warp
  const Weigher<Acc> wf = wf_s;
  const bool two_rows = wf.kind != kWeightPlain;
  const int warp = tid >> 5, lane = tid & 31;
  const int sub = 32 * VEC;                          // elements per sub-tile
  const int nsub = (n + sub - 1) / sub;
  // sub-tiles per tile (min_g > 1: fewer, longer tiles for short rows, fewer
  // per-tile reductions; every pass over the same row must use the same value)
  const int G = max(min_g, (nsub + kMaxTiles - 1) / kMaxTiles);
  const int ntiles = (nsub + G - 1) / G;
  const int per_warp = (ntiles + kConsumerWarps - 1) / kConsumerWarps;
  const int t0 = min(ntiles, warp * per_warp);
  const int t1 = min(ntiles, t0 + per_warp);

  // ---- one pass: tile sums -> shared memory (or the sums a previous call
  // over the same row and weights saved: tiles_in = [kMaxTiles] sums, W, last) ----
  int last = -1;
  double wsum = 0.0;
  if (tiles_in) {
    for (int t = tid; t < ntiles; t += kConsumerThreads) sh->tile[t] = tiles_in[t];
    if (tid == 0) {
      sh->warp_total[0] = tiles_in[kMaxTiles];
      sh->warp_last[0] = (int)tiles_in[kMaxTiles + 1];
    } else if (tid < kConsumerWarps) {
      sh->warp_total[tid] = 0.0;
      sh->warp_last[tid] = -1;
    }
  }
  for (int t = tiles_in ? t1 : t0; t < t1; t += U) {
    double ls[U];
#pragma unroll
    for (int k = 0; k < U; ++k) ls[k] = 0.0;
    for (int g = 0; g < G; ++g) {
      uint4 rt[U], rd[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int base = ((t + k) * G + g) * sub + lane * VEC;
        const bool ok = (t + k) < t1 && base < n;
        rt[k] = ok ? ldg128(row_t + base) : make_uint4(0, 0, 0, 0);
        rd[k] = (ok && two_rows) ? ldg128(row_d + base) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int base = ((t + k) * G + g) * sub + lane * VEC;
        if ((t + k) < t1 && base < n) {
          Acc w[VEC];
          if (base + VEC <= n)
            vec_weights<In, Acc, false>(rt[k], rd[k], base, n, wf, w);
          else
            vec_weights<In, Acc, true>(rt[k], rd[k], base, n, wf, w);
          // lane sum in the accumulation type, one conversion per vector; the
          // last vector with mass is kept (its last supported id is resolved
          // once, below)
          Acc lv = Acc(0);
#pragma unroll
          for (int e = 0; e < VEC; ++e) lv += w[e];
          // (max, not the latest: with several sub-tiles per tile the
          // processing order is not the id order)
          if (lv > Acc(0)) last = max(last, base);
          ls[k] += (double)lv;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (t + k < t1) {
        const double ts = warp_sum_f64(ls[k]);
        if (lane == 0) sh->tile[t + k] = ts;
        wsum += ts;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
  if (lane == 0 && !tiles_in) {
    sh->warp_total[warp] = wsum;
    sh->warp_last[warp] = last;
  }
  consumer_sync();

  // ---- warp 0: total, T = u W, crossing tile ----
  if (warp == 0) {
    double W = 0.0;
    int L = -1;
    for (int w = 0; w < kConsumerWarps; ++w) {
      W += sh->warp_total[w];
      L = max(L, sh->warp_last[w]);
    }
    if (!tiles_in && L >= 0) {
      // L is the base of the last vector with mass: its last supported id
      // (the rounding-gap fallback of sample_with_uniform)
      int e_last = 0;
      if (lane == 0) {
        const uint4 rt = ldg128(row_t + L);
        const uint4 rd = two_rows ? ldg128(row_d + L) : make_uint4(0, 0, 0, 0);
        Acc w[VEC];
        vec_weights<In, Acc, true>(rt, rd, L, n, wf, w);
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          if (w[e] > Acc(0)) e_last = e;
      }
      L += __shfl_sync(0xffffffffu, e_last, 0);
    }
    // t_override >= 0: the boundary was placed by the caller (a vocabulary
    // slice of a sharded row, T relative to this slice's first id)
    const double T = t_override >= 0.0 ? t_override : u * W;
    double run = 0.0;
    int found = -1;
    double base = 0.0;
    for (int c = 0; c < ntiles && found < 0; c += 32) {
      const int t = c + lane;
      const double x = t < ntiles ? sh->tile[t] : 0.0;
      double incl = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, t < ntiles && x > 0.0 && run + incl > T);
      if (hit) {
        const int src = __ffs(hit) - 1;
        found = c + src;
        base = run + __shfl_sync(0xffffffffu, incl - x, src);
      }
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tiles_out) {
      for (int t = lane; t < ntiles; t += 32) tiles_out[t] = sh->tile[t];
      if (lane == 0) {
        tiles_out[kMaxTiles] = W;
        tiles_out[kMaxTiles + 1] = (double)L;
      }
    }
    if (lane == 0) {
      sh->W = W;
      sh->T = T;
      sh->base = base;
      sh->crossing_tile = (W > 0.0 && !mass_only) ? found : -1;
      sh->result = (W > 0.0) ? L : -1;  // rounding-gap fallback: last supported id
      sh->near = (W > 0.0 && found < 0) ? 1 : 0;
    }
  }
  consumer_sync();

  // ---- warp 0: resolve lane and element inside the crossing tile ----
  const int ct = sh->crossing_tile;
  if (warp == 0 && ct >= 0) {
    const double T = sh->T, W = sh->W;
    double run = sh->base;
    bool done = false;
    // the first kPre sub-tiles' loads are issued together (one round trip)
    constexpr int kPre = 4;
    uint4 pre_t[kPre], pre_d[kPre];
#pragma unroll
    for (int k = 0; k < kPre; ++k) {
      const int base = (ct * G + k) * sub + lane * VEC;
      const bool ok = k < G && base < n;
      pre_t[k] = ok ? ldg128(row_t + base) : make_uint4(0, 0, 0, 0);
      pre_d[k] = (ok && two_rows) ? ldg128(row_d + base) : make_uint4(0, 0, 0, 0);
    }
    for (int g = 0; g < G && !done; ++g) {
      const int base = (ct * G + g) * sub + lane * VEC;
      Acc w[VEC];
      const bool ok = base < n;
      uint4 rt, rd;
      if (g < kPre) {
        // static selection (no dynamic index into the register arrays)
        rt = pre_t[0];
        rd = pre_d[0];
#pragma unroll
        for (int k = 1; k < kPre; ++k)
          if (g == k) {
            rt = pre_t[k];
            rd = pre_d[k];
          }
      } else {
        rt = ok ? ldg128(row_t + base) : make_uint4(0, 0, 0, 0);
        rd = (ok && two_rows) ? ldg128(row_d + base) : make_uint4(0, 0, 0, 0);
      }
      if (ok) {
        vec_weights<In, Acc>(rt, rd, base, n, wf, w);
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e) w[e] = Acc(0);
      }
      double ls = 0.0;
#pragma unroll
      for (int e = 0; e < VEC; ++e) ls += (double)w[e];
      double incl = ls;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const double excl = run + (incl - ls);
      const unsigned hit = __ballot_sync(0xffffffffu, ls > 0.0 && excl + ls > T);
      if (hit) {
        const int src = __ffs(hit) - 1;
        if (lane == src) {
          double c = excl, margin = 0.0;
          int idx = -1, lastsup = -1;
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            if (idx < 0 && w[e] > Acc(0)) {
              lastsup = e;
              const double nc = c + (double)w[e];
              if (T < nc) {
                idx = e;
                margin = fmin(T - c, nc - T);
              }
              c = nc;
            }
          }
          if (idx >= 0) {
            sh->result = base + idx;
            sh->near = (margin < eps * W) ? 1 : 0;
          } else {
            sh->result = base + lastsup;
            sh->near = 1;
          }
        }
        done = true;
      } else {
        const unsigned sup = __ballot_sync(0xffffffffu, ls > 0.0);
        if (sup && lane == 31 - __clz(sup)) {
          int lastsup = -1;
#pragma unroll
          for (int e = 0; e < VEC; ++e)
            if (w[e] > Acc(0)) lastsup = e;
          sh->result = base + lastsup;  // provisional: the tile's upper edge
        }
        run += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (!done && lane == 0) sh->near = 1;
  }
  consumer_sync();
  const int r = sh->result;
  if (near_out) *near_out = sh->near;
  consumer_sync();  // scratch reusable after return
  return r;
}

}  // namespace dsdv
