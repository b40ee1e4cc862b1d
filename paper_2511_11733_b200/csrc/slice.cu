// Vocabulary-slice statistics with one warp per item (dsdv_shard_stats,
// dsdv_shard_stats_peers).
//
// A rank of a vocabulary-sharded window reads slices of V/P ids, so its rows
// are P times shorter and there are P times more of them than in the
// unsharded window at the same bytes. In the fused kernel (verify.cu) all
// compute warps share each item, and every item's first chunk costs each of
// them a bound sort and a capture: at P=4 that first-chunk work was a third of
// the pass. Here each warp streams whole row pairs on its own:
//   * a private ring of kStages stages (1 KB of each row per stage) fed by
//     1-D bulk copies that the warp's lane 0 issues, one mbarrier per stage;
//     the next item's first chunks are issued while the current one drains;
//   * per lane: lazy-max online sums of e^l_t, e^l_d and of the softened mix
//     in log2 units (packed f32x2 for bf16 / fp32 rows);
//   * top-m per row: per-lane running maxima in registers, a bound derived
//     from them once per raise (one warp sort per row and raise, not one per
//     warp and item), and the elements that reach the bound captured into a
//     warp-private list, compacted when it fills; the final ranking is exact
//     (value desc, id asc, like top_ids, verifier.cpp:40-51), with a re-read
//     of the row as the fallback when the list overflowed;
//   * the partial record and the top lists are written exactly as the fused
//     kernel's write_partial does, including the stores into every peer's
//     exchange buffer.
// Work items (b, j) are claimed from a global ticket, one per warp at a time.
#include <cuda_runtime.h>

#include <climits>

#include "common.cuh"

namespace dsdv {
namespace slice {

#if defined(DSDV_SLICE_STATS) || defined(DSDV_SLICE_CYC)
// development counters (DSDV_SLICE_STATS): rows, blocks entering the capture
// path, sorts, captured elements, compactions, overflows; cycles per role
// (DSDV_SLICE_CYC, per-warp registers flushed at exit)
__device__ unsigned long long g_cnt[8];
__device__ unsigned long long g_cyc[4];  // issue, finish, wait_full, kernel
#endif
#ifdef DSDV_SLICE_STATS
#define SL_CNT(i, v) atomicAdd(&g_cnt[i], (unsigned long long)(v))
#else
#define SL_CNT(i, v) (void)0
#endif

constexpr int kWarps = 16;                     // item streams per CTA (one CTA per SM)
constexpr int kStages = 4;                     // per-warp ring depth
constexpr int kVecsW = 2;                      // 16-byte vectors per lane per row and stage
constexpr int kRowBytesW = 32 * 16 * kVecsW;   // 1 KB per row per stage
// captured top-m candidates per row (ties in bf16 rows can leave 100+
// elements at the bound)
template <class Acc>
constexpr int cap_w() {
  return sizeof(Acc) == 4 ? 256 : 128;
}
// rows of at most kMaxBlk stages (vocabulary slices: 64K bf16 ids) keep only
// per-block maxima while they stream and select the top M afterwards
constexpr int kMaxBlk = 128;
constexpr float kSlackW = 8.0f;                // lazy max: rescale past m + 8
constexpr float kFloorMW = -1e30f;             // finite "empty" maximum

template <class Acc>
struct WarpSmem {
  alignas(128) uint8_t ring[kStages][2][kRowBytesW];  // [stage][0 draft, 1 target]
  uint64_t full[kStages];
  int meta_item[kStages];
  int meta_chunk[kStages];
  int ncap_s[2];
  int bmax[2][kMaxBlk];  // deferred mode: per-block maximum keys of both rows
  int cap_id[2][cap_w<Acc>()];
  Acc cap_v[2][cap_w<Acc>()];
  int sel_id[2][32];
  Acc sel_v[2][32];
};

template <class Acc>
struct CtaSmem {
  WarpSmem<Acc> w[kWarps];
};

__device__ __forceinline__ int fkey(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ int fkey(double f) { return fkey(__double2float_rd(f)); }

__device__ __forceinline__ int warp_max_key(int key) {
  int r;
  asm volatile("redux.sync.max.s32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(key));
  return r;
}

// Descending bitonic sort of one int per lane; returns entry m - 1.
__device__ __noinline__ int mth_largest(int key, int m, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int pk = __shfl_xor_sync(0xffffffffu, key, j);
      const bool keep_max = ((lane & j) == 0) == ((lane & k) == 0);
      key = keep_max ? max(key, pk) : min(key, pk);
    }
  }
  return __shfl_sync(0xffffffffu, key, m - 1);
}

__device__ __forceinline__ unsigned long long bits_of(double x) {
  return (unsigned long long)__double_as_longlong(x);
}
__device__ __forceinline__ unsigned long long bits_of(float x) { return __float_as_uint(x); }

__device__ __forceinline__ float vmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ double vmax3(double a, double b, double c) { return fmax(fmax(a, b), c); }

// Per-lane online statistics of one item (sums relative to the log2 reference
// points mtL / mdL; see verify.cu ItemState for the conversion back).
template <class Acc>
struct LaneStats {
  Acc mt, md, mtL, mdL;
  Acc st, sd, sz;       // fp64 rows
  f32x2 pst, psd, psz;  // fp32 accumulation (bf16 / fp32 rows)
  uint32_t diff;
  __device__ __forceinline__ void reset() {
    mt = md = Acc(kFloorMW);
    mtL = mdL = Acc(kFloorMW) * log2e<Acc>();
    st = sd = sz = Acc(0);
    pst = psd = psz = 0ull;
    diff = 0;
  }
};

// Top-m capture state of one row (warp-uniform bound and count).
struct RowCap {
  int bin;    // this lane's running maximum key (over the blocks that reached th)
  int th;     // bound: every element of the final top M is >= th
  int ncap;   // entries in the list, -1 once the list overflowed
};

// Drop the entries below the current bound (in place, order kept).
template <class Acc>
__device__ __forceinline__ void compact(WarpSmem<Acc> &ws, int r, RowCap &rc, int lane) {
  const int n = rc.ncap;
  int out = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    Acc v = Acc(0);
    int id = 0;
    bool keep = false;
    if (i < n) {
      v = ws.cap_v[r][i];
      id = ws.cap_id[r][i];
      keep = fkey(v) >= rc.th;
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) {
      const int at = out + __popc(m & ((1u << lane) - 1u));
      ws.cap_v[r][at] = v;
      ws.cap_id[r][at] = id;
    }
    out += __popc(m);
    __syncwarp();
  }
  rc.ncap = out;
  if (lane == 0) ws.ncap_s[r] = out;
  __syncwarp();
}

__device__ __forceinline__ float fkey_inv(int k) {
  return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff);
}
// key(v) >= th <=> v >= key_floor(th) (keys of doubles round toward -inf)
template <class Acc>
__device__ __forceinline__ Acc key_floor(int th) {
  return th == INT_MIN ? neg_inf<Acc>() : (Acc)fkey_inv(th);
}

// This lane's elements of the block that can still be in the top M, as bits
// (element e of v is id id0 + (e / VEC) * 32 * VEC + e % VEC): v >= the
// bound th, and v > the bound th0 at the start of the block. A warp streams
// its row in id order, so th0 rests on M elements of earlier blocks, all with
// smaller ids: an element equal to th0 loses every tie against them
// ((value desc, id asc)). bf16 rows put many elements on the bound's value.
template <class Acc, int N, int VEC, bool TAIL>
__device__ __forceinline__ unsigned keep_bits(const Acc (&v)[N], int id0, int n, int th,
                                              int th0) {
  const Acc lo = key_floor<Acc>(th), lo0 = key_floor<Acc>(th0);
  unsigned keep = 0;
#pragma unroll
  for (int e = 0; e < N; ++e) {
    const bool ok = !TAIL || id0 + (e / VEC) * 32 * VEC + e % VEC < n;
    keep |= (ok && v[e] >= lo && (th0 == INT_MIN || v[e] > lo0) ? 1u : 0u) << e;
  }
  return keep;
}

// One block (this warp's share of a stage) of row r: bins, bound raises,
// capture. lkey = this lane's maximum key of the block; srow = the block's
// row in the stage (captured elements are re-read from it by index). A block
// that may not fit the list raises the bound and compacts first; if it still
// does not fit, the row is marked overflowed (ncap = -1) and finish_topm
// re-reads it.
template <class In, class Acc, int N, int VEC, bool TAIL>
__device__ __forceinline__ void topm_block(WarpSmem<Acc> &ws, int r, RowCap &rc, int lkey,
                                           const Acc (&v)[N], const uint8_t *srow, int id0,
                                           int n, int M, int lane) {
  const int bk = warp_max_key(lkey);
  const int th0 = rc.th;
  if (bk <= th0 && th0 != INT_MIN) return;
  if (lane == 0) SL_CNT(1, 1);
  rc.bin = max(rc.bin, lkey);
  if (th0 == INT_MIN || __popc(__ballot_sync(0xffffffffu, rc.bin > rc.th)) >= min(M + 8, 32)) {
    if (lane == 0) SL_CNT(2, 1);
    rc.th = max(rc.th, mth_largest(rc.bin, M, lane));
  }
  if (rc.ncap < 0 || bk < rc.th) return;
  unsigned keep = keep_bits<Acc, N, VEC, TAIL>(v, id0, n, rc.th, th0);
  int total = __reduce_add_sync(0xffffffffu, __popc(keep));
  if (lane == 0) SL_CNT(3, total);
  if (rc.ncap + total > cap_w<Acc>()) {
    if (lane == 0) SL_CNT(4, 1);
    rc.th = max(rc.th, mth_largest(rc.bin, M, lane));
    compact(ws, r, rc, lane);
    keep = keep_bits<Acc, N, VEC, TAIL>(v, id0, n, rc.th, th0);
    total = __reduce_add_sync(0xffffffffu, __popc(keep));
    if (rc.ncap + total > cap_w<Acc>()) {
      if (lane == 0) SL_CNT(5, 1);
      rc.ncap = -1;
      return;
    }
  }
  if (keep) {
    // this lane's slots (ws.ncap_s mirrors rc.ncap; the order of the entries
    // does not matter, the ranking in finish_topm is exact)
    int at = atomicAdd(&ws.ncap_s[r], __popc(keep));
    const In *src = reinterpret_cast<const In *>(srow);
    while (keep) {
      const int e = __ffs(keep) - 1;
      keep &= keep - 1;
      const int q = (e / VEC) * 32 + lane;  // vector index in the stage row
      ws.cap_v[r][at] = (Acc)load_smem_scalar(src + q * VEC + e % VEC);
      ws.cap_id[r][at] = id0 + (e / VEC) * 32 * VEC + e % VEC;
      ++at;
    }
  }
  rc.ncap += total;
  __syncwarp();
}

// Exact top M of one row from the captured candidates (or, after an
// overflow, from a re-read of the row), (value desc, id asc), into sel_*[r].
template <class In, class Acc>
__device__ __noinline__ void finish_topm(WarpSmem<Acc> &ws, int r, RowCap rc, const In *row,
                                         int n, int M, int lane) {
  constexpr int VEC = InTraits<In>::kVec;
  if (lane < M) {
    ws.sel_id[r][lane] = -1;
    ws.sel_v[r][lane] = neg_inf<Acc>();
  }
  rc.th = max(rc.th, mth_largest(rc.bin, M, lane));
  __syncwarp();
  if (lane == 0) SL_CNT(0, 1);
  if (rc.ncap >= 0) {
    compact(ws, r, rc, lane);
    const int nel = rc.ncap;
    if (lane == 0) SL_CNT(6, nel);
    for (int i = lane; i < nel; i += 32) {
      const Acc vi = ws.cap_v[r][i];
      const int ii = ws.cap_id[r][i];
      int rank = 0;
      for (int k = 0; k < nel; ++k) {
        const Acc vk = ws.cap_v[r][k];
        rank += (vk > vi || (vk == vi && ws.cap_id[r][k] < ii)) ? 1 : 0;
      }
      if (rank < M) {
        ws.sel_id[r][rank] = ii;
        ws.sel_v[r][rank] = vi;
      }
    }
    __syncwarp();
    return;
  }
  // overflow: the whole row again, every element at or above the bound
  TopList<Acc> L;
  L.reset();
  const int nvec = (n + VEC - 1) / VEC;
  for (int q0 = 0; q0 < nvec; q0 += 32) {
    const int q = q0 + lane;
    Acc v[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) v[e] = neg_inf<Acc>();
    if (q < nvec) unpack(ldg128(row + (size_t)q * VEC), v, (In *)nullptr);
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const bool c = q < nvec && q * VEC + e < n && fkey(v[e]) >= rc.th && v[e] >= L.theta;
      unsigned qq = __ballot_sync(0xffffffffu, c);
      while (qq) {
        const int src = __ffs(qq) - 1;
        qq &= qq - 1;
        const Acc cv = __shfl_sync(0xffffffffu, v[e], src);
        const int ci = __shfl_sync(0xffffffffu, q * VEC + e, src);
        if (cv >= L.theta) L.insert(cv, ci, M, lane);
      }
    }
  }
  if (lane < M && L.id != 0x7fffffff) {
    ws.sel_id[r][lane] = L.id;
    ws.sel_v[r][lane] = L.v;
  }
  __syncwarp();
}

// Deferred top M of one row (rows of at most kMaxBlk blocks): the bound is
// the best of the M-th largest lane maximum and, per group of 32 blocks, the
// M-th largest block maximum; only the blocks whose maximum reaches it are
// re-read (the row streamed a moment ago; about M of them), their elements at
// or above the bound go into the list, and the list is ranked exactly. Ties on
// the bound can overflow the list: then the whole row is scanned.
template <class In, class Acc>
__device__ __noinline__ void finish_topm_deferred(WarpSmem<Acc> &ws, int r, int bin,
                                                  const In *row, int n, int nblk, int M,
                                                  int lane) {
  constexpr int VEC = InTraits<In>::kVec;
  constexpr int CHE = kRowBytesW / (int)sizeof(In);
  constexpr int NE = kVecsW * VEC;
  RowCap rc{bin, mth_largest(bin, M, lane), 0};
  for (int g = 0; g < nblk; g += 32) {
    const int k = g + lane < nblk ? ws.bmax[r][g + lane] : INT_MIN;
    rc.th = max(rc.th, mth_largest(k, M, lane));
  }
  const Acc lo = key_floor<Acc>(rc.th);
  if (lane == 0) ws.ncap_s[r] = 0;
  __syncwarp();
  for (int g = 0; g < nblk && rc.ncap >= 0; g += 32) {
    unsigned q = __ballot_sync(0xffffffffu, g + lane < nblk && ws.bmax[r][g + lane] >= rc.th);
    while (q && rc.ncap >= 0) {
      // up to four blocks' loads in flight
      int blk[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        blk[k] = q ? g + __ffs(q) - 1 : -1;
        if (q) q &= q - 1;
      }
      uint4 raw[4][kVecsW];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int h = 0; h < kVecsW; ++h) {
          const int id = blk[k] * CHE + (h * 32 + lane) * VEC;
          raw[k][h] = (blk[k] >= 0 && id < n) ? ldg128(row + id) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (blk[k] < 0) break;
        Acc v[NE];
#pragma unroll
        for (int h = 0; h < kVecsW; ++h) {
          Acc t[VEC];
          unpack(raw[k][h], t, (In *)nullptr);
#pragma unroll
          for (int e = 0; e < VEC; ++e) v[h * VEC + e] = t[e];
        }
        const int id0 = blk[k] * CHE + lane * VEC;
        unsigned keep = 0;
#pragma unroll
        for (int e = 0; e < NE; ++e)
          keep |= (id0 + (e / VEC) * 32 * VEC + e % VEC < n && v[e] >= lo ? 1u : 0u) << e;
        const int total = __reduce_add_sync(0xffffffffu, __popc(keep));
        if (rc.ncap + total > cap_w<Acc>()) {
          rc.ncap = -1;
          break;
        }
        if (keep) {
          int at = atomicAdd(&ws.ncap_s[r], __popc(keep));
#pragma unroll
          for (int e = 0; e < NE; ++e)
            if (keep & (1u << e)) {
              ws.cap_v[r][at] = v[e];
              ws.cap_id[r][at] = id0 + (e / VEC) * 32 * VEC + e % VEC;
              ++at;
            }
        }
        rc.ncap += total;
      }
      __syncwarp();
    }
  }
  finish_topm<In, Acc>(ws, r, rc, row, n, M, lane);
}

// Exact log-sum-exp of the softened mix (two fp64 passes, one warp): the rare
// rows whose fp32 mix sum underflowed against its reference point.
template <class In>
__device__ __noinline__ double exact_lse_mix(const In *rt, const In *rd, int n, double omt,
                                             double tau, int lane) {
  constexpr int VEC = InTraits<In>::kVec;
  using Acc = typename InTraits<In>::Acc;
  const int nvec = (n + VEC - 1) / VEC;
  double zmax = -INFINITY;
  for (int q = lane; q < nvec; q += 32) {
    Acc t[VEC], d[VEC];
    unpack(ldg128(rt + (size_t)q * VEC), t, (In *)nullptr);
    unpack(ldg128(rd + (size_t)q * VEC), d, (In *)nullptr);
    for (int e = 0; e < VEC; ++e)
      if (q * VEC + e < n) zmax = fmax(zmax, omt * (double)t[e] + tau * (double)d[e]);
  }
  for (int o = 16; o > 0; o >>= 1) zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
  if (zmax == -INFINITY) return -INFINITY;
  double s = 0.0;
  for (int q = lane; q < nvec; q += 32) {
    Acc t[VEC], d[VEC];
    unpack(ldg128(rt + (size_t)q * VEC), t, (In *)nullptr);
    unpack(ldg128(rd + (size_t)q * VEC), d, (In *)nullptr);
    for (int e = 0; e < VEC; ++e)
      if (q * VEC + e < n) s += exp(omt * (double)t[e] + tau * (double)d[e] - zmax);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return zmax + log(s);
}

// Lane-stat merge (xor tree, accumulation precision), like verify.cu's
// merge_partials over the lanes of one warp.
template <class Acc>
__device__ __forceinline__ void merge_lanes(LaneStats<Acc> S, const DevParams &p,
                                            double (&out)[7]) {
  Acc mt = S.mt, md = S.md, mtL = S.mtL, mdL = S.mdL, st = S.st, sd = S.sd, sz = S.sz;
  const Acc omt = Acc(p.omt_f), tau = Acc(p.tau_f);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const Acc mt2 = __shfl_xor_sync(0xffffffffu, mt, off);
    const Acc md2 = __shfl_xor_sync(0xffffffffu, md, off);
    const Acc mtL2 = __shfl_xor_sync(0xffffffffu, mtL, off);
    const Acc mdL2 = __shfl_xor_sync(0xffffffffu, mdL, off);
    const Acc st2 = __shfl_xor_sync(0xffffffffu, st, off);
    const Acc sd2 = __shfl_xor_sync(0xffffffffu, sd, off);
    const Acc sz2 = __shfl_xor_sync(0xffffffffu, sz, off);
    const Acc ML = fmax(mtL, mtL2), DL = fmax(mdL, mdL2);
    st = st * fast_exp2(mtL - ML) + st2 * fast_exp2(mtL2 - ML);
    sd = sd * fast_exp2(mdL - DL) + sd2 * fast_exp2(mdL2 - DL);
    sz = sz * fast_exp2(omt * (mtL - ML) + tau * (mdL - DL)) +
         sz2 * fast_exp2(omt * (mtL2 - ML) + tau * (mdL2 - DL));
    mt = fmax(mt, mt2);
    md = fmax(md, md2);
    mtL = ML;
    mdL = DL;
  }
  out[0] = (double)mt;
  out[1] = (double)st;
  out[2] = (double)md;
  out[3] = (double)sd;
  out[4] = (double)sz;
  out[5] = (double)mtL;
  out[6] = (double)mdL;
}

template <class In, bool NEEDZ, bool DEFER>
__global__ void __launch_bounds__(kWarps * 32, 1)
    slice_stats_kernel(const __grid_constant__ DevParams p, const In *__restrict__ draft,
                       const In *__restrict__ target, const int32_t *__restrict__ tokens,
                       const DevOut o, unsigned int *ticket, unsigned int *exit_count) {
  using Acc = typename InTraits<In>::Acc;
  constexpr int VEC = InTraits<In>::kVec;
  constexpr int CHE = kRowBytesW / (int)sizeof(In);  // elements per row per stage
  constexpr int NE = kVecsW * VEC;                   // elements per lane per row per stage
  extern __shared__ __align__(128) unsigned char dsm[];
  CtaSmem<Acc> &cs = *reinterpret_cast<CtaSmem<Acc> *>(dsm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmem<Acc> &ws = cs.w[warp];
  const int G = p.gamma, G1 = G + 1, M = p.top_m, n = p.vocab_local;
  const int nch = (n + CHE - 1) / CHE;
  const size_t row_bytes = ((size_t)n * sizeof(In) + 15) & ~size_t(15);
  const int n_items = p.B * G1;

#ifdef DSDV_SLICE_CYC
  const long long tk0 = clock64();
  long long cyc_topm = 0, cyc_issue = 0, cyc_fin = 0, cyc_wait = 0;
#endif
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&ws.full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // ---- lane 0: the warp's copy stream. Items are claimed one ahead (the
  // claim's latency overlaps the current item); per stage only offsets move.
  int iss_item = n_items, nxt_item = n_items, iss_chunk = 0;
  const char *it_rt = nullptr, *it_rd = nullptr;
  auto start_item = [&]() {
    iss_item = nxt_item;
    iss_chunk = 0;
    if (iss_item < n_items) {
      nxt_item = (int)atomicAdd(ticket, 1u);
      const int bb = iss_item / G1, jj = iss_item - bb * G1;
      it_rt = reinterpret_cast<const char *>(target + ((size_t)bb * G1 + jj) * p.stride);
      it_rd = jj < G ? reinterpret_cast<const char *>(draft + ((size_t)bb * G + jj) * p.stride)
                     : nullptr;
    }
  };
  auto issue = [&](int seq) {
    const int stage = seq % kStages;
    if (iss_item >= n_items) {  // end of stream: an empty stage tells the lanes
      ws.meta_item[stage] = -1;
      mbar_arrive(&ws.full[stage]);
      return;
    }
    const size_t off = (size_t)iss_chunk * kRowBytesW;
    const uint32_t bytes = (uint32_t)min((size_t)kRowBytesW, row_bytes - off);
    ws.meta_item[stage] = iss_item;
    ws.meta_chunk[stage] = iss_chunk;
    mbar_arrive_expect_tx(&ws.full[stage], it_rd ? 2u * bytes : bytes);
    bulk_g2s(ws.ring[stage][1], it_rt + off, bytes, &ws.full[stage]);
    if (it_rd) bulk_g2s(ws.ring[stage][0], it_rd + off, bytes, &ws.full[stage]);
    if (++iss_chunk == nch) start_item();
  };
  if (lane == 0) {
    nxt_item = (int)atomicAdd(ticket, 1u);
    start_item();
    for (int s = 0; s < kStages; ++s) issue(s);
  }

  const Acc L = log2e<Acc>();
  const Acc ni = neg_inf<Acc>();
  LaneStats<Acc> S;
  RowCap cap[2];
  int b = 0, j = 0;
  bool pair = false;
  for (int seq = 0;; ++seq) {
    const int stage = seq % kStages;
#ifdef DSDV_SLICE_CYC
    const long long tq0 = clock64();
#endif
#ifdef DSDV_SLICE_SUSPEND
    mbar_wait(&ws.full[stage], (uint32_t)(seq / kStages) & 1u);
#else
    // plain probes: the data is usually there; a suspended warp wakes late
    mbar_wait_spin(&ws.full[stage], (uint32_t)(seq / kStages) & 1u);
#endif
#ifdef DSDV_SLICE_CYC
    cyc_wait += clock64() - tq0;
#endif
    const int item = ws.meta_item[stage];
    if (item < 0) break;
    const int c = ws.meta_chunk[stage];
    if (c == 0) {
      b = item / G1;
      j = item - b * G1;
      pair = j < G;
      S.reset();
      cap[0] = RowCap{INT_MIN, INT_MIN, 0};
      cap[1] = RowCap{INT_MIN, INT_MIN, 0};
      if (lane < 2) ws.ncap_s[lane] = 0;
      __syncwarp();
    }
    // ---- this lane's vectors: ids c*CHE + (h*32 + lane)*VEC + e ----
    const int id0 = c * CHE + lane * VEC;
    // the last stage of a row that is not a whole number of stages holds
    // stale bytes past the row: masked to -inf, compared element by element
    const bool tail = c == nch - 1 && n % CHE != 0;
    Acc vt[NE], vd[NE];
#pragma unroll
    for (int h = 0; h < kVecsW; ++h) {
      const uint4 a = lds128(ws.ring[stage][1] + (h * 32 + lane) * 16);
      Acc t[VEC];
      unpack(a, t, (In *)nullptr);
#pragma unroll
      for (int e = 0; e < VEC; ++e) vt[h * VEC + e] = t[e];
      if (pair) {
        const uint4 bb = lds128(ws.ring[stage][0] + (h * 32 + lane) * 16);
        Acc d[VEC];
        unpack(bb, d, (In *)nullptr);
#pragma unroll
        for (int e = 0; e < VEC; ++e) vd[h * VEC + e] = d[e];
        if (!tail) S.diff |= (a.x ^ bb.x) | (a.y ^ bb.y) | (a.z ^ bb.z) | (a.w ^ bb.w);
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e) vd[h * VEC + e] = Acc(0);
      }
    }
    if (tail) {
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int id = id0 + (e / VEC) * 32 * VEC + e % VEC;
        if (id >= n) {
          vt[e] = ni;
          if (pair) vd[e] = ni;
        } else if (pair && bits_of(vt[e]) != bits_of(vd[e])) {
          S.diff |= 1u;
        }
      }
    }
    // ---- chunk maxima, lazy reference update, exponential sums ----
    Acc cmt = ni, cmd = ni;
#pragma unroll
    for (int e = 0; e < NE; e += 2) {
      cmt = vmax3(cmt, vt[e], vt[e + 1]);
      if (pair) cmd = vmax3(cmd, vd[e], vd[e + 1]);
    }
    const bool up_t = cmt > S.mt + Acc(kSlackW);
    const bool up_d = pair && cmd > S.md + Acc(kSlackW);
    if (__any_sync(0xffffffffu, up_t || up_d)) {
      const Acc nt = up_t ? cmt : S.mt, nd = up_d ? cmd : S.md;
      const Acc ntL = nt * L, ndL = nd * L;
      const Acc ft = fast_exp2(S.mtL - ntL), fd = fast_exp2(S.mdL - ndL);
      const Acc fz = NEEDZ ? fast_exp2(Acc(p.omt_f) * (S.mtL - ntL) + Acc(p.tau_f) * (S.mdL - ndL))
                           : Acc(1);
      if constexpr (sizeof(Acc) == 4) {
        S.pst = mul2(S.pst, pk2(ft, ft));
        S.psd = mul2(S.psd, pk2(fd, fd));
        S.psz = mul2(S.psz, pk2(fz, fz));
      } else {
        S.st *= ft;
        S.sd *= fd;
        S.sz *= fz;
      }
      S.mt = nt;
      S.md = nd;
      S.mtL = ntL;
      S.mdL = ndL;
    }
#ifdef DSDV_SLICE_NOFOLD
    if (false) {  // development probe: sums off (results are wrong)
#else
    if constexpr (sizeof(Acc) == 4) {
#endif
      const f32x2 L2 = pk2(L, L), nmt2 = pk2(-S.mtL, -S.mtL), nmd2 = pk2(-S.mdL, -S.mdL);
      const f32x2 omt2 = pk2(p.omt_f, p.omt_f), tau2 = pk2(p.tau_f, p.tau_f);
      f32x2 at = 0ull, ad = 0ull, az = 0ull;
#pragma unroll
      for (int e = 0; e < NE; e += 2) {
        const f32x2 xt = fma2(pk2(vt[e], vt[e + 1]), L2, nmt2);
        at = add2(at, pk2(fast_exp2(lo2(xt)), fast_exp2(hi2(xt))));
        if (pair) {
          const f32x2 xd = fma2(pk2(vd[e], vd[e + 1]), L2, nmd2);
          ad = add2(ad, pk2(fast_exp2(lo2(xd)), fast_exp2(hi2(xd))));
          if (NEEDZ) {
            const f32x2 xz = fma2(omt2, xt, mul2(tau2, xd));
            az = add2(az, pk2(fast_exp2(lo2(xz)), fast_exp2(hi2(xz))));
          }
        }
      }
      S.pst = add2(S.pst, at);
      if (pair) {
        S.psd = add2(S.psd, ad);
        if (NEEDZ) S.psz = add2(S.psz, az);
      }
    } else {
      const double omt = (double)p.omt_f, tau = (double)p.tau_f;
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const double xt = vt[e] * L - S.mtL;
        S.st += exp2(xt);
        if (pair) {
          const double xd = vd[e] * L - S.mdL;
          S.sd += exp2(xd);
          if (NEEDZ) S.sz += exp2(omt * xt + tau * xd);
        }
      }
    }
    // ---- top-m bookkeeping of both rows ----
#ifdef DSDV_SLICE_CYC
    const long long tb0 = clock64();
#endif
#ifndef DSDV_SLICE_NOTOPM
    if (pair && DEFER) {
      // block maxima and lane maxima only; selection after the row
      const int lt = fkey(cmt), ld = fkey(cmd);
      const int bt = warp_max_key(lt), bd = warp_max_key(ld);
      if (lane == 0) {
        ws.bmax[0][c] = bt;
        ws.bmax[1][c] = bd;
      }
      cap[0].bin = max(cap[0].bin, lt);
      cap[1].bin = max(cap[1].bin, ld);
    } else if (pair) {
#else
    if (false) {  // development probe: top-m off (results are wrong)
#endif
      if (tail) {
        topm_block<In, Acc, NE, VEC, true>(ws, 0, cap[0], fkey(cmt), vt, ws.ring[stage][1], id0,
                                           n, M, lane);
        topm_block<In, Acc, NE, VEC, true>(ws, 1, cap[1], fkey(cmd), vd, ws.ring[stage][0], id0,
                                           n, M, lane);
      } else {
        topm_block<In, Acc, NE, VEC, false>(ws, 0, cap[0], fkey(cmt), vt, ws.ring[stage][1], id0,
                                            n, M, lane);
        topm_block<In, Acc, NE, VEC, false>(ws, 1, cap[1], fkey(cmd), vd, ws.ring[stage][0], id0,
                                            n, M, lane);
      }
    }
    __syncwarp();
#ifdef DSDV_SLICE_CYC
    cyc_topm += clock64() - tb0;
    const long long tw0 = clock64();
#endif
    if (lane == 0) issue(seq + kStages);  // refill this stage
#ifdef DSDV_SLICE_CYC
    cyc_issue += clock64() - tw0;
#endif
    if (c != nch - 1) continue;
#ifdef DSDV_SLICE_CYC
    const long long tf0 = clock64();
#endif

    // ---- item complete: partial record and top lists (write_partial) ----
    if constexpr (sizeof(Acc) == 4) {
      S.st = lo2(S.pst) + hi2(S.pst);
      S.sd = lo2(S.psd) + hi2(S.psd);
      S.sz = lo2(S.psz) + hi2(S.psz);
    }
    const uint32_t diff = __any_sync(0xffffffffu, S.diff != 0) ? 1u : 0u;
    double mrg[7];
    merge_lanes<Acc>(S, p, mrg);
    const In *rt = target + ((size_t)b * G1 + j) * p.stride;
    const In *rd = draft + ((size_t)b * G + (pair ? j : 0)) * p.stride;
    if (pair && DEFER) {
      __syncwarp();
      finish_topm_deferred<In, Acc>(ws, 0, cap[0].bin, rt, n, nch, M, lane);
      finish_topm_deferred<In, Acc>(ws, 1, cap[1].bin, rd, n, nch, M, lane);
    } else if (pair) {
      finish_topm<In, Acc>(ws, 0, cap[0], rt, n, M, lane);
      finish_topm<In, Acc>(ws, 1, cap[1], rd, n, M, lane);
    }
    const double Mt = mrg[0], St = mrg[1], Md = mrg[2], Sd = mrg[3], Sz = mrg[4];
    const double MtL = mrg[5], MdL = mrg[6];
    const double dd = (double)log2e<Acc>() * kLn2 - 1.0;
    const double omt = (double)p.omt_f, tau = (double)p.tau_f;
    double lsz = 0.0;
    if (pair && NEEDZ) {
      if (Sz > 1e-30 && isfinite(Sz)) {
        const double zL = omt * MtL + tau * MdL, z = omt * Mt + tau * Md;
        lsz = (zL + log2(Sz)) * kLn2 - dd * z - z;
      } else {
        lsz = exact_lse_mix<In>(rt, rd, n, omt, tau, lane) - (omt * Mt + tau * Md);
      }
    }
    auto put = [&](auto *addr, auto v) {
      *addr = v;
      for (int q = 0; q < o.npeer; ++q)
        *reinterpret_cast<decltype(addr)>(reinterpret_cast<char *>(addr) + o.peer_delta[q]) = v;
    };
    double wk = 0.0;
    if (lane < kRecordWords) {
      const int y = pair ? tokens[(size_t)b * G + j] : 0;
      const int yl = y - p.vocab_offset;
      const bool own = pair && yl >= 0 && yl < n;
      switch (lane) {
        case 0: wk = Mt; break;
        case 1: wk = (MtL + log2(St)) * kLn2 - dd * Mt - Mt; break;
        case 2: wk = pair ? Md : 0.0; break;
        case 3: wk = pair ? (MdL + log2(Sd)) * kLn2 - dd * Md - Md : 0.0; break;
        case 4: wk = pair ? lsz : 0.0; break;
        case 5: wk = own ? load_scalar<In>(rt + yl) : NAN; break;
        case 6: wk = own ? load_scalar<In>(rd + yl) : NAN; break;
        case 7: wk = pair ? (double)((diff ? 1 : 0) | (own ? 2 : 0)) : 0.0; break;
        default: break;
      }
      put(o.records + ((size_t)b * G1 + j) * kRecordWords + lane, wk);
    }
#ifdef DSDV_SLICE_CYC
    cyc_fin += clock64() - tf0;
#endif
    if (pair && lane < M) {
      const size_t base = ((size_t)b * G + j) * 2 * M;
      const int it = ws.sel_id[0][lane], id = ws.sel_id[1][lane];
      put(o.topv + base + lane, (double)ws.sel_v[0][lane]);
      put(o.topi + base + lane, it >= 0 ? p.vocab_offset + it : -1);
      put(o.topv + base + M + lane, (double)ws.sel_v[1][lane]);
      put(o.topi + base + M + lane, id >= 0 ? p.vocab_offset + id : -1);
    }
    __syncwarp();
  }
#ifdef DSDV_SLICE_CYC
  if (lane == 0) {
    atomicAdd(&g_cyc[0], (unsigned long long)cyc_issue);
    atomicAdd(&g_cyc[1], (unsigned long long)cyc_fin);
    atomicAdd(&g_cyc[2], (unsigned long long)cyc_wait);
    atomicAdd(&g_cyc[3], (unsigned long long)(clock64() - tk0));
    atomicAdd(&g_cnt[7], (unsigned long long)cyc_topm);
  }
#endif
  // last warp out re-arms the work counters for the next launch
  if (lane == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(exit_count, 1u);
    if (prev == gridDim.x * kWarps - 1) {
      *ticket = 0u;
      *exit_count = 0u;
      __threadfence();
    }
  }
}

}  // namespace slice

#if defined(DSDV_SLICE_STATS) || defined(DSDV_SLICE_CYC)
extern "C" int dsdv_debug_slice_counters(unsigned long long *out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, slice::g_cnt, sizeof(slice::g_cnt));
  cudaMemcpyFromSymbol(out + 8, slice::g_cyc, sizeof(slice::g_cyc));
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(slice::g_cnt, z, sizeof(z));
  cudaMemcpyToSymbol(slice::g_cyc, z, sizeof(slice::g_cyc));
  return 0;
}
#endif

template <class In>
cudaError_t launch_slice_stats(const DevParams &p, const void *draft, const void *target,
                               const int32_t *tokens, const DevOut &o, unsigned int *ticket,
                               unsigned int *exit_count, cudaStream_t stream) {
  using Acc = typename InTraits<In>::Acc;
  const size_t smem = sizeof(slice::CtaSmem<Acc>);
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (r != cudaSuccess) return r;
    kern<<<sms, slice::kWarps * 32, smem, stream>>>(p, (const In *)draft, (const In *)target,
                                                    tokens, o, ticket, exit_count);
    return cudaGetLastError();
  };
  const int nch = (p.vocab_local + slice::kRowBytesW / (int)sizeof(In) - 1) /
                  (slice::kRowBytesW / (int)sizeof(In));
  const bool defer = nch <= slice::kMaxBlk;
  if (p.need_z)
    return defer ? go(slice::slice_stats_kernel<In, true, true>)
                 : go(slice::slice_stats_kernel<In, true, false>);
  return defer ? go(slice::slice_stats_kernel<In, false, true>)
               : go(slice::slice_stats_kernel<In, false, false>);
}

template cudaError_t launch_slice_stats<__nv_bfloat16>(const DevParams &, const void *,
                                                       const void *, const int32_t *,
                                                       const DevOut &, unsigned int *,
                                                       unsigned int *, cudaStream_t);
template cudaError_t launch_slice_stats<float>(const DevParams &, const void *, const void *,
                                               const int32_t *, const DevOut &, unsigned int *,
                                               unsigned int *, cudaStream_t);
template cudaError_t launch_slice_stats<double>(const DevParams &, const void *, const void *,
                                                const int32_t *, const DevOut &, unsigned int *,
                                                unsigned int *, cudaStream_t);

}  // namespace dsdv
