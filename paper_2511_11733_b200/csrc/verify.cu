// Fused adaptive speculative verification for sm_100a (DSD, arXiv 2511.11733).
//
// One persistent, warp-specialised kernel (one CTA per SM) verifies a whole
// window for all B sequences. Work items are claimed from a global ticket in
// position-major order:
//   (b, j < gamma): the row pair (draft row j, target row j)
//   (b, gamma)    : target row gamma (bonus draw)
//
// Warp roles inside a CTA:
//   producer  (1 warp)  streams rows through a kStages-deep shared-memory ring
//                       with 1-D bulk copies (TMA engine, mbarrier completion);
//   compute   (16 warps) fold every 16-byte vector into per-thread online
//                       statistics — (max, sum exp) of l_t, l_d and of the
//                       softened mix (1-tau) l_t + tau l_d (soften,
//                       verifier.cpp:161-186, as a third accumulator sharing the
//                       row exponents), warp top-m lists of l_t and l_d in
//                       (value desc, id asc) order (top_ids, verifier.cpp:40-51;
//                       softmax is monotone so logit order is probability
//                       order) behind a one-compare threshold filter, and a
//                       bitwise row-equality flag (soften's short-circuit,
//                       verifier.cpp:172) — and at the end of an item publish a
//                       per-warp partial record into one of kSlots slots
//                       without ever waiting for the epilogue;
//   epilogue  (1 warp)  merges the partials, evaluates token_cross_entropy
//                       (:112-117), norm_match (:119-134), is_key (:136-159),
//                       the effective distribution (:231-233) and accept_prob
//                       (:188-196) in fp64, draws the Philox accept uniform and
//                       publishes a per-position flag.
//
// The extra draw (residual of a rejected position, :198-213, :245-246, or the
// bonus draw, :253-256) is needed by a position whose predecessors are not
// already known to have stopped the window. The epilogue posts it back to the
// producer as a "sample item": the rows are streamed again (from HBM: after
// 16+ stages of chip-wide streaming they are no longer in L2, see
// scripts/micro/l2keep.cu; this re-read is the traffic above the algorithmic
// bytes in profiles/) and
// the compute warps turn them into per-tile sums of the residual / bonus
// weights; the epilogue then scans the tile sums for u * W and resolves the
// crossing tile (sample_with_uniform, distribution.cpp:103-114). The last item
// of a sequence to finish (per-sequence counter) commits the round: first
// rejection (:223-250), k, extra token, key count.
#include <cuda_runtime.h>

#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "sample.cuh"

namespace dsdv {
namespace fz {

#ifndef DSDV_KCW
#define DSDV_KCW 16
#endif
constexpr int kCW = DSDV_KCW;        // compute warps
constexpr int kCT = kCW * 32;        // compute threads
#ifndef DSDV_KEW
#define DSDV_KEW 2
#endif
constexpr int kEW = DSDV_KEW;        // epilogue warps (alternate stream items)
constexpr int kEpiWarp = kCW;        // first epilogue warp index
constexpr int kProdWarp = kCW + kEW; // producer warp index
constexpr int kThreads = (kCW + kEW + 1) * 32;
#ifndef DSDV_KVECS
#define DSDV_KVECS 2
#endif
constexpr int kVecs = DSDV_KVECS;    // 16-byte vectors per compute thread per row and stage
constexpr int kRowBytes = kCT * 16 * kVecs;  // per row per ring stage (16 KB)
// 16-byte vector h (< kVecs) of (warp, lane) inside a row chunk: each warp owns
// kVecs * 32 consecutive vectors, so a (chunk, warp) block is a contiguous id
// range (block maxima, sample tiles), and each LDS.128 is conflict-free.
// Regular rows whose last chunk is short, ends on a whole 16-byte vector and
// leaves at most kPadMax bytes of the stage row unused: the producer fills the
// rest with -inf (a single lane: kept small) and the compute warps fold the
// chunk without per-element masks. One-chunk rows keep the masked path (their
// top-m capture starts unbounded, and padding must never enter it).
constexpr int kPadMax = 4096;
template <class In>
__device__ __forceinline__ bool pad_tail(const DevParams &p) {
  constexpr int CH = kRowBytes / (int)sizeof(In);
  const int rem = p.vocab_local % CH;
  return p.n_chunks > 1 && p.vocab_local % InTraits<In>::kVec == 0 && rem != 0 &&
         (CH - rem) * (int)sizeof(In) <= kPadMax;
}

__device__ __forceinline__ int vec_index(int h, int warp, int lane) {
  return (warp * kVecs + h) * 32 + lane;
}
#ifndef DSDV_SLOTS
#define DSDV_SLOTS 4
#endif
constexpr int kSlots = DSDV_SLOTS;  // items between the compute warps and the epilogue
// ring depth: 4 x 32 KB stages (3 for fp64 rows, whose slots are larger)
template <class Acc>
struct Ring {
#ifdef DSDV_STAGES  // development probe: ring depth
  static constexpr int kStages = DSDV_STAGES;
#else
  static constexpr int kStages = sizeof(Acc) == 8 ? 4 : 5;
#endif
};
// Blocks per slot, (chunk, warp) of kVecs*32*VEC ids each: per-slot block
// maxima (2 x int) or sample tiles (double). fp64 rows have 2048-id chunks,
// so their slots carry more (the fp64 ring is one stage shorter): the fused
// kernel takes V <= 64 * CH for bf16 / fp32 (524,288 / 262,144) and
// V <= 116 * 2048 = 237,568 for fp64.
template <class Acc>
struct Area {
#ifdef DSDV_TILES  // development probe: smaller slots (2 CTAs per SM)
  static constexpr int kTiles = DSDV_TILES;
#else
  static constexpr int kTiles = sizeof(Acc) == 8 ? 1856 : 1024;
#endif
  static constexpr int kBytes = 8 * kTiles;
};
#ifndef DSDV_KCAP
#define DSDV_KCAP 256
#endif
constexpr int kCap = DSDV_KCAP;      // captured top-m candidates per row and item
// Sample-request queue. Bound: a request is outstanding from its posting until
// the epilogue finishes its sample item. Stream items the producer issued but
// the epilogue has not finished are at most kSlots + kStages (slot reuse and
// the ring), and between two item boundaries of the producer (where it takes
// every pending request) the epilogue finishes at most that many regular
// items, so at most 2 (kSlots + kStages) + kEW < 32 requests are outstanding:
// the queue never overflows (no runtime check, no trap).
#ifndef DSDV_KREQ
#define DSDV_KREQ 32
#endif
constexpr int kReq = DSDV_KREQ;
constexpr float kSlack = 8.0f;       // lazy max: rescale when a value exceeds m by this much
constexpr float kFloorM = -1e30f;    // finite "empty" max (keeps (v - m) free of inf - inf)

enum ItemKind : int { kRegular = 0, kSample = 1, kAborted = 2 };
// StageMeta::kr bit 8: an early-exit abort stage (no data; ends its item)
constexpr int kAbortBit = 1 << 8;
// StageMeta::kr bit 9: the item is a row pair (draft + target), else a target row
constexpr int kPairBit = 1 << 9;

// Optional cycle accounting per CTA (compile with -DDSDV_TRACE; see
// scripts/trace_roles.py): where each warp role spends its time.
enum TraceWord : int {
  kTrComputeWaitFull = 0, kTrComputeFold, kTrComputeSample, kTrComputeWaitSlot, kTrComputeItemEnd,
  kTrEpiWaitFull, kTrEpiMerge, kTrEpiTopm, kTrEpiDecide, kTrEpiSample, kTrProdWaitEmpty,
  kTrProdDrain, kTrProdItems, kTrProdSamples, kTrKernel, kTrEpiItems, kTrTopmCand, kTrTopmIns,
  kTrTopmFallback, kTrMaxSurv, kTrNeedExact, kTrCapCalls, kTrCapLock, kTrCapCycles,
  kTrComputeLoop, kTrComputeA, kTrComputeB
};
#if defined(DSDV_TRACE_LOCAL)
// light tracing: per-thread counters in registers, one atomicAdd per word at
// the end of each role (scripts/trace_roles.py, TRACE_LOCAL=1)
#define TR_START(v) const long long v = clock64()
#define TR_ADD(tr, w, v) (trv[w] += (unsigned long long)(clock64() - (v)))
#define TR_INC(tr, w) (void)0
#define TR_ACC(tr, w, x) (void)0
#define TR_MAX(tr, w, x) (void)0
#define TR_DECL unsigned long long trv[kTraceWords] = {0}
#define TR_FLUSH(tr)                                              \
  do {                                                            \
    if (tr)                                                       \
      for (int i_ = 0; i_ < kTraceWords; ++i_)                    \
        if (trv[i_]) atomicAdd((tr) + i_, trv[i_]);               \
  } while (0)
#elif defined(DSDV_TRACE)
#define TR_DECL (void)0
#define TR_FLUSH(tr) (void)0
#define TR_START(v) const long long v = clock64()
#define TR_ADD(tr, w, v)                                                         \
  do {                                                                           \
    if (tr) atomicAdd((tr) + (w), (unsigned long long)(clock64() - (v)));       \
  } while (0)
#define TR_INC(tr, w)             \
  do {                            \
    if (tr) atomicAdd((tr) + (w), 1ull); \
  } while (0)
#define TR_ACC(tr, w, x)                                       \
  do {                                                         \
    if (tr) atomicAdd((tr) + (w), (unsigned long long)(x));    \
  } while (0)
#define TR_MAX(tr, w, x)                                       \
  do {                                                         \
    if (tr) atomicMax((tr) + (w), (unsigned long long)(x));    \
  } while (0)
#else
#define TR_DECL (void)0
#define TR_FLUSH(tr) (void)0
#define TR_START(v) (void)0
#define TR_ADD(tr, w, v) (void)0
#define TR_INC(tr, w) (void)0
#define TR_MAX(tr, w, x) (void)0
#define TR_ACC(tr, w, x) (void)0
#endif

struct alignas(16) StageMeta {  // one LDS.128 per chunk
  int item;   // global item id (b, j), -1 = end of stream
  int chunk;
  int n;      // CTA-local stream index (slot = n % kSlots)
  int kr;     // kind (kRegular / kSample) | sample request index << 1
  __device__ __forceinline__ int kind() const { return kr & 1; }
  __device__ __forceinline__ int req() const { return (kr >> 1) & 127; }
  __device__ __forceinline__ bool abort() const { return (kr & kAbortBit) != 0; }
  __device__ __forceinline__ bool pair() const { return (kr & kPairBit) != 0; }
};

template <class Acc>
struct WarpPartial {
  Acc mt, st, md, sd, sz;  // maxima (natural) and sums relative to mtL / mdL
  Acc mtL, mdL;            // log2 reference points (fl(max * log2 e))
  int diff;
};

template <class Acc>
struct Slot {
  int item;
  int kind;
  int req;
  WarpPartial<Acc> wp[kCW];
  // top-m capture per row: per-lane running maxima (capture_row), the bound
  // theta_run derived from them, and every element that reached theta_run
  int klist[2][32];
  int ktheta[2], ncap[2];
  int cap_id[2][kCap];
  Acc cap_v[2][kCap];
  // regular item: per-block max keys of l_t / l_d ([2][nblocks] ints, read only
  // by the capture-overflow fallback); sample item: per-tile weight sums
  // ([ntiles] doubles). See SlotView.
  alignas(16) uint8_t area[Area<Acc>::kBytes];
};

// Typed views of a slot's area for one launch shape.
struct SlotView {
  int *bmax[2];
  double *tiles;
  __device__ __forceinline__ SlotView(uint8_t *area, int nblocks) {
    int *a = reinterpret_cast<int *>(area);
    bmax[0] = a;
    bmax[1] = a + nblocks;
    tiles = reinterpret_cast<double *>(area);
  }
};

// Capture state of a slot back to empty (kernel start, and by the epilogue
// when it releases a regular item's slot). One warp.
template <class Acc>
__device__ __forceinline__ void reset_capture(Slot<Acc> &sl, int lane) {
  sl.klist[0][lane] = INT_MIN;
  sl.klist[1][lane] = INT_MIN;
  if (lane < 2) {
    sl.ktheta[lane] = INT_MIN;
    sl.ncap[lane] = 0;
  }
}

template <class Acc>
struct Request {
  int ready;  // set by the epilogue once the entry is complete
  int item;
  int rows;   // 2 = row pair (residual), 1 = target row (bonus)
  double u;
  Weigher<Acc> wf;
};

struct EpiScratch {
  int cand[32];          // candidate blocks of one 32-block batch
  int ev_id[128];        // surviving elements (id, value)
  double ev_key[128];
  int sel[2][kMaxTopM];     // top-m ids of the target / draft row
  double selv[2][kMaxTopM];  // and their values (sharded partial records)
};

template <class Acc>
struct alignas(128) Smem {
  static constexpr int kStages = Ring<Acc>::kStages;
  uint8_t ring[kStages][2][kRowBytes];  // [stage][0 = draft, 1 = target]
  Slot<Acc> slot[kSlots];
  Request<Acc> req[kReq];
  StageMeta meta[kStages];
  uint64_t full[kStages], empty[kStages];
  uint64_t part_full[kSlots], part_empty[kSlots];
  int req_head;            // producer: next request to stream
  int req_tail;            // epilogue warps: next request entry to fill (atomic)
  int req_done;            // sample items finished (entries free again)
  int epi_count;           // stream items the epilogue warps have finished
  int epi_exit;            // epilogue warps that have left
  EpiScratch epi[kEW];     // per epilogue warp: top-m selection scratch
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ bool bits_differ(float a, float b) {
  return __float_as_uint(a) != __float_as_uint(b);
}
__device__ __forceinline__ bool bits_differ(double a, double b) {
  return __double_as_longlong(a) != __double_as_longlong(b);
}
__device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double vmax(double a, double b) { return fmax(a, b); }
__device__ __forceinline__ float vmax3(float a, float b, float c) {  // FMNMX3
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ double vmax3(double a, double b, double c) { return fmax(fmax(a, b), c); }

// Order-preserving int key of a float (shared-memory atomicMax of thresholds).
__device__ __forceinline__ int fkey(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
// doubles round DOWN so the key stays a lower bound of the true threshold
__device__ __forceinline__ int fkey(double f) { return fkey(__double2float_rd(f)); }
__device__ __forceinline__ float fkey_inv(int k) {
  return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff);
}
constexpr int kKeyNegInf = (int)(0xff800000u ^ 0x7fffffffu);  // fkey(-inf)

__device__ __forceinline__ int vload(const int *p) { return *(const volatile int *)p; }
__device__ __forceinline__ void vstore(int *p, int v) { *(volatile int *)p = v; }

// Per-thread online statistics of one item. Sums are relative to log2-scaled
// reference points mtL = fl(mt * L), mdL = fl(md * L) (L = fp32 log2 e), so an
// exponent is one FFMA: x = v * L - mtL. The epilogue converts back exactly
// (lse_from_sum): ln sum 2^(v L) = (mtL + log2 s) ln 2, and the (1.3e-8)
// relative error of L is corrected to first order with the row maximum.
// fp32 sums are carried as packed f32x2 pairs (pst / psd / psz: one FADD2 per
// two exponentials, no per-chunk horizontal adds) and folded into st / sd / sz
// only at the end of an item (flush).
template <class Acc>
struct ItemState {
  Acc mt, st, md, sd, sz;  // natural-log maxima (lazy, within kSlack) and sums
  Acc mtL, mdL;            // log2 reference points of the sums
  uint32_t diff;
  f32x2 pst, psd, psz;     // packed fp32 sums (Acc = float only)
  __device__ __forceinline__ void reset() {
    mt = md = Acc(kFloorM);
    mtL = mdL = Acc(kFloorM) * log2e<Acc>();
    st = sd = sz = Acc(0);
    pst = psd = psz = 0ull;
    diff = 0;
  }
  __device__ __forceinline__ void flush() {
    if constexpr (sizeof(Acc) == 4) {
      st += lo2(pst) + hi2(pst);
      sd += lo2(psd) + hi2(psd);
      sz += lo2(psz) + hi2(psz);
      pst = psd = psz = 0ull;
    }
  }
};

__device__ __forceinline__ int warp_max_key(int key) {
  int r;
  asm volatile("redux.sync.max.s32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(key));
  return r;
}

// ------------------------------------------------------------------ compute warps
// Descending bitonic sort of one int per lane.
__device__ __forceinline__ int warp_sort_desc(int key, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int pk = __shfl_xor_sync(0xffffffffu, key, j);
      const bool keep_max = ((lane & j) == 0) == ((lane & k) == 0);
      key = keep_max ? max(key, pk) : min(key, pk);
    }
  }
  return key;
}

// ---- top-m capture (top_ids, verifier.cpp:40-51) ----
// Per slot and row, klist[r][l] holds the largest lane maximum seen so far from
// lane l of any (chunk, warp) block (shared-memory atomicMax, conflict-free).
// The 32 entries are distinct elements of the row, so their M-th largest never
// exceeds the row's M-th largest value; theta_run (ktheta) is a value that is
// at most that. Every element of the final top M is >= theta_run when its
// block streams, and a block whose maximum is below theta_run holds none of
// them. The compute warps append the elements that reach theta_run (ids,
// values) to the slot's capture buffer; the epilogue ranks only those.

// M-th largest of the 32 bins of a row (one warp, bitonic sort).
__device__ __noinline__ int theta_from_bins(const int *bins, int M, int lane) {
  const int sorted = warp_sort_desc(vload(bins + lane), lane);
  return __shfl_sync(0xffffffffu, sorted, M - 1);
}

// Epilogue warp, while it waits for a slot: re-derive theta_run of both rows
// of the item being folded into it (the bins only grow, so any value derived
// from them stays a valid bound).
template <class Acc>
__device__ __noinline__ void refresh_theta(Slot<Acc> &sl, int M, int lane) {
#pragma unroll 1
  for (int r = 0; r < 2; ++r) {
    const int th = vload(&sl.ktheta[r]);
    const int bin = vload(&sl.klist[r][lane]);
    if (__popc(__ballot_sync(0xffffffffu, bin > th)) >= M + 1) {
      const int sorted = warp_sort_desc(bin, lane);
      const int nth = __shfl_sync(0xffffffffu, sorted, M - 1);
      if (lane == 0 && nth > th) atomicMax(&sl.ktheta[r], nth);
    }
  }
}

// key(v) >= th  <=>  v >= fkey_inv(th) (keys round toward -inf)
template <class Acc>
__device__ __forceinline__ Acc key_floor(int th) {
  return th == INT_MIN ? neg_inf<Acc>() : (Acc)fkey_inv(th);
}

// Rare path of a block whose maximum reached theta_run (inline; the values
// are still in registers): fold the lane maxima into the bins, raise
// theta_run while it is far behind (one sort, out of line; small raises are
// left to the epilogue warps, refresh_theta), and capture the elements that
// reach it. Only lanes whose maximum reaches the bound enter the capture, and
// each captured element is re-read from the resident stage by its index, so
// the divergent part costs a few instructions per captured element.
template <class In, bool TAIL, class Acc>
__device__ __forceinline__ void capture_row(Slot<Acc> &sl, int r, int lkey, int th,
                                            const uint8_t *srow, int c, int tid, int lane,
                                            const DevParams &p, unsigned long long *trl) {
  constexpr int CH = kRowBytes / (int)sizeof(In);
  constexpr int VEC = InTraits<In>::kVec;
  TR_INC(trl, kTrCapCalls);
  int *bins = sl.klist[r];
  const int bin = vload(bins + lane);
  if (lkey > bin) atomicMax(bins + lane, lkey);
#ifndef DSDV_CAPSORT
#define DSDV_CAPSORT 8
#endif
  if (__popc(__ballot_sync(0xffffffffu, max(bin, lkey) > th)) >= p.top_m + DSDV_CAPSORT) {
    TR_INC(trl, kTrCapLock);
    __syncwarp();
    const int nth = theta_from_bins(bins, p.top_m, lane);
    if (nth > th) {
      th = nth;
      if (lane == 0) atomicMax(&sl.ktheta[r], nth);
    }
  }
  if (lkey >= th) {
    const Acc thv = key_floor<Acc>(th);
    unsigned keep = 0;
    Acc v[kVecs][VEC];  // this lane's elements, re-read from the resident stage
#pragma unroll
    for (int h = 0; h < kVecs; ++h)
      unpack(lds128(srow + vec_index(h, tid >> 5, lane) * 16), v[h], (In *)nullptr);
#pragma unroll
    for (int h = 0; h < kVecs; ++h)
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const bool ok = !TAIL || c * CH + vec_index(h, tid >> 5, lane) * VEC + e < p.vocab_local;
        keep |= (ok && v[h][e] >= thv ? 1u : 0u) << (h * VEC + e);
      }
    int at = atomicAdd(&sl.ncap[r], __popc(keep));
    while (keep) {
      const int bit = __ffs(keep) - 1;
      keep &= keep - 1;
      const int q = vec_index(bit / VEC, tid >> 5, lane), e = bit % VEC;
      const In *src = reinterpret_cast<const In *>(srow + q * 16) + e;
      if (at < kCap) {
        sl.cap_id[r][at] = c * CH + q * VEC + e;
        sl.cap_v[r][at] = (Acc)load_smem_scalar(src);
      }
      ++at;
    }
  }
}

#ifndef DSDV_ZMUFU
#define DSDV_ZMUFU 4
#endif
constexpr int kZMufu = DSDV_ZMUFU;

template <bool PAIR, bool NEEDZ, int VEC>
__device__ __forceinline__ void exp_sums(const float (&vt)[VEC], const float (&vd)[VEC],
                                         ItemState<float> &S, const DevParams &p) {
  const f32x2 L2 = pk2(kLog2eF, kLog2eF);
  const f32x2 nmt2 = pk2(-S.mtL, -S.mtL), nmd2 = pk2(-S.mdL, -S.mdL);
  const f32x2 omt2 = pk2(p.omt_f, p.omt_f), tau2 = pk2(p.tau_f, p.tau_f);
  f32x2 at = pk2(0.f, 0.f), ad = pk2(0.f, 0.f), az = pk2(0.f, 0.f);
#pragma unroll
  for (int e = 0; e < VEC; e += 2) {
    const f32x2 xt = fma2(pk2(vt[e], vt[e + 1]), L2, nmt2);
    at = add2(at, pk2(fast_exp2(lo2(xt)), fast_exp2(hi2(xt))));
    if (PAIR) {
      const f32x2 xd = fma2(pk2(vd[e], vd[e + 1]), L2, nmd2);
      ad = add2(ad, pk2(fast_exp2(lo2(xd)), fast_exp2(hi2(xd))));
      if (NEEDZ) {
        const f32x2 xz = fma2(omt2, xt, mul2(tau2, xd));
        // kZMufu of the VEC/2 pairs take the MUFU pipe, the rest the FMA pipe
        if (e / 2 < kZMufu)
          az = add2(az, pk2(fast_exp2(lo2(xz)), fast_exp2(hi2(xz))));
        else
          az = add2(az, poly_exp2x2(xz));
      }
    }
  }
  S.st += lo2(at) + hi2(at);
  if (PAIR) {
    S.sd += lo2(ad) + hi2(ad);
    if (NEEDZ) S.sz += lo2(az) + hi2(az);
  }
}

template <bool PAIR, bool NEEDZ, int VEC>
__device__ __forceinline__ void exp_sums(const double (&vt)[VEC], const double (&vd)[VEC],
                                         ItemState<double> &S, const DevParams &p) {
  const double L = kLog2e, omt = (double)p.omt_f, tau = (double)p.tau_f;
  double at = 0.0, ad = 0.0, az = 0.0;
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    const double xt = vt[e] * L - S.mtL;
    at += exp2(xt);
    if (PAIR) {
      const double xd = vd[e] * L - S.mdL;
      ad += exp2(xd);
      if (NEEDZ) az += exp2(omt * xt + tau * xd);
    }
  }
  S.st += at;
  if (PAIR) {
    S.sd += ad;
    if (NEEDZ) S.sz += az;
  }
}

// packed fp32 exponential sums of one 16-byte vector pair into the item's
// accumulators (the reference points are not changed here)
template <bool PAIR, bool NEEDZ, int VEC>
__device__ __forceinline__ void exp_acc(const float (&vt)[VEC], const float (&vd)[VEC],
                                        ItemState<float> &S, const DevParams &p) {
  const f32x2 L2 = pk2(kLog2eF, kLog2eF);
  const f32x2 nmt2 = pk2(-S.mtL, -S.mtL), nmd2 = pk2(-S.mdL, -S.mdL);
  const f32x2 omt2 = pk2(p.omt_f, p.omt_f), tau2 = pk2(p.tau_f, p.tau_f);
#pragma unroll
  for (int e = 0; e < VEC; e += 2) {
    const f32x2 xt = fma2(pk2(vt[e], vt[e + 1]), L2, nmt2);
    S.pst = add2(S.pst, pk2(fast_exp2(lo2(xt)), fast_exp2(hi2(xt))));
    if (PAIR) {
      const f32x2 xd = fma2(pk2(vd[e], vd[e + 1]), L2, nmd2);
      S.psd = add2(S.psd, pk2(fast_exp2(lo2(xd)), fast_exp2(hi2(xd))));
      if (NEEDZ) {
        const f32x2 xz = fma2(omt2, xt, mul2(tau2, xd));
        if (e / 2 < kZMufu)
          S.psz = add2(S.psz, pk2(fast_exp2(lo2(xz)), fast_exp2(hi2(xz))));
        else
          S.psz = add2(S.psz, poly_exp2x2(xz));
      }
    }
  }
}

// A chunk value above the reference by more than kGuard (natural-log units)
// could overflow the fp32 sums of a chunk folded against the old reference:
// 2^(kGuard * log2 e + log2 8192) stays below 2^128.
constexpr float kGuard = 60.0f;

// Fold this thread's kVecs 16-byte vectors per row of one ring stage (ids of
// vector h: c*CH + (h*kCT + tid)*VEC + e).
//
// fp32 accumulation (bf16 / fp32 rows): the exponentials go first, against the
// lane's current reference points, so the MUFU work of a chunk starts as soon
// as its vectors are unpacked; the chunk maximum, the block-maximum key
// (REDUX) of the top-m bookkeeping, the (rare) capture and the lazy
// reference update follow from the same registers. Only an item's first
// chunk takes its maximum first (no reference yet). A chunk that overshoots
// the reference by more than kGuard is folded again against the new one.
// fp64 rows keep the max-first order.
template <class In, bool PAIR, bool NEEDZ, bool TAIL>
__device__ __forceinline__ void fold_chunk(const uint8_t *sdraft, const uint8_t *starget, int tid,
                                           int c, ItemState<typename InTraits<In>::Acc> &S,
                                           const DevParams &p, int warp, int lane,
                                           Slot<typename InTraits<In>::Acc> &sl, int *bmax_t,
                                           int *bmax_d, unsigned long long *trl,
                                           const uint4 (&pre_t)[kVecs],
                                           const uint4 (&pre_d)[kVecs]) {
  using Acc = typename InTraits<In>::Acc;
  constexpr int VEC = InTraits<In>::kVec;
  constexpr int CH = kRowBytes / (int)sizeof(In);
  const Acc L = log2e<Acc>();
  const Acc ni = neg_inf<Acc>();

  Acc vt[kVecs][VEC], vd[kVecs][VEC];
  uint32_t diff = 0;
  auto load = [&]() {
#pragma unroll
    for (int h = 0; h < kVecs; ++h) {
      const uint4 a = pre_t[h];  // loaded with the stage descriptor (compute_loop)
      unpack(a, vt[h], (In *)nullptr);
      if (PAIR) {
        const uint4 bb = pre_d[h];
        unpack(bb, vd[h], (In *)nullptr);
        diff |= (a.x ^ bb.x) | (a.y ^ bb.y) | (a.z ^ bb.z) | (a.w ^ bb.w);
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e) vd[h][e] = Acc(0);
      }
    }
    if (TAIL) {
      // elements past the logical row are -inf in both rows (no mass, equal,
      // ranked after every real id); the equality flag sees real ids only
      diff = 0;
#pragma unroll
      for (int h = 0; h < kVecs; ++h) {
        const int id0 = c * CH + vec_index(h, warp, lane) * VEC;
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          if (id0 + e >= p.vocab_local) {
            vt[h][e] = ni;
            if (PAIR) vd[h][e] = ni;
          } else if (PAIR) {
            diff |= bits_differ(vt[h][e], vd[h][e]) ? 1u : 0u;
          }
        }
      }
    }
  };
  auto chunk_max = [&](Acc &cmt, Acc &cmd) {
    cmt = ni;
    cmd = ni;
#pragma unroll
    for (int h = 0; h < kVecs; ++h)
#pragma unroll
      for (int e = 0; e < VEC; e += 2) {
        cmt = vmax3(cmt, vt[h][e], vt[h][e + 1]);
        if (PAIR) cmd = vmax3(cmd, vd[h][e], vd[h][e + 1]);
      }
  };
  // new reference points for the lanes whose chunk maximum passed theirs by
  // more than kSlack; the sums are rescaled to them
  auto rescale = [&](bool up_t, bool up_d, Acc cmt, Acc cmd) {
    const Acc nt = up_t ? cmt : S.mt;
    const Acc nd = up_d ? cmd : S.md;
    const Acc ntL = nt * L, ndL = nd * L;
    const Acc ft = fast_exp2(S.mtL - ntL);
    const Acc fd = fast_exp2(S.mdL - ndL);
    const Acc fz = NEEDZ ? fast_exp2(Acc(p.omt_f) * (S.mtL - ntL) + Acc(p.tau_f) * (S.mdL - ndL))
                         : Acc(1);
    if constexpr (sizeof(Acc) == 4) {
      S.pst = mul2(S.pst, pk2(ft, ft));
      if (PAIR) S.psd = mul2(S.psd, pk2(fd, fd));
      if (NEEDZ) S.psz = mul2(S.psz, pk2(fz, fz));
    } else {
      S.st *= ft;
      if (PAIR) S.sd *= fd;
      if (NEEDZ) S.sz *= fz;
    }
    S.mt = nt;
    S.md = nd;
    S.mtL = ntL;
    S.mdL = ndL;
  };
  auto exps = [&]() {
#pragma unroll
    for (int h = 0; h < kVecs; ++h) {
      if constexpr (sizeof(Acc) == 4)
        exp_acc<PAIR, NEEDZ, VEC>(vt[h], vd[h], S, p);
      else
        exp_sums<PAIR, NEEDZ, VEC>(vt[h], vd[h], S, p);
    }
  };
  // top-m bookkeeping: one warp max per row (the key of block (chunk, warp))
  // against the row's running bound; the rare blocks that reach it are captured
  auto topm = [&](Acc cmt, Acc cmd) {
    if (!PAIR) return;
    S.diff |= diff;
    const int lt = fkey(cmt), ld = fkey(cmd);
    const int bt = warp_max_key(lt);
    const int bd = warp_max_key(ld);
    if (lane == 0) {
      bmax_t[c * kCW + warp] = bt;
      bmax_d[c * kCW + warp] = bd;
    }
    const int th0 = vload(&sl.ktheta[0]), th1 = vload(&sl.ktheta[1]);
#ifdef DSDV_XNOCAP
    if (false) {  // development probe: capture off (results are wrong)
#else
    if (bt >= th0 || bd >= th1) {
#endif
      TR_DECL;
      TR_START(tcap);
      if (bt >= th0) capture_row<In, TAIL>(sl, 0, lt, th0, starget, c, tid, lane, p, trl);
      if (bd >= th1) capture_row<In, TAIL>(sl, 1, ld, th1, sdraft, c, tid, lane, p, trl);
      TR_ADD(trl, kTrCapCycles, tcap);
    }
  };

#ifndef DSDV_ORDER
#define DSDV_ORDER 1
#endif
  load();
  Acc cmt, cmd;
  if (sizeof(Acc) == 8 || c == 0 || DSDV_ORDER < 2) {
    // max first: the item's first chunk sets the reference points
    chunk_max(cmt, cmd);
    if (DSDV_ORDER == 0) topm(cmt, cmd);
    const bool up_t = cmt > S.mt + Acc(kSlack);
    const bool up_d = PAIR && (cmd > S.md + Acc(kSlack));
    if (__any_sync(0xffffffffu, up_t || up_d)) rescale(up_t, up_d, cmt, cmd);
    exps();
    if (DSDV_ORDER != 0) topm(cmt, cmd);
    return;
  }
  // exponentials first, against the current reference points
  const f32x2 s0t = S.pst, s0d = S.psd, s0z = S.psz;
  exps();
  chunk_max(cmt, cmd);
  topm(cmt, cmd);
  const bool up_t = cmt > S.mt + Acc(kSlack);
  const bool up_d = PAIR && (cmd > S.md + Acc(kSlack));
  if (__any_sync(0xffffffffu, up_t || up_d)) {
    const bool over = cmt > S.mt + Acc(kGuard) || (PAIR && cmd > S.md + Acc(kGuard));
    if (__any_sync(0xffffffffu, over)) {
      // rare: this chunk may have overflowed against the old reference; fold
      // it again from the resident stage against the new one
      if constexpr (sizeof(Acc) == 4) {
        S.pst = s0t;
        S.psd = s0d;
        S.psz = s0z;
      }
      rescale(up_t, up_d, cmt, cmd);
      load();
      exps();
    } else {
      rescale(up_t, up_d, cmt, cmd);
    }
  }
}

// The same fold loading its own vectors (development probes: scripts/micro/).
template <class In, bool PAIR, bool NEEDZ, bool TAIL>
__device__ __forceinline__ void fold_chunk(const uint8_t *sdraft, const uint8_t *starget, int tid,
                                           int c, ItemState<typename InTraits<In>::Acc> &S,
                                           const DevParams &p, int warp, int lane,
                                           Slot<typename InTraits<In>::Acc> &sl, int *bmax_t,
                                           int *bmax_d, unsigned long long *trl) {
  uint4 pre_t[kVecs], pre_d[kVecs];
#pragma unroll
  for (int h = 0; h < kVecs; ++h) {
    const int q = vec_index(h, warp, lane);
    pre_t[h] = lds128(starget + q * 16);
    pre_d[h] = lds128(sdraft + q * 16);
  }
  fold_chunk<In, PAIR, NEEDZ, TAIL>(sdraft, starget, tid, c, S, p, warp, lane, sl, bmax_t, bmax_d,
                                    trl, pre_t, pre_d);
}

// Sample item: per-tile fp64 sums of the residual / bonus weights. Tile
// (chunk, warp) covers the warp's contiguous kVecs * 32 vectors of the chunk,
// ids [chunk*CH + warp*kVecs*32*VEC, +kVecs*32*VEC): tile index order is id
// order.
template <class In>
__device__ __forceinline__ void sample_chunk(const uint8_t *sdraft, const uint8_t *starget,
                                             int chunk, const Weigher<typename InTraits<In>::Acc> &wf,
                                             double *tiles, const DevParams &p, int tid, int warp,
                                             int lane, const uint4 (&pre_t)[kVecs],
                                             const uint4 (&pre_d)[kVecs]) {
  using Acc = typename InTraits<In>::Acc;
  constexpr int VEC = InTraits<In>::kVec;
  constexpr int CH = kRowBytes / (int)sizeof(In);
  double ls = 0.0;
#ifdef DSDV_XNOSAMPLE
  if (lane == 0) tiles[chunk * kCW + warp] = 1.0;  // development probe (wrong results)
  return;
#endif
#pragma unroll
  for (int h = 0; h < kVecs; ++h) {
    const int q = vec_index(h, warp, lane);
    const int id0 = chunk * CH + q * VEC;
    Acc vt[VEC], vd[VEC];
    unpack(pre_t[h], vt, (In *)nullptr);
    if (wf.kind != kWeightPlain) {
      unpack(pre_d[h], vd, (In *)nullptr);
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) vd[e] = Acc(0);
    }
    Acc w[VEC];
    weigh_vec<VEC>(wf, vt, vd, w);
    // ids past the row exist only in the row's last chunk
    if ((chunk + 1) * CH > p.vocab_local) {
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (id0 + e >= p.vocab_local) w[e] = Acc(0);
    }
    Acc lv = Acc(0);
#pragma unroll
    for (int e = 0; e < VEC; ++e) lv = add_rn(lv, w[e]);
    ls += (double)lv;
  }
  const double ts = warp_sum_f64(ls);
  if (lane == 0) tiles[chunk * kCW + warp] = ts;
}

template <class In, bool NEEDZ, bool EE>
__device__ void compute_loop(Smem<typename InTraits<In>::Acc> &sm, const DevParams &p,
                             const In *__restrict__ draft, const In *__restrict__ target, int tid,
                             unsigned long long *tr) {
  using Acc = typename InTraits<In>::Acc;
  constexpr int VEC = InTraits<In>::kVec;
  constexpr int CH = kRowBytes / (int)sizeof(In);
  const int warp = tid >> 5, lane = tid & 31;
  ItemState<Acc> S;
  S.reset();
  int stage = 0;
  uint32_t phase = 0;
  bool pair = false;
  int kind = kRegular, n = 0, s = 0;
  unsigned long long *trl = (tid & 31) == 0 ? tr : nullptr;
  TR_DECL;
  TR_START(tloop);
#if defined(DSDV_TRACE) || defined(DSDV_TRACE_LOCAL)
  long long tb = clock64();
#endif
  for (;;) {
    TR_ADD(trl, kTrComputeB, tb);
    TR_START(tw);
    mbar_wait(&sm.full[stage], phase);
    TR_ADD(trl, kTrComputeWaitFull, tw);
    TR_START(ta);
#ifdef DSDV_TIMELINE
    if (trl && warp == 0 && blockIdx.x == 0) {
      unsigned long long *tl = tr + 512 * kTraceWords;
      const unsigned q = (unsigned)tl[4094];
      if (q < 1000) {
        tl[q * 4 + 1] = clock64();
        tl[q * 4 + 2] = clock64() - tw;
      }
    }
#endif
    // the chunk's vectors of both rows go out together with the stage
    // descriptor: their latency overlaps the descriptor's instead of following it
    uint4 pre_t[kVecs], pre_d[kVecs];
#pragma unroll
    for (int h = 0; h < kVecs; ++h) {
      const int q = vec_index(h, warp, lane);
      pre_t[h] = lds128(sm.ring[stage][1] + q * 16);
      pre_d[h] = lds128(sm.ring[stage][0] + q * 16);
    }
    const StageMeta md = sm.meta[stage];
    if (md.item < 0) {
      // end of stream: one terminating slot per epilogue warp
      for (int k = 0; k < kEW; ++k) {
        const int nn = md.n + k, ns = nn % kSlots;
        mbar_wait(&sm.part_empty[ns], ((nn / kSlots) & 1) ^ 1);
        if (tid == 0) sm.slot[ns].item = -1;
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.part_full[ns]);
      }
      TR_ADD(trl, kTrComputeLoop, tloop);
      TR_FLUSH(trl);
      break;
    }
    const int c = md.chunk;
    if (c == 0) {
      kind = md.kind();
      n = md.n;
      s = n % kSlots;
      pair = md.pair();
      // the slot (partials + block maxima) must be free before this item runs
      TR_START(ts);
      mbar_wait(&sm.part_empty[s], ((n / kSlots) & 1) ^ 1);
      TR_ADD(trl, kTrComputeWaitSlot, ts);
    }
    const bool last = c == p.n_chunks - 1;
    TR_ADD(trl, kTrComputeA, ta);
    TR_START(tf);
#ifdef DSDV_NOFOLD
    // development probe: a fixed per-chunk busy time instead of the fold
    {
      const long long t0 = clock64();
      while (clock64() - t0 < DSDV_NOFOLD) {
      }
    }
    if (false) {
#else
    if (EE && md.abort()) {
      // early exit: the item's sequence already stopped at an earlier position;
      // no data, the item ends here
    } else if (kind == kRegular) {
#endif
      // a short last chunk is masked element by element unless the producer
      // padded it with -inf (pad_tail)
      const bool tail = last && (p.vocab_local % CH) != 0 && !pad_tail<In>(p);
      Slot<Acc> &sl = sm.slot[s];
      const SlotView sv(sl.area, p.n_chunks * kCW);
      const uint8_t *sd = sm.ring[stage][0], *st = sm.ring[stage][1];
      if (pair) {
        if (!tail)
          fold_chunk<In, true, NEEDZ, false>(sd, st, tid, c, S, p, warp, lane, sl, sv.bmax[0],
                                             sv.bmax[1], trl, pre_t, pre_d);
        else
          fold_chunk<In, true, NEEDZ, true>(sd, st, tid, c, S, p, warp, lane, sl, sv.bmax[0],
                                            sv.bmax[1], trl, pre_t, pre_d);
      } else if (!tail) {
        fold_chunk<In, false, false, false>(sd, st, tid, c, S, p, warp, lane, sl, sv.bmax[0],
                                            sv.bmax[1], trl, pre_t, pre_d);
      } else {
        fold_chunk<In, false, false, true>(sd, st, tid, c, S, p, warp, lane, sl, sv.bmax[0],
                                           sv.bmax[1], trl, pre_t, pre_d);
      }
    } else {
#ifndef DSDV_NOFOLD
      sample_chunk<In>(sm.ring[stage][0], sm.ring[stage][1], c, sm.req[md.req()].wf,
                       reinterpret_cast<double *>(sm.slot[s].area), p, tid, warp, lane, pre_t,
                       pre_d);
#endif
    }
    TR_ADD(trl, kind == kRegular ? kTrComputeFold : kTrComputeSample, tf);
#ifdef DSDV_TIMELINE
    if (trl && warp == 0 && blockIdx.x == 0) {
      unsigned long long *tl = tr + 512 * kTraceWords;
      const unsigned q = (unsigned)tl[4094]++;
      if (q < 1000) tl[q * 4 + 3] = clock64();
    }
#endif
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[stage]);
    if (++stage == Smem<Acc>::kStages) {
      stage = 0;
      phase ^= 1;
    }
#if defined(DSDV_TRACE) || defined(DSDV_TRACE_LOCAL)
    tb = clock64();
#endif
    if (!last) continue;

    // ---- item end: publish this warp's partial, never wait for the epilogue ----
    TR_START(te);
    Slot<Acc> &sl = sm.slot[s];
    if (kind == kRegular) {
      const Acc omt = Acc(p.omt_f), tau = Acc(p.tau_f);
      S.flush();
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const Acc mt2 = __shfl_xor_sync(0xffffffffu, S.mt, off);
        const Acc mtL2 = __shfl_xor_sync(0xffffffffu, S.mtL, off);
        const Acc st2 = __shfl_xor_sync(0xffffffffu, S.st, off);
        const Acc md2 = __shfl_xor_sync(0xffffffffu, S.md, off);
        const Acc mdL2 = __shfl_xor_sync(0xffffffffu, S.mdL, off);
        const Acc sd2 = __shfl_xor_sync(0xffffffffu, S.sd, off);
        const Acc sz2 = __shfl_xor_sync(0xffffffffu, S.sz, off);
        const Acc ML = vmax(S.mtL, mtL2), DL = vmax(S.mdL, mdL2);
        S.st = S.st * fast_exp2(S.mtL - ML) + st2 * fast_exp2(mtL2 - ML);
        S.sd = S.sd * fast_exp2(S.mdL - DL) + sd2 * fast_exp2(mdL2 - DL);
        S.sz = S.sz * fast_exp2(omt * (S.mtL - ML) + tau * (S.mdL - DL)) +
               sz2 * fast_exp2(omt * (mtL2 - ML) + tau * (mdL2 - DL));
        S.mt = vmax(S.mt, mt2);
        S.md = vmax(S.md, md2);
        S.mtL = ML;
        S.mdL = DL;
      }
      const int anydiff = __any_sync(0xffffffffu, S.diff != 0);
      if (lane == 0) {
        WarpPartial<Acc> w;
        w.mt = S.mt;
        w.st = S.st;
        w.md = S.md;
        w.sd = S.sd;
        w.sz = S.sz;
        w.mtL = S.mtL;
        w.mdL = S.mdL;
        w.diff = anydiff;
        sl.wp[warp] = w;
      }
      S.reset();
    }
    if (tid == 0) {
      sl.item = md.item;
      sl.kind = (EE && md.abort()) ? kAborted : kind;
      sl.req = md.req();
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.part_full[s]);
    TR_ADD(trl, kTrComputeItemEnd, te);
  }
}

// ------------------------------------------------------------------ epilogue warp
// Merge of the kCW warp partials (lanes 0..kCW-1, xor tree) in the
// accumulation precision. out = {mt, st, md, sd, sz, mtL, mdL}: maxima
// (natural), sums relative to the log2 reference points mtL / mdL (and
// (1-tau) mtL + tau mdL for sz).
template <class Acc>
__device__ __noinline__ void merge_partials(const Slot<Acc> &sl, const DevParams &p, int lane,
                                            double (&out)[7], int &diff) {
  Acc mt = Acc(kFloorM), md = Acc(kFloorM), st = Acc(0), sd = Acc(0), sz = Acc(0);
  Acc mtL = Acc(kFloorM) * log2e<Acc>(), mdL = mtL;
  int df = 0;
  if (lane < kCW) {
    const WarpPartial<Acc> w = sl.wp[lane];
    mt = w.mt;
    st = w.st;
    md = w.md;
    sd = w.sd;
    sz = w.sz;
    mtL = w.mtL;
    mdL = w.mdL;
    df = w.diff;
  }
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
    df |= __shfl_xor_sync(0xffffffffu, df, off);
    const Acc ML = vmax(mtL, mtL2), DL = vmax(mdL, mdL2);
    st = st * fast_exp2(mtL - ML) + st2 * fast_exp2(mtL2 - ML);
    sd = sd * fast_exp2(mdL - DL) + sd2 * fast_exp2(mdL2 - DL);
    sz = sz * fast_exp2(omt * (mtL - ML) + tau * (mdL - DL)) +
         sz2 * fast_exp2(omt * (mtL2 - ML) + tau * (mdL2 - DL));
    mt = vmax(mt, mt2);
    md = vmax(md, md2);
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
  diff = df;
}

// Exact top-M ids of one row, (value desc, id asc) like top_ids
// (verifier.cpp:40-51), from the compute warps' capture (capture_row): the
// captured elements whose key reaches the final theta_run are a superset of the
// top M; they are collected and each ranked against the others (ranks < M are
// the top M). If ties push more than 128 survivors past theta_run, a warp-list
// insertion over the capture takes over; if the capture buffer itself
// overflowed (e.g. rows sorted by id), the listed blocks whose maximum reaches
// theta_run are re-read. Both fallbacks are exact, only slower.
template <class In>
__device__ __noinline__ void select_topm(Slot<typename InTraits<In>::Acc> &sl, int r,
                                         const int *bmax, int nblocks, const In *row, int M,
                                         int nlocal, EpiScratch &es, int *sel, double *selv,
                                         int lane, unsigned long long *trl) {
  using Acc = typename InTraits<In>::Acc;
  constexpr int VEC = InTraits<In>::kVec;
  constexpr int CH = kRowBytes / (int)sizeof(In);
  // a vocabulary slice shorter than M leaves (-1, -inf) entries
  if (lane < M) {
    sel[lane] = -1;
    selv[lane] = -INFINITY;
  }
  __syncwarp();
#ifdef DSDV_XNOCAP
  return;  // development probe: capture off (results are wrong)
#endif
  // the final bins hold every block's lane maxima: the tightest bound
  int th = max(vload(&sl.ktheta[r]), theta_from_bins(sl.klist[r], M, lane));
  // short rows (vocabulary slices): the M-th largest block maximum of each group
  // of 32 blocks is a valid bound too and usually tighter -> fewer survivors
  if (nblocks <= 64 && nblocks % 32 == 0)
    for (int g = 0; g < nblocks; g += 32) th = max(th, theta_from_bins(bmax + g, M, lane));
  const int ncap = vload(&sl.ncap[r]);
  TR_ACC(trl, kTrTopmCand, ncap);
  if (ncap <= kCap) {
    int nel = 0;
    for (int base = 0; base < ncap; base += 32) {
      const int i = base + lane;
      Acc v = Acc(0);
      int id = 0;
      bool keep = false;
      if (i < ncap) {
        v = sl.cap_v[r][i];
        id = sl.cap_id[r][i];
        keep = fkey(v) >= th;
      }
      const unsigned q = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int at = nel + __popc(q & ((1u << lane) - 1u));
        if (at < 128) {
          es.ev_id[at] = id;
          es.ev_key[at] = (double)v;
        }
      }
      nel += __popc(q);
    }
    __syncwarp();
    TR_MAX(trl, kTrMaxSurv, nel);
    if (nel <= 128) {
      // rank every survivor against the others: (value desc, id asc)
      for (int i = lane; i < nel; i += 32) {
        const double vi = es.ev_key[i];
        const int ii = es.ev_id[i];
        int rank = 0;
        for (int k = 0; k < nel; ++k) {
          const double vk = es.ev_key[k];
          rank += (vk > vi || (vk == vi && es.ev_id[k] < ii)) ? 1 : 0;
        }
        if (rank < M) {
          sel[rank] = ii;
          selv[rank] = vi;
        }
      }
      __syncwarp();
      return;
    }
    TR_INC(trl, kTrTopmFallback);
    TopList<Acc> L;
    L.reset();
    for (int base = 0; base < ncap; base += 32) {
      const int i = base + lane;
      const Acc v = i < ncap ? sl.cap_v[r][i] : neg_inf<Acc>();
      const int id = i < ncap ? sl.cap_id[r][i] : 0;
      unsigned q = __ballot_sync(0xffffffffu, i < ncap && fkey(v) >= th && v >= L.theta);
      while (q) {
        const int src = __ffs(q) - 1;
        q &= q - 1;
        const Acc cv = __shfl_sync(0xffffffffu, v, src);
        const int ci = __shfl_sync(0xffffffffu, id, src);
        if (cv >= L.theta) L.insert(cv, ci, M, lane);
      }
    }
    if (lane < M && L.id != 0x7fffffff) {
      sel[lane] = L.id;
      selv[lane] = (double)L.v;
    }
    __syncwarp();
    return;
  }
  // capture overflow: re-read every block whose maximum reaches theta_run
  TR_INC(trl, kTrTopmFallback);
  TopList<Acc> L;
  L.reset();
  for (int b0 = 0; b0 < nblocks; b0 += 32) {
    const int bi = b0 + lane;
    unsigned q = __ballot_sync(0xffffffffu, bi < nblocks && bmax[bi] >= th);
    while (q) {
      const int blk = b0 + __ffs(q) - 1;
      q &= q - 1;
      const int cc = blk / kCW, w = blk - cc * kCW;
#pragma unroll 1
      for (int h = 0; h < kVecs; ++h) {
        const int id0 = cc * CH + vec_index(h, w, lane) * VEC;
        Acc v[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) v[e] = neg_inf<Acc>();
        if (id0 < nlocal) unpack(ldg128(row + id0), v, (In *)nullptr);
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const bool c = id0 + e < nlocal && fkey(v[e]) >= th && v[e] >= L.theta;
          unsigned qq = __ballot_sync(0xffffffffu, c);
          while (qq) {
            const int src = __ffs(qq) - 1;
            qq &= qq - 1;
            const Acc cv = __shfl_sync(0xffffffffu, v[e], src);
            const int ci = __shfl_sync(0xffffffffu, id0 + e, src);
            if (cv >= L.theta) L.insert(cv, ci, M, lane);
          }
        }
      }
    }
  }
  if (lane < M && L.id != 0x7fffffff) {
    sel[lane] = L.id;
    selv[lane] = (double)L.v;
  }
  __syncwarp();
}

// Exact log-sum-exp of the softened mix (two fp64 passes, one warp) for the
// rare rows whose online mix sum underflowed against its reference point.
template <class In>
__device__ __noinline__ double exact_lse_mix_warp(const In *rt, const In *rd, int n, double omt,
                                                  double tau, int lane) {
  constexpr int VEC = InTraits<In>::kVec;
  using Acc = typename InTraits<In>::Acc;
  const int nvec = (n + VEC - 1) / VEC;
  double zmax = -INFINITY;
  for (int q = lane; q < nvec; q += 32) {
    Acc t[VEC], d[VEC];
    unpack(ldg128(rt + q * VEC), t, (In *)nullptr);
    unpack(ldg128(rd + q * VEC), d, (In *)nullptr);
    for (int e = 0; e < VEC; ++e)
      if (q * VEC + e < n) zmax = fmax(zmax, omt * (double)t[e] + tau * (double)d[e]);
  }
  for (int o = 16; o > 0; o >>= 1) zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
  if (zmax == -INFINITY) return -INFINITY;
  double s = 0.0;
  for (int q = lane; q < nvec; q += 32) {
    Acc t[VEC], d[VEC];
    unpack(ldg128(rt + q * VEC), t, (In *)nullptr);
    unpack(ldg128(rd + q * VEC), d, (In *)nullptr);
    for (int e = 0; e < VEC; ++e)
      if (q * VEC + e < n) s += exp(omt * (double)t[e] + tau * (double)d[e] - zmax);
  }
  s = warp_sum_f64(s);
  return zmax + log(s);
}

// Lane 0: evaluate one position from merged statistics (token_cross_entropy
// :112-117, norm_match :119-134, is_key :136-159, effective distribution
// :231-233 with soften's short-circuits :170-172).
template <class In>
__device__ __noinline__ void evaluate_position(const double (&mrg)[7], int diff, double nm,
                                               const DevParams &p, const In *rt, const In *rd,
                                               int y, bool pair, PosEval &ev) {
  using Acc = typename InTraits<In>::Acc;
  const double Mt = mrg[0], St = mrg[1], Md = mrg[2], Sd = mrg[3], Sz = mrg[4];
  const double MtL = mrg[5], MdL = mrg[6];
  // sum 2^(v L - mL) = sum e^(v (1 + d)) e^(-mL ln2) with 1 + d = L ln 2; the
  // first-order correction of d uses the row maximum for E_P[v].
  const double d = (double)log2e<Acc>() * kLn2 - 1.0;
  const double omt = (double)p.omt_f, tau = (double)p.tau_f;
  ev.mt = Mt;
  ev.lst = (MtL + log2(St)) * kLn2 - d * Mt - Mt;
  ev.md = Md;
  ev.lsd = pair ? (MdL + log2(Sd)) * kLn2 - d * Md - Md : 0.0;
  ev.lsz = 0.0;
  ev.err = 0;
  ev.key = 0;
  ev.kind = DSDV_EFF_TARGET;
  ev.near = 0;
  ev.need_exact = 0;
  ev.accepted = 0;
  ev.h_t = ev.h_d = ev.p_t_y = ev.p_d_y = ev.nm = ev.p_eff = ev.a = ev.u = 0.0;
  ev.lt_y = ev.ld_y = -INFINITY;
  // Distribution invariants (distribution.cpp:29-63): finite, positive mass.
  if (!(St > 0.0 && isfinite(St))) ev.err = DSDV_E_INVARIANT;
  if (!pair) return;
  if (!(Sd > 0.0 && isfinite(Sd)) && !ev.err) ev.err = DSDV_E_INVARIANT;
  // check_token_in_vocab (verifier.cpp:32-37)
  const int yl = y - p.vocab_offset;
  const bool y_ok = y >= 0 && y < p.V && yl >= 0 && yl < p.vocab_local;
  if (!y_ok && !ev.err) ev.err = DSDV_E_INVARIANT;
  if (y_ok) {
    ev.lt_y = load_scalar<In>(rt + yl);
    ev.ld_y = load_scalar<In>(rd + yl);
  }
  const double lse_t = Mt + ev.lst, lse_d = Md + ev.lsd;
  ev.h_t = (ev.lt_y == -INFINITY) ? INFINITY : lse_t - ev.lt_y;
  ev.h_d = (ev.ld_y == -INFINITY) ? INFINITY : lse_d - ev.ld_y;
  ev.p_t_y = exp(ev.lt_y - lse_t);
  ev.p_d_y = exp(ev.ld_y - lse_d);
  const bool certain = ev.h_t < kCertainSurprisal;
  const bool ratio_cert = ev.h_d > 0.0;
  const bool ratio_rel = ev.h_d / ev.h_t > p.ratio_limit;
  const bool ratio = certain ? ratio_cert : ratio_rel;
  const double gap = fabs(ev.p_t_y - ev.p_d_y);
  const bool gapc = gap > p.gap_limit;
  ev.nm = nm;  // a double shared / m, compared as the reference does (:133, :156)
  const bool overlap = ev.nm < p.overlap_floor;
  ev.key = (ratio || gapc || overlap) ? 1 : 0;
  // near-threshold bookkeeping (fp32 statistics vs the fp64 reference)
  const double el = p.eps_lambda;
  if (ev.h_t < 1e-6 && (ratio_cert != ratio_rel || ev.h_d < 1e-6)) ev.near = 1;
  if (isfinite(p.ratio_limit) && ev.h_t >= 1e-6 && isfinite(ev.h_d) &&
      fabs(ev.h_d / ev.h_t - p.ratio_limit) < el * fmax(1.0, p.ratio_limit))
    ev.near = 1;
  if (fabs(gap - p.gap_limit) < el * fmax(1.0, p.gap_limit)) ev.near = 1;
  if (ev.key || p.tau == 0.0 || diff == 0)
    ev.kind = DSDV_EFF_TARGET;
  else if (p.tau == 1.0)
    ev.kind = DSDV_EFF_DRAFT;
  else
    ev.kind = DSDV_EFF_SOFTENED;
  if (ev.kind == DSDV_EFF_SOFTENED && !ev.err) {
    if (Sz > 1e-30 && isfinite(Sz)) {
      const double zL = omt * MtL + tau * MdL, z = omt * Mt + tau * Md;
      ev.lsz = (zL + log2(Sz)) * kLn2 - d * z - z;
    } else {
      ev.need_exact = 1;
    }
  }
}

// Lane 0: effective probability at y, accept_prob (verifier.cpp:188-196) and
// the strict accept test u < a (:237).
__device__ __forceinline__ void decide_position(const DevParams &p, int b, int j, PosEval &ev) {
  double p_eff = ev.p_t_y;
  if (ev.kind == DSDV_EFF_DRAFT) p_eff = ev.p_d_y;
  if (ev.kind == DSDV_EFF_SOFTENED && !ev.err) {
    const double lse_z = (double)p.omt_f * ev.mt + (double)p.tau_f * ev.md + ev.lsz;
    const double z_y = (1.0 - p.tau) * ev.lt_y + p.tau * ev.ld_y;
    p_eff = exp(z_y - lse_z);
  }
  if (!ev.err && !(ev.p_d_y > 0.0)) ev.err = DSDV_E_DRAFTING_CONTRACT;
  ev.p_eff = p_eff;
  ev.a = ev.err ? 0.0 : fmin(1.0, p_eff / ev.p_d_y);
  ev.u = 0.0;
  ev.accepted = 0;
  if (!p.stats_only) {
    ev.u = dsdv_philox_uniform(p.seed, p.window, p.seq_offset + (uint32_t)b,
                               (uint32_t)(p.gamma + j));
    ev.accepted = (!ev.err && ev.u < ev.a) ? 1 : 0;
    if (!ev.err && fabs(ev.u - ev.a) < p.eps_u) ev.near = 1;
  }
}

__device__ __forceinline__ void write_position(const DevOut &o, const DevParams &p, int b, int j,
                                               bool pair, const PosEval &ev) {
  const int G1 = p.gamma + 1;
  if (pair) {
    const size_t pos = (size_t)b * p.gamma + j;
    if (o.key_mask) o.key_mask[pos] = (uint8_t)ev.key;
    if (o.accepted) o.accepted[pos] = (uint8_t)ev.accepted;
    if (o.accept_prob) o.accept_prob[pos] = ev.a;
    if (o.h_target) o.h_target[pos] = ev.h_t;
    if (o.h_draft) o.h_draft[pos] = ev.h_d;
    if (o.p_target_y) o.p_target_y[pos] = ev.p_t_y;
    if (o.p_draft_y) o.p_draft_y[pos] = ev.p_d_y;
    if (o.norm_match) o.norm_match[pos] = ev.nm;
    if (o.p_effective_y) o.p_effective_y[pos] = ev.p_eff;
    if (o.uniform) o.uniform[pos] = ev.u;
  }
  if (o.records) {
    double *r = o.records + ((size_t)b * G1 + j) * kRecordWords;
    r[kRecMt] = ev.mt;
    r[kRecLst] = ev.lst;
    r[kRecMd] = pair ? ev.md : 0.0;
    r[kRecLsd] = pair ? ev.lsd : 0.0;
    r[kRecLsz] = pair ? ev.lsz : 0.0;
    r[kRecFlags] = (double)(ev.kind | (ev.err << 8) | (ev.key << 16));
  }
}

__device__ __forceinline__ uint32_t flag_word(const DevParams &p, const PosEval &ev,
                                              uint32_t outcome) {
  return (p.epoch << 4) | (ev.near << 3) | (ev.key << 2) | outcome;
}

// Early exit (positions after the first rejection are never
// evaluated): the smallest known stopping position of sequence b this launch.
__device__ __forceinline__ unsigned long long stop_key(const DevParams &p, int j) {
  return ((unsigned long long)p.epoch << 8) | (unsigned long long)(255 - j);
}
__device__ __forceinline__ void publish_stop(const DevScratch &s, const DevParams &p, int b, int j) {
  atomicMax(s.stop + b, stop_key(p, j));
}
// true when an earlier position than j is known to end sequence b's window
__device__ __forceinline__ bool stopped_before(const DevScratch &s, const DevParams &p, int b,
                                               int j) {
  const unsigned long long w = *(volatile const unsigned long long *)(s.stop + b);
  return (w >> 8) == (unsigned long long)p.epoch && 255 - (int)(w & 0xffu) < j;
}

// The last item of sequence b to finish commits the round (verifier.cpp:223-256).
__device__ void finalize_sequence(const DevOut &o, const DevScratch &s, const DevParams &p, int b) {
  const int G1 = p.gamma + 1;
  const unsigned int *fl = s.flags + (size_t)b * G1;
  const int2 *slots = s.slots + (size_t)b * G1;
  int keys = 0, nears = 0, k = p.gamma;
  uint32_t outcome = kOutAccepted;
  for (int j = 0; j < p.gamma; ++j) {
    const uint32_t f = ld_acquire(fl + j);
    keys += (f >> 2) & 1u;
    nears += (f >> 3) & 1u;
    outcome = f & 3u;
    if (outcome != kOutAccepted) {
      k = j;
      break;
    }
  }
  const int2 sl = slots[k];
  o.accepted_count[b] = k;
  o.key_count[b] = keys;
  o.extra_source[b] = (k < p.gamma) ? DSDV_EXTRA_RESIDUAL : DSDV_EXTRA_BONUS;
  o.extra_token[b] = sl.x;
  o.status[b] = sl.y & 0xff;
  o.near_threshold[b] = nears + ((sl.y >> 8) & 1);
}

__device__ __forceinline__ void complete_item(const DevOut &o, const DevScratch &s,
                                              const DevParams &p, int b) {
  __threadfence();
  const unsigned prev = atomicAdd(s.done + b, 1u);
  if (prev == (unsigned)p.gamma) {
    __threadfence();
    finalize_sequence(o, s, p, b);
    s.done[b] = 0u;  // re-armed for the next window
  }
}

// Weights of this lane's vector of one (chunk, warp, h) and their fp64 sum.
template <class In>
__device__ __forceinline__ double vector_weights(const In *rt, const In *rd,
                                                 const Weigher<typename InTraits<In>::Acc> &wf,
                                                 int id0, const DevParams &p,
                                                 typename InTraits<In>::Acc (&wt)[InTraits<In>::kVec]) {
  using Acc = typename InTraits<In>::Acc;
  constexpr int VEC = InTraits<In>::kVec;
  Acc vt[VEC], vd[VEC];
  const bool ok = id0 < p.vocab_local;
  if (ok) {
    unpack(ldg128(rt + id0), vt, (In *)nullptr);
    if (wf.kind != kWeightPlain) {
      unpack(ldg128(rd + id0), vd, (In *)nullptr);
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) vd[e] = Acc(0);
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) vt[e] = vd[e] = Acc(0);
  }
  weigh_vec<VEC>(wf, vt, vd, wt);
  double ls = 0.0;
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    if (!(ok && id0 + e < p.vocab_local)) wt[e] = Acc(0);
    ls += (double)wt[e];
  }
  return ls;
}

// Resolve the element of tile `t` = (chunk, warp) that holds T
// (warp-cooperative re-read): find the tile's vector whose running total
// passes T, then the lane and the element inside it.
template <class In>
__device__ __noinline__ int resolve_tile(const In *rt, const In *rd,
                                            const Weigher<typename InTraits<In>::Acc> &wf, int t,
                                            double run, double T, double W, double eps,
                                            const DevParams &p, int lane, int &near,
                                            bool want_last) {
  using Acc = typename InTraits<In>::Acc;
  constexpr int VEC = InTraits<In>::kVec;
  constexpr int CH = kRowBytes / (int)sizeof(In);
  const int c = t / kCW, w = t - c * kCW;
  int h = 0;
  {
    // the crossing vector of the tile (or, for the gap fallback, the last supported one)
    int last = -1, found = -1;
    double r = run;
#pragma unroll
    for (int hh = 0; hh < kVecs; ++hh) {
      Acc tmp[VEC];
      const double vs = warp_sum_f64(
          vector_weights<In>(rt, rd, wf, c * CH + vec_index(hh, w, lane) * VEC, p, tmp));
      if (vs > 0.0) last = hh;
      if (found < 0 && vs > 0.0 && r + vs > T) found = hh;
      if (found < 0) r += vs;
    }
    if (want_last || found < 0) {
      h = last < 0 ? kVecs - 1 : last;
      want_last = true;
    } else {
      h = found;
      // run before vector h
      double rr = run;
      for (int hh = 0; hh < h; ++hh) {
        Acc tmp[VEC];
        rr += warp_sum_f64(
            vector_weights<In>(rt, rd, wf, c * CH + vec_index(hh, w, lane) * VEC, p, tmp));
      }
      run = rr;
    }
  }
  const int id0 = c * CH + vec_index(h, w, lane) * VEC;
  Acc wt[VEC];
  const double ls = vector_weights<In>(rt, rd, wf, id0, p, wt);
  int result = -1;
  if (want_last) {
    // rounding-gap fallback: the last supported id of this tile
    const unsigned sup = __ballot_sync(0xffffffffu, ls > 0.0);
    const int src = sup ? 31 - __clz(sup) : -1;
    int lastsup = -1;
#pragma unroll
    for (int e = 0; e < VEC; ++e)
      if (wt[e] > Acc(0)) lastsup = id0 + e;
    result = src >= 0 ? __shfl_sync(0xffffffffu, lastsup, src) : -1;
    near = 1;
    return result;
  }
  double incl = ls;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const double excl = run + (incl - ls);
  const unsigned hit = __ballot_sync(0xffffffffu, ls > 0.0 && excl + ls > T);
  int idx = -1, nr = 1;
  if (hit) {
    const int src = __ffs(hit) - 1;
    if (lane == src) {
      double cum = excl, margin = 0.0;
      int lastsup = -1;
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        if (idx < 0 && wt[e] > Acc(0)) {
          lastsup = id0 + e;
          const double nc = cum + (double)wt[e];
          if (T < nc) {
            idx = id0 + e;
            margin = fmin(T - cum, nc - T);
          }
          cum = nc;
        }
      }
      if (idx >= 0) {
        nr = (margin < eps * W) ? 1 : 0;
      } else {
        idx = lastsup;
        nr = 1;
      }
    }
    idx = __shfl_sync(0xffffffffu, idx, src);
    nr = __shfl_sync(0xffffffffu, nr, src);
  } else {
    // fp64 re-association gap between tile total and lane scan: upper edge
    const unsigned sup = __ballot_sync(0xffffffffu, ls > 0.0);
    const int src = sup ? 31 - __clz(sup) : -1;
    int lastsup = -1;
#pragma unroll
    for (int e = 0; e < VEC; ++e)
      if (wt[e] > Acc(0)) lastsup = id0 + e;
    idx = src >= 0 ? __shfl_sync(0xffffffffu, lastsup, src) : -1;
    nr = 1;
  }
  near = nr;
  return idx;
}

// Sharded verifier (dsdv_shard_stats): the partial record of one position over
// this vocabulary slice, merged across slices by shard.cu (log-sum-exp of the
// per-slice normalisers, P-way merge of the top-m lists). Record words:
//   [0] m_t  [1] ln s_t  [2] m_d  [3] ln s_d  [4] ln s_z (relative to
//   (1-tau) m_t + tau m_d; -inf when the slice holds no mix mass)
//   [5] l_t(y) [6] l_d(y) (NaN unless y lies in this slice)
//   [7] rows differ | y in slice << 1
// and the slice's top-M (value, global id) of each row, (value desc, id asc).
template <class In>
__device__ __noinline__ void write_partial(const DevOut &o, const DevParams &p, int b, int j,
                                           bool pair, const double (&mrg)[7], int diff,
                                           const EpiScratch &es, const In *rt, const In *rd,
                                           const int32_t *tokens, int lane) {
  using Acc = typename InTraits<In>::Acc;
  const double Mt = mrg[0], St = mrg[1], Md = mrg[2], Sd = mrg[3], Sz = mrg[4];
  const double MtL = mrg[5], MdL = mrg[6];
  const double dd = (double)log2e<Acc>() * kLn2 - 1.0;
  const double omt = (double)p.omt_f, tau = (double)p.tau_f;
  double lsz = 0.0;
  if (pair && p.need_z) {
    if (Sz > 1e-30 && isfinite(Sz)) {
      const double zL = omt * MtL + tau * MdL, z = omt * Mt + tau * Md;
      lsz = (zL + log2(Sz)) * kLn2 - dd * z - z;
    } else {
      lsz = exact_lse_mix_warp<In>(rt, rd, p.vocab_local, omt, tau, lane) - (omt * Mt + tau * Md);
    }
  }
  const int G1 = p.gamma + 1;
  // one store here and one per peer (fused exchange: the records reach every
  // rank's buffer while the pass streams)
  auto put = [&](auto *addr, auto v) {
    *addr = v;
    for (int q = 0; q < o.npeer; ++q)
      *reinterpret_cast<decltype(addr)>(reinterpret_cast<char *>(addr) + o.peer_delta[q]) = v;
  };
  double w[kRecordWords];
  if (lane == 0) {
    w[0] = Mt;
    w[1] = (MtL + log2(St)) * kLn2 - dd * Mt - Mt;
    if (pair) {
      const int y = tokens[(size_t)b * p.gamma + j];
      const int yl = y - p.vocab_offset;
      const bool own = yl >= 0 && yl < p.vocab_local;
      w[2] = Md;
      w[3] = (MdL + log2(Sd)) * kLn2 - dd * Md - Md;
      w[4] = lsz;
      w[5] = own ? load_scalar<In>(rt + yl) : NAN;
      w[6] = own ? load_scalar<In>(rd + yl) : NAN;
      w[7] = (double)((diff ? 1 : 0) | (own ? 2 : 0));
    } else {
      w[2] = w[3] = w[4] = 0.0;
      w[5] = w[6] = NAN;
      w[7] = 0.0;
    }
  }
  // one coalesced store of the record per destination (lane k: word k)
  double wk = 0.0;
#pragma unroll
  for (int k = 0; k < kRecordWords; ++k) {
    const double t = __shfl_sync(0xffffffffu, w[k], 0);
    if (lane == k) wk = t;
  }
  if (lane < kRecordWords) put(o.records + ((size_t)b * G1 + j) * kRecordWords + lane, wk);
  const int M = p.top_m;
  if (pair && lane < M) {
    const size_t base = ((size_t)b * p.gamma + j) * 2 * M;
    const int it = es.sel[0][lane], id = es.sel[1][lane];
    put(o.topv + base + lane, es.selv[0][lane]);
    put(o.topi + base + lane, it >= 0 ? p.vocab_offset + it : -1);
    put(o.topv + base + M + lane, es.selv[1][lane]);
    put(o.topi + base + M + lane, id >= 0 ? p.vocab_offset + id : -1);
  }
  // (no fence per item: dsdv_peer_signal, after this kernel on the stream,
  // fences at system scope and releases the arrival flags)
}

template <class In, bool EE>
__device__ void epilogue_loop(Smem<typename InTraits<In>::Acc> &sm, const DevParams &p,
                              const In *__restrict__ draft, const In *__restrict__ target,
                              const int32_t *__restrict__ tokens, const DevOut &o,
                              const DevScratch &s, int ew, int lane, unsigned long long *tr) {
  using Acc = typename InTraits<In>::Acc;
  const int G1 = p.gamma + 1;
  const int M = p.top_m;
  const double omt_d = (double)p.omt_f, tau_d = (double)p.tau_f;
  const int nblocks = p.n_chunks * kCW;  // sample tiles (chunk, warp)
  unsigned long long *trl = lane == 0 ? tr : nullptr;
  TR_DECL;
  for (int n = ew;; n += kEW) {
    const int si = n % kSlots;
    TR_START(tw);
    // while the compute warps fold this slot's item, keep its top-m bound tight
#ifdef DSDV_EPI_BLOCK
    mbar_wait(&sm.part_full[si], (n / kSlots) & 1);
#else
#ifndef DSDV_EPI_SLEEP
#define DSDV_EPI_SLEEP 64
#endif
    while (!mbar_test(&sm.part_full[si], (n / kSlots) & 1)) {
      refresh_theta(sm.slot[si], M, lane);
      __nanosleep(DSDV_EPI_SLEEP);
    }
#endif
    TR_ADD(trl, kTrEpiWaitFull, tw);
    TR_START(tx);
    Slot<Acc> &sl = sm.slot[si];
    const int item = sl.item;
    if (item < 0) break;
    const int j = item / p.B, b = item - j * p.B;
    const bool pair = j < p.gamma;
    const In *rt = target + ((size_t)b * G1 + j) * (size_t)p.stride;
    const In *rd = draft + ((size_t)b * p.gamma + (pair ? j : 0)) * (size_t)p.stride;
    int2 *slotp = s.slots + (size_t)b * G1 + j;

    if (EE && sl.kind == kAborted) {
      // early exit: an item cut short after its sequence stopped earlier
      if (pair) reset_capture(sl, lane);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&sm.part_empty[si]);
        complete_item(o, s, p, b);
      }
    } else if (sl.kind == kRegular) {
      double mrg[7];
      int diff = 0;
      merge_partials(sl, p, lane, mrg, diff);
      TR_ADD(trl, kTrEpiMerge, tx);
      TR_START(tt);
      int shared = 0;
      if (pair) {
        EpiScratch &es = sm.epi[ew];
        const int nb = p.n_chunks * kCW;
        const SlotView sv(sl.area, nb);
        select_topm<In>(sl, 0, sv.bmax[0], nb, rt, M, p.vocab_local, es, es.sel[0], es.selv[0],
                        lane, trl);
        select_topm<In>(sl, 1, sv.bmax[1], nb, rd, M, p.vocab_local, es, es.sel[1], es.selv[1],
                        lane, trl);
        reset_capture(sl, lane);
        const int did = lane < M ? es.sel[1][lane] : -1;
        bool found = false;
        for (int k = 0; k < M; ++k) found |= (es.sel[0][k] == did);
        shared = __popc(__ballot_sync(0xffffffffu, found && lane < M));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.part_empty[si]);  // partials consumed
      TR_ADD(trl, kTrEpiTopm, tt);
      TR_START(td);
      TR_INC(trl, kTrEpiItems);
      if (p.partial) {
        // vocabulary-sharded verifier: this slice's partial record only
        const EpiScratch &es = sm.epi[ew];
        write_partial<In>(o, p, b, j, pair, mrg, diff, es, rt, rd, tokens, lane);
      } else {
      PosEval ev;
      if (lane == 0) {
        const int y = pair ? tokens[(size_t)b * p.gamma + j] : 0;
        // NormMatch of a top_m beyond the warp selection comes from the caller
        // (dsdv_window_stats_nm); otherwise from the selected top lists
        const double nm = (pair && p.nm_in) ? p.nm_in[(size_t)b * p.gamma + j]
                                            : (double)shared / (double)p.top_m;
        evaluate_position<In>(mrg, diff, nm, p, rt, rd, y, pair, ev);
      }
      const int need_exact = __shfl_sync(0xffffffffu, lane == 0 ? ev.need_exact : 0, 0);
      if (need_exact) {
        TR_INC(trl, kTrNeedExact);
        const double lse = exact_lse_mix_warp<In>(rt, rd, p.vocab_local, omt_d, tau_d, lane);
        if (lane == 0) {
          if (lse == -INFINITY)
            ev.err = DSDV_E_DEGENERATE_MIXTURE;  // disjoint supports (verifier.cpp:181-184)
          else
            ev.lsz = lse - (omt_d * ev.mt + tau_d * ev.md);
          ev.need_exact = 0;
        }
      }
      if (lane == 0) {
        if (pair) decide_position(p, b, j, ev);
        write_position(o, p, b, j, pair, ev);
        if (EE && pair && (ev.err || !ev.accepted)) publish_stop(s, p, b, j);  // positions past j are never needed (verifier.cpp:250)
        if (!p.stats_only) {
          const unsigned int *fl = s.flags + (size_t)b * G1;
          bool stopped_before = false;  // an earlier position already ends the window
          if (!(pair && ev.accepted)) {
            for (int jj = 0; jj < j && !stopped_before; ++jj) {
              const uint32_t f = ld_acquire(fl + jj);
              stopped_before = (f >> 4) == p.epoch && (f & 3u) != kOutAccepted;
            }
          }
          int want = 0;  // 1 residual, 2 bonus
          if (pair) {
            if (!ev.accepted && !stopped_before) {
              if (ev.err)
                *slotp = make_int2(-1, ev.err);
              else if (ev.kind == DSDV_EFF_DRAFT)
                *slotp = make_int2(-1, DSDV_E_EMPTY_RESIDUAL);  // verifier.cpp:209-211
              else
                want = 1;
            }
          } else if (!stopped_before) {
            if (ev.err)
              *slotp = make_int2(-1, ev.err);
            else
              want = 2;
          }
          if (want) {
            // the flag of a drawing position is published once its draw lands;
            // stash it in the slot until then
            if (pair) *slotp = make_int2(-2, (int)flag_word(p, ev, kOutRejected));
            const int t = atomicAdd(&sm.req_tail, 1);
            Request<Acc> &rq = sm.req[t % kReq];
            rq.item = item;
            rq.rows = want == 1 ? 2 : 1;
            rq.u = dsdv_philox_uniform(p.seed, p.window, p.seq_offset + (uint32_t)b,
                                       (uint32_t)(want == 1 ? p.gamma + j + 1 : 2 * p.gamma));
            set_weigher(rq.wf,
                        want == 2 ? kWeightPlain
                                  : (ev.kind == DSDV_EFF_SOFTENED ? kWeightResSoft
                                                                  : kWeightResTarget),
                        ev, omt_d, tau_d);
            __threadfence_block();
            vstore(&rq.ready, 1);
          } else {
            if (pair) {
              const uint32_t outcome =
                  ev.err ? kOutError : (ev.accepted ? kOutAccepted : kOutRejected);
              __threadfence();
              st_release(s.flags + (size_t)b * G1 + j, flag_word(p, ev, outcome));
            }
            complete_item(o, s, p, b);
          }
        }
      }
      }  // !p.partial
      TR_ADD(trl, kTrEpiDecide, td);
    } else {
      // ---- sample item: scan the tile sums for T = u W, resolve the tile ----
      const Request<Acc> &rq = sm.req[sl.req];
      const Weigher<Acc> wf = rq.wf;
      const double u = rq.u;
      const double *tiles = reinterpret_cast<const double *>(sl.area);
      double wpart = 0.0;
      for (int t = lane; t < nblocks; t += 32) wpart += tiles[t];
      const double W = warp_sum_f64(wpart);
      const double T = u * W;
      double run = 0.0, base = 0.0;
      int found = -1, lastpos = -1;
      for (int c0 = 0; c0 < nblocks; c0 += 32) {
        const int t = c0 + lane;
        const double x = t < nblocks ? tiles[t] : 0.0;
        const unsigned pos = __ballot_sync(0xffffffffu, x > 0.0);
        if (pos) lastpos = c0 + 31 - __clz(pos);
        if (found < 0) {
          double incl = x;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
          }
          const unsigned hit = __ballot_sync(0xffffffffu, t < nblocks && x > 0.0 && run + incl > T);
          if (hit) {
            const int src = __ffs(hit) - 1;
            found = c0 + src;
            base = run + __shfl_sync(0xffffffffu, incl - x, src);
          }
          run += __shfl_sync(0xffffffffu, incl, 31);
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&sm.part_empty[si]);  // tiles consumed
        atomicAdd(&sm.req_done, 1);       // request entry free again
      }
      int near = 0, idx = -1;
      if (W > 0.0) {
        if (found >= 0)
          idx = resolve_tile<In>(rt, rd, wf, found, base, T, W, p.eps_u, p, lane, near, false);
        else
          idx = resolve_tile<In>(rt, rd, wf, lastpos, 0.0, T, W, p.eps_u, p, lane, near, true);
      }
      if (lane == 0) {
        if (pair) {
          const int2 stash = *slotp;  // flag word stashed by the regular item
          *slotp = idx < 0 ? make_int2(-1, DSDV_E_EMPTY_RESIDUAL)
                           : make_int2(p.vocab_offset + idx, DSDV_OK | (near << 8));
          __threadfence();
          st_release(s.flags + (size_t)b * G1 + j, (uint32_t)stash.y);
        } else {
          *slotp = idx < 0 ? make_int2(-1, DSDV_E_EMPTY_RESIDUAL)
                           : make_int2(p.vocab_offset + idx, DSDV_OK | (near << 8));
        }
        complete_item(o, s, p, b);
      }
      TR_ADD(trl, kTrEpiSample, tx);
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      atomicAdd(&sm.epi_count, 1);
    }
  }
  // peer exchange: this warp's stores into the other ranks' buffers are
  // visible system-wide before the kernel ends (dsdv_peer_signal follows)
  if (o.npeer) __threadfence_system();
  TR_FLUSH(trl);
}

// ------------------------------------------------------------------ producer warp
template <class In, bool EE, class Acc = typename InTraits<In>::Acc>
__device__ __forceinline__ void stream_rows(Smem<Acc> &sm, const In *rt,
                                            const In *rd, bool two, int item, int kind, int n,
                                            int req, int n_chunks, int nlocal, bool pad, int &stage,
                                            uint32_t &phase, unsigned long long *tr,
                                            unsigned long long &copied, const DevScratch &sx,
                                            const DevParams &pp, int b, int j) {
  constexpr int CH = kRowBytes / (int)sizeof(In);
  TR_DECL;
  for (int c = 0; c < n_chunks; ++c) {
    TR_START(tw);
    mbar_wait_spin(&sm.empty[stage], phase ^ 1);
    TR_ADD(tr, kTrProdWaitEmpty, tw);
    if (EE && kind == kRegular && j > 0 && c > 0 && stopped_before(sx, pp, b, j)) {
      // early exit: the sequence stopped at an earlier position while this
      // item streamed; an empty stage ends the item
      StageMeta m;
      m.item = item;
      m.chunk = n_chunks - 1;
      m.n = n;
      m.kr = kind | (req << 1) | kAbortBit;
      sm.meta[stage] = m;
      mbar_arrive(&sm.full[stage]);
      if (++stage == Smem<Acc>::kStages) {
        stage = 0;
        phase ^= 1;
      }
      return;
    }
    StageMeta m;
    m.item = item;
    m.chunk = c;
    m.n = n;
    m.kr = kind | (req << 1) | (two ? kPairBit : 0);
    sm.meta[stage] = m;
    const int rem = nlocal - c * CH;
    const int elems = rem < CH ? rem : CH;
    const uint32_t bytes = ((uint32_t)(elems * (int)sizeof(In)) + 15u) & ~15u;
    copied += two ? 2u * bytes : bytes;
#ifdef DSDV_TIMELINE
    if (tr && blockIdx.x == 0) {
      unsigned long long *tl = tr + 512 * kTraceWords;
      const unsigned q = (unsigned)tl[4095]++;
      if (q < 1000) tl[q * 4 + 0] = clock64();
    }
#endif
    if (pad && bytes < (uint32_t)kRowBytes) {
      // short last chunk of a regular row: the rest of the stage reads as
      // -inf (no mass, never a maximum), so the compute warps fold it with
      // the unmasked code; the arrival (release) follows the fill while the
      // copies run
      mbar_expect_tx(&sm.full[stage], two ? 2u * bytes : bytes);
      bulk_g2s(sm.ring[stage][1], rt + (size_t)c * CH, bytes, &sm.full[stage]);
      if (two) bulk_g2s(sm.ring[stage][0], rd + (size_t)c * CH, bytes, &sm.full[stage]);
      const uint4 ninf = InTraits<In>::neg_inf_vec();
      for (uint32_t o = bytes; o < (uint32_t)kRowBytes; o += 16) {
        *reinterpret_cast<uint4 *>(sm.ring[stage][1] + o) = ninf;
        if (two) *reinterpret_cast<uint4 *>(sm.ring[stage][0] + o) = ninf;
      }
      mbar_arrive(&sm.full[stage]);
    } else {
      mbar_arrive_expect_tx(&sm.full[stage], two ? 2u * bytes : bytes);
      bulk_g2s(sm.ring[stage][1], rt + (size_t)c * CH, bytes, &sm.full[stage]);
      if (two) bulk_g2s(sm.ring[stage][0], rd + (size_t)c * CH, bytes, &sm.full[stage]);
    }
    if (++stage == Smem<Acc>::kStages) {
      stage = 0;
      phase ^= 1;
    }
  }
  TR_FLUSH(tr);
}

template <class In, bool EE>
__device__ void producer_loop(Smem<typename InTraits<In>::Acc> &sm, const DevParams &p,
                              const In *__restrict__ draft, const In *__restrict__ target,
                              const DevOut &o, const DevScratch &s, unsigned long long *tr) {
  TR_DECL;
  const int G1 = p.gamma + 1;
  unsigned long long copied = 0;
  int stage = 0;
  uint32_t phase = 0;
  int n = 0, next = -1;
  bool exhausted = false;
  for (;;) {
    // sample requests first: the sequence's completion waits on them
    const int head = vload(&sm.req_head);
    if (head != vload(&sm.req_tail)) {
      const int r = head % kReq;
      while (!vload(&sm.req[r].ready)) __nanosleep(32);  // entry still being written
      __threadfence_block();
      vstore(&sm.req[r].ready, 0);
      const int item = sm.req[r].item;
      const int two = sm.req[r].rows == 2;
      const int j = item / p.B, b = item - j * p.B;
      const In *rt = target + ((size_t)b * G1 + j) * (size_t)p.stride;
      const In *rd = draft + ((size_t)b * p.gamma + (j < p.gamma ? j : 0)) * (size_t)p.stride;
      stream_rows<In, EE>(sm, rt, rd, two, item, kSample, n, r, p.n_chunks, p.vocab_local, false, stage,
                      phase, tr, copied, s, p, b, j);
      TR_INC(tr, kTrProdSamples);
      ++n;
      vstore(&sm.req_head, head + 1);
      continue;
    }
    if (!exhausted) {
      const int item = next >= 0 ? next : (int)atomicAdd(s.ticket, 1u);
      next = -1;
      if (item < p.n_items) {
        // claim the following item now: the global atomic's round trip
        // overlaps this item's copies instead of delaying the next item
        next = (int)atomicAdd(s.ticket, 1u);
        const int j = item / p.B, b = item - j * p.B;  // position-major order
        const bool pair = j < p.gamma;
        if (EE && j > 0 && stopped_before(s, p, b, j)) {
          // early exit: an earlier position already ends this sequence's window
          // (verifier.cpp:250); the item is never streamed, only counted
          complete_item(o, s, p, b);
          continue;
        }
        const In *rt = target + ((size_t)b * G1 + j) * (size_t)p.stride;
        const In *rd = draft + ((size_t)b * p.gamma + (pair ? j : 0)) * (size_t)p.stride;
        stream_rows<In, EE>(sm, rt, rd, pair, item, kRegular, n, 0, p.n_chunks, p.vocab_local,
                        pad_tail<In>(p), stage, phase, tr, copied, s, p, b, j);
        TR_INC(tr, kTrProdItems);
        ++n;
        continue;
      }
      exhausted = true;
    }
    // drained: wait until the epilogue has seen everything streamed, then
    // re-check for requests it may have posted on the way
    TR_START(td);
    if (vload(&sm.epi_count) == n) {
      __threadfence_block();
      if (vload(&sm.req_head) == vload(&sm.req_tail)) break;
      continue;
    }
    __nanosleep(256);
    TR_ADD(tr, kTrProdDrain, td);
  }
  // end of stream
  TR_FLUSH(tr);
  if (s.streamed) atomicAdd(s.streamed, copied);
  mbar_wait(&sm.empty[stage], phase ^ 1);
  StageMeta m;
  m.item = -1;
  m.chunk = 0;
  m.n = n;
  m.kr = kRegular;
  sm.meta[stage] = m;
  mbar_arrive(&sm.full[stage]);
}

// ------------------------------------------------------------------ kernel
template <class In, bool EE>
#ifndef DSDV_CTAS
#define DSDV_CTAS 1  // resident CTAs per SM
#endif
__global__ void __launch_bounds__(kThreads, DSDV_CTAS)
    fused_verify_kernel(const __grid_constant__ DevParams p, const In *__restrict__ draft,
                        const In *__restrict__ target, const int32_t *__restrict__ tokens,
                        const __grid_constant__ DevOut o, const __grid_constant__ DevScratch s) {
  using Acc = typename InTraits<In>::Acc;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem<Acc> &sm = *reinterpret_cast<Smem<Acc> *>(smem_raw);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  unsigned long long *tr = s.trace ? s.trace + (size_t)blockIdx.x * kTraceWords : nullptr;
  TR_DECL;
  TR_START(tk);

  if (tid == 0) {
    for (int i = 0; i < Smem<Acc>::kStages; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], kCW);
    }
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&sm.part_full[i], kCW);
      mbar_init(&sm.part_empty[i], 1);
    }
    sm.req_head = sm.req_tail = sm.req_done = 0;
    sm.epi_count = sm.epi_exit = 0;
    for (int i = 0; i < kReq; ++i) sm.req[i].ready = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp < kSlots) reset_capture(sm.slot[warp], lane);
  __syncthreads();

  if (warp == kProdWarp) {
    if (lane == 0) producer_loop<In, EE>(sm, p, draft, target, o, s, tr);
  } else if (warp >= kEpiWarp) {
    epilogue_loop<In, EE>(sm, p, draft, target, tokens, o, s, warp - kEpiWarp, lane, tr);
    if (lane == 0 && atomicAdd(&sm.epi_exit, 1) == kEW - 1) {
      TR_ADD(tr, kTrKernel, tk);
      TR_FLUSH(tr);
      // last CTA out re-arms the work counters for the next launch
      __threadfence();
      const unsigned prev = atomicAdd(s.exit_count, 1u);
      if (prev == gridDim.x - 1) {
        *s.ticket = 0u;
        *s.exit_count = 0u;
        __threadfence();
      }
    }
  } else {
    if (p.need_z)
      compute_loop<In, true, EE>(sm, p, draft, target, tid, tr);
    else
      compute_loop<In, false, EE>(sm, p, draft, target, tid, tr);
  }
}

}  // namespace fz

// ------------------------------------------------------------------ launch
template <class In, bool EE>
cudaError_t launch_fused_t(const DevParams &q, const void *draft, const void *target,
                           const int32_t *tokens, const DevOut &o, const DevScratch &s,
                           cudaStream_t stream, int *grid_out) {
  using Acc = typename InTraits<In>::Acc;
  const size_t smem = sizeof(fz::Smem<Acc>);
  // occupancy is a property of (kernel, device): one query per device, the
  // cache guarded for concurrent host threads (sweep workers)
  static std::mutex mu;
  static int grid_cap[64] = {0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  int grid;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (grid_cap[dev] == 0) {
      e = cudaFuncSetAttribute(fz::fused_verify_kernel<In, EE>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      int per_sm = 0, sms = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fz::fused_verify_kernel<In, EE>,
                                                        fz::kThreads, smem);
      if (e != cudaSuccess) return e;
      e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (e != cudaSuccess) return e;
      if (per_sm < 1) return cudaErrorInvalidConfiguration;
      grid_cap[dev] = per_sm * sms;
    }
    grid = grid_cap[dev];
  }
  if (grid > q.n_items) grid = q.n_items;
  if (grid_out) *grid_out = grid;
  fz::fused_verify_kernel<In, EE><<<grid, fz::kThreads, smem, stream>>>(
      q, (const In *)draft, (const In *)target, tokens, o, s);
  return cudaGetLastError();
}

template <class In>
cudaError_t launch_fused(const DevParams &p, const void *draft, const void *target,
                         const int32_t *tokens, const DevOut &o, const DevScratch &s,
                         cudaStream_t stream, int *grid_out) {
  constexpr int CH = fz::kRowBytes / (int)sizeof(In);
  DevParams q = p;
  q.n_chunks = (p.vocab_local + CH - 1) / CH;
  const int ntiles = q.n_chunks * fz::kCW;
  if (ntiles > fz::Area<typename InTraits<In>::Acc>::kTiles)
    return cudaErrorInvalidValue;
  return q.early_exit ? launch_fused_t<In, true>(q, draft, target, tokens, o, s, stream, grid_out)
                      : launch_fused_t<In, false>(q, draft, target, tokens, o, s, stream, grid_out);
}

// Vocabulary limit of the fused kernel for a dtype (per-slot block maxima, or
// sample tiles, must fit the slot area).
int fused_max_vocab(int esize, int top_m) {
  (void)top_m;
  const int tiles = esize == 8 ? fz::Area<double>::kTiles : fz::Area<float>::kTiles;
  return tiles / fz::kCW * (fz::kRowBytes / esize);
}

template cudaError_t launch_fused<__nv_bfloat16>(const DevParams &, const void *, const void *,
                                                 const int32_t *, const DevOut &,
                                                 const DevScratch &, cudaStream_t, int *);
template cudaError_t launch_fused<float>(const DevParams &, const void *, const void *,
                                         const int32_t *, const DevOut &, const DevScratch &,
                                         cudaStream_t, int *);
template cudaError_t launch_fused<double>(const DevParams &, const void *, const void *,
                                          const int32_t *, const DevOut &, const DevScratch &,
                                          cudaStream_t, int *);

}  // namespace dsdv
