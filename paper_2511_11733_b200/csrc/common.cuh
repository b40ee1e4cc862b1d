// Shared device-side definitions for the dsdv sm_100a kernels.
//
// Element access is in 16-byte vectors (LDS.128 / LDG.128 / 1-D bulk copies);
// arithmetic is fp32 for f32/bf16 logits and fp64 for f64 logits.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dsdv/dsdv.h"
#include "dsdv/philox.h"

namespace dsdv {

constexpr int kConsumerWarps = 8;
constexpr int kConsumerThreads = kConsumerWarps * 32;
constexpr int kProducerWarps = 1;
constexpr int kFusedThreads = kConsumerThreads + 32 * kProducerWarps;
constexpr int kChunkBytes = 8192;  // per row per pipeline stage
constexpr int kStages = 4;
constexpr int kMaxTopM = 32;       // one warp lane per top-m list entry
constexpr int kRecordWords = DSDV_RECORD_WORDS;

// Record layout (double[kRecordWords]) per (sequence, position):
//   [0] m_t   max target logit (exact input value)      [1] ln s_t   (LSE_t = m_t + ln s_t)
//   [2] m_d   max draft logit                            [3] ln s_d
//   [4] ln s_z  (LSE_z = (1-tau) m_t + tau m_d + ln s_z)
//   [5] effective kind | error code << 8 | key << 16
constexpr int kRecMt = 0, kRecLst = 1, kRecMd = 2, kRecLsd = 3, kRecLsz = 4, kRecFlags = 5;

constexpr double kLn2 = 0.69314718055994530942;
constexpr double kLog2e = 1.44269504088896340736;
constexpr float kLog2eF = 1.44269504088896340736f;
constexpr double kCertainSurprisal = 1e-12;  // verifier.cpp:30

// Flag word per (sequence, position) published by the fused kernel:
//   bits 0-1 outcome (1 accepted, 2 rejected, 3 error), bit 2 key, bit 3 near,
//   bits 4-31 launch epoch (so flags never need clearing).
constexpr uint32_t kOutAccepted = 1, kOutRejected = 2, kOutError = 3;

struct DevParams {
  int B, gamma, V, stride, top_m, vocab_offset, vocab_local;
  int n_chunks;     // chunks per row
  int n_items;      // B * (gamma + 1)
  int stats_only;   // 1: dsdv_window_stats (no draws, no waits, no sampling)
  int partial;      // 1: dsdv_shard_stats (partial records of a vocabulary slice only)
  int need_z;       // 0 < tau < 1
  int early_exit;   // 1: dsdv_verify_early_exit (rows past a sequence's first rejection are skipped)
  const double *nm_in;  // dsdv_window_stats_nm: caller's NormMatch [B][gamma] (any top_m)
  float tau_f, omt_f;
  double tau, ratio_limit, gap_limit, overlap_floor, eps_u, eps_lambda;
  uint64_t seed, window;
  uint32_t seq_offset;
  uint32_t epoch;   // 28 bits used
};

struct DevOut {
  int32_t *accepted_count, *extra_token, *key_count, *status, *near_threshold;
  uint8_t *extra_source, *key_mask, *accepted;
  double *accept_prob, *h_target, *h_draft, *p_target_y, *p_draft_y, *norm_match,
      *p_effective_y, *uniform, *records;
  double *topv;    // sharded partial: [B][gamma][2][M] top-m values (target, draft)
  int32_t *topi;   //                  and global ids
  // peer exchange: every partial store is repeated at address + peer_delta[q]
  // (the same slot in rank q's mapped exchange buffer), q < npeer
  int npeer;
  long long peer_delta[8];
};

struct DevScratch {
  unsigned int *ticket;      // work counter (self-resetting)
  unsigned int *exit_count;  // CTAs finished (self-resetting)
  unsigned int *flags;       // [B][gamma+1] per-position outcome words (epoch-tagged)
  int2 *slots;               // [B][gamma+1] extra-token draws (token, status | near << 8)
  unsigned int *done;        // [B] items finished this window (reset by the finaliser)
  unsigned long long *trace; // [grid][kTraceWords] cycle counters (DSDV_TRACE builds only)
  unsigned long long *stop;  // [B] first known stop position, epoch << 8 | (255 - j) (atomicMax)
  unsigned long long *streamed;  // logit bytes the producers copied (accumulated across launches)
};
constexpr int kTraceWords = 28;

// ------------------------------------------------------------------ traits
template <class In>
struct InTraits;
template <>
struct InTraits<__nv_bfloat16> {
  static constexpr int kVec = 8;  // elements per 16-byte vector
  using Acc = float;
  __device__ static uint4 neg_inf_vec() { return make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u); }
};
template <>
struct InTraits<float> {
  static constexpr int kVec = 4;
  using Acc = float;
  __device__ static uint4 neg_inf_vec() { return make_uint4(0xff800000u, 0xff800000u, 0xff800000u, 0xff800000u); }
};
template <>
struct InTraits<double> {
  static constexpr int kVec = 2;
  using Acc = double;
  __device__ static uint4 neg_inf_vec() { return make_uint4(0u, 0xfff00000u, 0u, 0xfff00000u); }
};

// Unpack one 16-byte vector into accumulator-precision values.
__device__ __forceinline__ void unpack(const uint4 &r, float (&v)[8], __nv_bfloat16 *) {
  // bf16 -> f32 is a 16-bit shift; PRMT keeps it on the integer pipe
  v[0] = __uint_as_float(__byte_perm(r.x, 0u, 0x1044));
  v[1] = __uint_as_float(__byte_perm(r.x, 0u, 0x3244));
  v[2] = __uint_as_float(__byte_perm(r.y, 0u, 0x1044));
  v[3] = __uint_as_float(__byte_perm(r.y, 0u, 0x3244));
  v[4] = __uint_as_float(__byte_perm(r.z, 0u, 0x1044));
  v[5] = __uint_as_float(__byte_perm(r.z, 0u, 0x3244));
  v[6] = __uint_as_float(__byte_perm(r.w, 0u, 0x1044));
  v[7] = __uint_as_float(__byte_perm(r.w, 0u, 0x3244));
}
__device__ __forceinline__ void unpack(const uint4 &r, float (&v)[4], float *) {
  v[0] = __uint_as_float(r.x);
  v[1] = __uint_as_float(r.y);
  v[2] = __uint_as_float(r.z);
  v[3] = __uint_as_float(r.w);
}
__device__ __forceinline__ void unpack(const uint4 &r, double (&v)[2], double *) {
  v[0] = __hiloint2double((int)r.y, (int)r.x);
  v[1] = __hiloint2double((int)r.w, (int)r.z);
}

// One element from shared memory (the resident ring stage).
__device__ __forceinline__ float load_smem_scalar(const __nv_bfloat16 *p) {
  return __bfloat162float(*p);
}
__device__ __forceinline__ float load_smem_scalar(const float *p) { return *p; }
__device__ __forceinline__ double load_smem_scalar(const double *p) { return *p; }

template <class In>
__device__ __forceinline__ double load_scalar(const In *p);
template <>
__device__ __forceinline__ double load_scalar<__nv_bfloat16>(const __nv_bfloat16 *p) {
  return (double)__bfloat162float(*p);
}
template <>
__device__ __forceinline__ double load_scalar<float>(const float *p) {
  return (double)*p;
}
template <>
__device__ __forceinline__ double load_scalar<double>(const double *p) {
  return *p;
}

// ------------------------------------------------------------------ math
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ double fast_exp2(double x) { return exp2(x); }

// ---- packed fp32x2 arithmetic (FADD2 / FMUL2 / FFMA2: same element rate as
// scalar FP32, half the issue slots) ----
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo2(f32x2 a) { return __uint_as_float((unsigned)a); }
__device__ __forceinline__ float hi2(f32x2 a) { return __uint_as_float((unsigned)(a >> 32)); }
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// 2^x on the FMA pipe for two lanes at once (offloads the MUFU unit):
// x = n + f with n = rint(x) (1.5*2^23 magic), f in [-0.5, 0.5];
// 2^f by a relative-minimax polynomial (degree 4: max rel. error 2.7e-6 in
// fp32 Horner; -DDSDV_POLY5: degree 5, 2.3e-7), scaled by 2^n through the
// exponent field.
// x is clamped below at -126 (results under 2^-126 are negligible, like ex2.approx.ftz).
__device__ __forceinline__ f32x2 poly_exp2x2(f32x2 x) {
  // callers guarantee x <= ~12 (lazy-max slack); only the low end needs a clamp
  // clamp at -126: with n >= -126 the exponent add cannot wrap even when the
  // polynomial dips just below 1 at f = 0
  const float a = fmaxf(lo2(x), -126.0f);
  const float b = fmaxf(hi2(x), -126.0f);
  const f32x2 xc = pk2(a, b);
  const f32x2 magic = pk2(12582912.0f, 12582912.0f);
  const f32x2 j = add2(xc, magic);
  const f32x2 f = sub2(xc, sub2(j, magic));
#ifdef DSDV_POLY5
  f32x2 p = fma2(pk2(1.327647129073739e-3f, 1.327647129073739e-3f), f,
                 pk2(9.675540961325169e-3f, 9.675540961325169e-3f));
  p = fma2(p, f, pk2(5.550713092088699e-2f, 5.550713092088699e-2f));
  p = fma2(p, f, pk2(2.4022120237350464e-1f, 2.4022120237350464e-1f));
  p = fma2(p, f, pk2(6.931469440460205e-1f, 6.931469440460205e-1f));
  p = fma2(p, f, pk2(1.0000001192092896f, 1.0000001192092896f));
#else
  // degree 4: max relative error 2.7e-6 in fp32 Horner — within the 1e-5
  // tolerance on softened probabilities (the mix sum's relative error is at
  // most the per-term one), one FFMA2 per element pair cheaper
  f32x2 p = fma2(pk2(9.570101276040077e-3f, 9.570101276040077e-3f), f,
                 pk2(5.591785907745361e-2f, 5.591785907745361e-2f));
  p = fma2(p, f, pk2(2.40247443318367e-1f, 2.40247443318367e-1f));
  p = fma2(p, f, pk2(6.931217908859253e-1f, 6.931217908859253e-1f));
  p = fma2(p, f, pk2(9.999992847442627e-1f, 9.999992847442627e-1f));
#endif
  const unsigned jl = __float_as_uint(lo2(j)), jh = __float_as_uint(hi2(j));
  const float rl = __uint_as_float(__float_as_uint(lo2(p)) + (jl << 23));
  const float rh = __uint_as_float(__float_as_uint(hi2(p)) + (jh << 23));
  return pk2(rl, rh);
}

template <class Acc>
__device__ __forceinline__ Acc neg_inf();
template <>
__device__ __forceinline__ float neg_inf<float>() {
  return __int_as_float(0xff800000);
}
template <>
__device__ __forceinline__ double neg_inf<double>() {
  return __longlong_as_double(0xfff0000000000000ll);
}

template <class Acc>
__device__ __forceinline__ Acc log2e();
template <>
__device__ __forceinline__ float log2e<float>() {
  return kLog2eF;
}
template <>
__device__ __forceinline__ double log2e<double>() {
  return kLog2e;
}

// (m, s) online-softmax pair merge: s is relative to m (natural-log max).
template <class Acc>
__device__ __forceinline__ void merge_ms(Acc &m, Acc &s, Acc m2, Acc s2) {
  if (m2 > m) {
    s = (m == neg_inf<Acc>() ? Acc(0) : s * fast_exp2((m - m2) * log2e<Acc>())) + s2;
    m = m2;
  } else if (m2 != neg_inf<Acc>()) {
    s += s2 * fast_exp2((m2 - m) * log2e<Acc>());
  }
}

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
// Expect bytes on the barrier without arriving (the arrival follows later).
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t a = smem_addr(bar);
  do {
    // the suspend-time hint parks the warp in hardware until the phase flips,
    // instead of re-issuing the probe (spinning warps steal issue slots from
    // the compute warps)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, "
        "0, p; }"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(0x989680u)
        : "memory");
  } while (!done);
}
// Wait without a suspend hint: plain try_wait probes. For the producer, whose
// wake-up latency directly delays the next copy.
__device__ __forceinline__ void mbar_wait_spin(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t a = smem_addr(bar);
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, "
        "p; }"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
// One probe of an mbarrier phase (no suspend): true once the phase completed.
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, "
      "p; }"
      : "=r"(done)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
// 1-D bulk copy global -> shared (TMA engine), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ uint4 lds128(const void *p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_addr(p)));
  return r;
}
__device__ __forceinline__ uint4 ldg128(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// Barrier among the 256 consumer threads only (the producer warp keeps streaming).
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerThreads) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const unsigned int *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned int *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ------------------------------------------------------------------ top-m
// A warp-distributed sorted list of the best M (value desc, id asc) entries:
// lane l < M holds entry l. Empty slots are (-inf, INT_MAX), which every real
// element beats, so -inf logits still rank by id like zero probabilities do in
// the reference's stable sort (verifier.cpp:40-51).
template <class Acc>
struct TopList {
  Acc v;
  int id;
  Acc theta;  // value of entry M-1 (warp-uniform)
  __device__ __forceinline__ void reset() {
    v = neg_inf<Acc>();
    id = 0x7fffffff;
    theta = neg_inf<Acc>();
  }
  __device__ __forceinline__ bool full(int M) const {
    return __shfl_sync(0xffffffffu, id, M - 1) != 0x7fffffff;
  }
  // Warp-uniform (cv, cid). Inserts if it ranks inside the top M.
  __device__ __forceinline__ void insert(Acc cv, int cid, int M, int lane) {
    const bool beats = lane < M && (v > cv || (v == cv && id < cid));
    const int pos = __popc(__ballot_sync(0xffffffffu, beats));
    if (pos < M) {
      const Acc uv = __shfl_up_sync(0xffffffffu, v, 1);
      const int ui = __shfl_up_sync(0xffffffffu, id, 1);
      if (lane > pos && lane < M) {
        v = uv;
        id = ui;
      }
      if (lane == pos) {
        v = cv;
        id = cid;
      }
      theta = __shfl_sync(0xffffffffu, v, M - 1);
    }
  }
};

}  // namespace dsdv
