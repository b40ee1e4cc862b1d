// Row-level kernels around the fused verifier:
//   * sample_extra_kernel  — the extra draw from records of dsdv_window_stats,
//     for callers that own their UniformStream (residual_distribution + sample,
//     verifier.cpp:245-246; bonus draw :253-256);
//   * draft_sample_kernel  — the draft-side step, inverse-CDF draws from
//     softmax(draft row) (draft_window, verifier.cpp:93-110);
//   * synth_logits_kernel  — seeded benchmark/test inputs.
#include <cuda_runtime.h>

#include "common.cuh"
#include "sample.cuh"
#include "dsdv/synth.h"

namespace dsdv {

struct RowsSmem {
  SampleShared samp;
  double red_m[kConsumerWarps], red_s[kConsumerWarps];
};

template <class In>
__global__ void __launch_bounds__(kConsumerThreads)
    sample_extra_kernel(const __grid_constant__ DevParams p, const In *__restrict__ draft,
                        const In *__restrict__ target, const double *__restrict__ records,
                        const int32_t *__restrict__ position, const double *__restrict__ uniform,
                        int32_t *__restrict__ token_out, int32_t *__restrict__ status) {
  using Acc = typename InTraits<In>::Acc;
  __shared__ RowsSmem sm;
  __shared__ Weigher<Acc> wf;
  __shared__ int skip;
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  const int G1 = p.gamma + 1;
  const int j = position[b];
  if (tid == 0) {
    skip = 0;
    if (j < 0 || j > p.gamma) {
      token_out[b] = -1;
      status[b] = DSDV_E_INVARIANT;
      skip = 1;
    } else {
      const double *r = records + ((size_t)b * G1 + j) * kRecordWords;
      const int flags = (int)r[kRecFlags];
      const int kind = flags & 0xff, err = (flags >> 8) & 0xff;
      PosEval ev;
      ev.mt = r[kRecMt];
      ev.lst = r[kRecLst];
      ev.md = r[kRecMd];
      ev.lsd = r[kRecLsd];
      ev.lsz = r[kRecLsz];
      if (err) {
        token_out[b] = -1;
        status[b] = err;
        skip = 1;
      } else if (j == p.gamma) {
        set_weigher(wf, kWeightPlain, ev, (double)p.omt_f, (double)p.tau_f);
      } else if (kind == DSDV_EFF_DRAFT) {
        token_out[b] = -1;
        status[b] = DSDV_E_EMPTY_RESIDUAL;
        skip = 1;
      } else {
        set_weigher(wf, kind == DSDV_EFF_SOFTENED ? kWeightResSoft : kWeightResTarget, ev,
                    (double)p.omt_f, (double)p.tau_f);
      }
    }
  }
  __syncthreads();
  if (skip) return;
  const In *rt = target + ((size_t)b * G1 + j) * (size_t)p.stride;
  const In *rd = draft + ((size_t)b * p.gamma + (j < p.gamma ? j : 0)) * (size_t)p.stride;
  int near = 0;
  const int idx = cdf_sample<In, Acc>(rt, rd, wf, p.vocab_local, uniform[b], p.eps_u, &sm.samp,
                                      tid, &near);
  if (tid == 0) {
    if (idx < 0) {
      token_out[b] = -1;
      status[b] = DSDV_E_EMPTY_RESIDUAL;
    } else {
      token_out[b] = p.vocab_offset + idx;
      status[b] = DSDV_OK;
    }
  }
}

template <class In>
__global__ void __launch_bounds__(kConsumerThreads)
    draft_sample_kernel(const __grid_constant__ DevParams p, const In *__restrict__ draft,
                        int32_t *__restrict__ tokens, double temperature) {
  using Acc = typename InTraits<In>::Acc;
  constexpr int VEC = InTraits<In>::kVec;
  __shared__ RowsSmem sm;
  __shared__ Weigher<Acc> wf;
  const int row = blockIdx.x;  // b * gamma + j
  const int b = row / p.gamma, j = row - b * p.gamma;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const In *rd = draft + (size_t)row * p.stride;
  const Acc ni = neg_inf<Acc>();
  // temperature_scale (distribution.cpp:65-97): T = 1 identity, T = 0 one-hot
  // at the argmax (lowest id on ties), else p^(1/T) = softmax(l / T)
  const bool argmax = temperature == 0.0;
  const Acc it = (argmax || temperature == 1.0) ? Acc(1) : Acc(1.0 / temperature);
  const Acc itL = it * log2e<Acc>();
  Acc m = ni, s = Acc(0);
  int am = 0x7fffffff;  // argmax id (T = 0)
  const int nvec = (p.vocab_local + VEC - 1) / VEC;
  for (int q = tid; q < nvec; q += kConsumerThreads) {
    Acc v[VEC];
    unpack(ldg128(rd + (size_t)q * VEC), v, (In *)nullptr);
    Acc cm = ni;
    int ci = 0x7fffffff;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      if (q * VEC + e >= p.vocab_local) v[e] = ni;
      if (v[e] > cm) {  // strict: the lowest id keeps ties
        cm = v[e];
        ci = q * VEC + e;
      }
    }
    if (cm > m || (cm == m && ci < am)) am = ci;
    Acc cs = Acc(0);
    if (cm != ni) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) cs += fast_exp2((v[e] - cm) * itL);
    }
    // running (max, sum of exp((v - max) / T))
    if (cm > m) {
      s = (m == ni ? Acc(0) : s * fast_exp2((m - cm) * itL)) + cs;
      m = cm;
    } else if (cm != ni) {
      s += cs * fast_exp2((cm - m) * itL);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const Acc m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const Acc s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const int a2 = __shfl_xor_sync(0xffffffffu, am, o);
    if (m2 > m || (m2 == m && a2 < am)) am = a2;
    if (m2 > m) {
      s = (m == ni ? Acc(0) : s * fast_exp2((m - m2) * itL)) + s2;
      m = m2;
    } else if (m2 != ni) {
      s += s2 * fast_exp2((m2 - m) * itL);
    }
  }
  __shared__ int red_a[kConsumerWarps];
  if (lane == 0) {
    sm.red_m[warp] = (double)m;
    sm.red_s[warp] = (double)s;
    red_a[warp] = am;
  }
  __syncthreads();
  if (argmax) {
    if (tid == 0) {
      double M = sm.red_m[0];
      int A = red_a[0];
      for (int w = 1; w < kConsumerWarps; ++w)
        if (sm.red_m[w] > M || (sm.red_m[w] == M && red_a[w] < A)) {
          M = sm.red_m[w];
          A = red_a[w];
        }
      tokens[row] = (M == -INFINITY || A == 0x7fffffff) ? -1 : p.vocab_offset + A;
    }
    return;
  }
  if (tid == 0) {
    double M = sm.red_m[0], S = sm.red_s[0];
    for (int w = 1; w < kConsumerWarps; ++w) {
      const double m2 = sm.red_m[w], s2 = sm.red_s[w];
      if (m2 == -INFINITY) continue;
      if (m2 > M) {
        S = (M == -INFINITY ? 0.0 : S * exp((M - m2) * (double)it)) + s2;
        M = m2;
      } else {
        S += s2 * exp((m2 - M) * (double)it);
      }
    }
    PosEval ev;
    ev.mt = M;  // a row element: exact in Acc, so no rounding correction is scaled
    ev.lst = log(S);
    ev.md = ev.lsd = ev.lsz = 0.0;
    set_weigher(wf, kWeightPlain, ev, (double)p.omt_f, (double)p.tau_f);
    wf.itemp = it;
    wf.itL = (float)((double)it * kLog2e);
  }
  __syncthreads();
  const double u = dsdv_philox_uniform(p.seed, p.window, p.seq_offset + (uint32_t)b, (uint32_t)j);
  int near = 0;
  const int idx = cdf_sample<In, Acc>(rd, rd, wf, p.vocab_local, u, p.eps_u, &sm.samp, tid, &near);
  if (tid == 0) tokens[row] = idx < 0 ? -1 : p.vocab_offset + idx;
}

// ------------------------------------------------------------------ synth
template <class Out>
__device__ __forceinline__ Out to_out(float x);
template <>
__device__ __forceinline__ float to_out<float>(float x) {
  return x;
}
template <>
__device__ __forceinline__ __nv_bfloat16 to_out<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// Families by b mod 4; the element arithmetic lives in
// include/dsdv/synth.h, shared bit for bit with the host generator the CPU
// reference arm uses (oracle/dsd_oracle.c oracle_synth_logits).
template <class Out>
__global__ void __launch_bounds__(256)
    synth_logits_kernel(int B, int gamma, int V, int stride, uint64_t seed, Out *__restrict__ draft,
                        Out *__restrict__ target) {
  const int G1 = gamma + 1;
  const int item = blockIdx.x;  // b * (gamma + 1) + j
  const int b = item / G1, j = item - b * G1;
  const dsdv_synth_row rp = dsdv_synth_row_params(seed, (uint32_t)item, b, V);
  Out *rt = target + (size_t)item * stride;
  Out *rd = (j < gamma) ? draft + ((size_t)b * gamma + j) * stride : nullptr;
  const Out ninf = to_out<Out>(-INFINITY);
  for (int i = threadIdx.x; i < stride; i += blockDim.x) {
    if (i >= V) {
      rt[i] = ninf;
      if (rd) rd[i] = ninf;
      continue;
    }
    float lt, z1;
    dsdv_synth_element(seed, (uint32_t)item, &rp, V, i, &lt, &z1);
    // round the target first so that draft = stored target + noise
    const Out lt_o = to_out<Out>(lt);
    rt[i] = lt_o;
    if (rd) rd[i] = to_out<Out>(dsdv_synth_draft((float)lt_o, rp.delta, z1));
  }
}

// ------------------------------------------------------------------ launch
template <class In>
cudaError_t launch_sample_extra(const DevParams &p, const void *draft, const void *target,
                                const double *records, const int32_t *position,
                                const double *uniform, int32_t *token_out, int32_t *status,
                                cudaStream_t stream) {
  sample_extra_kernel<In><<<p.B, kConsumerThreads, 0, stream>>>(
      p, (const In *)draft, (const In *)target, records, position, uniform, token_out, status);
  return cudaGetLastError();
}

template <class In>
cudaError_t launch_draft_sample(const DevParams &p, const void *draft, int32_t *tokens,
                                double temperature, cudaStream_t stream) {
  draft_sample_kernel<In><<<p.B * p.gamma, kConsumerThreads, 0, stream>>>(p, (const In *)draft,
                                                                          tokens, temperature);
  return cudaGetLastError();
}

cudaError_t launch_synth(int dtype, int B, int gamma, int V, int stride, uint64_t seed, void *draft,
                         void *target, cudaStream_t stream) {
  const int grid = B * (gamma + 1);
  if (dtype == DSDV_DTYPE_BF16)
    synth_logits_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(
        B, gamma, V, stride, seed, (__nv_bfloat16 *)draft, (__nv_bfloat16 *)target);
  else
    synth_logits_kernel<float><<<grid, 256, 0, stream>>>(B, gamma, V, stride, seed, (float *)draft,
                                                          (float *)target);
  return cudaGetLastError();
}

// Whole-row mixture of two fp64 probability vectors (the drop-in soften,
// verifier.cpp:161-186, and residual_distribution, :198-213): w_i =
// a_i^(1-tau) b_i^tau (kind 0) or max(0, a_i - b_i) (kind 1), then w / sum(w)
// (Distribution::from_weights, distribution.cpp:54-63). One CTA; status is the
// error the reference throws when the mass is zero.
__global__ void __launch_bounds__(1024) mix_rows_kernel(int kind, int V, const double *a,
                                                         const double *b, double tau,
                                                         double *out, int32_t *status) {
  __shared__ double part[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const double w = kind == 0 ? pow(a[i], 1.0 - tau) * pow(b[i], tau) : fmax(0.0, a[i] - b[i]);
    out[i] = w;
    s += w;
  }
  s = warp_sum_f64(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
    t = warp_sum_f64(t);
    if (threadIdx.x == 0) part[0] = t;
  }
  __syncthreads();
  const double total = part[0];
  if (!(total > 0.0)) {
    if (threadIdx.x == 0)
      *status = kind == 0 ? DSDV_E_DEGENERATE_MIXTURE : DSDV_E_EMPTY_RESIDUAL;
    return;
  }
  for (int i = threadIdx.x; i < V; i += blockDim.x) out[i] /= total;
  if (threadIdx.x == 0) *status = DSDV_OK;
}

// In-place natural log of fp64 probability rows (the drop-in's Distribution
// rows become the logit rows the fused kernel folds: softmax(log p) = p);
// zero probabilities become -inf.
__global__ void log_rows_kernel(double *x, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    x[i] = v > 0.0 ? log(v) : -INFINITY;
  }
}

cudaError_t launch_log_rows(double *x, size_t n, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  size_t blocks = (n + 255) / 256;
  if (blocks > 4 * 148) blocks = 4 * 148;
  log_rows_kernel<<<(unsigned)blocks, 256, 0, stream>>>(x, n);
  return cudaGetLastError();
}


// Pipeline emulation: one thread holds the stream for `ns`
// nanoseconds of %globaltimer — a stage's compute step t0 or a link's
// injected latency t1.
__global__ void spin_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

cudaError_t launch_spin(unsigned long long ns, cudaStream_t stream) {
  spin_kernel<<<1, 1, 0, stream>>>(ns);
  return cudaGetLastError();
}

cudaError_t launch_mix_rows(int kind, int V, const double *a, const double *b, double tau,
                            double *out, int32_t *status, cudaStream_t stream) {
  mix_rows_kernel<<<1, 1024, 0, stream>>>(kind, V, a, b, tau, out, status);
  return cudaGetLastError();
}

#define DSDV_INST(T)                                                                             \
  template cudaError_t launch_sample_extra<T>(const DevParams &, const void *, const void *,     \
                                              const double *, const int32_t *, const double *,  \
                                              int32_t *, int32_t *, cudaStream_t);               \
  template cudaError_t launch_draft_sample<T>(const DevParams &, const void *, int32_t *,        \
                                              double, cudaStream_t);
DSDV_INST(__nv_bfloat16)
DSDV_INST(float)
DSDV_INST(double)
#undef DSDV_INST

}  // namespace dsdv
