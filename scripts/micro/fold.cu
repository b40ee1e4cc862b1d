// Compute-only rate of the fused kernel's fold step (development aid): 16
// compute warps fold ring stages that stay resident in shared memory (no
// producer, no HBM), so the cycles per chunk are the compute floor of
// fold_chunk. Top-m capture is disabled (theta_run pinned at +inf, and only
// chunks >= 8 are folded, which never seed or refresh the bound).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        scripts/micro/fold.cu -o scripts/micro/fold
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

#include "../../paper_2511_11733_b200/csrc/verify.cu"

using namespace dsdv;
using namespace dsdv::fz;

template <class In, bool NEEDZ, bool FORCE_CAPTURE>
__global__ void __launch_bounds__(kThreads, 1)
    fold_bench(const In *rows, int iters, const __grid_constant__ DevParams p,
               unsigned long long *cycles, float *sink) {
  using Acc = typename InTraits<In>::Acc;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem<Acc> &sm = *reinterpret_cast<Smem<Acc> *>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int S = Smem<Acc>::kStages;
  // stage s holds rows (2s, 2s+1) of the input
  for (int i = tid; i < S * 2 * kRowBytes / 16; i += blockDim.x) {
    const int s = i / (2 * kRowBytes / 16), r = (i / (kRowBytes / 16)) & 1, q = i % (kRowBytes / 16);
    reinterpret_cast<uint4 *>(sm.ring[s][r])[q] =
        reinterpret_cast<const uint4 *>(rows)[(size_t)(2 * s + r) * (kRowBytes / 16) + q];
  }
  if (warp < kSlots) {
    reset_capture(sm.slot[warp], lane);
    if (lane < 2) sm.slot[warp].ktheta[lane] = INT_MAX;
  }
  __syncthreads();
  if (warp >= kCW) return;
  ItemState<Acc> st;
  st.reset();
  Slot<Acc> &sl = sm.slot[0];
  const SlotView sv(sl.area, p.n_chunks * kCW);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    // chunks that neither seed nor refresh the top-m bound (capture stays off)
    const int stage = it % S, c = 8 + (it & 7);
    // FORCE_CAPTURE: every block of row 0 takes the capture path (with a sort)
    if (FORCE_CAPTURE && lane == 0) sl.ktheta[0] = INT_MIN;
    fold_chunk<In, true, NEEDZ, false>(sm.ring[stage][0], sm.ring[stage][1], tid, c, st, p, warp,
                                       lane, sl, sv.bmax[0], sv.bmax[1], nullptr);
    __syncwarp();
  }
  const long long t1 = clock64();
  if (lane == 0) atomicAdd(cycles, (unsigned long long)(t1 - t0));
  if (st.st == 12345.f) sink[tid] = st.st + st.sd + st.sz;
}

int main(int argc, char **argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 4096;
  using In = __nv_bfloat16;
  constexpr int CH = kRowBytes / 2;
  const int S = Smem<float>::kStages;
  std::vector<__nv_bfloat16> h((size_t)2 * S * CH);
  srand(1);
  for (size_t i = 0; i < h.size(); i += 2) {
    // target row / draft row pairs of correlated Gaussian logits (sigma 3)
    const float u1 = (rand() + 1.f) / (RAND_MAX + 2.f), u2 = (rand() + 1.f) / (RAND_MAX + 2.f);
    const float g = sqrtf(-2.f * logf(u1)) * cosf(6.2831853f * u2) * 3.f;
    h[i] = __float2bfloat16(g);
    h[i + 1] = __float2bfloat16(g + 0.5f * sqrtf(-2.f * logf(u2)) * sinf(6.2831853f * u1));
  }
  In *d;
  unsigned long long *cyc;
  float *sink;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 4096 * 4);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  DevParams p{};
  p.B = 1;
  p.gamma = 1;
  p.V = 128256;
  p.vocab_local = 128256;
  p.stride = 128256;
  p.top_m = 10;
  p.n_chunks = (128256 + CH - 1) / CH;
  p.tau_f = 0.2f;
  p.omt_f = 0.8f;
  const size_t smem = sizeof(Smem<float>);
  for (int z = 0; z < 3; ++z) {
    auto k = z == 2 ? fold_bench<In, true, true> : z ? fold_bench<In, true, false> : fold_bench<In, false, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(cyc, 0, 8);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k<<<148, kThreads, smem>>>(d, iters, p, cyc, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double per_chunk = (double)c / (148.0 * kCW) / iters;
      // bytes a chunk stands for: two 16 KB rows
      const double gbs = 148.0 * iters * 2.0 * kRowBytes / (ms * 1e6);
      printf("{\"mode\": %d, \"cycles_per_chunk_per_warp\": %.1f, \"ms\": %.3f, \"equiv_GBps\": %.0f, \"err\": \"%s\"}\n",
             z, per_chunk, ms, gbs, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
