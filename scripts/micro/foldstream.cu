// foldstream: the overlap probe with the verifier's real fold_chunk as the
// consumer work (capture pinned off). Does streaming slow the fold? (development aid). Producer: 1 warp, 1-D bulk copies of two
// 16 KB halves per stage into an S-stage ring, a global ticket over a 1 GB
// buffer. Consumers: per stage, `work` iterations of an FFMA2 + MUFU mix
// shaped like the verifier's fold. Reports GB/s with copies, and the time of
// the same consumer work with the copies skipped (compute only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2511_11733_b200/csrc/verify.cu"
using namespace dsdv;
using namespace dsdv::fz;
__constant__ DevParams cp;

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_hint(uint64_t *b, uint32_t ph) {
  uint32_t d = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0,1,0,p; }"
                 : "=r"(d) : "r"(sa(b)), "r"(ph), "r"(0x989680u) : "memory");
  } while (!d);
}
__device__ __forceinline__ void wait(uint64_t *b, uint32_t ph) {
  uint32_t d = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                 : "=r"(d) : "r"(sa(b)), "r"(ph) : "memory");
  } while (!d);
}

__global__ void __launch_bounds__(17 * 32, 1)
    kern(const uint8_t *src, size_t total, int stages, int work, int copy, unsigned *ticket,
         float *sink, int rowwise, int vary) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int SB = 32768;
  uint64_t *full = (uint64_t *)(sm + (size_t)SB * stages);
  uint64_t *empty = full + 16;
  long long *chunk_of = (long long *)(empty + 16);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[i])), "r"(16));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t nchunks = total / SB;
  if (warp == 16) {
    if (NOSYNC) return;
    if (lane == 0) {
      int st = 0; uint32_t ph = 0;
      size_t item = 0;
      int k = 16;
      for (;;) {
        size_t c;
        if (rowwise) {
          // like the verifier: claim a row pair, stream its 16 chunks in order
          if (k == 16) { item = atomicAdd(ticket, 1u); k = 0; }
          c = item * 16 + k++;
        } else {
          c = atomicAdd(ticket, 1u);
        }
#if PRODHINT
        wait_hint(&empty[st], ph ^ 1);
#else
        wait(&empty[st], ph ^ 1);
#endif
        chunk_of[st] = c < nchunks ? (long long)c : -1;
        if (c >= nchunks) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&full[st])) : "memory");
          break;
        }
        if (copy) {
          // (expect_tx posted after the addresses are known)
          const int half = SB / 2;
          // two rows far apart, like a (draft, target) row pair
          const uint8_t *a, *b;
          uint32_t nbytes = half;
          if (rowwise == 2) {
            // the verifier's C2 layout: rows of 128256 bf16 (256512 B), target
            // [256][9] rows, draft [256][8] rows, position-major items
            const size_t it2 = item % 2304, jj = it2 / 256, bb = it2 % 256;
            const size_t RB = 256512, off = (c % 16) * (size_t)half;
            a = src + (bb * 8 + (jj < 8 ? jj : 0)) * RB + off;
            b = src + 2048 * RB + (bb * 9 + jj) * RB + off;
            if (off + half > RB) nbytes = (uint32_t)(RB - off);
          } else if (rowwise) {  // rows of 256 KB: draft row in the first half, target row in the second
            a = src + (item * 262144 + (c % 16) * half) % (total / 2);
            b = src + total / 2 + (item * 262144 + (c % 16) * half) % (total / 2);
          } else {
            a = src + (c * half) % (total / 2);
            b = src + total / 2 + (c * half) % (total / 2);
          }
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])), "r"(2 * nbytes) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + (size_t)st * SB)), "l"(a), "r"(nbytes), "r"(sa(&full[st])) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + (size_t)st * SB + half)), "l"(b), "r"(nbytes), "r"(sa(&full[st])) : "memory");
        } else {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&full[st])) : "memory");
        }
        if (++st == stages) { st = 0; ph ^= 1; }
      }
    }
    return;
  }
  int st = 0; uint32_t ph = 0;
  float acc = 0.f;
  __shared__ Slot<float> slot0;
  __shared__ int bmt[1024], bmd[1024];
  Slot<float> *sl = &slot0;
  if (lane < 2) slot0.ktheta[lane] = INT_MAX;
  ItemState<float> S;
  S.reset();
  unsigned long long p = 0x3f8000003f800000ull;
  const unsigned long long m = 0x3f7fbe773f7fbe77ull, cc = 0x3a83126f3a83126full;
#if NOSYNC
  for (int it = 0; it < 221; ++it) {
    st = it % stages;
    fold_chunk<__nv_bfloat16, true, true, false>(sm + (size_t)st * SB, sm + (size_t)st * SB + SB / 2,
                                                threadIdx.x, 8 + (it & 7), S, cp, warp, lane,
                                                *sl, bmt, bmd, nullptr);
    __syncwarp();
  }
  if (S.st == 12345.f) sink[0] = S.st + S.sd + S.sz;
  return;
#endif
#if PAIRWAIT
  // two stages per synchronisation: wait for both, fold both, release both
  for (;;) {
    const int st2 = st + 1 == stages ? 0 : st + 1;
    const uint32_t ph2 = st + 1 == stages ? ph ^ 1 : ph;
    wait(&full[st], ph);
    if (chunk_of[st] < 0) break;
    wait(&full[st2], ph2);
    const bool second = chunk_of[st2] >= 0;
    fold_chunk<__nv_bfloat16, true, true, false>(sm + (size_t)st * SB, sm + (size_t)st * SB + SB / 2,
                                                threadIdx.x, 8 + (int)(chunk_of[st] & 7), S, cp, warp, lane,
                                                *sl, bmt, bmd, nullptr);
    if (second)
      fold_chunk<__nv_bfloat16, true, true, false>(sm + (size_t)st2 * SB, sm + (size_t)st2 * SB + SB / 2,
                                                  threadIdx.x, 8 + (int)(chunk_of[st2] & 7), S, cp, warp, lane,
                                                  *sl, bmt, bmd, nullptr);
    __syncwarp();
    if (lane == 0) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st])) : "memory");
      if (second) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st2])) : "memory");
    }
    if (!second) break;
    st = st2 + 1 == stages ? 0 : st2 + 1;
    if (st2 + 1 == stages || st + 0 == 0 && st2 != stages - 1) {}
    // phase flips whenever the index wraps
    if (st == 0 || st2 == 0) ph ^= 1;
  }
  if (S.st == 12345.f) sink[0] = S.st + S.sd + S.sz;
  return;
#endif
  for (;;) {
#if CONSHINT
    wait_hint(&full[st], ph);
#else
    wait(&full[st], ph);
#endif
    if (chunk_of[st] < 0) break;
    // read the whole stage like the fold does (4 x LDS.128 per thread)
    float x = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 v = *(const uint4 *)(sm + (size_t)st * SB + (q * 512 + threadIdx.x) * 16);
      x += __uint_as_float(v.x ^ v.y ^ v.z ^ v.w) * 1e-30f;
    }
    if (work) {
      fold_chunk<__nv_bfloat16, true, true, false>(sm + (size_t)st * SB, sm + (size_t)st * SB + SB / 2,
                                                  threadIdx.x, 8 + (int)(chunk_of[st] & 7), S, cp, warp, lane,
                                                  *sl, bmt, bmd, nullptr);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st])) : "memory");
    if (++st == stages) { st = 0; ph ^= 1; }
  }
  if (S.st == 12345.f) sink[0] = S.st + S.sd + S.sz + acc + (float)p;
}

int main() {
  const size_t total = (size_t)1 << 30;
  DevParams hp{};
  hp.B = 1; hp.gamma = 1; hp.V = 128256; hp.vocab_local = 128256; hp.stride = 128256; hp.top_m = 10;
  hp.n_chunks = 16; hp.tau_f = 0.2f; hp.omt_f = 0.8f;
  cudaMemcpyToSymbol(cp, &hp, sizeof(hp));
  uint8_t *src; unsigned *ticket; float *sink;
  const size_t alloc = (size_t)(2048 + 2304) * 256512 + (1 << 20);  // the C2 rows
  cudaMalloc(&src, alloc); cudaMemset(src, 1, alloc);
  cudaMalloc(&ticket, 4); cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int works[] = {0, 1};
  for (int vary : {0})
  for (int rowwise : {2})
  for (int stages : {STAGES}) {
    const size_t smem = (size_t)32768 * stages + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int w : works) {
      float t[2];
      for (int copy = 1; copy >= 0; --copy) {
        float best = 1e9f;
        for (int rep = 0; rep < 3; ++rep) {
          cudaMemset(ticket, 0, 4);
          cudaEventRecord(e0);
          kern<<<148, 17 * 32, smem>>>(src, total, stages, w, copy, ticket, sink, rowwise, vary);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        t[copy] = best;
      }
      printf("vary %d rowwise %d stages %d work %3d: with copies %.3f ms (%6.0f GB/s), compute only %.3f ms, err=%s\n",
             vary, rowwise, stages, w, t[1], total / t[1] / 1e6, t[0], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
