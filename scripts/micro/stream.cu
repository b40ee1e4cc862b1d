// Bulk-copy (TMA 1-D) streaming capacity per SM (development aid): one CTA per
// SM, one producer lane, NC consumer warps that only wait/arrive. Reports GB/s
// for a sweep of (stage bytes, stages).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t *b, uint32_t ph) {
  uint32_t d = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                 : "=r"(d) : "r"(sa(b)), "r"(ph) : "memory");
  } while (!d);
}

template <int NC>
__global__ void stream(const uint8_t *src, size_t total, int stage_bytes, int stages,
                       unsigned *ticket, float *sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t *full = (uint64_t *)(sm + (size_t)stage_bytes * stages);
  uint64_t *empty = full + 16;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[i])), "r"(NC));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t nchunks = total / stage_bytes;
  __shared__ long long chunk_of[16];
  if (warp == NC) {
    if (lane == 0) {
      int st = 0; uint32_t ph = 0;
      for (;;) {
        const size_t c = atomicAdd(ticket, 1u);
        wait(&empty[st], ph ^ 1);
        chunk_of[st] = c < nchunks ? (long long)c : -1;
        if (c >= nchunks) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&full[st])) : "memory");
          break;
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])), "r"(stage_bytes) : "memory");
        // two half copies (like a row pair)
        const int half = stage_bytes / 2;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + (size_t)st * stage_bytes)), "l"(src + c * stage_bytes), "r"(half), "r"(sa(&full[st])) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + (size_t)st * stage_bytes + half)), "l"(src + c * stage_bytes + half), "r"(half), "r"(sa(&full[st])) : "memory");
        if (++st == stages) { st = 0; ph ^= 1; }
      }
    }
    return;
  }
  int st = 0; uint32_t ph = 0;
  float acc = 0.f;
  for (;;) {
    wait(&full[st], ph);
    if (chunk_of[st] < 0) break;
    acc += (float)sm[(size_t)st * stage_bytes + threadIdx.x * 4];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st])) : "memory");
    if (++st == stages) { st = 0; ph ^= 1; }
  }
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  const size_t total = (size_t)1 << 30;
  uint8_t *src; unsigned *ticket; float *sink;
  cudaMalloc(&src, total); cudaMemset(src, 1, total);
  cudaMalloc(&ticket, 4); cudaMalloc(&sink, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int cfg[][2] = {{16384, 4}, {16384, 8}, {32768, 4}, {32768, 6}, {65536, 3}, {8192, 16}, {16384, 12}};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto &c : cfg) {
    const int sb = c[0], ns = c[1];
    const size_t smem = (size_t)sb * ns + 512;
    cudaFuncSetAttribute(stream<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(ticket, 0, 4);
      cudaEventRecord(e0);
      stream<8><<<sms, 9 * 32, smem>>>(src, total, sb, ns, ticket, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("stage %6d B x %2d stages (%4zu KB in flight/SM): %7.1f GB/s  err=%s\n", sb, ns,
           (size_t)sb * ns / 1024, total / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
