// Pipe-throughput microbenchmark (development aid): FFMA vs FFMA2 vs MUFU.EX2
// vs FADD2, warp-instructions per clock per SM, on the B200 box.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2(float a, float b) {
  return ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(a);
}

template <int MODE>
__global__ void bench(float *out, int iters, long long *cycles) {
  float a[8];
  unsigned long long p[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-7f + i; p[i] = f2(a[i], a[i] + 1); }
  const unsigned long long m = f2(0.999f, 0.998f), c = f2(1e-3f, 2e-3f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = fmaf(a[i], 0.999f, 1e-3f);
      if (MODE == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(m), "l"(c));
      if (MODE == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (MODE == 3) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(c));
      if (MODE == 4) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
                       asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(m), "l"(c)); }
      if (MODE == 5) a[i] = a[i] * 0.999f + 1e-3f;  // FFMA immediate form
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float((unsigned)p[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
  float *out; long long *cyc;
  const int blocks = 148, threads = 1024, iters = 4096;
  cudaMalloc(&out, blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  const char *names[] = {"FFMA", "FFMA2", "MUFU.EX2", "FADD2", "MUFU+FFMA2", "FFMA-imm"};
  for (int mode = 0; mode < 6; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (mode) {
        case 0: bench<0><<<blocks, threads>>>(out, iters, cyc); break;
        case 1: bench<1><<<blocks, threads>>>(out, iters, cyc); break;
        case 2: bench<2><<<blocks, threads>>>(out, iters, cyc); break;
        case 3: bench<3><<<blocks, threads>>>(out, iters, cyc); break;
        case 4: bench<4><<<blocks, threads>>>(out, iters, cyc); break;
        case 5: bench<5><<<blocks, threads>>>(out, iters, cyc); break;
      }
      cudaDeviceSynchronize();
    }
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double warp_instr = (double)(threads / 32) * iters * 8;  // per SM (1 block per SM)
    printf("%-12s %8.3f warp-instr/clk/SM  (%lld cycles)\n", names[mode], warp_instr / c, c);
  }
  return 0;
}
