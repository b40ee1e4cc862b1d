// Pipe rates of the integer / min-max instructions the fold uses, alone and
// mixed with FFMA2 / MUFU (development aid). warp-instr per clock per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void bench(unsigned *out, int iters, long long *cycles) {
  unsigned u[8];
  float f[8];
  unsigned long long p[8];
  for (int i = 0; i < 8; ++i) {
    u[i] = threadIdx.x * 2654435761u + i;
    f[i] = threadIdx.x * 1e-7f + i;
    p[i] = ((unsigned long long)__float_as_uint(f[i] + 1) << 32) | __float_as_uint(f[i]);
  }
  const unsigned long long m = 0x3f7fbe773f7fbe77ull, c = 0x3a83126f3a83126full;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("prmt.b32 %0, %0, 0, 0x1044;" : "+r"(u[i]));
      if (MODE == 1) asm volatile("lop3.b32 %0, %0, 0xffff0000, 0x12345, 0xea;" : "+r"(u[i]));
      if (MODE == 2) asm volatile("max.f32 %0, %0, 0fC2FE0000;" : "+f"(f[i]));
      if (MODE == 3) asm volatile("max.f32 %0, %0, %1, 0fC2FE0000;" : "+f"(f[i]) : "f"(f[(i + 1) & 7]));
      if (MODE == 4) asm volatile("mad.lo.u32 %0, %0, 8388608, 12345;" : "+r"(u[i]));
      if (MODE == 5) asm volatile("mad.lo.u32 %0, %0, 8388609, 12345;" : "+r"(u[i]));
      if (MODE == 6) asm volatile("shl.b32 %0, %0, 16;" : "+r"(u[i]));
      if (MODE == 7) {
        asm volatile("prmt.b32 %0, %0, 0, 0x1044;" : "+r"(u[i]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(m), "l"(c));
      }
      if (MODE == 8) {
        asm volatile("mad.lo.u32 %0, %0, 8388609, 12345;" : "+r"(u[i]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(m), "l"(c));
      }
      if (MODE == 9) {
        asm volatile("prmt.b32 %0, %0, 0, 0x1044;" : "+r"(u[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      }
      if (MODE == 10) {
        asm volatile("prmt.b32 %0, %0, 0, 0x1044;" : "+r"(u[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(m), "l"(c));
      }
      if (MODE == 11) asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, 0f3A83126F;" : "+f"(f[i]));
      if (MODE == 12) {
        asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, 0f3A83126F;" : "+f"(f[i]));
        asm volatile("prmt.b32 %0, %0, 0, 0x1044;" : "+r"(u[i]));
      }
    }
  }
  long long t1 = clock64();
  unsigned s = 0;
  for (int i = 0; i < 8; ++i) s += u[i] + __float_as_uint(f[i]) + (unsigned)p[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int M>
void run(const char *name, unsigned *out, long long *cyc, int ops_per_iter) {
  const int blocks = 148, threads = 1024, iters = 2048;
  for (int rep = 0; rep < 2; ++rep) {
    bench<M><<<blocks, threads>>>(out, iters, cyc);
    cudaDeviceSynchronize();
  }
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double wi = (double)(threads / 32) * iters * 8 * ops_per_iter;
  printf("%-22s %7.3f warp-instr/clk/SM\n", name, wi / c);
}

int main() {
  unsigned *out;
  long long *cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  run<0>("PRMT", out, cyc, 1);
  run<1>("LOP3", out, cyc, 1);
  run<2>("FMNMX", out, cyc, 1);
  run<3>("FMNMX3", out, cyc, 1);
  run<4>("IMAD x 2^23 (LEA?)", out, cyc, 1);
  run<5>("IMAD", out, cyc, 1);
  run<6>("SHL", out, cyc, 1);
  run<7>("PRMT+FFMA2", out, cyc, 2);
  run<8>("IMAD+FFMA2", out, cyc, 2);
  run<9>("PRMT+MUFU", out, cyc, 2);
  run<10>("PRMT+MUFU+FFMA2", out, cyc, 3);
  run<11>("FFMA", out, cyc, 1);
  run<12>("FFMA+PRMT", out, cyc, 2);
  return 0;
}
