// Instruction-throughput microbenchmark for the ops the fused MH sweep uses.
// One CTA of 1024 threads per SM, 8 independent dependency chains per thread;
// reports lane-ops per SM clock (clock64 inside the CTA).
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

#define ITERS 2048
#define CH 8

template <int OP>
__global__ void bench(float* out, long long* cyc, float seed) {
  float f[CH]; double d[CH]; unsigned u[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) { f[j] = seed * (threadIdx.x + j + 1) * 1e-3f; d[j] = f[j]; u[j] = threadIdx.x * 7 + j; }
  __shared__ float4 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[j]));
      if (OP == 1) asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(f[j]));
      if (OP == 2) asm volatile("cos.approx.ftz.f32 %0, %0;" : "+f"(f[j]));
      if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f[j]));
      if (OP == 4) { unsigned short h = (unsigned short)u[j]; asm volatile("fma.rn.f32.f16 %0, %1, %1, %0;" : "+f"(f[j]) : "h"(h)); }
      if (OP == 5) { unsigned r; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f[j]), "f"(f[(j+1)%CH])); f[j] = __uint_as_float(r); }
      if (OP == 6) { unsigned short h = (unsigned short)__float_as_uint(f[j]); asm volatile("cvt.f32.f16 %0, %1;" : "=f"(f[j]) : "h"(h)); }
      if (OP == 7) { float r; asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(r) : "d"(d[j])); d[j] = (double)__float_as_uint(r); }
      if (OP == 8) { unsigned short r; asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(r) : "d"(d[j])); d[j] += r; }
      if (OP == 9) asm volatile("add.rn.f64 %0, %0, %0;" : "+d"(d[j]));
      if (OP == 10) asm volatile("fma.rn.f64 %0, %0, %0, %0;" : "+d"(d[j]));
      if (OP == 11) { float r; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(r) : "r"(u[j])); u[j] = __float_as_uint(r); }
      if (OP == 12) asm volatile("mad.lo.u32 %0, %0, %0, %0;" : "+r"(u[j]));
      if (OP == 13) { float4 v = sm[(u[j] + it) & 2047]; f[j] += v.x; u[j] += 1; }
      if (OP == 14) { float2 v = reinterpret_cast<float2*>(sm)[(u[j] + it) & 4095]; f[j] += v.x; u[j] += 1; }
      if (OP == 15) f[j] = __shfl_xor_sync(0xffffffffu, f[j], 1);
      if (OP == 16) asm volatile("add.rn.f32 %0, %0, %0;" : "+f"(f[j]));
      if (OP == 17) { unsigned r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f[j]), "f"(f[(j+1)%CH])); f[j] = __uint_as_float(r); }
      if (OP == 18) { float r; asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(r) : "d"(d[j])); d[j] = r; }
      if (OP == 19) asm volatile("sin.approx.ftz.f32 %0, %0;" : "+f"(f[j]));
      if (OP == 20) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(f[j]));
      if (OP == 22) { int r; asm volatile("cvt.rni.s32.f32 %0, %1;" : "=r"(r) : "f"(f[j])); f[j] = __int_as_float(r); }
      if (OP == 23) { unsigned short h = (unsigned short)u[j]; asm volatile("fma.rn.f32.bf16 %0, %1, %1, %0;" : "+f"(f[j]) : "h"(h)); }
      if (OP == 24) { int r; asm volatile("cvt.rzi.s32.f32 %0, %1;" : "=r"(r) : "f"(f[j] * 1.5f)); f[j] = __int_as_float(r); }
      if (OP == 25) { double r; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(r) : "f"(f[j])); f[j] = (float)__double2loint(r) + f[j]; }
      if (OP == 26) { double r; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(r) : "f"(f[j])); d[j] += r; }
      if (OP == 21) { unsigned long long z = ((unsigned long long)u[j] << 32) | u[(j+1)%CH]; z *= 0xBF58476D1CE4E5B9ull; u[j] = (unsigned)(z >> 29); }
    }
  }
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < CH; ++j) s += f[j] + (float)d[j] + u[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP> void run(const char* name, float* out, long long* cyc, int nsm) {
  bench<OP><<<nsm, 1024>>>(out, cyc, 1.0f);
  bench<OP><<<nsm, 1024>>>(out, cyc, 1.0f);
  cudaDeviceSynchronize();
  long long h[1024]; cudaMemcpy(h, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
  double ops = 1024.0 * ITERS * CH;
  printf("%-28s %8.2f lane-ops/clk/SM\n", name, ops / mx);
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* cyc; cudaMalloc(&out, nsm * 1024 * 4); cudaMalloc(&cyc, nsm * 8);
  run<0>("ex2.approx.ftz.f32", out, cyc, nsm);
  run<1>("lg2.approx.ftz.f32", out, cyc, nsm);
  run<2>("cos.approx.ftz.f32", out, cyc, nsm);
  run<19>("sin.approx.ftz.f32", out, cyc, nsm);
  run<20>("rcp.approx.ftz.f32", out, cyc, nsm);
  run<3>("fma.rn.f32 (3-reg)", out, cyc, nsm);
  run<16>("add.rn.f32", out, cyc, nsm);
  run<4>("fma.rn.f32.f16 (mixed)", out, cyc, nsm);
  run<5>("cvt.rn.f16x2.f32 (pack)", out, cyc, nsm);
  run<17>("cvt.rn.bf16x2.f32 (pack)", out, cyc, nsm);
  run<6>("cvt.f32.f16 (unpack)", out, cyc, nsm);
  run<7>("cvt.rn.f32.f64", out, cyc, nsm);
  run<18>("cvt.rn.f32.f64 + cvt.f64.f32", out, cyc, nsm);
  run<8>("cvt.rn.f16.f64", out, cyc, nsm);
  run<9>("add.rn.f64", out, cyc, nsm);
  run<10>("fma.rn.f64", out, cyc, nsm);
  run<11>("cvt.rn.f32.s32", out, cyc, nsm);
  run<12>("mad.lo.u32", out, cyc, nsm);
  run<22>("cvt.rni.s32.f32", out, cyc, nsm);
  run<24>("fmul + cvt.rzi.s32.f32", out, cyc, nsm);
  run<23>("fma.rn.f32.bf16 (mixed)", out, cyc, nsm);
  run<26>("cvt.f64.f32 (+ dadd)", out, cyc, nsm);
  run<21>("u64 mul (splitmix step)", out, cyc, nsm);
  run<13>("lds.128", out, cyc, nsm);
  run<14>("lds.64", out, cyc, nsm);
  run<15>("shfl.bfly", out, cyc, nsm);
  cudaError_t e = cudaGetLastError(); printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
