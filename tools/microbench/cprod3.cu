// FP64 throughput of the local-energy product recurrence with everything in
// registers: isolates the arithmetic pattern from the shared-memory loads.
// Reports FP64 lane-ops per SM clock (peak 64).
#include <cstdio>
template <int MODE, int ST>
__global__ void __launch_bounds__(448, 2) k(double* out, long long* cyc, int rows, double seed) {
  double2 P[ST], tv[ST];
  double a[8], b[8], c[8];
#pragma unroll
  for (int j = 0; j < ST; ++j) { P[j] = make_double2(1.0, 0.0); tv[j] = make_double2(seed * (j + 1), seed * 0.5 * j); }
#pragma unroll
  for (int j = 0; j < 8; ++j) { a[j] = seed * j; b[j] = 1.0 - seed * j; c[j] = seed * 0.25 * j; }
  double2 tau0 = make_double2(seed * threadIdx.x, seed), tau1 = make_double2(seed, -seed * threadIdx.x);
  long long t0 = clock64();
#pragma unroll 1
  for (int r = 0; r < rows; ++r) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double2 tau = h ? tau1 : tau0;
      asm volatile("" : "+d"(tau.x), "+d"(tau.y));
#pragma unroll
      for (int j = 0; j < ST; ++j) asm volatile("" : "+d"(tv[j].x), "+d"(tv[j].y));
      if (MODE == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fma(b[j], c[j], a[j]);
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = fma(b[j], c[j], c[j]);
        // 16 DFMA per h
      } else {
#pragma unroll
        for (int j = 0; j < ST; ++j) {
          const double ux = fma(tv[j].x, tau.x, -tv[j].y * tau.y), uy = fma(tv[j].x, tau.y, tv[j].y * tau.x);
          const double px = P[j].x, py = P[j].y;
          if (MODE == 1) {
            P[j].x = fma(px, ux, fma(-py, uy, px));
            P[j].y = fma(px, uy, fma(py, ux, py));
          } else if (MODE == 2) {  // (1 + u) explicitly
            const double fx = 1.0 + ux;
            P[j].x = fma(px, fx, -py * uy);
            P[j].y = fma(px, uy, py * fx);
          } else if (MODE == 3) {  // P += P u with products first
            const double m1 = py * uy, m2 = py * ux;
            P[j].x = fma(px, ux, px - m1);
            P[j].y = fma(px, uy, py + m2);
          }
        }
        if (MODE == 4) {
#pragma unroll
          for (int j = 0; j < ST; ++j) {  // u only (4 FP64)
            tv[j].x = fma(tv[j].x, tau.x, -tv[j].y * tau.y);
            tv[j].y = fma(tv[j].x, tau.y, tv[j].y * tau.x);
          }
        }
      }
    }
  }
  long long t1 = clock64();
  double acc = 0;
#pragma unroll
  for (int j = 0; j < ST; ++j) acc += P[j].x + P[j].y + tv[j].x;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += a[j] + c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE, int ST>
void run(const char* name, int nsm, double* out, long long* cyc, int bps, int threads) {
  const int rows = 2000;
  k<MODE, ST><<<nsm * bps, threads>>>(out, cyc, rows, 1e-9);
  k<MODE, ST><<<nsm * bps, threads>>>(out, cyc, rows, 1e-9);
  cudaError_t e = cudaDeviceSynchronize();
  static long long h[4096];
  cudaMemcpy(h, cyc, nsm * bps * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < nsm * bps; ++i) mx = h[i] > mx ? h[i] : mx;
  const double per = MODE == 0 ? 32.0 : (MODE == 4 ? 8.0 * ST : (MODE == 2 ? 9.0 * ST : 16.0 * ST));  // per row (2 h)
  printf("%-34s ST=%d threads=%d CTAs/SM=%d err=%d: %6.2f FP64 lane-ops/clk/SM\n", name, ST, threads, bps, (int)e,
         per * threads * bps * rows / mx);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out; long long* cyc; cudaMalloc(&out, nsm * 4 * 1024 * 8); cudaMalloc(&cyc, nsm * 4 * 8);
  // (the complex-recurrence modes are measured with their shared-memory loads in cprod2.cu)
  run<0, 4>("16 independent DFMA chains", nsm, out, cyc, 2, 416);
  run<0, 4>("16 independent DFMA chains", nsm, out, cyc, 1, 1024);
  run<0, 4>("16 independent DFMA chains", nsm, out, cyc, 4, 256);
  return 0;
}
