// Complex running-product throughput probe (the local-energy phase-2 inner
// step): per row, u = tv * tau (complex), P += P * u, for ST independent
// products per thread; W warps per CTA, B CTAs per SM.  Reports FP64 lane-ops
// per SM clock (8 per factor) against the 64/clk peak.
#include <cstdio>
template <int ST>
__global__ void k(double* out, long long* cyc, int rows, double s) {
  double px[ST], py[ST], tx[ST], ty[ST];
#pragma unroll
  for (int j = 0; j < ST; ++j) { px[j] = 1.0; py[j] = 0.0; tx[j] = s * (j + 1); ty[j] = s * 0.5 * j; }
  double ax = s * threadIdx.x, ay = s;
  long long t0 = clock64();
#pragma unroll 2
  for (int r = 0; r < rows; ++r) {
#pragma unroll
    for (int j = 0; j < ST; ++j) {
      const double ux = fma(tx[j], ax, -ty[j] * ay), uy = fma(tx[j], ay, ty[j] * ax);
      const double x = px[j], y = py[j];
      px[j] = fma(x, ux, fma(-y, uy, x));
      py[j] = fma(x, uy, fma(y, ux, y));
    }
    ax = ax * 0.999;  // keep tau changing (one extra op per row)
  }
  long long t1 = clock64();
  double acc = 0;
#pragma unroll
  for (int j = 0; j < ST; ++j) acc += px[j] + py[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int ST> void run(int warps, int bps, double* out, long long* cyc, int nsm) {
  const int rows = 2000;
  k<ST><<<nsm * bps, warps * 32>>>(out, cyc, rows, 1e-3);
  k<ST><<<nsm * bps, warps * 32>>>(out, cyc, rows, 1e-3);
  cudaDeviceSynchronize();
  static long long h[4096];
  cudaMemcpy(h, cyc, nsm * bps * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < nsm * bps; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("ST=%d warps/CTA=%2d CTAs/SM=%d: %6.2f FP64 lane-ops/clk/SM\n", ST, warps, bps,
         (8.0 * ST + 1) * 32.0 * warps * bps * rows / mx);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out; long long* cyc; cudaMalloc(&out, nsm * 4 * 1024 * 8); cudaMalloc(&cyc, nsm * 4 * 8);
  for (int w : {8, 13, 16}) for (int b : {1, 2}) { run<2>(w, b, out, cyc, nsm); run<4>(w, b, out, cyc, nsm); run<8>(w, b, out, cyc, nsm); }
  return 0;
}
