// FP64 latency / ILP probe: each thread runs K independent DFMA chains; one CTA
// of W warps per SM.  Reports DFMA lane-ops per SM clock.
#include <cstdio>
template <int K>
__global__ void k(double* out, long long* cyc, double s) {
  double a[K];
#pragma unroll
  for (int j = 0; j < K; ++j) a[j] = s * (threadIdx.x + j);
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 4096; ++it) {
#pragma unroll
    for (int j = 0; j < K; ++j) a[j] = fma(a[j], 0.999999, 1e-9);
  }
  long long t1 = clock64();
  double r = 0;
#pragma unroll
  for (int j = 0; j < K; ++j) r += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int K> void run(int warps, double* out, long long* cyc, int nsm) {
  k<K><<<nsm, warps * 32>>>(out, cyc, 1.0);
  k<K><<<nsm, warps * 32>>>(out, cyc, 1.0);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, cyc, nsm * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("K=%2d warps/SM=%2d: %6.2f DFMA lanes/clk/SM, %6.1f cyc per dependent DFMA\n", K, warps,
         32.0 * warps * K * 4096 / mx, mx / 4096.0);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out; long long* cyc; cudaMalloc(&out, nsm * 1024 * 8); cudaMalloc(&cyc, nsm * 8);
  for (int w : {1, 4, 8, 16}) { run<1>(w, out, cyc, nsm); run<2>(w, out, cyc, nsm); run<4>(w, out, cyc, nsm); run<8>(w, out, cyc, nsm); run<16>(w, out, cyc, nsm); }
  return 0;
}
