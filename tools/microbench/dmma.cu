// DMMA (mma.sync m8n8k4 f64) throughput probe vs DFMA: K independent
// accumulator tiles per warp, W warps per SM.
#include <cstdio>
template <int K>
__global__ void k(double* out, long long* cyc, double s) {
  double c[K][2];
  double a = s * threadIdx.x, b = s + threadIdx.x;
#pragma unroll
  for (int j = 0; j < K; ++j) c[j][0] = c[j][1] = j;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 2048; ++it) {
#pragma unroll
    for (int j = 0; j < K; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double r = 0;
#pragma unroll
  for (int j = 0; j < K; ++j) r += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int K> void run(int warps, double* out, long long* cyc, int nsm) {
  k<K><<<nsm, warps * 32>>>(out, cyc, 1e-3);
  k<K><<<nsm, warps * 32>>>(out, cyc, 1e-3);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, cyc, nsm * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
  // one m8n8k4 = 256 FMA
  printf("DMMA K=%2d warps/SM=%2d: %7.2f FMA/clk/SM, %6.1f cyc per dependent DMMA\n", K, warps,
         256.0 * warps * K * 2048 / mx, mx / 2048.0);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out; long long* cyc; cudaMalloc(&out, nsm * 1024 * 8); cudaMalloc(&cyc, nsm * 8);
  for (int w : {1, 4, 8, 16}) { run<1>(w, out, cyc, nsm); run<2>(w, out, cyc, nsm); run<4>(w, out, cyc, nsm); run<8>(w, out, cyc, nsm); }
  return 0;
}
