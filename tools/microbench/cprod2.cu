// Phase-2 step of the local-energy kernel in isolation: per row, tau (per
// lane) and ST tanh(theta) values (broadcast) loaded from shared memory, the
// sign of d applied by LOP3 on the high words, u = tv*tau, P += P*u.
// Reports FP64 lane-ops per SM clock (8 per factor; peak 64).
#include <cstdio>
template <int ST, int SB, int MODE>
__global__ void __launch_bounds__(ST == 2 ? 832 : 448, ST == 8 ? 1 : 2) k(double* out, long long* cyc, int rows, int T) {
  extern __shared__ double2 sm[];
  double2* tt = sm;             // [rows][SB]
  double2* ts = sm + rows * SB;  // [rows][T]
  for (int i = threadIdx.x; i < rows * SB; i += blockDim.x) tt[i] = make_double2(1e-3 * (i % 17), 2e-3 * (i % 5));
  for (int i = threadIdx.x; i < rows * T; i += blockDim.x) ts[i] = make_double2(1e-3 * (i % 13), -1e-3 * (i % 7));
  __syncthreads();
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  double2 P[ST];
  unsigned sg[ST];
  double dj[ST];
#pragma unroll
  for (int j = 0; j < ST; ++j) { P[j] = make_double2(1.0, 0.0); sg[j] = ((threadIdx.x >> j) & 1) << 31; dj[j] = sg[j] ? -1.0 : 1.0; }
  long long t0 = clock64();
  for (int rep = 0; rep < 80; ++rep) {
    const double2* tp = ts + t;
    const double2* vp = tt + (g % (SB / ST)) * ST;
#pragma unroll 2
    for (int r = 0; r < rows; ++r) {
      const double2 tau = MODE == 2 ? make_double2(1e-3 * r, 2e-3) : *tp;
      double2 tv[ST];
#pragma unroll
      for (int j = 0; j < ST; ++j) tv[j] = MODE == 3 ? make_double2(1e-3 * (r + j), 1e-4 * j) : vp[j];
      tp += T;
      vp += SB;
#pragma unroll
      for (int j = 0; j < ST; ++j) {
        if (MODE == 4) {
          const long long m = (long long)sg[j] << 32;
          tv[j].x = __longlong_as_double(__double_as_longlong(tv[j].x) ^ m);
          tv[j].y = __longlong_as_double(__double_as_longlong(tv[j].y) ^ m);
        } else if (MODE == 5) {
          // sign as a multiply folded into the first product of each component
        } else if (MODE != 1) {
          tv[j].x = __hiloint2double(__double2hiint(tv[j].x) ^ (int)sg[j], __double2loint(tv[j].x));
          tv[j].y = __hiloint2double(__double2hiint(tv[j].y) ^ (int)sg[j], __double2loint(tv[j].y));
        }
        double ux, uy;
        if (MODE == 5) {
          const double dx = dj[j] * tv[j].x, dy = dj[j] * tv[j].y;  // (extra DMULs)
          ux = fma(dx, tau.x, -dy * tau.y); uy = fma(dx, tau.y, dy * tau.x);
        } else {
          ux = fma(tv[j].x, tau.x, -tv[j].y * tau.y); uy = fma(tv[j].x, tau.y, tv[j].y * tau.x);
        }
        const double px = P[j].x, py = P[j].y;
        P[j].x = fma(px, ux, fma(-py, uy, px));
        P[j].y = fma(px, uy, fma(py, ux, py));
      }
    }
  }
  long long t1 = clock64();
  double acc = 0;
#pragma unroll
  for (int j = 0; j < ST; ++j) acc += P[j].x + P[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int ST, int MODE>
void run(const char* name, int nsm, double* out, long long* cyc) {
  const int rows = 48, T = 100, SB = 16;
  const int threads = ((SB / ST) * T + 31) / 32 * 32;
  const int active = (SB / ST) * T;
  const size_t smem = (size_t)rows * (SB + T) * 16;
  cudaFuncSetAttribute(k<ST, 16, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int bps : {2}) {
    k<ST, 16, MODE><<<nsm * bps, threads, smem>>>(out, cyc, rows, T);
    k<ST, 16, MODE><<<nsm * bps, threads, smem>>>(out, cyc, rows, T);
    cudaError_t e = cudaDeviceSynchronize();
    static long long h[4096];
    cudaMemcpy(h, cyc, nsm * bps * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < nsm * bps; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%-28s ST=%d threads=%d CTAs/SM=%d err=%d: %6.2f FP64 lane-ops/clk/SM\n", name, ST, threads, bps, (int)e,
           8.0 * ST * active * bps * rows * 80 / mx);
  }
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out; long long* cyc; cudaMalloc(&out, nsm * 4 * 1024 * 8); cudaMalloc(&cyc, nsm * 4 * 8);
  run<4, 0>("full (lds tau+tv, lop3)", nsm, out, cyc);
  run<4, 1>("no lop3", nsm, out, cyc);
  run<4, 4>("xor.b64", nsm, out, cyc);
  run<4, 5>("dmul sign", nsm, out, cyc);
  run<4, 2>("tau in regs", nsm, out, cyc);
  run<4, 3>("tv in regs", nsm, out, cyc);
  run<8, 0>("full ST=8", nsm, out, cyc);
  run<2, 0>("full ST=2", nsm, out, cyc);
  return 0;
}
