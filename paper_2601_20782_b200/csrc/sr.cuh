// Stochastic-reconfiguration statistics and solve on the device (ref:
// vmc.py:145-229 forces / s_matrix / sr_step, vmc.py:592-604 the split-chain
// error, rbm.py:307-325 grad_log_psi_batch), all f64:
//
//  * dense O (optionally centred) and S = sum_s w_s conj(C_s) C_s^T for the
//    small-P dense path (the reference's Cholesky solve);
//  * the matrix-free conjugate-gradient solve of (S + lambda) g = F with the
//    scalars kept on the device: every iteration is a fixed kernel sequence
//    (O p with the weights fused, O^H u with sum_s u_s fused, then the vector
//    updates below) and the convergence test is a device flag, so the host
//    launches batches of iterations and synchronises once per batch;
//  * per-chain means and two-pass moments for the split-chain MC error.
// Every reduction runs in a fixed order: results are bit-reproducible.
#pragma once
#include "logderiv.cuh"

namespace mpv {

constexpr int kCgThreads = 256;
constexpr int kCgMaxBlocks = 296;  // 2 per SM; partial arrays hold <= kCgMaxBlocks values

// scalars of one CG solve (device, f64)
enum CgSlot { kCgRR = 0, kCgThr2 = 1, kCgIters = 2, kCgDone = 3, kCgMaxIter = 4, kCgSlots = 8 };

// Sum of n <= kCgMaxBlocks partials in a fixed order, identical in every block
// (warp 0: strided sequential sums, then a fixed xor tree); broadcast via smem.
__device__ __forceinline__ double block_sum_fixed(const double* part, int n) {
  __shared__ double res;
  if (threadIdx.x < 32) {
    double a = 0.0;
    for (int i = threadIdx.x; i < n; i += 32) a += part[i];
    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(kFull, a, off);
    if (threadIdx.x == 0) res = a;
  }
  __syncthreads();
  const double r = res;
  __syncthreads();
  return r;
}

// Block sum of one value per thread -> partial[blockIdx.x] (fixed order).
__device__ __forceinline__ void block_partial(double v, double* partial) {
  __shared__ double red[kCgThreads / 32];
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) a += red[i];
    partial[blockIdx.x] = a;
  }
}

// g = 0, r = p = f, rr = |f|^2 (partials), thresholds
__global__ void cg_init_kernel(int P, const double2* __restrict__ f, double2* g, double2* r, double2* p,
                               double* partial) {
  double a = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P; j += gridDim.x * blockDim.x) {
    const double2 v = f[j];
    g[j] = make_double2(0.0, 0.0);
    r[j] = v;
    p[j] = v;
    a = fma(v.x, v.x, fma(v.y, v.y, a));
  }
  block_partial(a, partial);
}

// rr = |f|^2; done = !(maxiter > 0 && fn > 0 && sqrt(rr) > tol fn)  (vmc CG loop guard)
__global__ void cg_init_scalars_kernel(const double* partial, int nb, double tol, double maxiter, double* sc) {
  const double rr = block_sum_fixed(partial, nb);
  if (threadIdx.x == 0) {
    const double thr = tol * sqrt(rr);  // tol * |f|
    sc[kCgRR] = rr;
    sc[kCgThr2] = thr;
    sc[kCgIters] = 0.0;
    sc[kCgMaxIter] = maxiter;
    sc[kCgDone] = (maxiter > 0.0 && rr > 0.0 && sqrt(rr) > thr) ? 0.0 : 1.0;
  }
}

// out = y - conj(obar) * ysum + lambda * v   (S v + lambda v from O^H (w O v));
// with pap_partial: partial Re <v, out>
__global__ void cg_ap_kernel(int P, const double2* __restrict__ y, const double2* __restrict__ ysum,
                             const double2* __restrict__ obar, double lambda, const double2* __restrict__ v,
                             double2* __restrict__ out, double* pap_partial) {
  const double2 sm = *ysum;
  double a = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P; j += gridDim.x * blockDim.x) {
    const double2 o = obar[j], yj = y[j], vj = v[j];
    // conj(o) * sm = (o.x sm.x + o.y sm.y) + i (o.x sm.y - o.y sm.x)
    const double re = fma(lambda, vj.x, yj.x - fma(o.x, sm.x, o.y * sm.y));
    const double im = fma(lambda, vj.y, yj.y - fma(o.x, sm.y, -o.y * sm.x));
    out[j] = make_double2(re, im);
    a = fma(vj.x, re, fma(vj.y, im, a));
  }
  if (pap_partial) block_partial(a, pap_partial);
}

// alpha = rr / pAp (0 once converged); g += alpha p; r -= alpha ap; partial |r|^2
__global__ void cg_update_kernel(int P, const double2* __restrict__ p, const double2* __restrict__ ap, double2* g,
                                 double2* r, const double* pap_partial, int nb, double* rr_partial,
                                 const double* sc) {
  const double pap = block_sum_fixed(pap_partial, nb);
  const bool done = sc[kCgDone] != 0.0;
  const double alpha = done ? 0.0 : sc[kCgRR] / pap;
  double a = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P; j += gridDim.x * blockDim.x) {
    const double2 pj = p[j], aj = ap[j];
    double2 gj = g[j], rj = r[j];
    gj.x = fma(alpha, pj.x, gj.x);
    gj.y = fma(alpha, pj.y, gj.y);
    rj.x = fma(-alpha, aj.x, rj.x);
    rj.y = fma(-alpha, aj.y, rj.y);
    g[j] = gj;
    r[j] = rj;
    a = fma(rj.x, rj.x, fma(rj.y, rj.y, a));
  }
  block_partial(a, rr_partial);
}

// p = r + (rr_new / rr) p   (unchanged once converged)
__global__ void cg_direction_kernel(int P, const double2* __restrict__ r, double2* p, const double* rr_partial, int nb,
                                    const double* sc) {
  const double rr_new = block_sum_fixed(rr_partial, nb);
  if (sc[kCgDone] != 0.0) return;
  const double beta = rr_new / sc[kCgRR];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P; j += gridDim.x * blockDim.x) {
    const double2 rj = r[j], pj = p[j];
    p[j] = make_double2(fma(beta, pj.x, rj.x), fma(beta, pj.y, rj.y));
  }
}

// rr = rr_new, iteration count, convergence flag (one block)
__global__ void cg_commit_kernel(const double* rr_partial, int nb, double* sc) {
  const double rr_new = block_sum_fixed(rr_partial, nb);
  if (threadIdx.x == 0 && sc[kCgDone] == 0.0) {
    const double it = sc[kCgIters] + 1.0;
    sc[kCgIters] = it;
    sc[kCgRR] = rr_new;
    sc[kCgDone] = (it < sc[kCgMaxIter] && sqrt(rr_new) > sc[kCgThr2]) ? 0.0 : 1.0;
  }
}

// Dense log-derivatives O_s = [x, t, t (x) x] - obar (ref: rbm.py:307-325), [U][P] complex
__global__ void ld_dense_kernel(const double2* __restrict__ t, const uint32_t* __restrict__ bits, int64_t U, int N,
                                int M, int words, const double2* __restrict__ obar, double2* __restrict__ o) {
  const int64_t P = (int64_t)N + M + (int64_t)M * N;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < U * P;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = idx / P;
    const int j = (int)(idx % P);
    double2 val;
    if (j < N) {
      val = make_double2((double)((bits[s * words + (j >> 5)] >> (j & 31)) & 1u), 0.0);
    } else if (j < N + M) {
      val = t[s * M + (j - N)];
    } else {
      const int i = (j - N - M) / N, k = (j - N - M) % N;
      val = ((bits[s * words + (k >> 5)] >> (k & 31)) & 1u) ? t[s * M + i] : make_double2(0.0, 0.0);
    }
    if (obar) {
      val.x -= obar[j].x;
      val.y -= obar[j].y;
    }
    o[idx] = val;
  }
}

// S = sum_s w_s conj(C_s) C_s^T for C [U][P] complex: 64x64 output tiles, 256
// threads with 4x4 complex entries each, samples staged 8 at a time in shared
// memory; the lower triangle is mirrored (Hermitian) by the tile owner.
constexpr int kSmT = 64, kSmK = 8;
__global__ void __launch_bounds__(256) sr_smatrix_kernel(const double2* __restrict__ c, const double* __restrict__ w,
                                                         int64_t U, int P, double2* __restrict__ s) {
  const int bj = blockIdx.y, bk = blockIdx.x;
  if (bk < bj) return;  // upper block triangle only
  __shared__ double2 aj[kSmK][kSmT + 1], ak[kSmK][kSmT + 1];
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const int j0 = bj * kSmT, k0 = bk * kSmT;
  double accr[4][4], acci[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) accr[a][b] = acci[a][b] = 0.0;
  for (int64_t s0 = 0; s0 < U; s0 += kSmK) {
    for (int e = tid; e < kSmK * kSmT; e += 256) {
      const int ss = e / kSmT, col = e % kSmT;
      const int64_t sidx = s0 + ss;
      double2 vj = make_double2(0.0, 0.0), vk = make_double2(0.0, 0.0);
      if (sidx < U) {
        const double ws = w ? w[sidx] : 1.0;
        if (j0 + col < P) {
          vj = c[sidx * P + j0 + col];
          vj.x *= ws;
          vj.y *= ws;
        }
        if (k0 + col < P) vk = c[sidx * P + k0 + col];
      }
      aj[ss][col] = vj;
      ak[ss][col] = vk;
    }
    __syncthreads();
#pragma unroll
    for (int ss = 0; ss < kSmK; ++ss) {
      double2 x[4], y[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) x[a] = aj[ss][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) y[b] = ak[ss][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          // conj(x) y
          accr[a][b] = fma(x[a].x, y[b].x, fma(x[a].y, y[b].y, accr[a][b]));
          acci[a][b] = fma(x[a].x, y[b].y, fma(-x[a].y, y[b].x, acci[a][b]));
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = j0 + ty + 16 * a, k = k0 + tx + 16 * b;
      if (j < P && k < P && j <= k) {
        s[(int64_t)j * P + k] = make_double2(accr[a][b], acci[a][b]);
        s[(int64_t)k * P + j] = make_double2(accr[a][b], -acci[a][b]);
      }
    }
}

// Hermitian part of the diagonal: Im S_jj = 0 exactly (the reference Hermitises S)
__global__ void sr_real_diag_kernel(int P, double2* s) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P; j += gridDim.x * blockDim.x) s[(int64_t)j * P + j].y = 0.0;
}

// Per-chain means of the local energies (ref: vmc.py:592-604): chain c (global
// id chain_offset + c) owns sample rows [c base + min(c, extra), ...) - row0;
// eps_u (complex, unique rows) indexed through `inverse`; + partial sums of the means.
__global__ void chain_means_kernel(const double2* __restrict__ eps_u, const int64_t* __restrict__ inverse,
                                   int64_t n_chains, int64_t chain_offset, int64_t base, int64_t extra,
                                   int64_t row0, double* __restrict__ means, double* partial) {
  double a = 0.0;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_chains;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = chain_offset + c;
    const int64_t r0 = g * base + (g < extra ? g : extra) - row0;
    const int64_t cnt = base + (g < extra ? 1 : 0);
    double sum = 0.0;
    for (int64_t r = 0; r < cnt; ++r) sum += eps_u[inverse ? inverse[r0 + r] : r0 + r].x;
    const double m = sum / (double)cnt;
    means[c] = m;
    a += m;
  }
  block_partial(a, partial);
}

// Two-pass moments of a vector: out = [mean, sum (x - mean)^2, n]; pass 1 in
// partial[0..nb), pass 2 in partial[nb..2nb).
__global__ void moments_pass2_kernel(const double* __restrict__ x, int64_t n, const double* partial, int nb,
                                     double* partial2) {
  const double mean = block_sum_fixed(partial, nb) / (double)n;
  double a = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = x[i] - mean;
    a = fma(d, d, a);
  }
  block_partial(a, partial2);
}
__global__ void moments_finish_kernel(const double* partial, int nb, const double* partial2, int64_t n,
                                      double* out) {
  const double sum = block_sum_fixed(partial, nb);
  const double ss = block_sum_fixed(partial2, nb);
  if (threadIdx.x == 0) {
    out[0] = sum / (double)n;
    out[1] = ss;
    out[2] = (double)n;
  }
}
__global__ void moments_pass1_kernel(const double* __restrict__ x, int64_t n, double* partial) {
  double a = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a += x[i];
  block_partial(a, partial);
}


// minSR sample-space matrix (beyond the reference; push-through form of
// vmc.py:202-229): K~ = W^1/2 (O - 1 obar^T)(O - 1 obar^T)^H W^1/2 + lambda I with
// (O O^H)_{ss'} = c_{ss'} + (T T^H)_{ss'} (1 + c_{ss'}),  c_{ss'} = popc(x_s & x_s')
// (a-block: common set bits; b-block: T T^H; W-block: (T T^H) * c), then
// K~_{ss'} = sqrt(w_s w_s') [(O O^H)_{ss'} - d_s - conj(d_s') + |obar|^2],
// d_s = (O conj(obar))_s.  Rows s of this rank (global row row0 + s) against all
// U_all columns: 64x64 tiles, T staged 8 units at a time; OutT = double2 or float2.
template <typename OutT>
__global__ void __launch_bounds__(256) minsr_gram_kernel(
    const double2* __restrict__ t_rows, const uint32_t* __restrict__ bits_rows, int64_t U_rows, int64_t row0,
    const double2* __restrict__ t_all, const uint32_t* __restrict__ bits_all, int64_t U_all, int M, int words,
    const double2* __restrict__ d_all, const double* __restrict__ w_all, double obar2, double lambda,
    OutT* __restrict__ out) {
  __shared__ double2 ta[kSmT][kSmK + 1], tb[kSmT][kSmK + 1];
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const int64_t s0 = (int64_t)blockIdx.y * kSmT, c0 = (int64_t)blockIdx.x * kSmT;
  double accr[4][4], acci[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) accr[a][b] = acci[a][b] = 0.0;
  for (int i0 = 0; i0 < M; i0 += kSmK) {
    for (int e = tid; e < kSmK * kSmT; e += 256) {
      const int rr = e / kSmK, ii = e % kSmK;
      const int i = i0 + ii;
      double2 va = make_double2(0.0, 0.0), vb = make_double2(0.0, 0.0);
      if (i < M) {
        if (s0 + rr < U_rows) va = t_rows[(s0 + rr) * M + i];
        if (c0 + rr < U_all) vb = t_all[(c0 + rr) * M + i];
      }
      ta[rr][ii] = va;
      tb[rr][ii] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int ii = 0; ii < kSmK; ++ii) {
      double2 x[4], y[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) x[a] = ta[ty + 16 * a][ii];
#pragma unroll
      for (int b = 0; b < 4; ++b) y[b] = tb[tx + 16 * b][ii];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {  // x conj(y)
          accr[a][b] = fma(x[a].x, y[b].x, fma(x[a].y, y[b].y, accr[a][b]));
          acci[a][b] = fma(x[a].y, y[b].x, fma(-x[a].x, y[b].y, acci[a][b]));
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t s = s0 + ty + 16 * a;
    if (s >= U_rows) continue;
    const int64_t gs = row0 + s;
    const double2 ds = d_all[gs];
    const double ws = sqrt(w_all[gs]);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t c = c0 + tx + 16 * b;
      if (c >= U_all) continue;
      int pc = 0;
      for (int wd = 0; wd < words; ++wd) pc += __popc(bits_rows[s * words + wd] & bits_all[c * words + wd]);
      const double2 dc = d_all[c];
      const double cc = (double)pc;
      const double sc = ws * sqrt(w_all[c]);
      double re = cc + accr[a][b] * (1.0 + cc) - ds.x - dc.x + obar2;
      double im = acci[a][b] * (1.0 + cc) - ds.y + dc.y;
      re *= sc;
      im *= sc;
      if (gs == c) {
        re += lambda;
        im = 0.0;
      }
      if constexpr (sizeof(OutT) == 16) out[s * U_all + c] = make_double2(re, im);
      else out[s * U_all + c] = make_float2((float)re, (float)im);
    }
  }
}

}  // namespace mpv
