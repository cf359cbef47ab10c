// Products with the RBM log-derivative matrix O (ref: rbm.py:307-325
// grad_log_psi_batch: O(x) = [x, tanh theta, tanh theta (x) x], columns a, b,
// W row-major) without forming O: the SR solve (vmc.py:145-229 estimators,
// solved matrix-free) needs O v and O^H u per conjugate-gradient iteration.
// X (samples x sites) is 0/1 and arrives bit-packed, T = tanh(theta) is a
// complex (U, M) matrix; both products are GEMMs over X on the FP64 tensor
// cores (DMMA m8n8k4), with the rest fused into their epilogues:
//
//   ov:  q_s = sum_k x_sk va_k + sum_i t_si (vb_i + (X vW^T)_si)
//        block = 16 samples; (X vW^T) as the energy kernel's theta GEMM
//        (A = sample bits, B = vW^T in the padded staging layout); the
//        epilogue multiplies by t and reduces over units in a fixed order.
//   ohu: out = [X^T u, T^H u, (conj(T) * u)^T X]  ==  A' B' with
//        A' rows (2i, 2i+1) = Re/Im conj(t_si) u_s, rows (2M, 2M+1) = Re/Im u_s,
//        B' = [X | 1]; split over sample chunks (K), partial sums reduced in a
//        fixed chunk order (deterministic).
#pragma once
#include <algorithm>

#include "common.cuh"

namespace mpv {

constexpr int kLdSB = 16;       // samples per ov block

__device__ __forceinline__ void ld_dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__host__ __device__ inline int ld_pitch(int M) { return 2 * M + 8; }  // doubles per vW^T row
__host__ __device__ inline int ld_rows(int N) { return (N + 3) / 4 * 4; }

// vW (row-major [M][N] complex, the W block of v) -> vWt[k][2i + c] padded
// `skip` (optional): a device flag; non-zero = the launch is a no-op (a converged
// CG solve's remaining batch iterations)
__global__ void ld_transpose_kernel(const double2* __restrict__ v, int N, int M, double* __restrict__ vwt,
                                    const double* __restrict__ skip = nullptr) {
  if (skip && *skip != 0.0) return;
  const int pitch = ld_pitch(M), rows = ld_rows(N);
  const double2* vw = v + N + M;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (int64_t)rows * pitch;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx / pitch), c = (int)(idx % pitch);
    double val = 0.0;
    if (k < N && c < 2 * M) {
      const double2 z = vw[(size_t)(c >> 1) * N + k];
      val = (c & 1) ? z.y : z.x;
    }
    vwt[idx] = val;
  }
}

// Complex tanh in f64: tanh(x + iy) = (sign(x)(1 - e^2) + 2i e sin 2y) / (1 + e^2 + 2e cos 2y),
// e = exp(-2|x|) (numerator and denominator of sinh 2x / (cosh 2x + cos 2y) scaled by 2e:
// no overflow for large |x|, and 1 - e^2 = -expm1(-4|x|) keeps small |x| accurate).
__device__ __forceinline__ double2 ctanh_f64(double x, double y) {
  const double ax = fabs(x);
  const double e = exp(-2.0 * ax);
  double s2, c2;
  sincos(2.0 * y, &s2, &c2);
  const double den = fma(2.0 * e, c2, fma(e, e, 1.0));
  return make_double2(copysign(-expm1(-4.0 * ax), x) / den, 2.0 * e * s2 / den);
}

// MODE 0 (ov):   q_s = w_s (O v)_s            (w NULL: 1)
// MODE 1 (tanh): t_si = tanh(b_i + (X W^T)_si) with v = the parameter vector [a | b | W]
// NW warps per block (the block's 16 samples are shared by all warps' n-tiles)
template <int KT, int MODE = 0, int NW = 8>
__global__ void __launch_bounds__(32 * NW, (KT >= 16 || NW > 8) ? (NW > 8 ? 2 : 1) : 2) ld_ov_kernel(const double2* __restrict__ t, const uint32_t* __restrict__ bits,
                                                    int64_t U, int N, int M, int words, const double2* __restrict__ v,
                                                    const double* __restrict__ vwt, double2* __restrict__ q,
                                                    const double* __restrict__ w = nullptr,
                                                    double2* __restrict__ t_out = nullptr,
                                                    const double* __restrict__ skip = nullptr) {
  if (skip && *skip != 0.0) return;
  __shared__ uint32_t smask[256 + 8];        // per-site masks of the block's 16 samples (N <= 256)
  __shared__ double2 red[NW][kLdSB];         // per-warp partial q
  __shared__ __align__(8) uint64_t tbar;
  extern __shared__ __align__(16) double2 tsm[];  // MODE 0: the block's T rows [16][M], bulk-copied
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t s0 = (int64_t)blockIdx.x * kLdSB;
  const int pitch = ld_pitch(M), rows = ld_rows(N);
  const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&tbar);
  if constexpr (MODE == 0) {
    // the epilogue's T rows stream in (TMA engine) under the GEMM
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      const uint32_t bytes = (uint32_t)((min((int64_t)kLdSB, U - s0)) * M * 16);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(bytes) : "memory");
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(tsm);
      for (uint32_t off = 0; off < bytes; off += 65536u) {
        const uint32_t n = min(bytes - off, 65536u);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         dst + off), "l"((const char*)(t + s0 * M) + off), "r"(n), "r"(sbar)
                     : "memory");
      }
    }
  }
  for (int k = tid; k < rows; k += blockDim.x) {
    uint32_t m = 0;
    if (k < N)
      for (int s = 0; s < kLdSB; ++s)
        if (s0 + s < U) m |= ((bits[(s0 + s) * words + (k >> 5)] >> (k & 31)) & 1u) << s;
    smask[k] = m;
  }
  __syncthreads();
  const int NT = (M + 3) / 4;
  const int qr = lane & 3, qc = lane >> 2;
  double acc[KT][2][2];
  int col[KT];
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    col[j] = min(warp + j * NW, NT - 1) * 8 + qc;
    acc[j][0][0] = acc[j][0][1] = acc[j][1][0] = acc[j][1][1] = 0.0;
  }
  // B fragments are prefetched one k-step ahead (L2 latency); n-tiles past NT
  // (clamped duplicates) are skipped (warp-uniform)
  double bf[KT], bn[KT];
#pragma unroll
  for (int j = 0; j < KT; ++j) bf[j] = __ldg(vwt + (size_t)qr * pitch + col[j]);
  for (int k0 = 0; k0 < rows; k0 += 4) {
    if (k0 + 4 < rows) {
      const double* brow = vwt + (size_t)(k0 + 4 + qr) * pitch;
#pragma unroll
      for (int j = 0; j < KT; ++j) bn[j] = __ldg(brow + col[j]);
    }
    const uint32_t mk = smask[k0 + qr];
    const double a0 = __hiloint2double((int)(((mk >> qc) & 1u) * 0x3ff00000u), 0);
    const double a1 = __hiloint2double((int)(((mk >> (8 + qc)) & 1u) * 0x3ff00000u), 0);
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      if (warp + j * NW < NT) {
        ld_dmma(acc[j][0][0], acc[j][0][1], a0, bf[j]);
        ld_dmma(acc[j][1][0], acc[j][1][1], a1, bf[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < KT; ++j) bf[j] = bn[j];
  }
  if constexpr (MODE == 1) {
    // D fragment (sample m*8 + qc, unit nt*4 + qr) = theta - b: write tanh(theta)
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      const int nt = warp + j * NW, i = nt * 4 + qr;
      if (nt < NT && i < M) {
        const double2 b = v[N + i];
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int64_t s = s0 + m * 8 + qc;
          if (s < U) t_out[s * M + i] = ctanh_f64(acc[j][m][0] + b.x, acc[j][m][1] + b.y);
        }
      }
    }
    return;
  }
  // epilogue: D fragment (sample m*8 + qc, unit nt*4 + qr) -> t * (Y + vb), summed over units
  asm volatile(
      "{.reg .pred p;\nWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(sbar)
      : "memory");
  double2 part[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    const int nt = warp + j * NW, i = nt * 4 + qr;
    if (nt < NT && i < M) {
      const double2 vb = v[N + i];
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int64_t s = s0 + m * 8 + qc;
        if (s < U) {
          const double2 ts = tsm[(m * 8 + qc) * M + i];
          const double yr = acc[j][m][0] + vb.x, yi = acc[j][m][1] + vb.y;
          part[m].x = fma(ts.x, yr, fma(-ts.y, yi, part[m].x));
          part[m].y = fma(ts.x, yi, fma(ts.y, yr, part[m].y));
        }
      }
    }
  }
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    for (int off = 1; off < 4; off <<= 1) {
      part[m].x += __shfl_xor_sync(kFull, part[m].x, off);
      part[m].y += __shfl_xor_sync(kFull, part[m].y, off);
    }
    if (qr == 0) red[warp][m * 8 + qc] = part[m];
  }
  __syncthreads();
  if (tid < kLdSB && s0 + tid < U) {
    const int64_t s = s0 + tid;
    double2 acc2 = make_double2(0.0, 0.0);
    for (int k = 0; k < N; ++k)  // sum_k x_sk va_k, ascending k
      if ((smask[k] >> tid) & 1u) {
        acc2.x += v[k].x;
        acc2.y += v[k].y;
      }
    for (int wp = 0; wp < NW; ++wp) {
      acc2.x += red[wp][tid].x;
      acc2.y += red[wp][tid].y;
    }
    if (w) {
      acc2.x *= w[s];
      acc2.y *= w[s];
    }
    q[s] = acc2;
  }
}

// ohu partials: block (row group x, chunk y, column group z); warp = one
// m-tile (8 rows of A'), NTC n-tiles (8*NTC columns of B' = [X | 1]).  The
// A' values of the next 64-sample tile are loaded into registers while the
// current tile's DMMAs run (double-buffered shared memory).
constexpr int kLdTile = 32;  // samples staged per sub-tile
__host__ __device__ inline int ld_rows_a(int M) { return (2 * M + 2 + 63) / 64 * 64; }  // A' rows, whole blocks
// n-tiles per column group: the smallest padding of N + 1 columns
__host__ __device__ inline int ld_ntc(int N) {
  const int c = N + 1;
  int best = 16, waste = 1 << 30;
  const int opts[4] = {16, 13, 8, 4};
  for (int k = 0; k < 4; ++k) {
    const int w = (c + 8 * opts[k] - 1) / (8 * opts[k]) * 8 * opts[k] - c;
    if (w < waste) { waste = w; best = opts[k]; }
  }
  return best;
}
__host__ __device__ inline int ld_cols(int N) { const int g = 8 * ld_ntc(N); return (N + 1 + g - 1) / g * g; }
// samples per K-chunk: about two blocks per SM over the (row, chunk, column) grid
inline int64_t ld_chunk(int64_t U, int N, int M) {
  const int64_t other = (int64_t)(ld_rows_a(M) / 64) * (ld_cols(N) / (8 * ld_ntc(N)));
  const int64_t target = std::max<int64_t>(1, 2 * 148 / std::max<int64_t>(1, other));
  const int64_t c = (U + target - 1) / target;
  return std::max<int64_t>(kLdTile, (c + kLdTile - 1) / kLdTile * kLdTile);
}

template <int NTC>
__global__ void __launch_bounds__(256, 2) ld_ohu_kernel(const double2* __restrict__ t, const uint32_t* __restrict__ bits,
                                                     int64_t U, int N, int M, int words, const double2* __restrict__ u,
                                                     double* __restrict__ partial, int64_t chunk,
                                                     const double* __restrict__ wts = nullptr,
                                                     const double* __restrict__ skip = nullptr) {
  if (skip && *skip != 0.0) return;
  __shared__ double as[2][64][kLdTile + 1];  // A' tiles [row][sample] (+1 pad: conflict-free column reads)
  // B' = [X | 1] of the tile as per-column sample masks: cms[buf][n] bit s =
  // X[tile sample s][site n] (built by warp ballots), column N = valid samples
  __shared__ uint32_t cms[2][264];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 2 * 264; i += 256) (&cms[0][0])[i] = 0u;  // columns past the packed words stay 0
  const int rows_a = 2 * M + 2;
  const int u0 = blockIdx.x * 32;  // first unit of this block (64 A' rows)
  const int64_t k_begin = (int64_t)blockIdx.y * chunk;
  const int64_t k_end = min(U, k_begin + chunk);
  const int c0 = blockIdx.z * 8 * NTC;  // first B' column of this block
  const int qr = lane & 3, qc = lane >> 2;
  constexpr int kPer = kLdTile * 32 / 256;  // (sample, unit) pairs staged per thread
  double2 pt[kPer], pu[kPer];
  uint32_t pb = 0;
  int pn = 0;
  auto load = [&](int64_t sb) {  // global -> registers for the tile at sb
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int idx = tid + r * 256, ls = idx >> 5, lu = idx & 31;
      const int64_t s = sb + ls;
      const int ui = u0 + lu;
      pt[r] = make_double2(0.0, 0.0);
      pu[r] = make_double2(0.0, 0.0);
      if (s < k_end) {
        pu[r] = u[s];
        if (wts) {
          const double ws = wts[s];
          pu[r].x *= ws;
          pu[r].y *= ws;
        }
        pt[r] = ui < M ? t[s * M + ui] : make_double2(2 * ui < rows_a ? 1.0 : 0.0, 0.0);  // rows 2M, 2M+1: u itself
      }
    }
    if (warp < words) pb = (sb + lane < k_end) ? bits[(sb + lane) * words + warp] : 0u;  // warp w: word w, lane: sample
    pn = (int)min((int64_t)kLdTile, k_end - sb);  // valid samples of the tile
  };
  auto store = [&](int buf) {  // registers -> shared: A' = (Re, Im) conj(t) u
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int idx = tid + r * 256, ls = idx >> 5, lu = idx & 31;
      as[buf][2 * lu][ls] = fma(pt[r].x, pu[r].x, pt[r].y * pu[r].y);
      as[buf][2 * lu + 1][ls] = fma(pt[r].x, pu[r].y, -pt[r].y * pu[r].x);
    }
    if (warp < words) {  // transpose word `warp` of the 32 samples into 32 column masks
#pragma unroll 8
      for (int b = 0; b < 32; ++b) {
        const uint32_t m = __ballot_sync(kFull, (pb >> b) & 1u);
        if (lane == b && warp * 32 + b != N) cms[buf][warp * 32 + b] = m;
      }
    }
    if (tid == 0) cms[buf][N] = pn >= 32 ? 0xFFFFFFFFu : ((1u << pn) - 1u);  // the ones column
  };
  double acc[NTC][2];
#pragma unroll
  for (int j = 0; j < NTC; ++j) acc[j][0] = acc[j][1] = 0.0;
  int cur = 0;
  load(k_begin);
  store(0);
  __syncthreads();
  for (int64_t sb = k_begin; sb < k_end; sb += kLdTile) {
    const bool more = sb + kLdTile < k_end;
    if (more) load(sb + kLdTile);  // in flight during the DMMAs below
    uint32_t mj[NTC];  // the lane's B' columns c0 + 8 j + qc of this tile
#pragma unroll
    for (int j = 0; j < NTC; ++j) {
      const int n = c0 + j * 8 + qc;
      mj[j] = n < 264 ? cms[cur][n] : 0u;
    }
#pragma unroll 4
    for (int k0 = 0; k0 < kLdTile; k0 += 4) {
      const double av = as[cur][warp * 8 + qc][k0 + qr];
#pragma unroll
      for (int j = 0; j < NTC; ++j) {
        const uint32_t bit = (mj[j] >> (k0 + qr)) & 1u;
        ld_dmma(acc[j][0], acc[j][1], av, __hiloint2double((int)(bit * 0x3ff00000u), 0));
      }
    }
    if (more) store(cur ^ 1);
    __syncthreads();
    cur ^= 1;
  }
  // D fragment: row 2*u0 + warp*8 + qc, columns c0 + j*8 + 2*qr (+1) -> partial[chunk][row][col]
  const int cols = ld_cols(N);
  double* out = partial + (size_t)blockIdx.y * ld_rows_a(M) * cols;
  const int row = 2 * u0 + warp * 8 + qc;
#pragma unroll
  for (int j = 0; j < NTC; ++j) {
    out[(size_t)row * cols + c0 + j * 8 + 2 * qr] = acc[j][0];
    out[(size_t)row * cols + c0 + j * 8 + 2 * qr + 1] = acc[j][1];
  }
}

// fixed-order reduction of the chunk partials -> out (complex P-vector); with
// sum_out, also sum_s u_s (rows 2M, 2M+1 of A' against the ones column N)
__global__ void ld_ohu_reduce_kernel(const double* __restrict__ partial, int chunks, int N, int M,
                                     double2* __restrict__ out, double2* __restrict__ sum_out = nullptr,
                                     const double* __restrict__ skip = nullptr) {
  if (skip && *skip != 0.0) return;
  const int rows_pad = ld_rows_a(M), cols = ld_cols(N);
  const int P = N + M + M * N;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < P + 1; idx += gridDim.x * blockDim.x) {
    if (idx == P && !sum_out) break;
    int r, c;  // (row pair, column) of the entry
    if (idx == P) { r = M; c = N; }                         // sum_s u_s
    else if (idx < N) { r = M; c = idx; }                   // a-part: rows 2M, 2M+1 (u), column k
    else if (idx < N + M) { r = idx - N; c = N; }          // b-part: unit i, ones column
    else { r = (idx - N - M) / N; c = (idx - N - M) % N; }  // W-part: unit i, site k
    double re = 0.0, im = 0.0;
    for (int ch = 0; ch < chunks; ++ch) {
      const double* p = partial + (size_t)ch * rows_pad * cols;
      re += p[(size_t)(2 * r) * cols + c];
      im += p[(size_t)(2 * r + 1) * cols + c];
    }
    if (idx == P) *sum_out = make_double2(re, im);
    else out[idx] = make_double2(re, im);
  }
}

}  // namespace mpv
