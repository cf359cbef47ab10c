// f64 local energies (ref: vmc.py:52-108 local_energies, _diagonal_energy).
//
//   eps(x) = J sum_bonds s_i s_j + c * sum_terms psi(x')/psi(x),  s = 1 - 2 bit
//   TFIM:       terms = all N single flips, c = h
//   Heisenberg: terms = bonds (i,j) with x_i != x_j (swap), c = 2J
//
// The reference forms every connected x' and runs a full forward on it
// (O(N * N * M) per sample).  Here a ratio is an O(M) product over hidden
// units of cosh(theta_i + d w_i) / cosh(theta_i) = C_i + d tanh(theta_i) S_i
// with C = cosh(w), S = sinh(w) tabulated once per parameter snapshot
// (w = W_:k for a flip of k, w = W_:i - W_:j for a swap of bond (i,j); d = +-1),
// times exp(d a_k) (or exp(d (a_i - a_j))).  theta and tanh(theta) are formed
// once per sample.  Terms whose table has |Re w| > kSafeRe (where C - S would
// cancel against tanh ~ +-1) use the log-cosh difference instead.
#pragma once
#include "common.cuh"

namespace mpv {

constexpr double kSafeRe = 4.0;
constexpr int kEnergyWarps = 8;     // warps per block
constexpr int kSamplesPerWarp = 2;  // samples per warp (reuses each table load twice)
constexpr int kTermsPerLane = 8;    // register budget per lane per sample

struct EnergyArgs {
  int N, M, words, ham, n_bonds, n_terms;
  const double2 *a, *b, *w_t;  // w_t [N][M]
  const int32_t* bonds;        // [n_bonds][2]
  double J, h;
  const double2* C;  // [M][n_terms]
  const double2* S;  // [M][n_terms]
  const double2* ea; // [n_terms][2]: exp(+a_t), exp(-a_t)
  const int32_t* slow;  // [n_terms]
  const uint32_t* bits;
  int64_t B;
  double2* out;
  int64_t* status;
};

__device__ __forceinline__ double2 cmul(double2 p, double2 q) {
  return make_double2(fma(p.x, q.x, -p.y * q.y), fma(p.x, q.y, p.y * q.x));
}
__device__ __forceinline__ double2 ccosh(double2 z) {
  double s, c;
  sincos(z.y, &s, &c);
  return make_double2(cosh(z.x) * c, sinh(z.x) * s);
}
__device__ __forceinline__ double2 csinh(double2 z) {
  double s, c;
  sincos(z.y, &s, &c);
  return make_double2(sinh(z.x) * c, cosh(z.x) * s);
}
__device__ __forceinline__ double2 cexp_(double2 z) {
  double s, c;
  sincos(z.y, &s, &c);
  const double m = exp(z.x);
  return make_double2(m * c, m * s);
}
// tanh(x+iy) = (sinh 2x + i sin 2y) / (cosh 2x + cos 2y)
__device__ __forceinline__ double2 ctanh(double2 z) {
  if (fabs(z.x) > 20.0) return make_double2(z.x > 0 ? 1.0 : -1.0, 0.0);
  double s, c;
  sincos(2.0 * z.y, &s, &c);
  const double den = cosh(2.0 * z.x) + c;
  return make_double2(sinh(2.0 * z.x) / den, s / den);
}
// complex log cosh, principal branch (ref: rbm.py:130-140)
__device__ __forceinline__ double2 clogcosh(double2 z) {
  const double u = fabs(z.x);
  const double v = z.x < 0.0 ? -z.y : z.y;
  const double t = exp(-2.0 * u);
  double s, c;
  sincos(v, &s, &c);
  const double wr = (1.0 + t) * c, wi = (1.0 - t) * s;
  return make_double2(u - 0.69314718055994530942 + 0.5 * log(wr * wr + wi * wi), atan2(wi, wr));
}

// ---- per-snapshot tables ----
__global__ void energy_tables_kernel(const EnergyArgs a, double2* C, double2* S, double2* ea,
                                     int32_t* slow) {
  const int T = a.n_terms;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (int64_t)a.M * T;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / T), t = (int)(idx % T);
    double2 w;
    if (a.ham == MPV_HAM_TFIM) {
      w = a.w_t[(size_t)t * a.M + i];
    } else {
      const int p = a.bonds[2 * t], q = a.bonds[2 * t + 1];
      const double2 wp = a.w_t[(size_t)p * a.M + i], wq = a.w_t[(size_t)q * a.M + i];
      w = make_double2(wp.x - wq.x, wp.y - wq.y);
    }
    C[(size_t)i * T + t] = ccosh(w);
    S[(size_t)i * T + t] = csinh(w);
  }
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    double2 av;
    int bad = 0;
    if (a.ham == MPV_HAM_TFIM) {
      av = a.a[t];
      for (int i = 0; i < a.M; ++i) bad |= fabs(a.w_t[(size_t)t * a.M + i].x) > kSafeRe;
    } else {
      const int p = a.bonds[2 * t], q = a.bonds[2 * t + 1];
      av = make_double2(a.a[p].x - a.a[q].x, a.a[p].y - a.a[q].y);
      for (int i = 0; i < a.M; ++i)
        bad |= fabs(a.w_t[(size_t)p * a.M + i].x - a.w_t[(size_t)q * a.M + i].x) > kSafeRe;
    }
    ea[2 * t] = cexp_(av);
    ea[2 * t + 1] = cexp_(make_double2(-av.x, -av.y));
    slow[t] = bad;
  }
}

// Scale p by 2^-e (exact), e = exponent of max(|re|, |im|); accumulate e.
__device__ __forceinline__ void renorm(double2& p, int& e) {
  const double m = fmax(fabs(p.x), fabs(p.y));
  if (m == 0.0 || !isfinite(m)) return;
  const int k = ilogb(m);
  const double sc = __longlong_as_double((long long)(1023 - k) << 52);  // 2^-k, |k| < 1023
  p.x *= sc;
  p.y *= sc;
  e += k;
}

__global__ void __launch_bounds__(kEnergyWarps * 32) energy_kernel(const EnergyArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M = a.M, T = a.n_terms;
  double2* th = reinterpret_cast<double2*>(smem_raw) + (size_t)warp * kSamplesPerWarp * 2 * M;
  double2* tt = th + kSamplesPerWarp * M;
  const int64_t s_base = ((int64_t)blockIdx.x * kEnergyWarps + warp) * kSamplesPerWarp;

  uint32_t word[kSamplesPerWarp];
  bool valid[kSamplesPerWarp];
#pragma unroll
  for (int q = 0; q < kSamplesPerWarp; ++q) {
    const int64_t s = s_base + q;
    valid[q] = s < a.B;
    word[q] = (valid[q] && lane < a.words) ? a.bits[s * a.words + lane] : 0u;
  }
  // theta = b + W x, tanh(theta) for both samples; the packed words go
  // through shared memory so the unit loop needs no shuffles.
  uint32_t* wsm = reinterpret_cast<uint32_t*>(smem_raw + (size_t)kEnergyWarps * kSamplesPerWarp * 2 *
                                                             M * sizeof(double2)) +
                  warp * kSamplesPerWarp * 32;
#pragma unroll
  for (int q = 0; q < kSamplesPerWarp; ++q) wsm[q * 32 + lane] = word[q];
  __syncwarp();
  for (int i = lane; i < M; i += 32) {
#pragma unroll
    for (int q = 0; q < kSamplesPerWarp; ++q) {
      double2 z = a.b[i];
      for (int w = 0; w < a.words; ++w) {
        uint32_t wd = wsm[q * 32 + w];
        while (wd) {
          const int k = w * 32 + __ffs(wd) - 1;
          wd &= wd - 1;
          const double2 e = a.w_t[(size_t)k * M + i];
          z.x += e.x;
          z.y += e.y;
        }
      }
      th[q * M + i] = z;
      tt[q * M + i] = ctanh(z);
    }
  }
  __syncwarp();

  auto bit_of = [&](int q, int k) -> int {
    const uint32_t wd = __shfl_sync(kFull, word[q], k >> 5);
    return (wd >> (k & 31)) & 1u;
  };

  double2 sum[kSamplesPerWarp];
  double diag[kSamplesPerWarp];
#pragma unroll
  for (int q = 0; q < kSamplesPerWarp; ++q) {
    sum[q] = make_double2(0.0, 0.0);
    diag[q] = 0.0;
  }
  // diagonal J sum s_i s_j (ref: vmc.py:52-57)
  for (int b0 = 0; b0 < a.n_bonds; b0 += 32) {
    const int b = b0 + lane;
    const int p = b < a.n_bonds ? a.bonds[2 * b] : 0, r = b < a.n_bonds ? a.bonds[2 * b + 1] : 0;
#pragma unroll
    for (int q = 0; q < kSamplesPerWarp; ++q) {
      const int xp = bit_of(q, p), xr = bit_of(q, r);
      if (b < a.n_bonds) diag[q] += (double)((1 - 2 * xp) * (1 - 2 * xr));
    }
  }
  const bool any_terms = (a.ham == MPV_HAM_HEISENBERG) || (a.h != 0.0);
  for (int t0 = 0; any_terms && t0 < T; t0 += 32 * kTermsPerLane) {
    double2 P[kSamplesPerWarp][kTermsPerLane];
    int E[kSamplesPerWarp][kTermsPerLane];
    double dd[kSamplesPerWarp][kTermsPerLane];
    bool on[kSamplesPerWarp][kTermsPerLane];
#pragma unroll
    for (int r = 0; r < kTermsPerLane; ++r) {
      const int t = t0 + r * 32 + lane;
      const bool inr = t < T;
      int p = 0, qq = 0;
      if (a.ham == MPV_HAM_TFIM) p = inr ? t : 0;
      else if (inr) { p = a.bonds[2 * t]; qq = a.bonds[2 * t + 1]; }
#pragma unroll
      for (int q = 0; q < kSamplesPerWarp; ++q) {
        int d;
        if (a.ham == MPV_HAM_TFIM) d = 1 - 2 * bit_of(q, p);
        else d = bit_of(q, qq) - bit_of(q, p);
        dd[q][r] = (double)d;
        on[q][r] = inr && valid[q] && d != 0;
        P[q][r] = make_double2(1.0, 0.0);
        E[q][r] = 0;
      }
    }
    for (int i = 0; i < M; ++i) {
      double2 tv[kSamplesPerWarp];
#pragma unroll
      for (int q = 0; q < kSamplesPerWarp; ++q) tv[q] = tt[q * M + i];
#pragma unroll
      for (int r = 0; r < kTermsPerLane; ++r) {
        const int t = t0 + r * 32 + lane;
        if (t < T) {
          const double2 c = a.C[(size_t)i * T + t], sv = a.S[(size_t)i * T + t];
#pragma unroll
          for (int q = 0; q < kSamplesPerWarp; ++q) {
            const double2 ts = cmul(tv[q], sv);
            const double2 f = make_double2(fma(dd[q][r], ts.x, c.x), fma(dd[q][r], ts.y, c.y));
            P[q][r] = cmul(P[q][r], f);
          }
        }
      }
      if ((i & 15) == 15) {
#pragma unroll
        for (int r = 0; r < kTermsPerLane; ++r)
#pragma unroll
          for (int q = 0; q < kSamplesPerWarp; ++q) renorm(P[q][r], E[q][r]);
      }
    }
#pragma unroll
    for (int r = 0; r < kTermsPerLane; ++r) {
      const int t = t0 + r * 32 + lane;
#pragma unroll
      for (int q = 0; q < kSamplesPerWarp; ++q) {
        if (!on[q][r]) continue;
        double2 ratio;
        if (a.slow[t]) {
          // log-cosh difference (ref formulation), O(M) complex logs
          double2 lsum = make_double2(0.0, 0.0);
          int p = 0, pq = 0;
          if (a.ham == MPV_HAM_TFIM) p = t;
          else { p = a.bonds[2 * t]; pq = a.bonds[2 * t + 1]; }
          for (int i = 0; i < M; ++i) {
            double2 w = a.w_t[(size_t)p * M + i];
            if (a.ham != MPV_HAM_TFIM) {
              const double2 w2 = a.w_t[(size_t)pq * M + i];
              w = make_double2(w.x - w2.x, w.y - w2.y);
            }
            const double2 z = th[q * M + i];
            const double2 l1 = clogcosh(make_double2(z.x + dd[q][r] * w.x, z.y + dd[q][r] * w.y));
            const double2 l0 = clogcosh(z);
            lsum.x += l1.x - l0.x;
            lsum.y += l1.y - l0.y;
          }
          double2 av = a.ea[2 * t];  // exp(a_t): recover a_t via log-free route below
          (void)av;
          double2 at;
          if (a.ham == MPV_HAM_TFIM) at = a.a[t];
          else at = make_double2(a.a[p].x - a.a[pq].x, a.a[p].y - a.a[pq].y);
          ratio = cexp_(make_double2(lsum.x + dd[q][r] * at.x, lsum.y + dd[q][r] * at.y));
        } else {
          const double2 e = a.ea[2 * t + (dd[q][r] > 0 ? 0 : 1)];
          double2 v = cmul(e, P[q][r]);
          const int k = E[q][r];
          // v * 2^k without overflow in the scale factor
          const int k1 = max(-1000, min(1000, k));
          v.x = ldexp(v.x, k1);
          v.y = ldexp(v.y, k1);
          if (k != k1) {
            v.x = ldexp(v.x, k - k1);
            v.y = ldexp(v.y, k - k1);
          }
          ratio = v;
        }
        sum[q].x += ratio.x;
        sum[q].y += ratio.y;
      }
    }
  }
  const double coef = (a.ham == MPV_HAM_TFIM) ? a.h : 2.0 * a.J;
#pragma unroll
  for (int q = 0; q < kSamplesPerWarp; ++q) {
    const double dg = segment_sum(diag[q], 32);
    const double sr = segment_sum(sum[q].x, 32);
    const double si = segment_sum(sum[q].y, 32);
    if (lane == 0 && valid[q]) {
      const int64_t s = s_base + q;
      const double2 eps = make_double2(a.J * dg + coef * sr, coef * si);
      a.out[s] = eps;
      if ((!isfinite(eps.x) || !isfinite(eps.y)) && a.status) {
        atomicMin((unsigned long long*)&a.status[1], (unsigned long long)s);
        atomicExch((unsigned long long*)&a.status[0], (unsigned long long)MPV_ERR_NONFINITE);
      }
    }
  }
}

}  // namespace mpv
