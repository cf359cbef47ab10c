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

// One block = SB samples x all terms.  Thread t owns term t (and t + blockDim,
// ...), keeps the SB running products in registers and streams its column
// of the C/S tables once per block (each load reused by SB samples); the
// SB x M table of tanh(theta) sits in shared memory and is read as a
// broadcast.  Sums over terms are reduced in a fixed order (deterministic).
template <int SB>
__global__ void __launch_bounds__(512) energy_kernel(const EnergyArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int M = a.M, T = a.n_terms, words = a.words;
  double2* tt = reinterpret_cast<double2*>(smem_raw);                 // [SB][M]
  uint32_t* wsm = reinterpret_cast<uint32_t*>(tt + (size_t)SB * M);   // [SB][32]
  double* red = reinterpret_cast<double*>(wsm + SB * 32);             // [SB][32 warps][2]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int64_t s0 = (int64_t)blockIdx.x * SB;

  for (int idx = tid; idx < SB * 32; idx += blockDim.x) {
    const int s = idx >> 5, w = idx & 31;
    wsm[idx] = (w < words && s0 + s < a.B) ? a.bits[(s0 + s) * words + w] : 0u;
  }
  __syncthreads();
  for (int idx = tid; idx < SB * M; idx += blockDim.x) {
    const int s = idx / M, i = idx % M;
    double2 z = a.b[i];
    for (int w = 0; w < words; ++w) {
      uint32_t wd = wsm[s * 32 + w];
      while (wd) {
        const int k = w * 32 + __ffs(wd) - 1;
        wd &= wd - 1;
        const double2 e = a.w_t[(size_t)k * M + i];
        z.x += e.x;
        z.y += e.y;
      }
    }
    tt[idx] = ctanh(z);
  }
  __syncthreads();

  auto bit_of = [&](int s, int k) -> int { return (wsm[s * 32 + (k >> 5)] >> (k & 31)) & 1u; };
  double sr[SB], si[SB];
#pragma unroll
  for (int s = 0; s < SB; ++s) sr[s] = si[s] = 0.0;
  const bool any_terms = (a.ham == MPV_HAM_HEISENBERG) || (a.h != 0.0);
  for (int t = tid; any_terms && t < T; t += blockDim.x) {
    int p, q = 0;
    if (a.ham == MPV_HAM_TFIM) p = t;
    else { p = a.bonds[2 * t]; q = a.bonds[2 * t + 1]; }
    double dd[SB];
    double2 P[SB];
    int E[SB];
#pragma unroll
    for (int s = 0; s < SB; ++s) {
      dd[s] = (a.ham == MPV_HAM_TFIM) ? (double)(1 - 2 * bit_of(s, p)) : (double)(bit_of(s, q) - bit_of(s, p));
      P[s] = make_double2(1.0, 0.0);
      E[s] = 0;
    }
    const bool slow = a.slow[t] != 0;
    if (!slow) {
      const double2* Cc = a.C + t;
      const double2* Sc = a.S + t;
      for (int i = 0; i < M; ++i) {
        const double2 c = Cc[(size_t)i * T], sv = Sc[(size_t)i * T];
#pragma unroll
        for (int s = 0; s < SB; ++s) {
          const double2 tv = tt[s * M + i];
          const double2 ts = cmul(tv, sv);
          P[s] = cmul(P[s], make_double2(fma(dd[s], ts.x, c.x), fma(dd[s], ts.y, c.y)));
        }
        if ((i & 15) == 15) {
#pragma unroll
          for (int s = 0; s < SB; ++s) renorm(P[s], E[s]);
        }
      }
    }
#pragma unroll
    for (int s = 0; s < SB; ++s) {
      if (s0 + s >= a.B || dd[s] == 0.0) continue;
      double2 ratio;
      if (slow) {
        // log-cosh difference (ref formulation) with theta recomputed here
        double2 lsum = make_double2(0.0, 0.0);
        for (int i = 0; i < M; ++i) {
          double2 z = a.b[i];
          for (int w = 0; w < words; ++w) {
            uint32_t wd = wsm[s * 32 + w];
            while (wd) {
              const int k = w * 32 + __ffs(wd) - 1;
              wd &= wd - 1;
              const double2 e = a.w_t[(size_t)k * M + i];
              z.x += e.x;
              z.y += e.y;
            }
          }
          double2 w = a.w_t[(size_t)p * M + i];
          if (a.ham != MPV_HAM_TFIM) {
            const double2 w2 = a.w_t[(size_t)q * M + i];
            w = make_double2(w.x - w2.x, w.y - w2.y);
          }
          const double2 l1 = clogcosh(make_double2(z.x + dd[s] * w.x, z.y + dd[s] * w.y));
          const double2 l0 = clogcosh(z);
          lsum.x += l1.x - l0.x;
          lsum.y += l1.y - l0.y;
        }
        double2 at;
        if (a.ham == MPV_HAM_TFIM) at = a.a[p];
        else at = make_double2(a.a[p].x - a.a[q].x, a.a[p].y - a.a[q].y);
        ratio = cexp_(make_double2(lsum.x + dd[s] * at.x, lsum.y + dd[s] * at.y));
      } else {
        const double2 e = a.ea[2 * t + (dd[s] > 0 ? 0 : 1)];
        double2 v = cmul(e, P[s]);
        const int k = E[s];
        const int k1 = max(-1000, min(1000, k));
        v.x = ldexp(v.x, k1);
        v.y = ldexp(v.y, k1);
        if (k != k1) {
          v.x = ldexp(v.x, k - k1);
          v.y = ldexp(v.y, k - k1);
        }
        ratio = v;
      }
      sr[s] += ratio.x;
      si[s] += ratio.y;
    }
  }
  // fixed-order reduction over threads: warp butterfly, then warps in order
#pragma unroll
  for (int s = 0; s < SB; ++s) {
    const double vr = segment_sum(sr[s], 32), vi = segment_sum(si[s], 32);
    if (lane == 0) {
      red[(s * 32 + warp) * 2] = vr;
      red[(s * 32 + warp) * 2 + 1] = vi;
    }
  }
  __syncthreads();
  if (tid < SB && s0 + tid < a.B) {
    const int s = tid;
    double er = 0.0, ei = 0.0;
    for (int w = 0; w < nwarps; ++w) {
      er += red[(s * 32 + w) * 2];
      ei += red[(s * 32 + w) * 2 + 1];
    }
    double diag = 0.0;  // ref vmc.py:52-57
    for (int b = 0; b < a.n_bonds; ++b) {
      const int xp = bit_of(s, a.bonds[2 * b]), xq = bit_of(s, a.bonds[2 * b + 1]);
      diag += (double)((1 - 2 * xp) * (1 - 2 * xq));
    }
    const double coef = (a.ham == MPV_HAM_TFIM) ? a.h : 2.0 * a.J;
    const double2 eps = make_double2(a.J * diag + coef * er, coef * ei);
    a.out[s0 + s] = eps;
    if ((!isfinite(eps.x) || !isfinite(eps.y)) && a.status) {
      atomicMin((unsigned long long*)&a.status[1], (unsigned long long)(s0 + s));
      atomicExch((unsigned long long*)&a.status[0], (unsigned long long)MPV_ERR_NONFINITE);
    }
  }
}

constexpr int kEnergySB = 8;

}  // namespace mpv
