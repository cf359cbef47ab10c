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

// Scale p by 2^-k (exact), k = biased-exponent of max(|re|, |im|) - 1023;
// accumulate k.  Bit arithmetic only (no libm call).
__device__ __forceinline__ void renorm(double2& p, int& e) {
  const double m = fmax(fabs(p.x), fabs(p.y));
  const int be = (int)((__double_as_longlong(m) >> 52) & 0x7ff);
  if (be == 0 || be == 0x7ff) return;  // zero / subnormal / inf / nan: leave as is
  const int k = be - 1023;
  const double sc = __longlong_as_double((long long)(1023 - k) << 52);  // 2^-k
  p.x *= sc;
  p.y *= sc;
  e += k;
}

// One block = NG groups x ST samples x all terms (NG * ST = SB samples).
// Thread (g, t) owns term t for the ST samples of group g: it keeps ST
// running products in registers and streams its column of the C/S tables
// (the NG threads of a term read the same addresses: one L1 fill).  theta
// is formed per unit with one coalesced load of W_t[k][i] per (site, unit)
// shared by all SB samples (per-site sample masks), then tanh(theta) sits in
// shared memory, read as a broadcast.  Sums over terms are reduced in a fixed
// order (deterministic).
constexpr int kRows = 6;   // C/S rows per staged chunk
constexpr int kMaxSB = 16;  // samples per block (NG * ST)

// Bulk-async (TMA engine) staging of contiguous global chunks into a double
// buffer in shared memory, one mbarrier per buffer.  Thread 0 issues; every
// thread waits; a block barrier after consumption frees the buffer.
struct Stager {
  uint32_t buf_addr[2], bar_addr[2];
  unsigned char* buf[2];
  int uses[2];
  __device__ void init(unsigned char* base, size_t bytes, uint64_t* bars, int tid) {
    for (int b = 0; b < 2; ++b) {
      buf[b] = base + b * bytes;
      buf_addr[b] = (uint32_t)__cvta_generic_to_shared(buf[b]);
      bar_addr[b] = (uint32_t)__cvta_generic_to_shared(bars + b);
      uses[b] = 0;
    }
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_addr[0]));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_addr[1]));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  // one or two copies completing the same buffer
  __device__ void issue(int b, const void* src1, uint32_t bytes1, const void* src2, uint32_t off2, uint32_t bytes2) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_addr[b]), "r"(bytes1 + bytes2)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     buf_addr[b]), "l"(src1), "r"(bytes1), "r"(bar_addr[b]) : "memory");
    if (bytes2)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       buf_addr[b] + off2), "l"(src2), "r"(bytes2), "r"(bar_addr[b]) : "memory");
  }
  __device__ void wait(int b) {
    const uint32_t parity = uses[b] & 1;
    asm volatile(
        "{.reg .pred p;\nWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            bar_addr[b]), "r"(parity) : "memory");
    ++uses[b];
  }
};

// One block = NG groups x ST samples x all terms (SB = NG*ST samples).
// Phase 1: theta = b + W x, thread i owns unit i for all SB samples; W_t
// rows are staged by bulk copies and shared by the block (per-site sample
// bit masks select the adds).  tanh(theta) goes to shared memory.
// Phase 2: thread (g, t) owns term t for the ST samples of group g and keeps
// ST running products of (C + d tanh(theta) S) in registers; C/S rows are
// staged the same way and read conflict-free.  Sums over terms reduce in a
// fixed order (deterministic).
template <int ST>
__global__ void __launch_bounds__(512) energy_kernel(const EnergyArgs a, int NG, int stage_bytes) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int M = a.M, T = a.n_terms, words = a.words, N = a.N;
  const int SB = ST * NG;
  const int TT = (T + 31) / 32 * 32;  // threads per group
  double2* tt = reinterpret_cast<double2*>(smem_raw);                  // [M][SB]
  uint32_t* wsm = reinterpret_cast<uint32_t*>(tt + (size_t)SB * M);    // [SB][32]
  uint32_t* smask = wsm + SB * 32;                                     // [N], padded to 16 B
  double* red = reinterpret_cast<double*>(smask + ((N + 3) / 4) * 4);  // [SB][16 warps][2]
  unsigned char* stage_base = reinterpret_cast<unsigned char*>(red + kMaxSB * 16 * 2);
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage_base + 2 * (size_t)stage_bytes);
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t s0 = (int64_t)blockIdx.x * SB;
  Stager st;
  st.init(stage_base, stage_bytes, bars, tid);

  for (int idx = tid; idx < SB * 32; idx += blockDim.x) {
    const int s = idx >> 5, w = idx & 31;
    wsm[idx] = (w < words && s0 + s < a.B) ? a.bits[(s0 + s) * words + w] : 0u;
  }
  __syncthreads();
  for (int k = tid; k < N; k += blockDim.x) {
    uint32_t m = 0;
    for (int s = 0; s < SB; ++s) m |= ((wsm[s * 32 + (k >> 5)] >> (k & 31)) & 1u) << s;
    smask[k] = m;
  }
  // 0/1 multipliers x[k][s] as doubles (theta phase uses DFMA, no selects)
  double* xk = reinterpret_cast<double*>(stage_base + 2 * (size_t)stage_bytes + 16);  // [N][kMaxSB]
  for (int idx = tid; idx < N * kMaxSB; idx += blockDim.x) {
    const int k = idx / kMaxSB, s2 = idx % kMaxSB;
    xk[idx] = (s2 < SB) ? (double)((wsm[s2 * 32 + (k >> 5)] >> (k & 31)) & 1u) : 0.0;
  }
  // ---- phase 1: theta ----
  {
    const int rW = stage_bytes / (M * (int)sizeof(double2));
    const int nW = (N + rW - 1) / rW;
    auto issueW = [&](int c) {
      const int k0 = c * rW, nr = min(rW, N - k0);
      st.issue(c & 1, a.w_t + (size_t)k0 * M, (uint32_t)(nr * M * sizeof(double2)), nullptr, 0, 0);
    };
    if (tid == 0) {
      issueW(0);
      if (nW > 1) issueW(1);
    }
    __syncthreads();  // masks ready
    double zr[kMaxSB], zi[kMaxSB];
    const int i = tid;
    if (i < M) {
      const double2 b = a.b[i];
#pragma unroll
      for (int s = 0; s < kMaxSB; ++s) { zr[s] = b.x; zi[s] = b.y; }
    }
    for (int c = 0; c < nW; ++c) {
      const int b = c & 1;
      st.wait(b);
      if (i < M) {
        const double2* wr = reinterpret_cast<const double2*>(stage_base + (size_t)b * stage_bytes) + i;
        const int k0 = c * rW, nr = min(rW, N - k0);
        for (int r = 0; r < nr; ++r) {
          const double2 w = wr[r * M];
          const double* xr = xk + (k0 + r) * kMaxSB;
#pragma unroll
          for (int s = 0; s < kMaxSB; ++s) {
            const double x = xr[s];
            zr[s] = fma(x, w.x, zr[s]);
            zi[s] = fma(x, w.y, zi[s]);
          }
        }
      }
      __syncthreads();
      if (tid == 0 && c + 2 < nW) issueW(c + 2);
    }
    if (i < M) {
#pragma unroll
      for (int s = 0; s < kMaxSB; ++s)
        if (s < SB) tt[i * SB + s] = ctanh(make_double2(zr[s], zi[s]));
    }
  }
  __syncthreads();

  auto bit_of = [&](int s, int k) -> int { return (wsm[s * 32 + (k >> 5)] >> (k & 31)) & 1u; };
  const int g = tid / TT, t = tid % TT;
  const bool any_terms = (a.ham == MPV_HAM_HEISENBERG) || (a.h != 0.0);
  double2 ratio[ST];
  double dd[ST];
  double2 P[ST];
  int E[ST];
#pragma unroll
  for (int j = 0; j < ST; ++j) {
    ratio[j] = make_double2(0.0, 0.0);
    dd[j] = 0.0;
    P[j] = make_double2(1.0, 0.0);
    E[j] = 0;
  }
  const bool active = any_terms && g < NG && t < T;
  bool slow = false;
  const double2* tg = tt;
  int p = 0, q = 0;
  if (active) {
    if (a.ham == MPV_HAM_TFIM) p = t;
    else { p = a.bonds[2 * t]; q = a.bonds[2 * t + 1]; }
#pragma unroll
    for (int j = 0; j < ST; ++j) {
      const int s = g * ST + j;
      dd[j] = (a.ham == MPV_HAM_TFIM) ? (double)(1 - 2 * bit_of(s, p)) : (double)(bit_of(s, q) - bit_of(s, p));
    }
    slow = a.slow[t] != 0;
    tg = tt + g * ST;
  }
  // ---- phase 2: products over hidden units ----
  if (any_terms) {
    const int nchunks = (M + kRows - 1) / kRows;
    const uint32_t row_bytes = (uint32_t)T * sizeof(double2);
    auto issueCS = [&](int c) {
      const int r0 = c * kRows, nr = min(kRows, M - r0);
      st.issue(c & 1, a.C + (size_t)r0 * T, nr * row_bytes, a.S + (size_t)r0 * T, kRows * row_bytes, nr * row_bytes);
    };
    if (tid == 0) {
      issueCS(0);
      if (nchunks > 1) issueCS(1);
    }
    for (int c = 0; c < nchunks; ++c) {
      const int b = c & 1;
      st.wait(b);
      if (active && !slow) {
        // shared-space pointers derived from the dynamic smem array (LDS, not generic LD)
        const double2* Cs = reinterpret_cast<const double2*>(stage_base + (size_t)b * stage_bytes) + t;
        const double2* Ss = Cs + kRows * T;
        const int r0 = c * kRows, nr = min(kRows, M - r0);
        const double2* trow = tg + (size_t)r0 * SB;
        for (int r = 0; r < nr; ++r, trow += SB) {
          const double2 cv = Cs[r * T], sv = Ss[r * T];
          // three independent phases over the ST samples: ts = tanh*S, f = C + d ts, P *= f
          double2 f[ST];
#pragma unroll
          for (int j = 0; j < ST; ++j) {
            const double2 tv = trow[j];
            f[j] = make_double2(fma(tv.x, sv.x, -tv.y * sv.y), fma(tv.x, sv.y, tv.y * sv.x));
          }
#pragma unroll
          for (int j = 0; j < ST; ++j) f[j] = make_double2(fma(dd[j], f[j].x, cv.x), fma(dd[j], f[j].y, cv.y));
#pragma unroll
          for (int j = 0; j < ST; ++j) P[j] = cmul(P[j], f[j]);
        }
        if ((c & 3) == 3) {
#pragma unroll
          for (int j = 0; j < ST; ++j) renorm(P[j], E[j]);
        }
      }
      __syncthreads();  // buffer b consumed by every thread
      if (tid == 0 && c + 2 < nchunks) issueCS(c + 2);
    }
  }
  if (active) {
#pragma unroll
    for (int j = 0; j < ST; ++j) {
      const int s = g * ST + j;
      if (s0 + s >= a.B || dd[j] == 0.0) continue;
      if (slow) {
        // log-cosh difference (ref formulation) with theta recomputed here
        double2 lsum = make_double2(0.0, 0.0);
        for (int i = 0; i < M; ++i) {
          double2 z = a.b[i];
          for (int k = 0; k < N; ++k)
            if (bit_of(s, k)) {
              const double2 e = a.w_t[(size_t)k * M + i];
              z.x += e.x;
              z.y += e.y;
            }
          double2 w = a.w_t[(size_t)p * M + i];
          if (a.ham != MPV_HAM_TFIM) {
            const double2 w2 = a.w_t[(size_t)q * M + i];
            w = make_double2(w.x - w2.x, w.y - w2.y);
          }
          const double2 l1 = clogcosh(make_double2(z.x + dd[j] * w.x, z.y + dd[j] * w.y));
          const double2 l0 = clogcosh(z);
          lsum.x += l1.x - l0.x;
          lsum.y += l1.y - l0.y;
        }
        double2 at;
        if (a.ham == MPV_HAM_TFIM) at = a.a[p];
        else at = make_double2(a.a[p].x - a.a[q].x, a.a[p].y - a.a[q].y);
        ratio[j] = cexp_(make_double2(lsum.x + dd[j] * at.x, lsum.y + dd[j] * at.y));
      } else {
        const double2 e = a.ea[2 * t + (dd[j] > 0 ? 0 : 1)];
        double2 v = cmul(e, P[j]);
        const int k = E[j];
        const int k1 = max(-1000, min(1000, k));
        v.x = ldexp(v.x, k1);
        v.y = ldexp(v.y, k1);
        if (k != k1) {
          v.x = ldexp(v.x, k - k1);
          v.y = ldexp(v.y, k - k1);
        }
        ratio[j] = v;
      }
    }
  }
  // fixed-order reduction: warp butterfly, then the group's warps in order
  const int wg = t >> 5;  // warp index within the group
#pragma unroll
  for (int j = 0; j < ST; ++j) {
    const double vr = segment_sum(ratio[j].x, 32), vi = segment_sum(ratio[j].y, 32);
    if (lane == 0 && g < NG) {
      red[((g * ST + j) * 16 + wg) * 2] = vr;
      red[((g * ST + j) * 16 + wg) * 2 + 1] = vi;
    }
  }
  __syncthreads();
  if (tid < SB && s0 + tid < a.B) {
    const int s = tid;
    double er = 0.0, ei = 0.0;
    if (any_terms)
      for (int w = 0; w < TT / 32; ++w) {
        er += red[(s * 16 + w) * 2];
        ei += red[(s * 16 + w) * 2 + 1];
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

constexpr int kEnergyST = 8;  // samples per thread

}  // namespace mpv
