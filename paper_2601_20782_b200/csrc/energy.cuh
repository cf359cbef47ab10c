// f64 local energies (ref: vmc.py:52-108 local_energies, _diagonal_energy).
//
//   eps(x) = J sum_bonds s_i s_j + c * sum_terms psi(x')/psi(x),  s = 1 - 2 bit
//   TFIM:       terms = all N single flips, c = h
//   Heisenberg: terms = bonds (i,j) with x_i != x_j (swap), c = 2J
//
// The reference forms every connected x' and runs a full forward on it
// (O(N * N * M) per sample).  Here a ratio is an O(M) product over hidden
// units of cosh(theta_i + d w_i) / cosh(theta_i) = cosh(w_i) (1 + d tanh(theta_i) tau_i),
// tau = tanh(w), tabulated once per parameter snapshot (w = W_:k for a flip of
// k, w = W_:i - W_:j for a swap of bond (i,j); d = +-1).  The term constant
// exp(d a) prod_i cosh(w_i) (mantissa + binary exponent) is tabulated too, so a
// factor costs one complex multiply plus one complex multiply-add (8 FP64
// ops).  theta = b + W x is a 0/1 x f64 GEMM on the FP64 tensor cores (DMMA).
// Terms with |Re w| > kSafeRe (tanh ~ +-1 cancels in 1 - tanh tanh) or
// |cosh w| < kMinCosh (tau near a pole) use the log-cosh difference instead.
#pragma once
#include "common.cuh"

namespace mpv {

constexpr double kSafeRe = 4.0;
constexpr double kMinCosh2 = 1.0 / 16.0;  // |cosh w|^2 below this -> slow path

struct EnergyArgs {
  int N, M, words, ham, n_bonds, n_terms;
  const double2 *a, *b, *w_t;  // w_t [N][M]
  const int32_t* bonds;        // [n_bonds][2]
  double J, h;
  const double2* tau;   // [M][n_terms]: tanh(w)
  const double2* ea;    // [n_terms][2]: exp(+-a_t) prod_i cosh(w_it), mantissa
  const int32_t* ec;    // [n_terms]: binary exponent of prod_i cosh(w_it)
  const int32_t* slow;  // [n_terms]
  const double* term_coef;  // [n_terms] off-diagonal coefficient (NULL: h for TFIM, 2J for Heisenberg)
  const double* bond_j;     // [n_bonds] diagonal couplings (NULL: J for every bond)
  const double* wp;     // [roundup(N, 8)][2M + 8]: W_t in the staging layout
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

__device__ __forceinline__ double2 term_w(const EnergyArgs& a, int t, int i) {
  if (a.ham == MPV_HAM_TFIM) return a.w_t[(size_t)t * a.M + i];
  const int p = a.bonds[2 * t], q = a.bonds[2 * t + 1];
  const double2 wp = a.w_t[(size_t)p * a.M + i], wq = a.w_t[(size_t)q * a.M + i];
  return make_double2(wp.x - wq.x, wp.y - wq.y);
}

__global__ void energy_tables_kernel(const EnergyArgs a, double2* tau, double2* ea, int32_t* ec, int32_t* slow,
                                     double* wp) {
  const int T = a.n_terms;
  // W_t copied to the staging layout: rows padded to a multiple of 8 (zero
  // rows), pitch 2M + 8 doubles (zero pad)
  const int pitch = 2 * a.M + 8, np = (a.N + 7) / 8 * 8;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (int64_t)np * pitch;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx / pitch), c = (int)(idx % pitch);
    wp[idx] = (k < a.N && c < 2 * a.M) ? reinterpret_cast<const double*>(a.w_t)[(size_t)k * 2 * a.M + c] : 0.0;
  }
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (int64_t)a.M * T;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / T), t = (int)(idx % T);
    tau[(size_t)i * T + t] = ctanh(term_w(a, t, i));
  }
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    double2 av;
    if (a.ham == MPV_HAM_TFIM) {
      av = a.a[t];
    } else {
      const int p = a.bonds[2 * t], q = a.bonds[2 * t + 1];
      av = make_double2(a.a[p].x - a.a[q].x, a.a[p].y - a.a[q].y);
    }
    int bad = 0, e = 0;
    double2 cp = make_double2(1.0, 0.0);
    for (int i = 0; i < a.M; ++i) {
      const double2 w = term_w(a, t, i);
      const double2 c = ccosh(w);
      bad |= fabs(w.x) > kSafeRe || c.x * c.x + c.y * c.y < kMinCosh2;
      cp = cmul(cp, c);
      renorm(cp, e);
    }
    ea[2 * t] = cmul(cexp_(av), cp);
    ea[2 * t + 1] = cmul(cexp_(make_double2(-av.x, -av.y)), cp);
    ec[t] = e;
    slow[t] = bad;
  }
}

// Block layout (dynamic shared memory, 16-B aligned offsets):
//   pool:  tt [M][SB] double2 (theta, then tanh theta) followed by nbt tau
//          staging buffers of `rows` rows.  During phase 1 the whole pool is
//          nbw W staging buffers of 8 padded rows; after phase 2 it holds the
//          per-(sample, term) ratios [SB][T] double2.
//   wsm [SB][32] packed sample bits, smask [energy_mask_pad(N)] per-site
//   sample masks (zero beyond N), 16 mbarriers (two Pipes).
constexpr int kMaxSB = 16;  // samples per block
constexpr int kWRows = 8;   // W rows per staged chunk (two DMMA k-steps)
constexpr int kMaxBufs = 8; // ring depth limit per Pipe

struct EnergyPlan {
  int SB, rows, nbt, nbw;          // samples/block, tau rows/chunk, tau buffers, W buffers
  int tbuf_bytes, wbuf_bytes, pool_bytes;
  int skip;  // profiling only (MPV_ENERGY_SKIP): bit 0 phase 1, bit 1 tanh, bit 2 phase 2, bit 3 ratios, bit 4 sums
};
__host__ __device__ inline int energy_mask_pad(int N) { return (N + 15) / 16 * 16 + 16; }
__host__ __device__ inline int energy_w_pitch(int M) { return 2 * M + 8; }  // doubles per staged W row
__host__ __device__ inline int energy_w_rows(int N) { return (N + kWRows - 1) / kWRows * kWRows; }
// fills pool/buffer sizes; returns the dynamic shared memory bytes
inline size_t energy_plan(int N, int M, int T, int SB, int rows, int nbt, EnergyPlan* p) {
  p->SB = SB;
  p->rows = rows;
  p->nbt = nbt;
  p->tbuf_bytes = rows * T * 16;
  p->wbuf_bytes = kWRows * energy_w_pitch(M) * 8;
  size_t pool = (size_t)SB * M * 16 + (size_t)nbt * p->tbuf_bytes;
  if ((size_t)SB * T * 16 > pool) pool = (size_t)SB * T * 16;
  if ((size_t)2 * p->wbuf_bytes > pool) pool = (size_t)2 * p->wbuf_bytes;
  pool = (pool + 127) / 128 * 128;
  p->pool_bytes = (int)pool;
  p->nbw = (int)(pool / p->wbuf_bytes);
  if (p->nbw > kMaxBufs) p->nbw = kMaxBufs;
  // + the Heisenberg compaction's per-term active masks and unit offsets
  return pool + (size_t)SB * 32 * 4 + (size_t)energy_mask_pad(N) * 4 + 4 * kMaxBufs * 8 + (size_t)(2 * T + 1) * 4;
}

// Bulk-async (TMA engine) ring of nb <= kMaxBufs buffers in shared memory.  Per
// buffer a "full" mbarrier (count 1 + transaction bytes; thread 0 issues) and
// an "empty" mbarrier (one arrival per warp once the warp has read the chunk).
// Chunk c uses buffer c % nb, that buffer's (c / nb)-th completion, so waits
// are on parity (c / nb) & 1 (tracked incrementally by Pos).  No block-wide barrier per chunk: only the
// producer thread waits for the slowest warp before refilling a buffer.
struct Pipe {
  uint32_t buf_addr0, bar_addr0, bytes;  // bars: full[kMaxBufs], empty[kMaxBufs]
  int nb;
  __device__ void init(const unsigned char* base, uint32_t buf_bytes, int n_buf, const uint64_t* bars) {
    buf_addr0 = (uint32_t)__cvta_generic_to_shared(base);
    bar_addr0 = (uint32_t)__cvta_generic_to_shared(bars);
    bytes = buf_bytes;
    nb = n_buf;
  }
  __device__ static void init_bars(const uint64_t* bars, int n_pipes, int n_warps) {
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(bars);
    for (int p = 0; p < n_pipes; ++p)
      for (int k = 0; k < 2 * kMaxBufs; ++k)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b0 + 8 * (2 * kMaxBufs * p + k)),
                     "r"(k < kMaxBufs ? 1 : n_warps));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __device__ uint32_t full(int b) const { return bar_addr0 + 8 * b; }
  __device__ uint32_t empty(int b) const { return bar_addr0 + 8 * kMaxBufs + 8 * b; }
  __device__ uint32_t buf(int b) const { return buf_addr0 + b * bytes; }
  __device__ void expect(int b, uint32_t total) const {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full(b)), "r"(total) : "memory");
  }
  __device__ void copy(int b, uint32_t dst_off, const void* src, uint32_t n) const {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     buf(b) + dst_off), "l"(src), "r"(n), "r"(full(b)) : "memory");
  }
  __device__ static void wait_parity(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{.reg .pred p;\nWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            bar), "r"(parity) : "memory");
  }
  // consumers: chunk in buffer b, that buffer's use with parity ph
  __device__ void wait_full(int b, uint32_t ph) const { wait_parity(full(b), ph); }
  __device__ void release(int b, int lane) const {
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty(b)) : "memory");
  }
  // producer: buffer b was released by every warp for its use with parity ph
  __device__ void wait_empty(int b, uint32_t ph) const { wait_parity(empty(b), ph); }
  // ring position of a chunk sequence: slot and use parity, advanced per chunk
  struct Pos {
    int slot;
    uint32_t ph;
  };
  __device__ void advance(Pos& p) const {
    if (++p.slot == nb) {
      p.slot = 0;
      p.ph ^= 1u;
    }
  }
};

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// tanh(x+iy) = (sinh 2x + i sin 2y) / (cosh 2x + cos 2y) with one expm1, one
// sincos and one division: m = expm1(2|x|), sinh 2|x| = m (m + 2) / (2 (m + 1)),
// cosh 2|x| = 1 + m^2 / (2 (m + 1)), 1 + cos 2y = 2 cos^2 y, so
//   tanh = (m (m + 2) + i 4 (m + 1) sin y cos y) / (4 (m + 1) cos^2 y + m^2)
// (a sum of non-negative terms in the denominator: no cancellation).
__device__ __forceinline__ double2 ctanh_fast(double2 z) {
  const double ax = fmin(fabs(z.x), 40.0);  // tanh(40) == 1 in f64
  const double m = expm1(2.0 * ax);
  double s, c;
  sincos(z.y, &s, &c);
  const double m1 = 4.0 * (m + 1.0);
  const double inv = 1.0 / fma(m1 * c, c, m * m);
  return make_double2(copysign(m * (m + 2.0) * inv, z.x), m1 * s * c * inv);
}

// Ratio of term t for one sample through the log-cosh difference (ref
// formulation, rbm.py:130-140), theta recomputed from W: the path for terms
// whose tau table would cancel or blow up (slow[t]).
__device__ __noinline__ double2 slow_ratio(int N, int M, int ham, const double2* __restrict__ av,
                                           const double2* __restrict__ bv, const double2* __restrict__ w_t,
                                           const int32_t* __restrict__ bonds, const uint32_t* xbits, int t, double d) {
  double2 lsum = make_double2(0.0, 0.0);
  int p = t, q = 0;
  if (ham != MPV_HAM_TFIM) {
    p = bonds[2 * t];
    q = bonds[2 * t + 1];
  }
  for (int i = 0; i < M; ++i) {
    double2 z = bv[i];
    for (int k = 0; k < N; ++k)
      if ((xbits[k >> 5] >> (k & 31)) & 1u) {
        const double2 e = w_t[(size_t)k * M + i];
        z.x += e.x;
        z.y += e.y;
      }
    double2 w = w_t[(size_t)p * M + i];
    if (ham != MPV_HAM_TFIM) {
      const double2 w2 = w_t[(size_t)q * M + i];
      w = make_double2(w.x - w2.x, w.y - w2.y);
    }
    const double2 l1 = clogcosh(make_double2(z.x + d * w.x, z.y + d * w.y));
    const double2 l0 = clogcosh(z);
    lsum.x += l1.x - l0.x;
    lsum.y += l1.y - l0.y;
  }
  double2 at;
  if (ham == MPV_HAM_TFIM) at = av[t];
  else at = make_double2(av[p].x - av[q].x, av[p].y - av[q].y);
  return cexp_(make_double2(lsum.x + d * at.x, lsum.y + d * at.y));
}

// One block = SB samples x all terms.  Thread (g, t) = (tid / T, tid % T)
// owns term t for the ST samples of group g (groups and terms are flattened
// over the block, so only the last warp has idle lanes).
// Phase 1: theta[s][i] = b_i + sum_k x[s][k] W_t[k][i] as a real GEMM
//   X[SB x N] (0/1) . Wr[N x 2M] on DMMA m8n8k4 tiles; W_t rows are staged by
//   bulk copies into a padded pitch (2M + 8 doubles: the four k-rows of a
//   fragment land on disjoint bank halves); A fragments come from the per-site
//   sample masks.  The D fragment (row s, cols 2i, 2i+1) is exactly theta_i(s).
//   tanh(theta) is then formed in place by one rolled loop.
// Phase 2: each thread keeps ST running products of (1 + d tanh(theta) tau)
//   in registers; tau rows are staged by bulk copies and read per lane,
//   tanh(theta) as broadcasts.  Ratios go to shared memory and one warp per
//   sample sums the terms in a fixed order (deterministic).
// ST samples per thread, KT DMMA n-tiles per warp, launch bounds (TMAX threads, MINB blocks/SM)
template <int ST, int KT, int TMAX, int MINB, bool COMPACT>
__global__ void __launch_bounds__(TMAX, MINB) energy_kernel(const EnergyArgs a, const EnergyPlan pl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int M = a.M, T = a.n_terms, words = a.words, N = a.N;
  const int SB = pl.SB, NG = SB / ST, rows = pl.rows;
  double2* tt = reinterpret_cast<double2*>(smem_raw);  // [M][SB]
  unsigned char* tstage = smem_raw + (size_t)SB * M * sizeof(double2);
  uint32_t* wsm = reinterpret_cast<uint32_t*>(smem_raw + pl.pool_bytes);  // [SB][32]
  uint32_t* smask = wsm + SB * 32;                                         // [energy_mask_pad(N)]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smask + energy_mask_pad(N));  // 4 * kMaxBufs
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int64_t s0 = (int64_t)blockIdx.x * SB;
  if (tid == 0) Pipe::init_bars(bars, 2, nwarps);
  Pipe pw, pt;
  pw.init(smem_raw, (uint32_t)pl.wbuf_bytes, pl.nbw, bars);
  pt.init(tstage, (uint32_t)pl.tbuf_bytes, pl.nbt, bars + 2 * kMaxBufs);
  const int pitch = energy_w_pitch(M);
  const int nW = energy_w_rows(N) / kWRows;
  auto issueW = [&](int c, int b) {
    pw.expect(b, (uint32_t)pl.wbuf_bytes);
    pw.copy(b, 0, a.wp + (size_t)c * kWRows * pitch, (uint32_t)pl.wbuf_bytes);
  };
  __syncthreads();  // barriers initialised
  if (tid == 0 && !(pl.skip & 1))
    for (int c = 0; c < min(pl.nbw, nW); ++c) issueW(c, c);

  for (int idx = tid; idx < SB * 32; idx += blockDim.x) {
    const int s = idx >> 5, w = idx & 31;
    wsm[idx] = (w < words && s0 + s < a.B) ? a.bits[(s0 + s) * words + w] : 0u;
  }
  __syncthreads();
  for (int k = tid; k < energy_mask_pad(N); k += blockDim.x) {
    uint32_t m = 0;
    if (k < N)
      for (int s = 0; s < SB; ++s) m |= ((wsm[s * 32 + (k >> 5)] >> (k & 31)) & 1u) << s;
    smask[k] = m;
  }
  __syncthreads();
  // ---- phase 1: theta on DMMA (one pass: the launch gives every warp <= KT tiles) ----
  const int NT = (M + 3) / 4;  // n-tiles of 8 real columns (4 units)
  const int MT = SB / 8;       // m-tiles of 8 samples
  const int qr = lane & 3, qc = lane >> 2;
  double acc[KT][2][2];
  int col[KT];  // B column of tile j (clamped: surplus tiles compute and are dropped)
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    const int nt = warp + j * nwarps;
    col[j] = min(nt, NT - 1) * 8 + qc;
    const int i = nt * 4 + qr;
    const double2 bi = i < M ? a.b[i] : make_double2(0.0, 0.0);
#pragma unroll
    for (int m = 0; m < 2; ++m) { acc[j][m][0] = bi.x; acc[j][m][1] = bi.y; }
  }
  Pipe::Pos wpos{0, 0u};
  for (int c = 0; c < ((pl.skip & 1) ? 0 : nW); ++c) {
    pw.wait_full(wpos.slot, wpos.ph);
    const double* wbuf = reinterpret_cast<const double*>(smem_raw + (size_t)wpos.slot * pl.wbuf_bytes);
#pragma unroll
    for (int kk = 0; kk < kWRows; kk += 4) {
      const double* brow = wbuf + (kk + qr) * pitch;
      double bf[KT];
#pragma unroll
      for (int j = 0; j < KT; ++j) bf[j] = brow[col[j]];
      const uint32_t mk = smask[c * kWRows + kk + qr];  // zero past N
      double af[2];
#pragma unroll
      for (int m = 0; m < 2; ++m)
        af[m] = __hiloint2double((int)(((mk >> (m * 8 + qc)) & 1u) * 0x3ff00000u), 0);
#pragma unroll
      for (int j = 0; j < KT; ++j) dmma_8x8x4(acc[j][0][0], acc[j][0][1], af[0], bf[j]);
      if (MT > 1) {
#pragma unroll
        for (int j = 0; j < KT; ++j) dmma_8x8x4(acc[j][1][0], acc[j][1][1], af[1], bf[j]);
      }
    }
    pw.release(wpos.slot, lane);
    if (tid == 0 && c + pl.nbw < nW) {
      pw.wait_empty(wpos.slot, wpos.ph);
      issueW(c + pl.nbw, wpos.slot);
    }
    pw.advance(wpos);
  }
  __syncthreads();  // every W read done: the pool is free
  const bool any_terms = (a.ham == MPV_HAM_HEISENBERG) || (a.h != 0.0);
  const int nchunks = (M + rows - 1) / rows;
  const uint32_t trow_bytes = (uint32_t)T * sizeof(double2);
  auto issueT = [&](int c, int b) {
    const int r0 = c * rows, nr = min(rows, M - r0);
    pt.expect(b, nr * trow_bytes);
    pt.copy(b, 0, a.tau + (size_t)r0 * T, nr * trow_bytes);
  };
  if (any_terms && !(pl.skip & 4) && tid == 0)
    for (int c = 0; c < min(pl.nbt, nchunks); ++c) issueT(c, c);
  // D fragment (row s = m*8 + qc, cols 2i, 2i+1) = theta_i(s): tanh formed in
  // registers (the lane's 2 KT fragments are independent chains) -> tt[i][s]
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    const int nt = warp + j * nwarps, i = nt * 4 + qr;
    if (nt < NT && i < M) {
#pragma unroll
      for (int m = 0; m < 2; ++m)
        if (m < MT) {
          const double2 z = make_double2(acc[j][m][0], acc[j][m][1]);
          tt[i * SB + m * 8 + qc] = (pl.skip & 2) ? z : ctanh_fast(z);
        }
    }
  }
  __syncthreads();

  auto bit_of = [&](int s, int k) -> int { return (wsm[s * 32 + (k >> 5)] >> (k & 31)) & 1u; };
  // Heisenberg / J1-J2: a (sample, bond) pair with aligned spins (d = 0) has no
  // off-diagonal term (about half of them).  The active pairs of each bond are
  // packed into units of ST samples, term-major, one unit per thread, so whole
  // warps at the end of the block idle instead of half the lanes of every warp.
  // TFIM: every pair is active; thread (g, t) takes samples g ST .. g ST + ST - 1.
  constexpr bool compact = COMPACT;  // launched for Heisenberg / J1-J2 terms
  uint32_t* cmask = reinterpret_cast<uint32_t*>(bars + 4 * kMaxBufs);  // [T] active samples per term
  int* coff = reinterpret_cast<int*>(cmask + T);                       // [T + 1] first unit per term
  if constexpr (compact) {
    for (int x = tid; x < T; x += blockDim.x) {
      const int p = a.bonds[2 * x], q = a.bonds[2 * x + 1];
      uint32_t m = 0;
      for (int ss = 0; ss < SB; ++ss)
        if (s0 + ss < a.B && bit_of(ss, p) != bit_of(ss, q)) m |= 1u << ss;
      cmask[x] = m;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of ceil(active / ST) over the terms
      int carry = 0;
      for (int x0 = 0; x0 < T; x0 += 32) {
        const int x = x0 + lane;
        const int cnt = x < T ? (__popc(cmask[x]) + ST - 1) / ST : 0;
        int inc = cnt;
        for (int off = 1; off < 32; off <<= 1) {
          const int y = __shfl_up_sync(kFull, inc, off);
          if (lane >= off) inc += y;
        }
        if (x < T) coff[x] = carry + inc - cnt;
        carry += __shfl_sync(kFull, inc, 31);
      }
      if (lane == 0) coff[T] = carry;
    }
    __syncthreads();
  }
  int g = 0, t = 0;
  int sidx[ST];       // block sample of slot j
  uint32_t live = 0;  // bit j: slot j carries an active pair
  bool have = false;
  if constexpr (compact) {
    if (tid < coff[T]) {
      int lo = 0, hi = T - 1;  // last term whose first unit is <= tid
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (coff[mid] <= tid) lo = mid;
        else hi = mid - 1;
      }
      t = lo;
      have = true;
      uint32_t m = cmask[t];
      for (int k = (tid - coff[t]) * ST; k > 0; --k) m &= m - 1;
#pragma unroll
      for (int j = 0; j < ST; ++j) {
        sidx[j] = m ? __ffs(m) - 1 : 0;
        live |= (m ? 1u : 0u) << j;
        m &= m - 1;
      }
    }
  } else {
    g = tid / T;
    t = tid - g * T;
    have = g < NG;
#pragma unroll
    for (int j = 0; j < ST; ++j) {
      sidx[j] = g * ST + j;
      live |= 1u << j;
    }
  }
  double2 P[ST];
  int E[ST];
  uint32_t sg[ST];  // sign bit of d on the high word (d = -1 -> flip tanh(theta))
  uint32_t nz = 0;       // bit j: d_j != 0
  uint32_t sg_bits = 0;  // bit j: d_j < 0
#pragma unroll
  for (int j = 0; j < ST; ++j) {
    P[j] = make_double2(1.0, 0.0);
    E[j] = 0;
    sg[j] = 0;
  }
  const bool active = any_terms && have;
  bool slow = false;
  if (active) {
    int p = t, q = 0;
    if (a.ham != MPV_HAM_TFIM) { p = a.bonds[2 * t]; q = a.bonds[2 * t + 1]; }
#pragma unroll
    for (int j = 0; j < ST; ++j) {
      const int s = sidx[j];
      const int d = (a.ham == MPV_HAM_TFIM) ? 1 - 2 * bit_of(s, p) : bit_of(s, q) - bit_of(s, p);
      sg[j] = d < 0 ? 0x80000000u : 0u;
      sg_bits |= (d < 0 ? 1u : 0u) << j;
      nz |= (d != 0 && ((live >> j) & 1u) ? 1u : 0u) << j;
    }
    slow = a.slow[t] != 0;
  }
  // ---- phase 2: products over hidden units ----
  if (any_terms && !(pl.skip & 4)) {
    Pipe::Pos tpos{0, 0u};
    for (int c = 0; c < nchunks; ++c) {
      pt.wait_full(tpos.slot, tpos.ph);
      if (active && !slow) {
        // shared-space pointers derived from the dynamic smem array (LDS, not generic LD)
        const double2* tp = reinterpret_cast<const double2*>(tstage + (size_t)tpos.slot * pl.tbuf_bytes) + t;
        const int r0 = c * rows, nr = min(rows, M - r0);
        const double2* vp = tt + (size_t)r0 * SB + (compact ? 0 : g * ST);
#pragma unroll 2
        for (int r = 0; r < nr; ++r) {
          // all loads of the row first (tau per lane, tanh(theta) broadcasts)
          const double2 tau = *tp;
          double2 tv[ST];
#pragma unroll
          for (int j = 0; j < ST; ++j) tv[j] = vp[compact ? sidx[j] : j];
          tp += T;
          vp += SB;
          // u = (d tanh theta) tau, P += P u
#pragma unroll
          for (int j = 0; j < ST; ++j) {
            tv[j].x = __hiloint2double(__double2hiint(tv[j].x) ^ (int)sg[j], __double2loint(tv[j].x));
            tv[j].y = __hiloint2double(__double2hiint(tv[j].y) ^ (int)sg[j], __double2loint(tv[j].y));
            const double2 u = cmul(tv[j], tau);
            const double px = P[j].x, py = P[j].y;
            P[j].x = fma(px, u.x, fma(-py, u.y, px));
            P[j].y = fma(px, u.y, fma(py, u.x, py));
          }
        }
        if (c & 1) {
#pragma unroll
          for (int j = 0; j < ST; ++j) renorm(P[j], E[j]);
        }
      }
      pt.release(tpos.slot, lane);
      if (tid == 0 && c + pl.nbt < nchunks) {
        pt.wait_empty(tpos.slot, tpos.ph);
        issueT(c + pl.nbt, tpos.slot);
      }
      pt.advance(tpos);
    }
  }
  __syncthreads();  // all reads of tt and the staging buffers done
  // R [SB][T] (reuses tt + staging: all reads of them are done): thread (g, t)
  // writes coef_t * ratio_t plus the diagonal of bonds b = t, t + T, ...
  // (ref vmc.py:52-57: J_b s_p s_q), so one fixed-order sum over t gives eps.
  double2* R = tt;
  // diagonal of bonds x, x + T, ... (bond x's J s_p s_q rides on term x's entry)
  auto diag_of = [&](int s, int x) {
    double dg = 0.0;
    for (int b = x; b < a.n_bonds; b += T)
      dg += (bit_of(s, a.bonds[2 * b]) ^ bit_of(s, a.bonds[2 * b + 1])) ? -(a.bond_j ? a.bond_j[b] : a.J)
                                                                        : (a.bond_j ? a.bond_j[b] : a.J);
    return dg;
  };
  if (COMPACT && !(pl.skip & 8)) {  // pairs without an off-diagonal term: the diagonal only
    for (int idx = tid; idx < SB * T; idx += blockDim.x) {
      const int ss = idx / T, x = idx - ss * T;
      if (!((cmask[x] >> ss) & 1u)) R[ss * T + x] = make_double2(diag_of(ss, x), 0.0);
    }
  }
  if (have && !(pl.skip & 8)) {
    // the first two bonds of this term in registers (TFIM: 2N bonds over N terms)
    const int b0 = t, b1 = t + T;
    const bool h0 = b0 < a.n_bonds, h1 = b1 < a.n_bonds;
    const int p0 = h0 ? a.bonds[2 * b0] : 0, q0 = h0 ? a.bonds[2 * b0 + 1] : 0;
    const int p1 = h1 ? a.bonds[2 * b1] : 0, q1 = h1 ? a.bonds[2 * b1 + 1] : 0;
    const double j0 = h0 ? (a.bond_j ? a.bond_j[b0] : a.J) : 0.0;
    const double j1 = h1 ? (a.bond_j ? a.bond_j[b1] : a.J) : 0.0;
    const double ct = a.term_coef ? a.term_coef[t] : (a.ham == MPV_HAM_TFIM ? a.h : 2.0 * a.J);
    const double2 eap = a.ea[2 * t], eam = a.ea[2 * t + 1];
    const int ect = a.ec[t];
    // diagonal of bonds t, t + T (and further bonds, not in practice)
    auto diag = [&](int s) {
      double dg = 0.0;
      if (h0) dg += (bit_of(s, p0) ^ bit_of(s, q0)) ? -j0 : j0;
      if (h1) dg += (bit_of(s, p1) ^ bit_of(s, q1)) ? -j1 : j1;
      for (int b = t + 2 * T; b < a.n_bonds; b += T)
        dg += (bit_of(s, a.bonds[2 * b]) ^ bit_of(s, a.bonds[2 * b + 1])) ? -(a.bond_j ? a.bond_j[b] : a.J)
                                                                          : (a.bond_j ? a.bond_j[b] : a.J);
      return dg;
    };
    if (active && slow) {
#pragma unroll
      for (int j = 0; j < ST; ++j) {  // unrolled (sidx stays in registers); slow_ratio is not inlined
        if (!((live >> j) & 1u)) continue;
        const int s = sidx[j];
        double2 v = make_double2(0.0, 0.0);
        if (s0 + s < a.B && ((nz >> j) & 1u)) v = slow_ratio(a.N, a.M, a.ham, a.a, a.b, a.w_t, a.bonds, wsm + s * 32, t,
                                                                ((sg_bits >> j) & 1u) ? -1.0 : 1.0);
        R[s * T + t] = make_double2(fma(ct, v.x, diag(s)), ct * v.y);
      }
    } else {
#pragma unroll
      for (int j = 0; j < ST; ++j) {
        if (!((live >> j) & 1u)) continue;
        const int s = sidx[j];
        double2 v = make_double2(0.0, 0.0);
        if (active && ((nz >> j) & 1u)) {
          v = cmul(sg[j] ? eam : eap, P[j]);
          const int k = E[j] + ect;
          if (k >= -1022 && k <= 1023) {  // exact power-of-two scale (correctly rounded, like ldexp)
            const double f = __longlong_as_double((long long)(k + 1023) << 52);
            v.x *= f;
            v.y *= f;
          } else {
            const int k1 = max(-1000, min(1000, k));
            v.x = ldexp(ldexp(v.x, k1), k - k1);
            v.y = ldexp(ldexp(v.y, k1), k - k1);
          }
        }
        R[s * T + t] = make_double2(fma(ct, v.x, diag(s)), ct * v.y);
      }
    }
  }
  __syncthreads();
  // fixed-order sums: warp w takes samples w, w + nwarps, ...; lane l sums
  // terms l, l + 32, ... then a butterfly
  for (int s = warp; s < ((pl.skip & 16) ? 0 : SB); s += nwarps) {
    if (s0 + s >= a.B) continue;
    double er = 0.0, ei = 0.0;
    for (int u = lane; u < T; u += 32) {
      er += R[s * T + u].x;
      ei += R[s * T + u].y;
    }
    er = segment_sum(er, 32);
    ei = segment_sum(ei, 32);
    if (lane == 0) {
      const double2 eps = make_double2(er, ei);
      a.out[s0 + s] = eps;
      if ((!isfinite(eps.x) || !isfinite(eps.y)) && a.status) {
        atomicMin((unsigned long long*)&a.status[1], (unsigned long long)(s0 + s));
        atomicExch((unsigned long long*)&a.status[0], (unsigned long long)MPV_ERR_NONFINITE);
      }
    }
  }
}

}  // namespace mpv
