// Fused Metropolis–Hastings sweep (ref: sampler.py:111-133 ChainEnsemble.step,
// repeated n_steps times; sampler.py:142-167 collect) for the RBM log-probability
// (ref: rbm.py:361-405 log_prob_evaluator) — one launch runs many proposals per
// chain with the chain's state on chip.
//
// Layout: a chain is owned by a segment of G lanes of one warp (32/G chains
// per warp).  Hidden unit i = u*G + gl lives in lane gl of the segment, slot u
// (U slots per lane), so a flip of site k reads the contiguous column
// table[k*Mpad + ...] with conflict-free shared-memory loads.  The packed
// configuration is spread over the segment (word w in lane w).  theta = b + W x
// is kept EXACT in registers (X1 / X2 / F64 accumulators), the
// log p of a proposal is a fixed function of the proposed configuration, and
// the accept test is the reference's f64 `log(u) < lp_new - lp_old`.
#pragma once
#ifndef MPV_XI_FOLD
#define MPV_XI_FOLD 1  // experiments: 0 scales bf16 XI theta by q before rounding
#endif
#ifndef MPV_SWEEP_UNDO
#define MPV_SWEEP_UNDO 1  // experiments: 0 evaluates theta' aside and commits accepted moves
#endif
#include "common.cuh"

namespace mpv {

struct SweepArgs {
  // snapshot
  int N, M, Mpad, G, words;
  const void* table;  // global copy of the table
  const void* bias;
  const void* vis;
  size_t table_bytes;
  int table_in_smem;
  // chains
  int64_t n_chains, chain_offset;
  uint32_t* bits;
  double* log_probs;
  int64_t* accepted;
  int64_t* status;
  // schedule
  uint64_t key;
  int64_t init_draws, step_index, n_steps, thin;
  uint32_t* samples;
  int64_t sample_base, sample_extra, round_offset, row0;
  // persistent work queue: items (segment, chain group), segment-major
  int64_t seg_len, n_groups, n_items;
  float xi_scale;     // quantum q of the XI variant (theta = integer * q)
  int* queue;         // [1], zero at launch
  int* done;          // [n_groups] segments finished, zero at launch
  float* save;        // [n_groups][save_words][32] theta between segments
  void* vis_save;     // [n_chains] visible term between segments
  uint64_t noise_key;  // frozen log-density noise (f64 arithmetic, N <= 64); sigma 0 = off
  double noise_sigma;
  // cluster split (CS > 1): rank block bytes in global (16-aligned), vis bytes,
  // and the shared-memory offset of the exchange buffers
  size_t rank_block_bytes, vis_bytes, xchg_off;
};

// ------------------------------------------------------------------------
// Cluster exchange of per-rank partial sums (CS ranks split the hidden units).
// Per warp: two data slots [parity][rank][32 lanes] and two mbarriers (one per
// slot parity, CS - 1 arrivals each).  Every rank writes its partial into every
// other rank's slot (st.shared::cluster) and arrives on their barrier
// (release.cluster); after its own barrier completes it sums the CS partials
// in rank order, so all ranks hold the identical total.  A slot is rewritten
// two exchanges later, after the writer has seen the reader's next arrival,
// i.e. after the reader consumed it.
// ------------------------------------------------------------------------
template <int CS, typename T>
struct ClusterXchg {
  uint32_t data0;  // shared address of this warp's slots in this CTA: [2][CS][32] T
  uint32_t bar0;   // shared address of this warp's two mbarriers
  int rank;
  uint32_t count;  // exchanges done by this warp
  __device__ static uint32_t mapa(uint32_t addr, int r) {
    uint32_t out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(r));
    return out;
  }
  __device__ T sum(T v, int lane) {
    if constexpr (CS == 1) {
      return v;
    } else {
      const uint32_t par = count & 1u;
      const uint32_t slot = data0 + (uint32_t)((par * CS + rank) * 32 + lane) * (uint32_t)sizeof(T);
#pragma unroll
      for (int r = 0; r < CS; ++r) {
        if (r == rank) continue;
        const uint32_t dst = mapa(slot, r);
        if constexpr (sizeof(T) == 8)
          asm volatile("st.shared::cluster.b64 [%0], %1;" ::"r"(dst), "l"(__double_as_longlong((double)v)) : "memory");
        else
          asm volatile("st.shared::cluster.b32 [%0], %1;" ::"r"(dst), "r"(__float_as_uint((float)v)) : "memory");
      }
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int r = 0; r < CS; ++r) {
          if (r == rank) continue;
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(bar0 + 8 * par, r))
                       : "memory");
        }
      }
      const uint32_t ph = (count >> 1) & 1u;
      asm volatile(
          "{.reg .pred p;\nXW_%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra XW_%=;\n}" ::"r"(
              bar0 + 8 * par),
          "r"(ph)
          : "memory");
      T total = T(0);
#pragma unroll
      for (int r = 0; r < CS; ++r) {
        T x;
        if (r == rank) {
          x = v;
        } else {
          const uint32_t src = data0 + (uint32_t)((par * CS + r) * 32 + lane) * (uint32_t)sizeof(T);
          if constexpr (sizeof(T) == 8) {
            unsigned long long b;
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(b) : "r"(src) : "memory");
            x = (T)__longlong_as_double((long long)b);
          } else {
            uint32_t b;
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(b) : "r"(src) : "memory");
            x = (T)__uint_as_float(b);
          }
        }
        total += x;
      }
      ++count;
      return total;
    }
  }
};

// code(x) of the configuration spread over a segment's lanes (word w in lane w)
__device__ __forceinline__ uint64_t segment_code(uint32_t word, int words, int G) {
  const uint32_t w0 = __shfl_sync(kFull, word, 0, G);
  const uint32_t w1 = __shfl_sync(kFull, word, 1 % G, G);
  return (uint64_t)w0 | (words > 1 ? (uint64_t)w1 << 32 : 0ull);
}

// ------------------------------------------------------------------------
// Unit evaluators: Re log cosh of one hidden unit in the snapshot's arithmetic.
// ------------------------------------------------------------------------

// f16 / bf16 NATIVE: theta' rounded once to the format, Re log cosh in f32 with
// 3 MUFU ops  ½ log(1 + t² + 2 t cos 2y) + |x| - ln2,  t = e^{-2|x|}
// (the same closed form as ref _logcosh_pair, rbm.py:130-140), result rounded
// to the format by the caller (pairs of units share one F2FP).
constexpr float kLcK = -2.8853900817779268f;  // -2 log2(e) in f32
__device__ __forceinline__ float lc_fast(float x, float y2, float& vmin) {
  const float ax = fabsf(x);
  const float t = ex2_approx(ax * kLcK);  // e^{-2|x|}
  const float c = cos_approx(y2);                          // cos 2y
  const float s = fmaf(2.0f, c, t);
  const float v = fmaf(t, s, 1.0f);                        // 4 e^{-2|x|} |cosh z|^2
  vmin = fminf(vmin, v);
  return fmaf(lg2_approx(v), 0.34657359027997264f, ax - 0.69314718055994531f);
}

// lc_fast(m q, y2) for a power-of-two q folded into the constants (bf16 XI:
// RN_bf16(m q) = RN_bf16(m) q over bf16's f32 exponent range): |m| (k q) and
// |m| q - ln 2 are the same real numbers as |x| k and |x| - ln 2, so the
// results are bit-identical to lc_fast(m q, y2) with one multiply fewer per
// component.  ksc = k q with k the f32 constant of lc_fast.
__device__ __forceinline__ float lc_fast_sc(float m, float y2, float q, float ksc, float& vmin) {
  const float am = fabsf(m);
  const float t = ex2_approx(am * ksc);
  const float c = cos_approx(y2);
  const float s = fmaf(2.0f, c, t);
  const float v = fmaf(t, s, 1.0f);
  vmin = fminf(vmin, v);
  return fmaf(lg2_approx(v), 0.34657359027997264f, fmaf(am, q, -0.69314718055994531f));
}
// Near a zero of cosh (v = 1 + t^2 + 2t cos 2y -> 0) the MUFU form cancels.
// There |x| < 0.02 and cos^2 y < 2.5e-4, and Re log cosh = ½ log(sinh^2 x +
// cos^2 y) is evaluated with a short sinh series and cos y = ±sin r,
// r = y - (k+½)π reduced in f64 (rare path, taken by a warp only when one of
// its units is this close to a zero).
// Threshold on v below which the MUFU error (~1e-6 absolute in v) exceeds the
// format's rounding of log cosh: f16 (2^-11) -> 2e-3, bf16 (2^-8) -> 2e-4.
template <int FMT> struct NearZero { static constexpr float kV = FMT == MPV_FMT_BF16 ? 2e-4f : 2e-3f; };
constexpr float kNearZeroV = 2e-3f;
__device__ __forceinline__ float lc_near_zero(float x, float y) {
  const float ax = fabsf(x);
  const float x2 = ax * ax;
  const float sh = ax * fmaf(x2, fmaf(x2, 1.0f / 120.0f, 1.0f / 6.0f), 1.0f);
  const double q = rint((double)y * 0.31830988618379067 - 0.5) + 0.5;
  const float r = (float)fma(-q, 3.141592653589793, (double)y);
  const float r2 = r * r;
  const float sr = r * fmaf(r2, fmaf(r2, 1.0f / 120.0f, -1.0f / 6.0f), 1.0f);
  return 0.34657359027997264f * lg2_approx(fmaf(sh, sh, sr * sr));
}

// f32 NATIVE: Re log cosh(x + iy) = 1/2 log(sinh^2 x + cos^2 y):
// both terms are computed to a few f32 ulps *relative*, so the sum has no
// cancellation, near the zeros of cosh included; branch-free (the lanes of a
// warp hold different units).  sinh: odd series through x^9 for |x| < 1/2,
// (e - 1/e)/2 from MUFU ex2 / rcp above (relative error < 3e-7 there);
// cos^2 y: Cody-Waite reduction to [-pi/4, pi/4] and the quadrant's sin or cos
// polynomial (< 1 ulp); log through MUFU lg2 (absolute error ~6e-8 per unit).
// |x| > 40: |x| - ln 2 (the correction is < 1e-34).  (A two-MUFU variant with
// the e^{-2|x|}-scaled form above |x| = 1/2 measured 13% slower: issue-bound.)
__device__ __forceinline__ float lc_f32(float x, float y) {
  const float ax = fabsf(x);
  const float x2 = ax * ax;
  const float sh_s =
      ax * fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, 2.7557319e-6f, 1.9841270e-4f), 8.3333333e-3f), 0.16666667f), 1.0f);
  const float e = ex2_approx(ax * 1.4426950408889634f);
  const float sh_l = 0.5f * (e - rcp_approx(e));
  const float sh = ax < 0.5f ? sh_s : sh_l;
  const float k = rintf(y * 0.63661977236758134f);  // y / (pi/2)
  float r = fmaf(-k, 1.5707963705062866f, y);
  r = fmaf(-k, -4.3711388286737929e-8f, r);
  const float r2 = r * r;
  const float sr = r * fmaf(r2, fmaf(r2, fmaf(r2, -1.9841270e-4f, 8.3333333e-3f), -0.16666667f), 1.0f);
  const float cr = fmaf(r2, fmaf(r2, fmaf(r2, fmaf(r2, 2.4801587e-5f, -1.3888889e-3f), 4.1666667e-2f), -0.5f), 1.0f);
  const float cy = (((int)k) & 1) ? sr : cr;  // |cos y|
  const float v = fmaf(sh, sh, cy * cy);
  const float lc = 0.34657359027997264f * lg2_approx(v);
  return ax > 40.0f ? ax - 0.69314718055994531f : lc;
}

// f64: the reference formula op for op (rbm.py:130-140 / _kernels.py:101-106).
__device__ __forceinline__ double lc_f64(double tr, double ti) {
  const double u = fabs(tr);
  const double v = tr >= 0.0 ? ti : -ti;
  const double t = exp(-2.0 * u);
  double sv, cv;
  sincos(v, &sv, &cv);  // one shared argument reduction (same values as cos(v), sin(v))
  const double wr = __dmul_rn(__dadd_rn(1.0, t), cv);
  const double wi = __dmul_rn(__dadd_rn(1.0, -t), sv);
  const double q = __dadd_rn(__dmul_rn(wr, wr), __dmul_rn(wi, wi));
  return __dadd_rn(__dadd_rn(u, -0.69314718055994530942), __dmul_rn(0.5, log(q)));
}

// ------------------------------------------------------------------------
// Accumulator variants.  Each provides:
//   Entry      table element type;  Vis  visible-bias element type
//   init(b)    theta = bias;         add(e, d) theta += d*e (d in {-1,0,1})
//   eval/lc    contribution of the unit for theta + d*e (proposal)
// ------------------------------------------------------------------------

template <int FMT, int VAR> struct Acc;

// ---- X1, f16/bf16: theta in one f32 per component (exact by planner check) ----
template <int FMT> struct Acc<FMT, MPV_ACC_X1> {
  using H = Half<FMT>;
  using Entry = uint32_t;
  using Vis = float;
  using Sign = uint16_t;
  float re, im;
  __device__ __forceinline__ static Sign sign(int d) {
    return d > 0 ? H::kOne : (d < 0 ? H::kMinusOne : (uint16_t)0);
  }
  __device__ __forceinline__ void init(Entry b) { re = H::lo(b); im = H::hi(b); }
  __device__ __forceinline__ void value(float sc, float& xr, float& xi) const { xr = re; xi = im; }
  __device__ __forceinline__ void add(Entry e, Sign d) {
    re = H::fma_lo(e, d, re);
    im = H::fma_hi(e, d, im);
  }
  // theta' for a one-column move
  __device__ __forceinline__ void prop1(Entry e, Sign d, float sc, float& xr, float& xi) const {
    xr = H::fma_lo(e, d, re);
    xi = H::fma_hi(e, d, im);
  }
  __device__ __forceinline__ void prop2(Entry e1, Entry e2, Sign d, Sign md, float sc, float& xr,
                                        float& xi) const {
    xr = H::fma_lo(e1, d, H::fma_lo(e2, md, re));
    xi = H::fma_hi(e1, d, H::fma_hi(e2, md, im));
  }
};

// ---- X2, f16/bf16: hi/lo f32 accumulators on a fixed split grid ----
template <int FMT> struct Acc<FMT, MPV_ACC_X2> {
  using H = Half<FMT>;
  using Entry = uint2;  // x: hi pair, y: lo pair
  using Vis = float2;
  using Sign = uint16_t;
  float hr, hi_, lr, li;
  __device__ __forceinline__ static Sign sign(int d) {
    return d > 0 ? H::kOne : (d < 0 ? H::kMinusOne : (uint16_t)0);
  }
  __device__ __forceinline__ void init(Entry b) {
    hr = H::lo(b.x); hi_ = H::hi(b.x); lr = H::lo(b.y); li = H::hi(b.y);
  }
  __device__ __forceinline__ void value(float sc, float& xr, float& xi) const { xr = hr + lr; xi = hi_ + li; }
  __device__ __forceinline__ void add(Entry e, Sign d) {
    hr = H::fma_lo(e.x, d, hr); hi_ = H::fma_hi(e.x, d, hi_);
    lr = H::fma_lo(e.y, d, lr); li = H::fma_hi(e.y, d, li);
  }
  __device__ __forceinline__ void prop1(Entry e, Sign d, float sc, float& xr, float& xi) const {
    xr = H::fma_lo(e.x, d, hr) + H::fma_lo(e.y, d, lr);
    xi = H::fma_hi(e.x, d, hi_) + H::fma_hi(e.y, d, li);
  }
  __device__ __forceinline__ void prop2(Entry e1, Entry e2, Sign d, Sign md, float sc, float& xr,
                                        float& xi) const {
    xr = H::fma_lo(e1.x, d, H::fma_lo(e2.x, md, hr)) + H::fma_lo(e1.y, d, H::fma_lo(e2.y, md, lr));
    xi = H::fma_hi(e1.x, d, H::fma_hi(e2.x, md, hi_)) + H::fma_hi(e1.y, d, H::fma_hi(e2.y, md, li));
  }
};

// ---- XI, f16/bf16: theta as an exact int32 multiple of the snapshot quantum q
// (host planner: B/q < 2^31); one IMAD per component, the f32 value is the
// correctly rounded I2F of the integer times q (a power of two: exact).
// bf16 (kFold): the values are returned unscaled and the evaluator applies q
// (lc_fast_sc), exact over bf16's exponent range (host planner: q >= 2^-100).
template <int FMT> struct Acc<FMT, MPV_ACC_XI> {
  using Entry = int2;
  using Vis = int;
  using Sign = int;
  static constexpr bool kFold = MPV_XI_FOLD && FMT == MPV_FMT_BF16;
  int re, im;
  __device__ __forceinline__ static Sign sign(int d) { return d; }
  __device__ __forceinline__ static float scaled(int v, float sc) {
    return kFold ? __int2float_rn(v) : __int2float_rn(v) * sc;
  }
  __device__ __forceinline__ void init(Entry b) { re = b.x; im = b.y; }
  __device__ __forceinline__ void value(float sc, float& xr, float& xi) const {
    xr = scaled(re, sc);
    xi = scaled(im, sc);
  }
  __device__ __forceinline__ void add(Entry e, Sign d) { re += d * e.x; im += d * e.y; }
  // theta + ea - eb (exchange with the columns ordered by the move's sign: one IADD3 per component)
  __device__ __forceinline__ void add_diff(Entry ea, Entry eb) { re += ea.x - eb.x; im += ea.y - eb.y; }
  __device__ __forceinline__ void prop1(Entry e, Sign d, float sc, float& xr, float& xi) const {
    xr = scaled(re + d * e.x, sc);
    xi = scaled(im + d * e.y, sc);
  }
  __device__ __forceinline__ void prop2(Entry e1, Entry e2, Sign d, Sign md, float sc, float& xr,
                                        float& xi) const {
    xr = scaled(re + d * e1.x + md * e2.x, sc);
    xi = scaled(im + d * e1.y + md * e2.y, sc);
  }
};
template <int FMT, int VAR> struct FoldsScale { static constexpr bool value = false; };
template <int FMT> struct FoldsScale<FMT, MPV_ACC_XI> { static constexpr bool value = Acc<FMT, MPV_ACC_XI>::kFold; };

// ---- X1, f32 format: float pairs ----
template <> struct Acc<MPV_FMT_F32, MPV_ACC_X1> {
  using Entry = float2;
  using Vis = float;
  using Sign = float;
  float re, im;
  __device__ __forceinline__ static Sign sign(int d) { return (float)d; }
  __device__ __forceinline__ void init(Entry b) { re = b.x; im = b.y; }
  __device__ __forceinline__ void value(float sc, float& xr, float& xi) const { xr = re; xi = im; }
  __device__ __forceinline__ void add(Entry e, Sign d) { re = fmaf(e.x, d, re); im = fmaf(e.y, d, im); }
  __device__ __forceinline__ void prop1(Entry e, Sign d, float sc, float& xr, float& xi) const {
    xr = fmaf(e.x, d, re);
    xi = fmaf(e.y, d, im);
  }
  __device__ __forceinline__ void prop2(Entry e1, Entry e2, Sign d, Sign md, float sc, float& xr,
                                        float& xi) const {
    xr = fmaf(e1.x, d, fmaf(e2.x, md, re));
    xi = fmaf(e1.y, d, fmaf(e2.y, md, im));
  }
};

// ---- X2, f32 format ----
template <> struct Acc<MPV_FMT_F32, MPV_ACC_X2> {
  using Entry = float4;  // hi re, hi im, lo re, lo im
  using Vis = float2;
  using Sign = float;
  float hr, hi_, lr, li;
  __device__ __forceinline__ static Sign sign(int d) { return (float)d; }
  __device__ __forceinline__ void init(Entry b) { hr = b.x; hi_ = b.y; lr = b.z; li = b.w; }
  __device__ __forceinline__ void value(float sc, float& xr, float& xi) const { xr = hr + lr; xi = hi_ + li; }
  __device__ __forceinline__ void add(Entry e, Sign d) {
    hr = fmaf(e.x, d, hr); hi_ = fmaf(e.y, d, hi_); lr = fmaf(e.z, d, lr); li = fmaf(e.w, d, li);
  }
  __device__ __forceinline__ void prop1(Entry e, Sign d, float sc, float& xr, float& xi) const {
    xr = fmaf(e.x, d, hr) + fmaf(e.z, d, lr);
    xi = fmaf(e.y, d, hi_) + fmaf(e.w, d, li);
  }
  __device__ __forceinline__ void prop2(Entry e1, Entry e2, Sign d, Sign md, float sc, float& xr,
                                        float& xi) const {
    xr = fmaf(e1.x, d, fmaf(e2.x, md, hr)) + fmaf(e1.z, d, fmaf(e2.z, md, lr));
    xi = fmaf(e1.y, d, fmaf(e2.y, md, hi_)) + fmaf(e1.w, d, fmaf(e2.w, md, li));
  }
};

// ---- F64 accumulators (any format; f64/storage-only evaluate in f64) ----
template <int FMT> struct Acc<FMT, MPV_ACC_F64> {
  using Entry = double2;
  using Vis = double;
  using Sign = double;
  double re, im;
  __device__ __forceinline__ static Sign sign(int d) { return (double)d; }
  __device__ __forceinline__ void init(Entry b) { re = b.x; im = b.y; }
  __device__ __forceinline__ void value(float sc, double& xr, double& xi) const { xr = re; xi = im; }
  __device__ __forceinline__ void add(Entry e, Sign d) { re = fma(e.x, d, re); im = fma(e.y, d, im); }
  __device__ __forceinline__ void prop1(Entry e, Sign d, float sc, double& xr, double& xi) const {
    xr = fma(e.x, d, re);
    xi = fma(e.y, d, im);
  }
  __device__ __forceinline__ void prop2(Entry e1, Entry e2, Sign d, Sign md, float sc, double& xr,
                                        double& xi) const {
    xr = fma(e1.x, d, fma(e2.x, md, re));
    xi = fma(e1.y, d, fma(e2.y, md, im));
  }
};

// ------------------------------------------------------------------------
// Per-unit contribution and the final log p for each (FMT, VAR) combination.
// The f64 path (FMT == F64, or STORAGE_ONLY passed as FMT_F64) sums in f64;
// the reduced formats sum in f32.
// ------------------------------------------------------------------------
template <int FMT, int VAR> struct Eval {
  using A = Acc<FMT, VAR>;
  static constexpr bool kF64 = (FMT == MPV_FMT_F64);
  using Sum = typename std::conditional<kF64, double, float>::type;

  // Contribution of two units (u0, u1) given proposed theta in f32 (or f64).
  // Reduced formats: theta rounded to fmt, lc in f32, lc rounded to fmt, then
  // accumulated in f32 (mask 0 for padded units).
  static constexpr bool kFold = FoldsScale<FMT, VAR>::value;
  // the unit's log cosh from the packed rounded pair (kFold: unscaled by q)
  __device__ __forceinline__ static float lc_packed(uint32_t p, float sc, float& vmin) {
    using H = Half<FMT>;
    if constexpr (kFold)
      return lc_fast_sc(H::lo(p), H::fma_hi(p, (uint16_t)(__float_as_uint(2.0f * sc) >> 16), -0.0f), sc, kLcK * sc,
                        vmin);
    else
      return lc_fast(H::lo(p), H::hi2(p), vmin);
  }
  template <typename T>
  __device__ __forceinline__ static void pair(T xr0, T xi0, T xr1, T xi1, Sum& acc, float& vmin, float sc) {
    if constexpr (kF64) {
      acc += lc_f64(xr0, xi0);
      acc += lc_f64(xr1, xi1);
    } else {
      float a0 = (float)xr0, b0 = (float)xi0, a1 = (float)xr1, b1 = (float)xi1;
      if constexpr (FMT == MPV_FMT_F32) {
        acc += lc_f32(a0, b0);
        acc += lc_f32(a1, b1);
      } else {
        using H = Half<FMT>;
        const uint32_t p0 = H::pack(a0, b0), p1 = H::pack(a1, b1);
        const float l0 = lc_packed(p0, sc, vmin);
        const float l1 = lc_packed(p1, sc, vmin);
        const uint32_t lp = H::pack(l0, l1);
        acc = H::acc_lo(lp, acc);
        acc = H::acc_hi(lp, acc);
      }
    }
  }
  template <typename T>
  __device__ __forceinline__ static void single(T xr, T xi, Sum& acc, float& vmin, float sc) {
    if constexpr (kF64) {
      acc += lc_f64(xr, xi);
    } else if constexpr (FMT == MPV_FMT_F32) {
      acc += lc_f32((float)xr, (float)xi);
    } else {
      using H = Half<FMT>;
      const uint32_t p = H::pack((float)xr, (float)xi);
      const uint32_t lp = H::pack(lc_packed(p, sc, vmin), 0.0f);
      acc = H::acc_lo(lp, acc);
    }
  }
  // Correction for units near a cosh zero: h += q(lc_near_zero) - q(lc_fast)
  // (both rounded to the format), in unit order.  Deterministic in theta.
  template <typename T>
  __device__ __forceinline__ static void fix(T xr, T xi, Sum& acc, float sc) {
    if constexpr (!kF64 && FMT != MPV_FMT_F32) {
      using H = Half<FMT>;
      const uint32_t p = H::pack((float)xr, (float)xi);
      float v = 1e30f;
      const float lf = lc_packed(p, sc, v);
      if (v < NearZero<FMT>::kV) {
        const float la = kFold ? lc_near_zero(H::lo(p) * sc, H::hi(p) * sc) : lc_near_zero(H::lo(p), H::hi(p));
        const uint32_t q = H::pack(lf, la);
        acc += H::hi(q) - H::lo(q);
      }
    }
  }
  static constexpr bool kFix = !kF64 && FMT != MPV_FMT_F32;
  // log p is f64 for the f64 arithmetic and f32 for the NATIVE reduced
  // formats (an f32 number: 2 * RN32(RN32(a.x) + H)); the NATIVE accept test
  // is then made in f32.
  using Lp = typename std::conditional<kF64, double, float>::type;
  __device__ __forceinline__ static Lp finalize(typename A::Vis vis, Sum h, float xi_scale_) {
    if constexpr (kF64) {
      return 2.0 * (vis + h);
    } else if constexpr (VAR == MPV_ACC_F64) {
      return 2.0f * __fadd_rn(__double2float_rn(vis), h);
    } else if constexpr (VAR == MPV_ACC_X2) {
      return 2.0f * __fadd_rn(__fadd_rn(vis.x, vis.y), h);
    } else if constexpr (VAR == MPV_ACC_XI) {
      return 2.0f * __fadd_rn(__int2float_rn(vis) * xi_scale_, h);
    } else {
      return 2.0f * __fadd_rn(vis, h);
    }
  }
};

template <typename V> __device__ __forceinline__ V vis_add(V v, V a, int d);
template <> __device__ __forceinline__ float vis_add(float v, float a, int d) { return fmaf(a, (float)d, v); }
template <> __device__ __forceinline__ float2 vis_add(float2 v, float2 a, int d) {
  return make_float2(fmaf(a.x, (float)d, v.x), fmaf(a.y, (float)d, v.y));
}
template <> __device__ __forceinline__ double vis_add(double v, double a, int d) { return fma(a, (double)d, v); }
template <> __device__ __forceinline__ int vis_add(int v, int a, int d) { return v + d * a; }
template <typename V> __device__ __forceinline__ V vis_zero();
template <> __device__ __forceinline__ float vis_zero<float>() { return 0.0f; }
template <> __device__ __forceinline__ float2 vis_zero<float2>() { return make_float2(0.f, 0.f); }
template <> __device__ __forceinline__ double vis_zero<double>() { return 0.0; }
template <> __device__ __forceinline__ int vis_zero<int>() { return 0; }

// Record the first (lowest step, then lowest chain) non-finite evaluation.
__device__ __forceinline__ void report_nonfinite(int64_t* status, int64_t step, int64_t chain) {
  if (!status) return;
  atomicMin((unsigned long long*)&status[1], (unsigned long long)((step << 32) | chain));
  atomicExch((unsigned long long*)&status[0], (unsigned long long)MPV_ERR_NONFINITE);
}


// ------------------------------------------------------------------------
// The kernel: persistent warps pull (segment, chain-group) items from a
// segment-major queue, so the last wave is balanced to within one segment.
// A group's segment s+1 waits for segment s (already handed out, hence
// running or finished on a resident warp: no deadlock).
// ------------------------------------------------------------------------

template <int FMT, int VAR, int G, int U, int PROP, bool SMEM, int CS = 1>
__global__ void __launch_bounds__((PROP == MPV_PROPOSAL_FLIP) ? 512 : 256, (PROP == MPV_PROPOSAL_FLIP || SMEM) ? 1 : 2)
    sweep_kernel(const SweepArgs a) {
  static_assert(CS == 1 || SMEM, "cluster-split sweeps keep their rank block in shared memory");
  using A = Acc<FMT, VAR>;
  using E = Eval<FMT, VAR>;
  using Entry = typename A::Entry;
  using VisT = typename A::Vis;
  using Sign = typename A::Sign;
  using Sum = typename E::Sum;
  using Lp = typename E::Lp;
  using Theta = typename std::conditional<VAR == MPV_ACC_F64, double, float>::type;
  constexpr int CPW = 32 / G;
  // keep each unit's proposed theta in registers and commit it by select
  // (exchange: no second column read; table beyond shared memory: no L1/L2 re-read)
  // (not for the f64 arithmetic's flip sweep: 26 doubles per lane spill there, -13%)
  constexpr bool kKeep = (PROP == MPV_PROPOSAL_EXCHANGE) || (!SMEM && FMT != MPV_FMT_F64);
  // Flip sweeps with exact accumulators (X1 / X2 / XI): theta' is formed in
  // place, so an accepted move needs no commit; a warp with a rejecting chain
  // restores theta = theta' - d w exactly (every partial sum is exact).
  constexpr bool kUndo = MPV_SWEEP_UNDO && PROP == MPV_PROPOSAL_FLIP && !kKeep && VAR != MPV_ACC_F64;
  constexpr int SW = (int)(sizeof(A) / sizeof(float));

  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Entry* tab;
  const VisT* visv;
  int rank = 0;
  if constexpr (CS > 1) {
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    // this rank's block of hidden units, then the visible biases; the exchange
    // barriers are initialised before any rank can arrive on them (cluster barrier)
    __shared__ __align__(8) uint64_t bar;
    const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&bar);
    const uint32_t rb = (uint32_t)a.rank_block_bytes, vb = (uint32_t)((a.vis_bytes + 15) & ~(size_t)15);
    uint64_t* xbars = reinterpret_cast<uint64_t*>(smem_raw + a.xchg_off);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
        for (int k = 0; k < 2; ++k)
          asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(
                           xbars + 2 * w + k)),
                       "r"(CS - 1));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(rb + vb) : "memory");
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem_raw);
      const char* src = (const char*)a.table + (size_t)rank * rb;
      for (uint32_t off = 0; off < rb; off += 65536u)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst + off),
            "l"(src + off), "r"(min(rb - off, 65536u)), "r"(sbar)
            : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst + rb),
          "l"((const char*)a.vis), "r"(vb), "r"(sbar)
          : "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile(
        "{.reg .pred p;\nWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(
            sbar)
        : "memory");
    tab = reinterpret_cast<const Entry*>(smem_raw);
    visv = reinterpret_cast<const VisT*>(smem_raw + rb);
  } else if constexpr (SMEM) {
    // Stage the snapshot (column table, then visible biases) into shared memory
    // with bulk async copies (TMA engine, cp.async.bulk) on one mbarrier.
    __shared__ __align__(8) uint64_t bar;
    const uint32_t bytes = (uint32_t)a.table_bytes;
    const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(bytes)
                   : "memory");
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem_raw);
      uint32_t off = 0;
      while (off < bytes) {
        const uint32_t chunk = min(bytes - off, 65536u);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                dst + off),
            "l"((const char*)a.table + off), "r"(chunk), "r"(sbar)
            : "memory");
        off += chunk;
      }
    }
    asm volatile(
        "{.reg .pred p;\nWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(
            sbar)
        : "memory");
    tab = reinterpret_cast<const Entry*>(smem_raw);
    visv = reinterpret_cast<const VisT*>(smem_raw + (((size_t)a.N * (G * U) * sizeof(Entry) + 15) & ~(size_t)15));
  } else {
    tab = reinterpret_cast<const Entry*>(a.table);
    visv = reinterpret_cast<const VisT*>((const char*)a.table + (((size_t)a.N * (G * U) * sizeof(Entry) + 15) & ~(size_t)15));
  }
  constexpr int Mpad = G * U;
  const float sc = a.xi_scale;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int slot = lane / G;
  const int N = a.N;
  const int words = a.words;
  const double n_pairs = 0.5 * (double)N * (double)(N - 1);
  const Entry* bias = reinterpret_cast<const Entry*>(a.bias) + rank * Mpad;  // this rank's units
  VisT* vsave = reinterpret_cast<VisT*>(a.vis_save);
  const int warp = threadIdx.x >> 5;
  ClusterXchg<CS, Sum> xchg;
  if constexpr (CS > 1) {
    xchg.rank = rank;
    xchg.count = 0;
    xchg.bar0 = (uint32_t)__cvta_generic_to_shared(smem_raw + a.xchg_off) + 16u * warp;
    xchg.data0 = (uint32_t)__cvta_generic_to_shared(smem_raw + a.xchg_off) + 16u * (blockDim.x >> 5) +
                 (uint32_t)(warp * 2 * CS * 32 * sizeof(Sum));
  }
  // parked theta of this rank; per-rank segment counters
  float* const save_r = a.save + (size_t)rank * a.n_groups * (U * SW) * 32;
  int* const done_r = a.done + (size_t)rank * a.n_groups;
  const bool writer = rank == 0;  // rank 0 owns the chain state (bits, log p, counters, samples)
  // CS > 1: static item order (the ranks of a cluster walk the same items in
  // lockstep); a group's earlier segment always has a smaller item index, so
  // the persistent grid cannot deadlock
  const int64_t gwarp = (int64_t)(blockIdx.x / CS) * (blockDim.x >> 5) + warp;
  const int64_t gstride = (int64_t)(gridDim.x / CS) * (blockDim.x >> 5);
  int64_t next_item = gwarp;

  for (;;) {
    int64_t item = 0;
    if constexpr (CS == 1) {
      int it = 0;
      if (lane == 0) it = atomicAdd(a.queue, 1);
      item = __shfl_sync(kFull, it, 0);
    } else {
      item = next_item;
      next_item += gstride;
    }
    if (item >= a.n_items) break;
    const int64_t seg = item / a.n_groups;
    const int64_t grp = item % a.n_groups;
    const int64_t chain = grp * CPW + slot;
    const bool live = chain < a.n_chains;
    const int64_t cidx = live ? chain : 0;  // tail lanes mirror chain 0 and never write
    const int64_t gchain = a.chain_offset + cidx;
    if (seg > 0) {
      if (lane == 0) {
        // this rank's parked theta, and (CS > 1) the chain state written by rank 0
        for (int r = 0; r < (CS > 1 && rank != 0 ? 2 : 1); ++r) {
          const int* flag = (r == 0 ? done_r : a.done) + grp;
          int d;
          for (;;) {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(d) : "l"(flag) : "memory");
            if (d >= seg) break;
            __nanosleep(100);
          }
        }
      }
      __syncwarp();
    }
    uint32_t myword = (gl < words) ? a.bits[cidx * words + gl] : 0u;

    A acc[U];
    VisT vis;
    Lp lp;
    if (seg == 0) {
      // refresh: theta = b + W x, vis = a.x, log p (set_evaluator semantics)
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u].init(bias[u * G + gl]);
      vis = vis_zero<VisT>();
      const Sign one = A::sign(1);
      for (int w = 0; w < words; ++w) {
        uint32_t word = __shfl_sync(kFull, myword, w, G);
        while (word) {
          const int k = w * 32 + __ffs(word) - 1;
          word &= word - 1;
          const Entry* col = tab + (size_t)k * Mpad + gl;
#pragma unroll
          for (int u = 0; u < U; ++u) acc[u].add(col[u * G], one);
          vis = vis_add(vis, visv[k], 1);
        }
      }
      Sum h0 = Sum(0);
      float vmin0 = 1e30f;
#pragma unroll
      for (int u = 0; u + 1 < U; u += 2) {
        Theta xr0, xi0, xr1, xi1;
        acc[u].prop1(Entry{}, A::sign(0), sc, xr0, xi0);
        acc[u + 1].prop1(Entry{}, A::sign(0), sc, xr1, xi1);
        E::pair(xr0, xi0, xr1, xi1, h0, vmin0, sc);
      }
      if constexpr (U & 1) {
        Theta xr, xi;
        acc[U - 1].prop1(Entry{}, A::sign(0), sc, xr, xi);
        E::single(xr, xi, h0, vmin0, sc);
      }
      if constexpr (E::kFix) {
        if (vmin0 < NearZero<FMT>::kV) {  // rare: a unit is near a cosh zero
          // the accumulators go through this lane's parking slot so the
          // correction loop is a compact rolled loop (no register pressure)
          float* sv = save_r + (size_t)grp * (U * SW) * 32 + lane;
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < SW; ++j) sv[(u * SW + j) * 32] = reinterpret_cast<const float*>(&acc[u])[j];
#pragma unroll 1
          for (int u = 0; u < U; ++u) {
            A au;
#pragma unroll
            for (int j = 0; j < SW; ++j) reinterpret_cast<float*>(&au)[j] = sv[(u * SW + j) * 32];
            Theta xr, xi;
            au.prop1(Entry{}, A::sign(0), sc, xr, xi);
            E::fix(xr, xi, h0, sc);
          }
        }
      }
      h0 = xchg.sum(segment_sum(h0, G), lane);
      lp = E::finalize(vis, h0, sc);
      if (a.noise_sigma != 0.0) lp = (Lp)((double)lp + noise_zeta(a.noise_key, segment_code(myword, words, G), a.noise_sigma));
      if (!isfinite(lp)) {
        if (live && gl == 0 && writer) report_nonfinite(a.status, 0, cidx);
        lp = Lp(NAN);  // NaN marks a frozen chain
      }
    } else {
      const float* sv = save_r + (size_t)grp * (U * SW) * 32 + lane;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float* dst = reinterpret_cast<float*>(&acc[u]);
#pragma unroll
        for (int j = 0; j < SW; ++j) dst[j] = sv[(u * SW + j) * 32];
      }
      vis = vsave[cidx];
      lp = (Lp)a.log_probs[cidx];
    }
    bool dead = isnan(lp);

    A nxt[kKeep ? U : 1];  // exchange / global table: theta after the proposed move
    const uint64_t s0 = stream_state(a.key, (uint64_t)gchain);
    const int64_t count_c = a.sample_base + ((gchain < a.sample_extra) ? 1 : 0);
    const int64_t offset_c =
        gchain * a.sample_base + (gchain < a.sample_extra ? gchain : a.sample_extra) - a.row0;
    int n_acc = 0;
    int sel_c = 0;    // cached selection (site, or pair i | j<<16)
    Lp logu_c = 0;    // cached log(u_accept) (f32 for the NATIVE reduced formats)
    const int s_begin = (int)(seg * a.seg_len);
    const int s_end = (int)min(a.n_steps, (int64_t)s_begin + a.seg_len);
    const int thin = (int)a.thin;
    int next_record = -1;
    if (a.samples && thin > 0) next_record = (s_begin / thin + 1) * thin;
    const int64_t t_base = a.init_draws + 2 * a.step_index;

    for (int s = s_begin; s < s_end; ++s) {
      const int src = s & (G - 1);
      if (src == 0) {
        // lane gl draws the two uniforms of step s+gl (ref: sampler.py:113,127)
        const uint64_t t = (uint64_t)(t_base + 2 * (int64_t)(s + gl));
        const double us = stream_draw(s0, t);
        const double ua = stream_draw(s0, t + 1);
        if (PROP == MPV_PROPOSAL_FLIP) {
          sel_c = (int)floor_scaled(us, (double)N);
        } else {
          int i, j;
          pair_of(floor_scaled(us, n_pairs), N, i, j);
          sel_c = i | (j << 16);
        }
        logu_c = (Lp)log(ua);
      }
      const int sel = __shfl_sync(kFull, sel_c, src, G);
      const Lp logu = __shfl_sync(kFull, logu_c, src, G);

      int dsign, k1, k2 = 0;
      uint32_t flip;  // this lane's word bits that change if the move is accepted
      if (PROP == MPV_PROPOSAL_FLIP) {
        k1 = sel;
        const uint32_t m1 = 1u << (k1 & 31);
        const uint32_t wd = __shfl_sync(kFull, myword, k1 >> 5, G);
        dsign = (wd & m1) ? -1 : 1;
        flip = (gl == (k1 >> 5)) ? m1 : 0u;
      } else {
        k1 = sel & 0xFFFF;
        k2 = sel >> 16;
        const uint32_t m1 = 1u << (k1 & 31), m2 = 1u << (k2 & 31);
        const uint32_t wi = __shfl_sync(kFull, myword, k1 >> 5, G);
        const uint32_t wj = __shfl_sync(kFull, myword, k2 >> 5, G);
        dsign = ((wj & m2) ? 1 : 0) - ((wi & m1) ? 1 : 0);  // x_i' = x_j: theta' = theta + d (W_:i - W_:j)
        flip = ((gl == (k1 >> 5)) ? m1 : 0u) ^ ((gl == (k2 >> 5)) ? m2 : 0u);
      }
      // Every segment evaluates (no divergence around the segment shuffles); an
      // exchange of equal bits (dsign == 0) is accepted unconditionally: the
      // reference evaluator returns the cached value, Δ = 0, log u < 0
      // (sampler.py:119-131).
      // A warp whose chains all drew an exchange of equal bits has nothing to
      // evaluate this step: every chain accepts without moving (the reference
      // returns the cached value, sampler.py:119-131); only the counters and the
      // sample record advance.  (Flip proposals always have dsign != 0.)
      if (PROP == MPV_PROPOSAL_EXCHANGE && !__any_sync(kFull, dsign != 0)) {
        n_acc += dead ? 0 : 1;
        if (s + 1 == next_record) {
          next_record += thin;
          const int64_t r = a.round_offset + (s + 1) / thin - 1;
          if (live && writer && r < count_c && gl < words) a.samples[(offset_c + r) * words + gl] = myword;
        }
        continue;
      }
      const Sign d = A::sign(dsign);
      const Sign md = A::sign(-dsign);
      const Entry* c1 = tab + (size_t)k1 * Mpad + gl;
      const Entry* c2 = tab + (size_t)k2 * Mpad + gl;
      // exchange, XI: theta' = theta + ca - cb with the columns ordered by the sign
      // of the move (cb = ca when the bits are equal: theta' = theta)
      const Entry* ca = dsign >= 0 ? c1 : c2;
      const Entry* cb = dsign > 0 ? c2 : (dsign < 0 ? c1 : ca);
      auto xmove = [&](A& n, int u) {
        if constexpr (VAR == MPV_ACC_XI) {
          n.add_diff(ca[u * G], cb[u * G]);
        } else {
          n.add(c2[u * G], md);
          n.add(c1[u * G], d);
        }
      };
      Sum h = Sum(0);
      float vmin = 1e30f;
#pragma unroll
      for (int u = 0; u + 1 < U; u += 2) {
        Theta xr0, xi0, xr1, xi1;
        if constexpr (PROP == MPV_PROPOSAL_FLIP && kKeep) {  // table in L1/L2: keep theta' for the commit
          nxt[u] = acc[u];
          nxt[u].add(c1[u * G], d);
          nxt[u].value(sc, xr0, xi0);
          nxt[u + 1] = acc[u + 1];
          nxt[u + 1].add(c1[(u + 1) * G], d);
          nxt[u + 1].value(sc, xr1, xi1);
        } else if constexpr (kUndo) {
          acc[u].add(c1[u * G], d);
          acc[u].value(sc, xr0, xi0);
          acc[u + 1].add(c1[(u + 1) * G], d);
          acc[u + 1].value(sc, xr1, xi1);
        } else if constexpr (PROP == MPV_PROPOSAL_FLIP) {
          acc[u].prop1(c1[u * G], d, sc, xr0, xi0);
          acc[u + 1].prop1(c1[(u + 1) * G], d, sc, xr1, xi1);
        } else {  // exchange: the proposed theta is kept for the commit (nxt)
          nxt[u] = acc[u];
          xmove(nxt[u], u);
          nxt[u].value(sc, xr0, xi0);
          nxt[u + 1] = acc[u + 1];
          xmove(nxt[u + 1], u + 1);
          nxt[u + 1].value(sc, xr1, xi1);
        }
        E::pair(xr0, xi0, xr1, xi1, h, vmin, sc);
      }
      if constexpr (U & 1) {
        Theta xr, xi;
        if constexpr (PROP == MPV_PROPOSAL_FLIP && kKeep) {
          nxt[U - 1] = acc[U - 1];
          nxt[U - 1].add(c1[(U - 1) * G], d);
          nxt[U - 1].value(sc, xr, xi);
        } else if constexpr (kUndo) {
          acc[U - 1].add(c1[(U - 1) * G], d);
          acc[U - 1].value(sc, xr, xi);
        } else if constexpr (PROP == MPV_PROPOSAL_FLIP) {
          acc[U - 1].prop1(c1[(U - 1) * G], d, sc, xr, xi);
        } else {
          nxt[U - 1] = acc[U - 1];
          xmove(nxt[U - 1], U - 1);
          nxt[U - 1].value(sc, xr, xi);
        }
        E::single(xr, xi, h, vmin, sc);
      }
      if constexpr (E::kFix) {
        if (vmin < NearZero<FMT>::kV) {  // rare: a unit of this lane is near a cosh zero
          float* sv = save_r + (size_t)grp * (U * SW) * 32 + lane;
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < SW; ++j) sv[(u * SW + j) * 32] = reinterpret_cast<const float*>(&acc[u])[j];
#pragma unroll 1
          for (int u = 0; u < U; ++u) {
            A au;
#pragma unroll
            for (int j = 0; j < SW; ++j) reinterpret_cast<float*>(&au)[j] = sv[(u * SW + j) * 32];
            Theta xr, xi;
            if (kUndo) au.value(sc, xr, xi);  // acc already holds theta'
            else if (PROP == MPV_PROPOSAL_FLIP) au.prop1(c1[u * G], d, sc, xr, xi);
            else au.prop2(c1[u * G], c2[u * G], d, md, sc, xr, xi);
            E::fix(xr, xi, h, sc);
          }
        }
      }
      h = xchg.sum(segment_sum(h, G), lane);
      VisT vnew = vis_add(vis, visv[k1], dsign);
      if (PROP == MPV_PROPOSAL_EXCHANGE) vnew = vis_add(vnew, visv[k2], -dsign);
      Lp lp_new = E::finalize(vnew, h, sc);
      if (a.noise_sigma != 0.0)
        lp_new = (Lp)((double)lp_new + noise_zeta(a.noise_key, segment_code(myword ^ flip, words, G), a.noise_sigma));
      // ref sampler.py:128-129: NaN compares false (reject); the reference raises
      // EvaluationFailureError on any non-finite proposal (rbm.py:242-251): the
      // chain freezes and the first failure is reported.
      if (!isfinite(lp_new) && dsign != 0 && !dead) {
        dead = true;
        if (live && gl == 0 && writer) report_nonfinite(a.status, a.step_index + s + 1, cidx);
      }
      const bool accept = !dead && (dsign == 0 || logu < lp_new - lp);
      const bool moved = accept && dsign != 0;
      vis = moved ? vnew : vis;
      lp = moved ? lp_new : lp;
      myword ^= moved ? flip : 0u;
      n_acc += accept ? 1 : 0;
      // commit (flip): the column entries are re-read from shared memory (cheaper than
      // keeping U entries live in registers across the evaluation)
      if constexpr (kUndo) {
        if (__any_sync(kFull, !moved)) {  // warp-uniform: restore the rejecting chains' theta
          const Sign dund = moved ? A::sign(0) : md;
#pragma unroll
          for (int u = 0; u < U; ++u) acc[u].add(c1[u * G], dund);
        }
      } else if constexpr (PROP == MPV_PROPOSAL_FLIP && !kKeep) {
        const Sign dacc = moved ? d : A::sign(0);
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u].add(c1[u * G], dacc);
      } else {  // exchange: the evaluated theta becomes the state (no column re-read)
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = moved ? nxt[u] : acc[u];
      }
      if (s + 1 == next_record) {
        next_record += thin;
        const int64_t r = a.round_offset + (s + 1) / thin - 1;
        if (live && writer && r < count_c && gl < words) a.samples[(offset_c + r) * words + gl] = myword;
      }
    }
    if (dead) lp = Lp(NAN);

    if (live && writer) {
      if (gl < words) a.bits[cidx * words + gl] = myword;
      if (gl == 0) {
        a.log_probs[cidx] = (double)lp;
        if (a.accepted) a.accepted[cidx] += n_acc;
      }
    }
    if (s_end < a.n_steps) {  // more segments follow: park theta and vis
      float* sv = save_r + (size_t)grp * (U * SW) * 32 + lane;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float* src = reinterpret_cast<const float*>(&acc[u]);
#pragma unroll
        for (int j = 0; j < SW; ++j) sv[(u * SW + j) * 32] = src[j];
      }
      if (live && gl == 0 && writer) vsave[cidx] = vis;
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(done_r + grp), "r"((int)(seg + 1)) : "memory");
  }
  if constexpr (CS > 1) {  // no rank leaves while another may still address its shared memory
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}

}  // namespace mpv
