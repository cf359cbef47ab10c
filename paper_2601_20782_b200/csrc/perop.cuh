// Reference-emulation ("per_operation") forward and sampler, plus the f64
// forward.  These recompute log p of every proposal from scratch, exactly in
// the reference's canonical operation order (ref: _kernels.py:51-129,
// precision.py:287-338): visible term and every theta_i accumulated over the
// set bits in ascending k with one rounding per add, log cosh in f64 rounded
// once, hidden sum rounded sequentially in ascending i, then the rounded
// total and doubling.  Native f16/bf16/f32 adds reproduce the reference's
// f64-add-then-round bit for bit (double rounding is innocuous for p <= 24);
// only a CUDA-vs-glibc f64 libm ulp at a rounding boundary can differ.
#pragma once
#include "common.cuh"

namespace mpv {

// fmt-specific scalar ops on values stored as the table's element type.
template <int FMT> struct PerOp;
template <> struct PerOp<MPV_FMT_F16> {
  using Entry = uint32_t;
  using S = uint16_t;
  __device__ static S re(Entry e) { return (S)(e & 0xFFFF); }
  __device__ static S im(Entry e) { return (S)(e >> 16); }
  __device__ static S add(S a, S b) { return Half<MPV_FMT_F16>::add(a, b); }
  __device__ static double f64(S a) { return Half<MPV_FMT_F16>::to_f64(a); }
  __device__ static S q(double v) { return Half<MPV_FMT_F16>::from_f64(v); }
  __device__ static S from_vis(float v) { return __half_as_ushort(__float2half_rn(v)); }
};
template <> struct PerOp<MPV_FMT_BF16> {
  using Entry = uint32_t;
  using S = uint16_t;
  __device__ static S re(Entry e) { return (S)(e & 0xFFFF); }
  __device__ static S im(Entry e) { return (S)(e >> 16); }
  __device__ static S add(S a, S b) { return Half<MPV_FMT_BF16>::add(a, b); }
  __device__ static double f64(S a) { return Half<MPV_FMT_BF16>::to_f64(a); }
  __device__ static S q(double v) { return Half<MPV_FMT_BF16>::from_f64(v); }
  __device__ static S from_vis(float v) { return __bfloat16_as_ushort(__float2bfloat16_rn(v)); }
};
template <> struct PerOp<MPV_FMT_F32> {
  using Entry = float2;
  using S = float;
  __device__ static S re(Entry e) { return e.x; }
  __device__ static S im(Entry e) { return e.y; }
  __device__ static S add(S a, S b) { return __fadd_rn(a, b); }
  __device__ static double f64(S a) { return (double)a; }
  __device__ static S q(double v) { return __double2float_rn(v); }
  __device__ static S from_vis(float v) { return v; }
};

struct FwdArgs {
  int N, M, Mpad, words;
  int GU;             // units per rank block (Mpad for an unsplit snapshot)
  int64_t RB;         // elements per rank block (16-byte padded)
  const void* table;  // rank blocks [Mpad / GU][N][GU] entries (include/mpvmc_b200.h)
  const void* bias;   // [Mpad] entries
  const void* vis;    // [N] float (per-op: a_re exact) or double (f64)
  const double* vis_im;
  const uint32_t* bits;  // [B][words]
  int64_t B;
  double *out_lp, *out_re, *out_im;
  int64_t* status;
};

// One warp evaluates one configuration (packed words in shared memory `wbuf`).
// hbuf: per-warp scratch of 2*M doubles.  Returns lp in every lane; re/im if want_im.
template <int FMT>
__device__ double warp_forward_perop(const FwdArgs& a, const uint32_t* wbuf, double* hbuf,
                                     bool want_im, double* out_re, double* out_im) {
  using P = PerOp<FMT>;
  using Entry = typename P::Entry;
  using S = typename P::S;
  const int lane = threadIdx.x & 31;
  const Entry* tab = reinterpret_cast<const Entry*>(a.table);
  const Entry* bias = reinterpret_cast<const Entry*>(a.bias);
  for (int i = lane; i < a.M; i += 32) {
    const Entry b = bias[i];
    S tr = P::re(b), ti = P::im(b);
    for (int w = 0; w < a.words; ++w) {
      uint32_t word = wbuf[w];
      while (word) {
        const int k = w * 32 + __ffs(word) - 1;
        word &= word - 1;
        const Entry e = tab[(size_t)(i / a.GU) * a.RB + (size_t)k * a.GU + i % a.GU];
        tr = P::add(tr, P::re(e));
        ti = P::add(ti, P::im(e));
      }
    }
    // _kernels.py:101-106 in f64, one rounding of the result
    const double dtr = P::f64(tr), dti = P::f64(ti);
    const double u = fabs(dtr);
    const double v = dtr >= 0.0 ? dti : -dti;
    const double t = exp(-2.0 * u);
    double sv, cv;
    sincos(v, &sv, &cv);  // one shared argument reduction (same values as cos(v), sin(v))
    const double wr = __dmul_rn(__dadd_rn(1.0, t), cv);
    const double wi = __dmul_rn(__dadd_rn(1.0, -t), sv);
    const double qq = __dadd_rn(__dmul_rn(wr, wr), __dmul_rn(wi, wi));
    const double hr = __dadd_rn(__dadd_rn(u, -0.69314718055994530942), __dmul_rn(0.5, log(qq)));
    hbuf[i] = P::f64(P::q(hr));
    if (want_im) hbuf[a.M + i] = P::f64(P::q(atan2(wi, wr)));
  }
  __syncwarp();
  double lp = 0.0, re = 0.0, im = 0.0;
  if (lane == 0) {
    const float* visr = reinterpret_cast<const float*>(a.vis);
    S vr = P::q(0.0), vi = P::q(0.0);
    for (int w = 0; w < a.words; ++w) {
      uint32_t word = wbuf[w];
      while (word) {
        const int k = w * 32 + __ffs(word) - 1;
        word &= word - 1;
        vr = P::add(vr, P::from_vis(visr[k]));
        if (want_im) vi = P::add(vi, P::q(a.vis_im[k]));
      }
    }
    S hs = P::q(hbuf[0]), his = want_im ? P::q(hbuf[a.M]) : P::q(0.0);
    for (int i = 1; i < a.M; ++i) {
      hs = P::add(hs, P::q(hbuf[i]));
      if (want_im) his = P::add(his, P::q(hbuf[a.M + i]));
    }
    const S tot = P::add(vr, hs);
    lp = P::f64(P::add(tot, tot));  // q(2*total) == RN(total + total)
    re = P::f64(tot);
    im = want_im ? P::f64(P::add(vi, his)) : 0.0;
  }
  __syncwarp();
  lp = __shfl_sync(kFull, lp, 0);
  if (want_im) {
    *out_re = __shfl_sync(kFull, re, 0);
    *out_im = __shfl_sync(kFull, im, 0);
  }
  return lp;
}

// f64 forward (ref: rbm.py:143-150): theta in f64, complex log cosh
// (rbm.py:130-140), f64 sums.  Table entries are double2, vis double.
__device__ double warp_forward_f64(const FwdArgs& a, const uint32_t* wbuf, double* hbuf,
                                   bool want_im, double* out_re, double* out_im) {
  const int lane = threadIdx.x & 31;
  const double2* tab = reinterpret_cast<const double2*>(a.table);
  const double2* bias = reinterpret_cast<const double2*>(a.bias);
  double hr_part = 0.0, hi_part = 0.0;
  for (int i = lane; i < a.M; i += 32) {
    double2 th = bias[i];
    for (int w = 0; w < a.words; ++w) {
      uint32_t word = wbuf[w];
      while (word) {
        const int k = w * 32 + __ffs(word) - 1;
        word &= word - 1;
        const double2 e = tab[(size_t)(i / a.GU) * a.RB + (size_t)k * a.GU + i % a.GU];
        th.x += e.x;
        th.y += e.y;
      }
    }
    const double u = fabs(th.x);
    const double v = th.x < 0.0 ? -th.y : th.y;
    const double t = exp(-2.0 * u);
    double sv, cv;
    sincos(v, &sv, &cv);  // one shared argument reduction (same values as cos(v), sin(v))
    const double wr = __dmul_rn(__dadd_rn(1.0, t), cv);
    const double wi = __dmul_rn(__dadd_rn(1.0, -t), sv);
    const double qq = __dadd_rn(__dmul_rn(wr, wr), __dmul_rn(wi, wi));
    hr_part += __dadd_rn(__dadd_rn(u, -0.69314718055994530942), __dmul_rn(0.5, log(qq)));
    if (want_im) hi_part += atan2(wi, wr);
  }
  (void)hbuf;
  double vr = 0.0, vi = 0.0;
  const double* visr = reinterpret_cast<const double*>(a.vis);
  for (int w = 0; w < a.words; ++w) {
    uint32_t word = wbuf[w];
    while (word) {
      const int k = w * 32 + __ffs(word) - 1;
      word &= word - 1;
      vr += visr[k];
      if (want_im) vi += a.vis_im[k];
    }
  }
  hr_part = segment_sum(hr_part, 32);
  if (want_im) {
    hi_part = segment_sum(hi_part, 32);
    *out_re = vr + hr_part;
    *out_im = vi + hi_part;
  }
  return 2.0 * (vr + hr_part);
}

template <int FMT>  // FMT_F64 selects the f64 forward
__global__ void __launch_bounds__(256) forward_kernel(const FwdArgs a, int want_im) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  uint32_t* wbuf = reinterpret_cast<uint32_t*>(smem_raw) + warp * 32;
  double* hbuf = reinterpret_cast<double*>(smem_raw + nw * 32 * sizeof(uint32_t)) +
                 (size_t)warp * 2 * a.M;
  for (int64_t row = (int64_t)blockIdx.x * nw + warp; row < a.B; row += (int64_t)gridDim.x * nw) {
    if (lane < a.words) wbuf[lane] = a.bits[row * a.words + lane];
    __syncwarp();
    double re = 0.0, im = 0.0, lp;
    if constexpr (FMT == MPV_FMT_F64) lp = warp_forward_f64(a, wbuf, hbuf, want_im, &re, &im);
    else lp = warp_forward_perop<FMT>(a, wbuf, hbuf, want_im, &re, &im);
    if (lane == 0) {
      a.out_lp[row] = lp;
      if (a.out_re) a.out_re[row] = re;
      if (a.out_im) a.out_im[row] = im;
      const bool bad = !isfinite(lp) || (want_im && (!isfinite(re) || !isfinite(im)));
      if (bad && a.status) {
        atomicMin((unsigned long long*)&a.status[1], (unsigned long long)row);
        atomicExch((unsigned long long*)&a.status[0], (unsigned long long)MPV_ERR_NONFINITE);
      }
    }
    __syncwarp();
  }
}

// Per-operation MH sweep: one warp per chain, full per-op forward of every
// proposal (ref: sampler.py:111-133 with rbm.log_prob_evaluator(..., PER_OPERATION)).
struct PerOpSweepArgs {
  FwdArgs f;
  int64_t n_chains, chain_offset;
  uint32_t* bits;
  double* log_probs;
  int64_t* accepted;
  int64_t* status;
  uint64_t key;
  int64_t init_draws, step_index, n_steps, thin;
  uint32_t* samples;
  int64_t sample_base, sample_extra, round_offset, row0;
};

template <int FMT, int PROP>
__global__ void __launch_bounds__(128) perop_sweep_kernel(const PerOpSweepArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int words = a.f.words, N = a.f.N;
  uint32_t* cur = reinterpret_cast<uint32_t*>(smem_raw) + warp * 64;
  uint32_t* prop = cur + 32;
  double* hbuf = reinterpret_cast<double*>(smem_raw + nw * 64 * sizeof(uint32_t)) +
                 (size_t)warp * 2 * a.f.M;
  const int64_t chain = (int64_t)blockIdx.x * nw + warp;
  if (chain >= a.n_chains) return;  // whole warp exits together
  const int64_t gchain = a.chain_offset + chain;
  if (lane < words) cur[lane] = a.bits[chain * words + lane];
  __syncwarp();
  double dummy_re, dummy_im;
  double lp = warp_forward_perop<FMT>(a.f, cur, hbuf, false, &dummy_re, &dummy_im);
  bool dead = !isfinite(lp);
  if (dead && lane == 0 && a.status) {
    atomicMin((unsigned long long*)&a.status[1], (unsigned long long)((0ll << 32) | chain));
    atomicExch((unsigned long long*)&a.status[0], (unsigned long long)MPV_ERR_NONFINITE);
  }
  const uint64_t s0 = stream_state(a.key, (uint64_t)gchain);
  const int64_t count_c = a.sample_base + (gchain < a.sample_extra ? 1 : 0);
  const int64_t offset_c =
      gchain * a.sample_base + (gchain < a.sample_extra ? gchain : a.sample_extra) - a.row0;
  const double n_pairs = 0.5 * (double)N * (double)(N - 1);
  int64_t n_acc = 0;
  for (int64_t s = 0; s < a.n_steps; ++s) {
    const uint64_t t = (uint64_t)(a.init_draws + 2 * (a.step_index + s));
    const double us = stream_draw(s0, t);
    int k1, k2 = -1;
    if (PROP == MPV_PROPOSAL_FLIP) {
      k1 = (int)floor_scaled(us, (double)N);
    } else {
      pair_of(floor_scaled(us, n_pairs), N, k1, k2);
    }
    if (lane < words) {
      uint32_t w = cur[lane];
      if (PROP == MPV_PROPOSAL_FLIP) {
        if (lane == (k1 >> 5)) w ^= 1u << (k1 & 31);
      } else {
        const int bi = (cur[k1 >> 5] >> (k1 & 31)) & 1u, bj = (cur[k2 >> 5] >> (k2 & 31)) & 1u;
        if (bi != bj) {
          if (lane == (k1 >> 5)) w ^= 1u << (k1 & 31);
          if (lane == (k2 >> 5)) w ^= 1u << (k2 & 31);
        }
      }
      prop[lane] = w;
    }
    __syncwarp();
    const double lp_new = warp_forward_perop<FMT>(a.f, prop, hbuf, false, &dummy_re, &dummy_im);
    const double ua = stream_draw(s0, t + 1);
    if (!isfinite(lp_new) && !dead) {
      dead = true;
      if (lane == 0 && a.status) {
        atomicMin((unsigned long long*)&a.status[1],
                  (unsigned long long)(((a.step_index + s + 1) << 32) | chain));
        atomicExch((unsigned long long*)&a.status[0], (unsigned long long)MPV_ERR_NONFINITE);
      }
    }
    const bool accept = !dead && (log(ua) < lp_new - lp);
    if (accept) {
      lp = lp_new;
      ++n_acc;
      if (lane < words) cur[lane] = prop[lane];
    }
    __syncwarp();
    if (a.samples && a.thin > 0 && ((s + 1) % a.thin) == 0) {
      const int64_t r = a.round_offset + (s + 1) / a.thin - 1;
      if (r < count_c && lane < words) a.samples[(offset_c + r) * words + lane] = cur[lane];
    }
  }
  if (lane < words) a.bits[chain * words + lane] = cur[lane];
  if (lane == 0) {
    a.log_probs[chain] = lp;
    if (a.accepted) a.accepted[chain] += n_acc;
  }
}

}  // namespace mpv
