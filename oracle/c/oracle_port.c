/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference CPU algorithm for the hot path of
 * arXiv 2601.20782's `mpvmc` package (reference tree: /root/reference/pkg/src/mpvmc).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  The product path
 * (paper_2601_20782_b200) never calls it.
 *
 * What is restated (each function cites the reference lines it follows):
 *   orc_mix64 / orc_stream_uniform   rng.py:21-27, 50-53, 63-77 (closed form of StreamSet)
 *   orc_quantize                     _kernels.py:27-48 (Veltkamp split + magic-constant RNE)
 *   orc_quantize_array               rbm.py:91-101 (round_parameters, elementwise)
 *   orc_rounded_forward              _kernels.py:51-92
 *   orc_rounded_log_prob             _kernels.py:95-129
 *   orc_f64_forward                  rbm.py:130-150 (_logcosh_pair / _fast_forward; the
 *                                    reference sums through BLAS/numpy pairwise, here the
 *                                    sums are sequential, so f64 agrees to ~1e-15, not bitwise)
 *   orc_chains_init / orc_chains_step sampler.py:67-88, 111-133 (ChainEnsemble)
 *   orc_local_energies               vmc.py:52-108 (full forward per connected state)
 *
 * Built with -ffp-contract=off so no FMA contraction changes the rounding of
 * the f64 intermediates (numba compiles the reference kernel with fastmath off,
 * _kernels.py:7-8).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL
static const double LOG2 = 0.69314718055994530942;
static const double MAGIC = 6755399441055744.0; /* 1.5 * 2^52, _kernels.py:24 */

uint64_t orc_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static double uniform_from_bits(uint64_t z) { /* rng.py:50-53 */
  return (double)(z >> 12) * 0x1p-52 + 0x1p-53;
}

/* StreamSet(key, n).next_uniform() called t+1 times, stream `chain` (rng.py:71-77):
 * state0 = mix64(key ^ (chain+1)*G); draw t = u(mix64(state0 + (t+1)*G)). */
double orc_stream_uniform(uint64_t key, uint64_t chain, uint64_t t) {
  uint64_t s0 = orc_mix64(key ^ ((chain + 1) * GOLDEN));
  return uniform_from_bits(orc_mix64(s0 + (t + 1) * GOLDEN));
}

void orc_stream_uniforms(uint64_t key, int64_t n_chains, int64_t chain0, int64_t t0, int64_t n_draws,
                         double* out /* [n_draws][n_chains] */) {
  for (int64_t t = 0; t < n_draws; ++t)
    for (int64_t c = 0; c < n_chains; ++c)
      out[t * n_chains + c] = orc_stream_uniform(key, (uint64_t)(chain0 + c), (uint64_t)(t0 + t));
}

/* Quantizer constants of one reduced format (rbm.py:187-200). */
typedef struct {
  double spl, mn, iq, qq, maxf;
  int is_f64;
} qfmt;

static double orc_quantize(double value, const qfmt* f) { /* _kernels.py:27-48 */
  if (f->is_f64) return value;
  if (value == 0.0 || !isfinite(value)) return value;
  double mag = fabs(value);
  if (mag >= f->mn) {
    double y = f->spl * value;
    double r = y - (y - value);
    if (fabs(r) > f->maxf) return copysign(INFINITY, r);
    return r;
  }
  double z = value * f->iq;
  double rounded = (z + MAGIC) - MAGIC;
  return rounded * f->qq;
}

/* fmt: 0=f64 1=f32 2=f16 3=bf16 (precision.py:64-67) */
static qfmt make_qfmt(int fmt) {
  qfmt q;
  memset(&q, 0, sizeof q);
  int mbits, emin, emax;
  switch (fmt) {
    case 1: mbits = 23; emin = -126; emax = 127; break;
    case 2: mbits = 10; emin = -14; emax = 15; break;
    case 3: mbits = 7; emin = -126; emax = 127; break;
    default: q.is_f64 = 1; return q;
  }
  double quantum = ldexp(1.0, emin - mbits);
  q.spl = ldexp(1.0, 52 - mbits) + 1.0;
  q.mn = ldexp(1.0, emin);
  q.iq = 1.0 / quantum;
  q.qq = quantum;
  q.maxf = (2.0 - ldexp(1.0, -mbits)) * ldexp(1.0, emax);
  return q;
}

double orc_quantize_fmt(double v, int fmt) {
  qfmt q = make_qfmt(fmt);
  return orc_quantize(v, &q);
}

/* Elementwise RNE rounding of an array to fmt: the two-copy snapshot of
 * rbm.round_parameters (rbm.py:91-101), applied to Re and Im separately. */
void orc_quantize_array(const double* in, int64_t n, int fmt, double* out) {
  qfmt q = make_qfmt(fmt);
  for (int64_t i = 0; i < n; ++i) out[i] = orc_quantize(in[i], &q);
}

/* One row of _kernels.rounded_forward (_kernels.py:58-92); im lanes skipped when
 * want_im == 0 (that is rounded_log_prob, _kernels.py:95-129). */
static void rounded_row(const uint8_t* x, int N, int M, const double* a_re, const double* a_im,
                        const double* b_re, const double* b_im, const double* w_re,
                        const double* w_im, const qfmt* f, int want_im, double* lp, double* re,
                        double* im) {
  double vr = 0.0, vi = 0.0;
  for (int k = 0; k < N; ++k)
    if (x[k]) {
      vr = orc_quantize(vr + a_re[k], f);
      if (want_im) vi = orc_quantize(vi + a_im[k], f);
    }
  double hr_sum = 0.0, hi_sum = 0.0;
  for (int i = 0; i < M; ++i) {
    double tr = b_re[i], ti = b_im[i];
    const double* wr_row = w_re + (size_t)i * N;
    const double* wi_row = w_im + (size_t)i * N;
    for (int k = 0; k < N; ++k)
      if (x[k]) {
        tr = orc_quantize(tr + wr_row[k], f);
        ti = orc_quantize(ti + wi_row[k], f);
      }
    double u = fabs(tr);
    double v = tr >= 0.0 ? ti : -ti;
    double t = exp(-2.0 * u);
    double wr = (1.0 + t) * cos(v);
    double wi = (1.0 - t) * sin(v);
    double hr = orc_quantize(u - LOG2 + 0.5 * log(wr * wr + wi * wi), f);
    double hi = want_im ? orc_quantize(atan2(wi, wr), f) : 0.0;
    if (i == 0) {
      hr_sum = hr;
      hi_sum = hi;
    } else {
      hr_sum = orc_quantize(hr_sum + hr, f);
      if (want_im) hi_sum = orc_quantize(hi_sum + hi, f);
    }
  }
  double total_re = orc_quantize(vr + hr_sum, f);
  *lp = orc_quantize(2.0 * total_re, f);
  if (want_im) {
    *re = total_re;
    *im = orc_quantize(vi + hi_sum, f);
  }
}

void orc_rounded_forward(const uint8_t* bits, int64_t B, int N, int M, const double* a_re,
                         const double* a_im, const double* b_re, const double* b_im,
                         const double* w_re, const double* w_im, int fmt, double* out_lp,
                         double* out_re, double* out_im, int nthreads) {
  qfmt f = make_qfmt(fmt);
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t s = 0; s < B; ++s)
    rounded_row(bits + s * N, N, M, a_re, a_im, b_re, b_im, w_re, w_im, &f, 1, out_lp + s,
                out_re + s, out_im + s);
}

void orc_rounded_log_prob(const uint8_t* bits, int64_t B, int N, int M, const double* a_re,
                          const double* b_re, const double* b_im, const double* w_re,
                          const double* w_im, int fmt, double* out_lp, int nthreads) {
  qfmt f = make_qfmt(fmt);
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t s = 0; s < B; ++s)
    rounded_row(bits + s * N, N, M, a_re, NULL, b_re, b_im, w_re, w_im, &f, 0, out_lp + s, NULL,
                NULL);
}

/* f64 forward, rbm.py:143-150 with _logcosh_pair rbm.py:130-140. */
static void f64_row(const uint8_t* x, int N, int M, const double* a_re, const double* a_im,
                    const double* b_re, const double* b_im, const double* w_re,
                    const double* w_im, double* re, double* im) {
  double vr = 0.0, vi = 0.0;
  for (int k = 0; k < N; ++k)
    if (x[k]) {
      vr += a_re[k];
      vi += a_im[k];
    }
  double hr_sum = 0.0, hi_sum = 0.0;
  for (int i = 0; i < M; ++i) {
    double tr = b_re[i], ti = b_im[i];
    for (int k = 0; k < N; ++k)
      if (x[k]) {
        tr += w_re[(size_t)i * N + k];
        ti += w_im[(size_t)i * N + k];
      }
    double u = fabs(tr);
    double v = tr < 0.0 ? -ti : ti;
    double t = exp(-2.0 * u);
    double wr = (1.0 + t) * cos(v);
    double wi = (1.0 - t) * sin(v);
    hr_sum += u - LOG2 + 0.5 * log(wr * wr + wi * wi);
    hi_sum += atan2(wi, wr);
  }
  *re = vr + hr_sum;
  *im = vi + hi_sum;
}

void orc_f64_forward(const uint8_t* bits, int64_t B, int N, int M, const double* a_re,
                     const double* a_im, const double* b_re, const double* b_im,
                     const double* w_re, const double* w_im, double* out_lp, double* out_re,
                     double* out_im, int nthreads) {
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t s = 0; s < B; ++s) {
    double re, im;
    f64_row(bits + s * N, N, M, a_re, a_im, b_re, b_im, w_re, w_im, &re, &im);
    if (out_re) out_re[s] = re;
    if (out_im) out_im[s] = im;
    if (out_lp) out_lp[s] = 2.0 * re;
  }
}

/* ---- ChainEnsemble (sampler.py:48-167), one OpenMP thread per chain block. ---- */

typedef struct {
  int N, M, fmt; /* fmt as above; 0 -> f64 forward */
  const double *a_re, *a_im, *b_re, *b_im, *w_re, *w_im;
} orc_model;

static double model_lp(const orc_model* m, const uint8_t* x, const qfmt* f) {
  if (m->fmt == 0) {
    double re, im;
    f64_row(x, m->N, m->M, m->a_re, m->a_im, m->b_re, m->b_im, m->w_re, m->w_im, &re, &im);
    return 2.0 * re;
  }
  double lp;
  rounded_row(x, m->N, m->M, m->a_re, NULL, m->b_re, m->b_im, m->w_re, m->w_im, f, 0, &lp, NULL,
              NULL);
  return lp;
}

/* _initial_bits (sampler.py:67-88).  proposal 0 = flip (N draws), 1 = exchange
 * (Fisher-Yates over a weight-w template, N-1 draws).  Returns the number of
 * draws consumed per chain. */
int64_t orc_chains_init(uint64_t key, int64_t n_chains, int64_t chain0, int N, int proposal,
                        int weight, uint8_t* bits) {
  for (int64_t c = 0; c < n_chains; ++c) {
    uint8_t* x = bits + c * N;
    uint64_t gc = (uint64_t)(chain0 + c);
    if (proposal == 0) {
      for (int k = 0; k < N; ++k) x[k] = orc_stream_uniform(key, gc, (uint64_t)k) < 0.5;
    } else {
      for (int k = 0; k < N; ++k) x[k] = k < weight;
      uint64_t t = 0;
      for (int i = N - 1; i > 0; --i) {
        int64_t j = (int64_t)(orc_stream_uniform(key, gc, t++) * (double)(i + 1));
        uint8_t vi = x[i];
        x[i] = x[j];
        x[j] = vi;
      }
    }
  }
  return proposal == 0 ? N : N - 1;
}

void orc_log_probs(const orc_model* m, const uint8_t* bits, int64_t B, double* out, int nthreads) {
  qfmt f = make_qfmt(m->fmt);
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t s = 0; s < B; ++s) out[s] = model_lp(m, bits + s * m->N, &f);
}

/* n_steps of ChainEnsemble.step (sampler.py:111-133).  `t_draw` is the draw
 * index of the first step's selection draw (init draws + 2 * steps done).
 * Optional sample recording reproduces collect() (sampler.py:142-167): after
 * every `thin` steps round r is recorded for chains with r < count_c into row
 * offset_c + r of `samples` (global chain ids, base/extra of n_samples). */
void orc_chains_step(const orc_model* m, uint64_t key, int64_t n_chains, int64_t chain0,
                     int proposal, uint8_t* bits, double* logp, int64_t* accepted,
                     int64_t t_draw, int64_t n_steps, int64_t thin, int64_t base, int64_t extra,
                     uint8_t* samples, int nthreads) {
  const int N = m->N;
  const int64_t n_pairs = (int64_t)N * (N - 1) / 2;
  qfmt f = make_qfmt(m->fmt);
#pragma omp parallel num_threads(nthreads)
  {
    uint8_t* prop = (uint8_t*)malloc((size_t)N);
#pragma omp for schedule(static)
    for (int64_t c = 0; c < n_chains; ++c) {
      uint64_t gc = (uint64_t)(chain0 + c);
      uint64_t s0 = orc_mix64(key ^ ((gc + 1) * GOLDEN));
      uint8_t* x = bits + c * N;
      int64_t acc = 0;
      int64_t count = base + ((int64_t)gc < extra ? 1 : 0);
      int64_t offset = (int64_t)gc * base + ((int64_t)gc < extra ? (int64_t)gc : extra);
      for (int64_t st = 0; st < n_steps; ++st) {
        uint64_t t = (uint64_t)(t_draw + 2 * st);
        double u_sel = uniform_from_bits(orc_mix64(s0 + (t + 1) * GOLDEN));
        memcpy(prop, x, (size_t)N);
        if (proposal == 0) {
          int64_t site = (int64_t)(u_sel * (double)N);
          prop[site] ^= 1;
        } else {
          int64_t idx = (int64_t)(u_sel * (double)n_pairs);
          /* lexicographic (i<j) pair table, sampler.py:42-45 */
          int i = 0;
          int64_t rem = idx;
          while (rem >= N - 1 - i) {
            rem -= N - 1 - i;
            ++i;
          }
          int j = i + 1 + (int)rem;
          uint8_t vi = prop[i];
          prop[i] = prop[j];
          prop[j] = vi;
        }
        double lp_new = model_lp(m, prop, &f);
        double u_acc = uniform_from_bits(orc_mix64(s0 + (t + 2) * GOLDEN));
        if (log(u_acc) < lp_new - logp[c]) { /* NaN compares false: reject */
          memcpy(x, prop, (size_t)N);
          logp[c] = lp_new;
          ++acc;
        }
        if (samples && thin > 0 && (st + 1) % thin == 0) {
          int64_t r = (st + 1) / thin - 1;
          if (r < count) memcpy(samples + (offset + r) * N, x, (size_t)N);
        }
      }
      accepted[c] += acc;
    }
    free(prop);
  }
}

/* vmc.local_energies (vmc.py:60-108) for one configuration with the f64 forward:
 * eps = J sum_bonds s_i s_j + sum_{x'} H(x,x') exp(logpsi(x') - logpsi(x)).
 * ham: 0 = TFIM (flip every site, H = h), 1 = Heisenberg (swap differing bonds, H = 2J).
 * Returns 0, or 1 when a ratio or eps is non-finite (EvaluationFailureError). */
int orc_local_energies(const orc_model* m, int ham, const int64_t* bonds, int n_bonds, double J,
                       double h, const uint8_t* bits, int64_t B, double* eps_re, double* eps_im,
                       int nthreads) {
  const int N = m->N;
  int bad = 0;
#pragma omp parallel num_threads(nthreads) reduction(| : bad)
  {
    uint8_t* y = (uint8_t*)malloc((size_t)N);
#pragma omp for schedule(static)
    for (int64_t s = 0; s < B; ++s) {
      const uint8_t* x = bits + s * N;
      double br, bi;
      f64_row(x, N, m->M, m->a_re, m->a_im, m->b_re, m->b_im, m->w_re, m->w_im, &br, &bi);
      double diag = 0.0;
      for (int b = 0; b < n_bonds; ++b) {
        double si = 1.0 - 2.0 * x[bonds[2 * b]], sj = 1.0 - 2.0 * x[bonds[2 * b + 1]];
        diag += si * sj;
      }
      double er = J * diag, ei = 0.0;
      if (ham == 0 && h != 0.0) {
        double sr = 0.0, si_ = 0.0;
        for (int k = 0; k < N; ++k) {
          memcpy(y, x, (size_t)N);
          y[k] ^= 1;
          double yr, yi;
          f64_row(y, N, m->M, m->a_re, m->a_im, m->b_re, m->b_im, m->w_re, m->w_im, &yr, &yi);
          double mag = exp(yr - br);
          if (!isfinite(mag)) bad = 1;
          sr += mag * cos(yi - bi);
          si_ += mag * sin(yi - bi);
        }
        er += h * sr;
        ei += h * si_;
      } else if (ham == 1) {
        for (int b = 0; b < n_bonds; ++b) {
          int i = (int)bonds[2 * b], k = (int)bonds[2 * b + 1];
          if (x[i] == x[k]) continue;
          memcpy(y, x, (size_t)N);
          y[i] = x[k];
          y[k] = x[i];
          double yr, yi;
          f64_row(y, N, m->M, m->a_re, m->a_im, m->b_re, m->b_im, m->w_re, m->w_im, &yr, &yi);
          double mag = exp(yr - br);
          if (!isfinite(mag)) bad = 1;
          er += 2.0 * J * mag * cos(yi - bi);
          ei += 2.0 * J * mag * sin(yi - bi);
        }
      }
      if (!isfinite(er) || !isfinite(ei)) bad = 1;
      eps_re[s] = er;
      eps_im[s] = ei;
    }
    free(y);
  }
  return bad;
}
