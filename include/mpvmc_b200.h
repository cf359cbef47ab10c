/*
 * mpvmc_b200 — C ABI of the B200 (sm_100a) hot path for arXiv 2601.20782:
 * batched Metropolis–Hastings sampling of an RBM neural quantum state in
 * reduced precision, plus the local energies that consume the samples.
 *
 * Every entry point takes caller-owned DEVICE pointers and a cudaStream_t
 * (passed as void*), launches asynchronously on that stream and returns an
 * int status (MPV_OK ... MPV_ERR_NONFINITE).  The library never allocates
 * device memory and keeps no state except a thread-local error string
 * (mpv_last_error).  Citations "ref:" are into the reference package
 * /root/reference/pkg/src/mpvmc/ (file:line) — the interface each function
 * replaces; INTEGRATION.md shows the ctypes binding the reference would add.
 */
#ifndef MPVMC_B200_H
#define MPVMC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define MPV_OK 0
#define MPV_ERR_ARGS 1
#define MPV_ERR_CUDA 2
#define MPV_ERR_NONFINITE 3

/* float formats (ref: precision.py:64-67) */
#define MPV_FMT_F64 0
#define MPV_FMT_F32 1
#define MPV_FMT_F16 2
#define MPV_FMT_BF16 3

/* rounding modes (ref: precision.py:158-169, plus the device NATIVE mode) */
#define MPV_MODE_NATIVE 0
#define MPV_MODE_PER_OPERATION 1
#define MPV_MODE_STORAGE_ONLY 2

/* exact-theta accumulator variants of the fused sweep */
#define MPV_ACC_X1 0  /* one f32 accumulator per component, exact by host planner check */
#define MPV_ACC_X2 1  /* hi/lo f32 accumulators on a fixed split grid, exact */
#define MPV_ACC_F64 2 /* f64 accumulators */
#define MPV_ACC_XI 3  /* int32 accumulators in units of the snapshot quantum (exact) */

/* proposals (ref: sampler.py:24-39) */
#define MPV_PROPOSAL_FLIP 0
#define MPV_PROPOSAL_EXCHANGE 1

/* Hamiltonians (ref: hamiltonians.py:28-46) */
#define MPV_HAM_TFIM 0
#define MPV_HAM_HEISENBERG 1

/*
 * A prepared parameter snapshot in kernel layout (the device counterpart of
 * ref: rbm.py:161-200 _PreparedRounded, built by the host from
 * round_parameters(params, fmt), ref: rbm.py:91-101).  Column-major by site
 * so one flip reads one contiguous column.  The hidden units are split into
 * `cluster` rank blocks of GU = lanes_per_chain * units_per_lane units
 * (hidden_pad = cluster * GU): entry (k, i) of rank block r = i / GU sits at
 * element r * RB + k * GU + i % GU, RB = round_up(N * GU * entry, 16) / entry
 * (cluster = 1: table[k * hidden_pad + i]).  With cluster > 1 the fused sweep
 * runs as thread-block clusters: CTA rank r stages block r in shared memory
 * and the ranks exchange partial log-cosh sums over distributed shared memory
 * every step (tables beyond one SM's shared memory stay on chip).
 *   entry type      table/bias element            vis element
 *   X1, PER_OP      fmt pair (re,im): 4 B f16/bf16, 8 B f32      float (a_re)
 *   X2              two fmt pairs (hi, lo)                       float2 (hi, lo)
 *   F64             double2 (re, im)                             double
 *   XI              int2 (re, im) = value / quantum              int
 * `vis_im` (double[N], a_im) is only read by mpv_snapshot_forward (log psi).
 * For the fused sweep `vis` must sit at table + cluster * RB * entry:
 * [table | vis] is staged into shared memory with bulk copies.
 */
typedef struct {
  int32_t n_visible, n_hidden, hidden_pad;
  int32_t fmt, mode, variant;
  int32_t lanes_per_chain, units_per_lane;
  int32_t cluster; /* 1, 2 or 4 rank blocks (mpv_plan_cluster) */
  const void* table;
  const void* bias;
  const void* vis;
  const double* vis_im;
  double quantum; /* XI: table integers are multiples of this power of two (>= 2^-100) */
  /* Frozen Gaussian log-density noise (ref: rbm.py:333-352 NoiseField,
   * rbm.py:408-416 noisy_log_prob_evaluator): log p(x) += noise_sigma *
   * ndtri(counter_uniform(noise_key, code(x))) with code(x) = sum_k bit_k 2^k
   * (rng.py:56-60, 86-96).  noise_sigma == 0 disables it; only for f64
   * arithmetic (fmt F64 / STORAGE_ONLY) and n_visible <= 64. */
  uint64_t noise_key;
  double noise_sigma;
} mpv_snapshot;

/* ---- snapshot build on the device (ref: rbm.py:91-101 round_parameters and
 *      rbm.py:161-200 _PreparedRounded) ----
 * mpv_snapshot_bytes: out[0] = bytes of the [table | vis] blob, out[1] = offset
 * of vis in it, out[2] = bias bytes, for the layout (fmt, mode, variant, hidden_pad).
 * mpv_snapshot_round: params = [a (N) | b (M) | w_t (N x M)] complex f64 (re, im)
 * on the device; writes every component rounded RNE to fmt into `rounded` (same
 * layout) and plan[0..3] = {finest power-of-two quantum of a_re, b, w (1 if all
 * zero), max_i |b_re_i| + sum_k |w_re_ki|, the same for im, sum_k |a_re_k|}
 * (`plan` >= 8 doubles of device scratch): the inputs of the exact-accumulator
 * planner (paper_2601_20782_b200/rbm.py plan_exact).
 * mpv_snapshot_fill: writes table/bias/vis (and vis_im if set) of `snap`, whose
 * layout fields and buffers the caller has set, from `rounded`; split = X2 grid. */
int mpv_snapshot_bytes(int n_visible, int hidden_pad, int fmt, int mode, int variant, int cluster, size_t* out);
int mpv_snapshot_round(int N, int M, int fmt, const double* params, double* rounded, double* plan,
                       void* stream);
int mpv_snapshot_fill(const mpv_snapshot* snap, const double* rounded, double split, void* stream);

/* Chain state of one shard (device pointers; ref: sampler.py:55-65 state). */
typedef struct {
  int64_t n_chains;     /* chains in this shard */
  int64_t chain_offset; /* global id of chain 0: draws depend on global ids only */
  int32_t n_sites, words; /* words = ceil(n_sites / 32) */
  uint32_t* bits;        /* [n_chains][words], bit k of a chain in word k>>5, bit k&31 */
  double* log_probs;     /* [n_chains] */
  int64_t* accepted;     /* [n_chains] accepted proposals since reset */
  int64_t* status;       /* [2]: {code, step*2^32 + chain of the first non-finite log p} */
  void* scratch;         /* work queue + parked theta: mpv_sweep_scratch_bytes(snap, n_chains) */
  size_t scratch_bytes;
} mpv_chains;

/* ---- RNG (ref: rng.py:63-77 StreamSet.next_uniform, closed form) ---- */
/* out[t][c] = draw t0+t of stream chain0+c of `key`. */
int mpv_stream_uniforms(uint64_t key, int64_t n_chains, int64_t chain0, int64_t t0,
                        int64_t n_draws, double* out, void* stream);

/* ---- chain initialisation (ref: sampler.py:67-88 ChainEnsemble._initial_bits) ----
 * flip: bit_k = u_k < 0.5 (N draws); exchange: Fisher–Yates of a weight-w
 * template (N-1 draws).  Writes ch->bits; zeroes accepted/status. */
int mpv_chains_init(const mpv_chains* ch, uint64_t key, int proposal, int sector_weight,
                    void* stream);

/* ---- fused MH sweep (ref: sampler.py:111-133 ChainEnsemble.step x n_steps,
 *      sampler.py:142-167 collect) ----
 * Runs n_steps proposals per chain.  step_index = proposals already made by
 * this ensemble (the draw counter is init_draws + 2*step_index).  The cached
 * log p is recomputed from the bits at launch start (set_evaluator
 * semantics, ref: sampler.py:90-93) and written back at the end.
 * If samples != NULL: after every `thin` steps round r = round_offset + j is
 * recorded for chain c (global id) when r < count_c, into row offset_c + r
 * relative to the shard's first row `row0` (count_c, offset_c from
 * n_samples_total over n_chains_total, ref: sampler.py:152-166). */
size_t mpv_sweep_scratch_bytes(const mpv_snapshot* snap, int64_t n_chains);
int mpv_mh_sweep(const mpv_snapshot* snap, const mpv_chains* ch, uint64_t key, int proposal,
                 int64_t init_draws, int64_t step_index, int64_t n_steps, int64_t thin,
                 uint32_t* samples, int64_t n_samples_total, int64_t n_chains_total,
                 int64_t round_offset, int64_t row0, void* stream);

/* ---- MH sweep over a dense log-probability table (ref: sampler.py:254-268
 *      table_log_prob / uniform_log_prob driven by ChainEnsemble.step) ----
 * table: f64[2^n_sites] (device), indexed by the configuration code (bit k of
 * the code = site k); n_sites <= 30, ch->words == 1.  Same draw schedule,
 * sample layout and f64 accept test as mpv_mh_sweep; no finiteness check
 * (the reference's table evaluator has none: -inf targets are never entered). */
int mpv_table_sweep(const double* table, const mpv_chains* ch, uint64_t key, int proposal,
                    int64_t init_draws, int64_t step_index, int64_t n_steps, int64_t thin,
                    uint32_t* samples, int64_t n_samples_total, int64_t n_chains_total,
                    int64_t round_offset, int64_t row0, void* stream);

/* ---- batched log-probability / log-psi in the snapshot's arithmetic ----
 * bits: packed [B][words].  PER_OPERATION reproduces ref: _kernels.py:51-129
 * (rounded_forward / rounded_log_prob) bit for bit; F64/STORAGE_ONLY follow
 * ref: rbm.py:143-150 (_fast_forward); NATIVE is the fused sweep's arithmetic.
 * out_re/out_im (log psi, may be NULL) are only produced by PER_OPERATION and F64.
 * NATIVE needs `scratch` of mpv_sweep_scratch_bytes(snap, B) (unused otherwise). */
int mpv_snapshot_forward(const mpv_snapshot* snap, const uint32_t* bits, int64_t B,
                         double* out_lp, double* out_re, double* out_im, int64_t* status,
                         void* scratch, size_t scratch_bytes, void* stream);

/* Drop-in for ref: _kernels.py:95-129 rounded_log_prob(bits, a_re, b_re, b_im,
 * w_re, w_im, spl, mn, iq, qq, maxf): uint8 bits [B][N], f64 parameters already
 * on fmt's grid in the reference layout (w row-major [M][N]); the quantizer
 * constants are implied by fmt.  `scratch` >= mpv_rounded_scratch_bytes(B, N, M, fmt). */
size_t mpv_rounded_scratch_bytes(int64_t B, int N, int M, int fmt);
int mpv_rounded_log_prob(const uint8_t* bits, int64_t B, int N, int M, const double* a_re,
                         const double* b_re, const double* b_im, const double* w_re,
                         const double* w_im, int fmt, double* out_lp, void* scratch,
                         void* stream);

/* ---- local energies (ref: vmc.py:52-108 local_energies) ----
 * eps(x) = J sum_bonds s_i s_j + sum_{x'} H(x,x') psi(x')/psi(x) in f64 with
 * the master (unrounded) parameters.  params: a [N], b [M] double2 (re,im);
 * w_t [N][M] double2 (column-major by site).  `tables` is a caller workspace
 * of mpv_energy_tables_bytes(...) filled by mpv_energy_prepare. */
size_t mpv_energy_tables_bytes(int N, int M, int ham, int n_bonds);
int mpv_energy_prepare(int N, int M, const double* a, const double* b, const double* w_t,
                       int ham, const int32_t* bonds, int n_bonds, void* tables, void* stream);
int mpv_local_energies(int N, int M, const double* a, const double* b, const double* w_t,
                       int ham, const int32_t* bonds, int n_bonds, double J, double h,
                       const void* tables, const uint32_t* bits, int64_t B, double* out_eps,
                       int64_t* status, void* stream);
/* General couplings (beyond the reference: J1-J2 bond classes, Marshall sign):
 * eps(x) = sum_b bond_j[b] s_p s_q + sum_t term_coef[t] psi(x_t)/psi(x), with
 * x_t the connected configuration of term t (TFIM: flip of site t; Heisenberg:
 * swap of bond t).  NULL term_coef = h (TFIM) / 2J (Heisenberg) for every term,
 * NULL bond_j = J for every bond (then identical to mpv_local_energies).
 * Marshall sign: term_coef[t] = -2 J_t for bonds joining the two sublattices. */
int mpv_local_energies_ex(int N, int M, const double* a, const double* b, const double* w_t,
                          int ham, const int32_t* bonds, int n_bonds, double J, double h,
                          const double* term_coef, const double* bond_j, const void* tables,
                          const uint32_t* bits, int64_t B, double* out_eps, int64_t* status,
                          void* stream);

/* ---- products with the log-derivative matrix O (ref: rbm.py:307-325
 *      grad_log_psi_batch, O(x) = [x, tanh theta, tanh theta (x) x]; the SR
 *      estimators of vmc.py:145-229 evaluated matrix-free) ----
 * t: tanh(theta) complex [U][M]; bits: packed [U][ceil(N/32)]; v, out:
 * complex P-vectors (P = N + M + M N, order a, b, W row-major); q, u:
 * complex U-vectors.  mpv_logderiv_ov: q = O v.  mpv_logderiv_ohu:
 * out = O^H u = sum_s conj(O_s) u_s (deterministic: fixed-order chunk sums).
 * `scratch` >= mpv_logderiv_scratch_bytes(U, N, M).  N <= 256, M <= 512. */
size_t mpv_logderiv_scratch_bytes(int64_t U, int N, int M);
/* q_s = w_s (O v)_s (w: real [U], NULL = 1) */
int mpv_logderiv_ov(const double* t, const uint32_t* bits, int64_t U, int N, int M, const double* v,
                    const double* w, double* q, void* scratch, void* stream);
/* out = sum_s conj(O_s) w_s u_s; sum_out (NULL = skip) = sum_s w_s u_s */
int mpv_logderiv_ohu(const double* t, const uint32_t* bits, int64_t U, int N, int M, const double* u,
                     const double* w, double* out, double* sum_out, void* scratch, void* stream);
/* t = tanh(b + W x_s) complex [U][M] (ref: rbm.py:316) for params = [a | b | W row-major]
 * complex (the order of RbmParameters.flatten, rbm.py:64-67); same scratch. */
int mpv_logderiv_tanh(const double* params, const uint32_t* bits, int64_t U, int N, int M, double* t,
                      void* scratch, void* stream);
/* dense O_s - obar (obar NULL = uncentred), complex [U][P] (ref: rbm.py:307-325) */
int mpv_logderiv_dense(const double* t, const uint32_t* bits, int64_t U, int N, int M, const double* obar,
                       double* o, void* stream);

/* ---- SR statistics and solve on the device (ref: vmc.py:145-229) ----
 * mpv_sr_smatrix: S = sum_s w_s conj(C_s) C_s^T (Hermitian, real diagonal) for
 * the centred dense C [U][P] complex (w NULL = 1), s [P][P] complex
 * (ref: vmc.py:168-188 s_matrix). */
int mpv_sr_smatrix(const double* c, const double* w, int64_t U, int P, double* s, void* stream);

/* Matrix-free conjugate gradients for (S + lambda) g = F with S v =
 * O^H (w O v) - conj(obar) (obar . v) and obar = sum_s w_s O_s; the
 * vmc.py:202-229 system solved without forming S.  The CG scalars live in
 * `scalars` (double[8]: rr, tol |F|, iterations, done flag, maxiter); every
 * reduction runs in a fixed order.  Single process: mpv_cg_init, then
 * mpv_cg_run(k) batches (read scalars[2..3] between batches).  Across ranks:
 * per iteration mpv_cg_apply(p -> y, ysum), all-reduce [y | ysum], mpv_cg_step. */
typedef struct {
  int32_t n_visible, n_hidden;
  int64_t n_samples;
  const double* t;       /* tanh theta, complex [U][M] */
  const uint32_t* bits;  /* packed [U][ceil(N/32)] */
  const double* w;       /* sample weights, real [U] */
  const double* obar;    /* sum_s w_s O_s (all ranks), complex [P] */
  double lambda;
  double *g, *r, *p, *ap; /* complex [P] */
  double *y, *ysum;       /* complex [P], [1]: O^H (w O p) and sum_s w_s (O p)_s */
  double* q;              /* complex [U] */
  double* partials;       /* double[mpv_cg_partials_len()] */
  double* scalars;        /* double[8] */
  void* scratch;          /* >= mpv_logderiv_scratch_bytes(U, N, M) */
  size_t scratch_bytes;
} mpv_cg;
size_t mpv_cg_partials_len(void);
int mpv_cg_init(const mpv_cg* cg, const double* f, double tol, int64_t maxiter, void* stream);
int mpv_cg_apply(const mpv_cg* cg, const double* v, double* y, double* ysum, void* stream);
int mpv_cg_apply_finish(const mpv_cg* cg, const double* v, const double* y, const double* ysum, double* out,
                        void* stream);
int mpv_cg_step(const mpv_cg* cg, void* stream);
int mpv_cg_run(const mpv_cg* cg, int n_iter, void* stream);

/* minSR sample-space matrix (beyond the reference: the SR step of vmc.py:202-229
 * solved in sample space by the push-through identity) for this rank's rows
 * [row0, row0 + U_rows) of the all-rank sample set against all U_all columns:
 * K = W^1/2 (O - 1 obar^T)(O - 1 obar^T)^H W^1/2 + lambda I, with O O^H formed from
 * the factors (common set bits of the packed rows, T T^H) and d = O conj(obar),
 * obar2 = |obar|^2.  out: [U_rows][U_all] complex, f64 (out_f32 = 0) or f32. */
int mpv_minsr_gram(const double* t_rows, const uint32_t* bits_rows, int64_t U_rows, int64_t row0,
                   const double* t_all, const uint32_t* bits_all, int64_t U_all, int N, int M, const double* d_all,
                   const double* w_all, double obar2, double lambda, int out_f32, void* out, void* stream);

/* Split-chain statistics (ref: vmc.py:592-604, mc_error vmc.py:311-317): per-chain
 * means of Re eps over each chain's sample rows (rows of chain c = global id
 * chain_offset + c: [c base + min(c, extra), ...) - row0, eps_u[inverse[row]]),
 * then out = [mean of the means, sum of squared deviations, n_chains] (two-pass,
 * fixed order).  mpv_moments: the same three numbers for a real vector.
 * partials: double[mpv_cg_partials_len()]. */
int mpv_chain_stats(const double* eps_u, const int64_t* inverse, int64_t n_chains, int64_t chain_offset,
                    int64_t base, int64_t extra, int64_t row0, double* means, double* partials, double* out,
                    void* stream);
int mpv_moments(const double* x, int64_t n, double* partials, double* out, void* stream);

/* ---- batched forward on the tensor cores (north_star (2); ref: rbm.py:130-150
 *      _fast_forward over a batch, i.e. log_psi_batch / log_prob_batch) ----
 * theta = b + W x as a tcgen05 GEMM (f16/bf16 operands, f32 accumulators in
 * TMEM) with the log-cosh sum as its epilogue.  mpv_forward_tc_prepare rounds
 * params = [a (N) | b (M) | w_t (N x M)] complex (re, im) f64 (the layout of
 * mpv_snapshot_round) to fmt (MPV_FMT_F16 / MPV_FMT_BF16, round-to-nearest-
 * even as round_parameters, rbm.py:91-101) into `weights` (device, >=
 * mpv_forward_tc_weights_bytes(N, M); 0 = unsupported shape, N <= 1024).
 * mpv_forward_tc: bits packed [B][ceil(N/32)]; any of out_lp (= 2 Re log psi),
 * out_re, out_im (double[B]) may be NULL but not all; max_ctas <= 0 = one CTA
 * per SM.  Agrees with the f64 forward of the rounded parameters to f32
 * accumulation error (tests/test_gpu_forward_tc.py). */
size_t mpv_forward_tc_weights_bytes(int N, int M);
int mpv_forward_tc_prepare(int N, int M, int fmt, const double* params, void* weights, void* stream);
int mpv_forward_tc(int N, int M, int fmt, const void* weights, const uint32_t* bits, int64_t B, double* out_lp,
                   double* out_re, double* out_im, int max_ctas, void* stream);

/* ---- ResCNN ansatz (beyond the reference: PAPER.md:876-890, BASELINE configs[3]) ----
 * log psi(x) = sum LN(h_n), h_0 = Conv(1 - 2x), h_{l+1} = h_l + Conv(GELU(Conv(GELU(LN(h_l)))))
 * on an L x L periodic lattice (3 <= L <= 30), 16 channels, 3x3 kernels, n_res <= 8 blocks.
 * `blob` (>= mpv_rescnn_blob_bytes(L, n_res), built by rescnn.py from the f64
 * parameters): per convolution and tap a 16 x 16 f16/bf16 B operand in the
 * tcgen05 K-major core-matrix layout, then f32 vectors (per LN: running
 * residual bias, gain, shift; per block: the first convolution's bias).
 * mpv_rescnn_forward: tcgen05 forward (f16/bf16 operands, f32 accumulation),
 * out_lp = 2 log psi.  mpv_rescnn_forward_f64: the f64 forward on the CUDA cores
 * (theta = the flat parameter vector of oracle/rescnn.py), out = log psi.
 * mpv_rescnn_mh_sweep: n_steps MH steps (ref: sampler.py:111-133, the
 * reference's streams and f64 accept test) with the tcgen05 evaluator, one
 * fused propose / evaluate / accept launch per step, samples recorded as
 * mpv_mh_sweep does; the cached log p is refreshed first.  Exchange steps
 * with ch->scratch of >= mpv_rescnn_mh_scratch_bytes(n_chains) bytes first
 * settle the chains whose swap exchanges equal bits (the identity, always
 * accepted) and evaluate only the others on the tensor cores. */
size_t mpv_rescnn_blob_bytes(int L, int n_res);
size_t mpv_rescnn_mh_scratch_bytes(int64_t n_chains);
int mpv_rescnn_forward(int L, int n_res, int fmt, const void* blob, const uint32_t* bits, int64_t B, double* out_lp,
                       int64_t* status, void* stream);
int mpv_rescnn_forward_f64(const double* theta, int L, int n_res, const uint32_t* bits, int64_t B, double* out,
                           void* stream);
int mpv_rescnn_mh_sweep(int L, int n_res, int fmt, const void* blob, const mpv_chains* ch, uint64_t key, int proposal,
                        int64_t init_draws, int64_t step_index, int64_t n_steps, int64_t thin, uint32_t* samples,
                        int64_t n_samples_total, int64_t n_chains_total, int64_t round_offset, int64_t row0,
                        void* stream);

/* ---- helpers ---- */
int mpv_unpack_bits(const uint32_t* words, int64_t B, int N, uint8_t* out, void* stream);
int mpv_pack_bits(const uint8_t* bits, int64_t B, int N, uint32_t* out, void* stream);
/* per-chain -> total accepted (int64 sum) */
int mpv_sum_i64(const int64_t* x, int64_t n, int64_t* out, void* stream);

/* Layout of the fused sweep for N sites, M hidden units: lanes per chain G
 * (power of two, >= ceil(N/32)) and hidden units per lane U; hidden_pad = G*U.
 * U is capped by the accumulator's register footprint (25 for X1 f16/bf16).
 * The f32 summation order of NATIVE log p follows (G, U): a fixed function of
 * (N, M, fmt, variant), hence of the snapshot. */
int mpv_plan_layout(int n_visible, int n_hidden, int fmt, int variant, int32_t* lanes_per_chain,
                    int32_t* units_per_lane);
/* Layout of the fused sweep including the cluster split: the smallest cluster
 * size (1, 2, 4) whose per-CTA rank block (+ visible biases and exchange
 * buffers) fits in shared memory, and the (G, U) of one rank block's
 * ceil(M / cluster) units; cluster = 1 with a table beyond shared memory when
 * none fits (read through L1/L2). */
int mpv_plan_cluster(int n_visible, int n_hidden, int fmt, int mode, int variant, int32_t* cluster,
                     int32_t* lanes_per_chain, int32_t* units_per_lane);
/* As mpv_plan_cluster with at least `min_lanes` lanes per chain (a power of
 * two <= 32).  Exchange sweeps plan with 32: a warp then holds one chain, and
 * a step whose exchange swaps equal bits (about half of them in a balanced
 * sector) is skipped by the whole warp.  The f32 summation order of NATIVE
 * log p follows the layout, so it is a function of (snapshot, min_lanes). */
int mpv_plan_cluster_ex(int n_visible, int n_hidden, int fmt, int mode, int variant, int min_lanes,
                        int32_t* cluster, int32_t* lanes_per_chain, int32_t* units_per_lane);

const char* mpv_last_error(void);
const char* mpv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MPVMC_B200_H */
