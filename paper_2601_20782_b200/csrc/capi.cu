// C ABI of libmpvmc_b200 (include/mpvmc_b200.h): argument checks, launch
// configuration and the small helper kernels.  No device allocation happens
// here: every buffer is caller-owned.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>
#include <unordered_map>

#include "energy.cuh"
#include "logderiv.cuh"
#include "ov_tc.h"
#include "perop.cuh"
#include "snapshot.cuh"
#include "sr.cuh"
#include "sweep.cuh"

namespace mpv {
#define MPV_DECL(f, v) void* sweep_kernel_ptr_##f##_##v(int G, int U, int prop, int smem, int cs);
MPV_DECL(f16, x1) MPV_DECL(f16, x2) MPV_DECL(f16, f64) MPV_DECL(f16, xi)
MPV_DECL(bf16, x1) MPV_DECL(bf16, x2) MPV_DECL(bf16, f64) MPV_DECL(bf16, xi)
MPV_DECL(f32, x1) MPV_DECL(f32, x2) MPV_DECL(f32, f64)
MPV_DECL(f64, f64)
#undef MPV_DECL

size_t forward_tc_weights_bytes(int N, int M);
size_t rescnn_blob_bytes(int L, int n_res);
cudaError_t rescnn_launch(int L, int n_res, int fmt, const void* blob, uint32_t* bits, int64_t B, int words,
                          double* lp, int64_t* accepted, int64_t* status, int mh, uint64_t key, int64_t chain_offset,
                          int64_t init_draws, int64_t step_index, int proposal, uint32_t* samples, int64_t thin,
                          int64_t sample_base, int64_t sample_extra, int64_t round_offset, int64_t row0,
                          int64_t local_step1, cudaStream_t st, int32_t* list = nullptr,
                          int32_t* count = nullptr);
cudaError_t rescnn_f64_launch(const double* theta, int L, int n_res, const uint32_t* bits, int64_t B, int words,
                              double* out, cudaStream_t st);
cudaError_t forward_tc_prepare(int N, int M, int fmt, const double* params, void* weights, cudaStream_t st);
cudaError_t forward_tc_launch(int N, int M, int fmt, const void* weights, const uint32_t* bits, int64_t B,
                              double* out_lp, double* out_re, double* out_im, int max_ctas, cudaStream_t st);

void* sweep_kernel_ptr(int fmt, int variant, int G, int U, int prop, int smem, int cs) {
  switch (fmt) {
    case MPV_FMT_F16:
      return variant == MPV_ACC_X1 ? sweep_kernel_ptr_f16_x1(G, U, prop, smem, cs)
           : variant == MPV_ACC_X2 ? sweep_kernel_ptr_f16_x2(G, U, prop, smem, cs)
           : variant == MPV_ACC_XI ? sweep_kernel_ptr_f16_xi(G, U, prop, smem, cs)
                                   : sweep_kernel_ptr_f16_f64(G, U, prop, smem, cs);
    case MPV_FMT_BF16:
      return variant == MPV_ACC_X1 ? sweep_kernel_ptr_bf16_x1(G, U, prop, smem, cs)
           : variant == MPV_ACC_X2 ? sweep_kernel_ptr_bf16_x2(G, U, prop, smem, cs)
           : variant == MPV_ACC_XI ? sweep_kernel_ptr_bf16_xi(G, U, prop, smem, cs)
                                   : sweep_kernel_ptr_bf16_f64(G, U, prop, smem, cs);
    case MPV_FMT_F32:  // (no integer accumulators for f32 snapshots)
      return variant == MPV_ACC_X1    ? sweep_kernel_ptr_f32_x1(G, U, prop, smem, cs)
           : variant == MPV_ACC_X2    ? sweep_kernel_ptr_f32_x2(G, U, prop, smem, cs)
           : variant == MPV_ACC_F64   ? sweep_kernel_ptr_f32_f64(G, U, prop, smem, cs)
                                      : nullptr;
    default:
      return sweep_kernel_ptr_f64_f64(G, U, prop, smem, cs);
  }
}
}  // namespace mpv

using namespace mpv;

namespace {

thread_local std::string g_error;

int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MPV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return MPV_OK;
}

int max_smem_optin() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return v;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) raised to the largest size
// requested so far for each kernel.
int ensure_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> done;
  if (bytes <= 48 * 1024) return MPV_OK;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(fn);
  if (it != done.end() && it->second >= bytes) return MPV_OK;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return fail(MPV_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  done[fn] = bytes;
  return MPV_OK;
}

constexpr int kUnits[] = {4, 8, 13, 16, 20, 25};
constexpr int MAX_WORDS_INIT = 32;  // n_sites <= 1024

size_t entry_bytes(int fmt, int variant) {
  if (variant == MPV_ACC_F64 || fmt == MPV_FMT_F64) return 16;
  if (variant == MPV_ACC_XI) return 8;
  const size_t pair = (fmt == MPV_FMT_F32) ? 8 : 4;
  return variant == MPV_ACC_X2 ? 2 * pair : pair;
}
size_t acc_bytes(int fmt, int variant) {  // sizeof(Acc<FMT, VAR>)
  if (variant == MPV_ACC_F64 || fmt == MPV_FMT_F64) return 16;
  if (variant == MPV_ACC_XI) return 8;
  return variant == MPV_ACC_X2 ? 16 : 8;
}
size_t vis_bytes(int fmt, int variant) {
  if (variant == MPV_ACC_F64 || fmt == MPV_FMT_F64) return 8;
  if (variant == MPV_ACC_XI) return 4;
  return variant == MPV_ACC_X2 ? 8 : 4;
}

// B200 shared memory per block (opt-in) used by the layout planner (the
// launch checks the device's own value)
constexpr size_t kSmemPlan = 232448;
constexpr int kFlipThreads = 512, kExchangeThreads = 256;
size_t rank_block_bytes(int N, int GU, size_t entry) { return ((size_t)N * GU * entry + 15) & ~(size_t)15; }
size_t vis16(int N, size_t vb) { return ((size_t)N * vb + 15) & ~(size_t)15; }
// exchange buffers of a cluster-split sweep: per warp 2 mbarriers + [2][CS][32] partial sums
size_t xchg_bytes(int cs, int warps, size_t sum_bytes) { return (size_t)warps * (16 + 2 * cs * 32 * sum_bytes); }
size_t sum_bytes(int kfmt) { return kfmt == MPV_FMT_F64 ? 8 : 4; }

// ---------------- helper kernels ----------------

__global__ void stream_uniforms_kernel(uint64_t key, int64_t n_chains, int64_t chain0, int64_t t0,
                                       int64_t n_draws, double* out) {
  const int64_t n = n_chains * n_draws;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = idx / n_chains, c = idx % n_chains;
    out[idx] = stream_draw(stream_state(key, (uint64_t)(chain0 + c)), (uint64_t)(t0 + t));
  }
}

// ref: sampler.py:67-88
__global__ void chains_init_kernel(mpv_chains ch, uint64_t key, int proposal, int weight) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ch.n_chains) return;
  const uint64_t s0 = stream_state(key, (uint64_t)(ch.chain_offset + c));
  uint32_t w[MAX_WORDS_INIT];
  const int N = ch.n_sites;
  for (int i = 0; i < ch.words; ++i) w[i] = 0u;
  if (proposal == MPV_PROPOSAL_FLIP) {
    for (int k = 0; k < N; ++k)
      if (stream_draw(s0, (uint64_t)k) < 0.5) w[k >> 5] |= 1u << (k & 31);
  } else {
    for (int k = 0; k < weight; ++k) w[k >> 5] |= 1u << (k & 31);
    uint64_t t = 0;
    for (int i = N - 1; i > 0; --i) {
      const int j = (int)floor_scaled(stream_draw(s0, t++), (double)(i + 1));
      const uint32_t bi = (w[i >> 5] >> (i & 31)) & 1u, bj = (w[j >> 5] >> (j & 31)) & 1u;
      if (bi != bj) {
        w[i >> 5] ^= 1u << (i & 31);
        w[j >> 5] ^= 1u << (j & 31);
      }
    }
  }
  for (int i = 0; i < ch.words; ++i) ch.bits[c * ch.words + i] = w[i];
  if (ch.log_probs) ch.log_probs[c] = 0.0;
  if (ch.accepted) ch.accepted[c] = 0;
}

__global__ void unpack_kernel(const uint32_t* words, int64_t B, int N, int nw, uint8_t* out) {
  const int64_t n = B * N;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / N;
    const int k = (int)(idx % N);
    out[idx] = (uint8_t)((words[r * nw + (k >> 5)] >> (k & 31)) & 1u);
  }
}

__global__ void pack_kernel(const uint8_t* bits, int64_t B, int N, int nw, uint32_t* out) {
  const int64_t n = B * nw;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / nw;
    const int w = (int)(idx % nw);
    uint32_t v = 0;
    for (int b = 0; b < 32 && w * 32 + b < N; ++b) v |= (uint32_t)(bits[r * N + w * 32 + b] & 1u) << b;
    out[idx] = v;
  }
}

// MH sweep over a dense log-probability table (ref: sampler.py:254-268
// table_log_prob / uniform_log_prob as the evaluator of ChainEnsemble.step,
// sampler.py:111-133): one thread per chain, configuration = its code (N <= 30),
// the reference's draw schedule and f64 accept test (NaN / -inf reject).
__global__ void table_sweep_kernel(const double* __restrict__ table, int N, mpv_chains ch, uint64_t key,
                                   int proposal, int64_t init_draws, int64_t step_index, int64_t n_steps,
                                   int64_t thin, uint32_t* samples, int64_t base, int64_t extra,
                                   int64_t round_offset, int64_t row0) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ch.n_chains) return;
  const int64_t gchain = ch.chain_offset + c;
  const uint64_t s0 = mpv::stream_state(key, (uint64_t)gchain);
  uint32_t word = ch.bits[c];
  double lp = table[word];
  const int64_t count_c = base + (gchain < extra ? 1 : 0);
  const int64_t offset_c = gchain * base + (gchain < extra ? gchain : extra) - row0;
  const double n_pairs = 0.5 * (double)N * (double)(N - 1);
  int64_t n_acc = 0;
  for (int64_t s = 0; s < n_steps; ++s) {
    const uint64_t t = (uint64_t)(init_draws + 2 * (step_index + s));
    const double us = mpv::stream_draw(s0, t), ua = mpv::stream_draw(s0, t + 1);
    uint32_t prop = word;
    if (proposal == MPV_PROPOSAL_FLIP) {
      prop ^= 1u << (int)mpv::floor_scaled(us, (double)N);
    } else {
      int i, j;
      mpv::pair_of(mpv::floor_scaled(us, n_pairs), N, i, j);
      if (((word >> i) ^ (word >> j)) & 1u) prop ^= (1u << i) | (1u << j);
    }
    const double lp_new = table[prop];
    if (log(ua) < lp_new - lp) {
      word = prop;
      lp = lp_new;
      ++n_acc;
    }
    if (samples && thin > 0 && (s + 1) % thin == 0) {
      const int64_t r = round_offset + (s + 1) / thin - 1;
      if (r < count_c) samples[offset_c + r] = word;
    }
  }
  ch.bits[c] = word;
  ch.log_probs[c] = lp;
  if (ch.accepted) ch.accepted[c] += n_acc;
}

__global__ void noise_add_kernel(const uint32_t* bits, int64_t B, int words, uint64_t key, double sigma,
                                 double* out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < B; r += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t code = (uint64_t)bits[r * words] | (words > 1 ? (uint64_t)bits[r * words + 1] << 32 : 0ull);
    out[r] += mpv::noise_zeta(key, code, sigma);
  }
}

__global__ void sum_i64_kernel(const int64_t* x, int64_t n, int64_t* out) {
  __shared__ long long part[32];
  long long acc = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += x[i];
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(kFull, acc, off);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = (threadIdx.x < (blockDim.x >> 5)) ? part[threadIdx.x] : 0;
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(kFull, acc, off);
    if (threadIdx.x == 0) *out = acc;
  }
}

// Table of a reference-layout parameter set for mpv_rounded_log_prob.
template <int FMT>
__global__ void perop_table_kernel(int N, int M, const double* a_re, const double* b_re,
                                   const double* b_im, const double* w_re, const double* w_im,
                                   void* table, void* bias, float* vis) {
  using P = PerOp<FMT>;
  using Entry = typename P::Entry;
  Entry* T = reinterpret_cast<Entry*>(table);
  Entry* Bv = reinterpret_cast<Entry*>(bias);
  const int64_t n = (int64_t)N * M;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n + M + N;
       idx += (int64_t)gridDim.x * blockDim.x) {
    if (idx < n) {
      const int k = (int)(idx / M), i = (int)(idx % M);
      const double re = w_re[(size_t)i * N + k], im = w_im[(size_t)i * N + k];
      if constexpr (FMT == MPV_FMT_F32) T[idx] = make_float2((float)re, (float)im);
      else T[idx] = (uint32_t)P::q(re) | ((uint32_t)P::q(im) << 16);
    } else if (idx < n + M) {
      const int i = (int)(idx - n);
      if constexpr (FMT == MPV_FMT_F32) Bv[i] = make_float2((float)b_re[i], (float)b_im[i]);
      else Bv[i] = (uint32_t)P::q(b_re[i]) | ((uint32_t)P::q(b_im[i]) << 16);
    } else {
      const int k = (int)(idx - n - M);
      vis[k] = (float)a_re[k];
    }
  }
}

}  // namespace

extern "C" {
#pragma GCC visibility push(default)

size_t mpv_sweep_scratch_bytes(const mpv_snapshot* snap, int64_t n_chains);

int mpv_pack_bits(const uint8_t* bits, int64_t B, int N, uint32_t* out, void* stream);

const char* mpv_last_error(void) { return g_error.c_str(); }
const char* mpv_version(void) { return "mpvmc_b200 0.1.0 (sm_100a)"; }

// Units-per-lane cap by accumulator footprint: registers per hidden unit are
// theta + the kept column entry (3 for X1 f16/bf16, 4-6 for X1 f32 / X2, 8 for F64).
static int units_cap(int fmt, int variant) {
  if (fmt == MPV_FMT_F64 || variant == MPV_ACC_F64) return 13;
  if (variant == MPV_ACC_XI) return 25;
  if (variant == MPV_ACC_X1) return fmt == MPV_FMT_F32 ? 16 : 25;
  return fmt == MPV_FMT_F32 ? 13 : 16;
}

static int plan_layout(int n_visible, int n_hidden, int fmt, int variant, int min_lanes, int32_t* lanes_per_chain,
                       int32_t* units_per_lane) {
  if (n_visible < 1 || n_visible > 1024 || n_hidden < 1 || !lanes_per_chain || !units_per_lane ||
      min_lanes < 1 || min_lanes > 32 || (min_lanes & (min_lanes - 1)))
    return fail(MPV_ERR_ARGS, "plan: bad args");
  const int words = (n_visible + 31) / 32;
  const int cap = units_cap(fmt, variant);
  int G = min_lanes;
  while (G < 32 && ((n_hidden + G - 1) / G > cap || G < words)) G *= 2;
  const int need = (n_hidden + G - 1) / G;
  for (int u : kUnits)
    if (u >= need && u <= cap) {
      *lanes_per_chain = G;
      *units_per_lane = u;
      return MPV_OK;
    }
  return fail(MPV_ERR_ARGS, "plan: too many hidden units for the fused sweep");
}

int mpv_plan_layout(int n_visible, int n_hidden, int fmt, int variant, int32_t* lanes_per_chain,
                    int32_t* units_per_lane) {
  return plan_layout(n_visible, n_hidden, fmt, variant, 1, lanes_per_chain, units_per_lane);
}

int mpv_stream_uniforms(uint64_t key, int64_t n_chains, int64_t chain0, int64_t t0, int64_t n_draws,
                        double* out, void* stream) {
  if (n_chains < 0 || n_draws < 0 || (!out && n_chains * n_draws > 0)) return fail(MPV_ERR_ARGS, "stream_uniforms: bad args");
  if (n_chains * n_draws == 0) return MPV_OK;
  const int64_t n = n_chains * n_draws;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  stream_uniforms_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(key, n_chains, chain0, t0, n_draws, out);
  return check_launch("stream_uniforms");
}

int mpv_snapshot_bytes(int n_visible, int hidden_pad, int fmt, int mode, int variant, int cluster, size_t* out) {
  if (n_visible < 1 || hidden_pad < 1 || fmt < MPV_FMT_F64 || fmt > MPV_FMT_BF16 || !out ||
      (cluster != 1 && cluster != 2 && cluster != 4) || hidden_pad % cluster)
    return fail(MPV_ERR_ARGS, "snapshot_bytes: bad args");
  const bool f64arith = (fmt == MPV_FMT_F64) || (mode == MPV_MODE_STORAGE_ONLY);
  const int kfmt = f64arith ? MPV_FMT_F64 : fmt, var = f64arith ? MPV_ACC_F64 : variant;
  const size_t t16 = cluster * rank_block_bytes(n_visible, hidden_pad / cluster, entry_bytes(kfmt, var));
  out[0] = t16 + vis16(n_visible, vis_bytes(kfmt, var));                     // [rank blocks | vis]
  out[1] = t16;                                                             // vis offset
  out[2] = ((size_t)hidden_pad * entry_bytes(kfmt, var) + 15) & ~(size_t)15;  // bias
  return MPV_OK;
}

int mpv_plan_cluster(int n_visible, int n_hidden, int fmt, int mode, int variant, int32_t* cluster,
                     int32_t* lanes_per_chain, int32_t* units_per_lane) {
  return mpv_plan_cluster_ex(n_visible, n_hidden, fmt, mode, variant, 1, cluster, lanes_per_chain, units_per_lane);
}

int mpv_plan_cluster_ex(int n_visible, int n_hidden, int fmt, int mode, int variant, int min_lanes, int32_t* cluster,
                        int32_t* lanes_per_chain, int32_t* units_per_lane) {
  if (!cluster || !lanes_per_chain || !units_per_lane) return fail(MPV_ERR_ARGS, "plan_cluster: null output");
  const bool f64arith = (fmt == MPV_FMT_F64) || (mode == MPV_MODE_STORAGE_ONLY);
  const int kfmt = f64arith ? MPV_FMT_F64 : fmt, var = f64arith ? MPV_ACC_F64 : variant;
  const size_t eb = entry_bytes(kfmt, var), vb = vis_bytes(kfmt, var);
  int32_t G = 0, U = 0;
  // The cluster split is opt-in (MPV_CLUSTER_SPLIT=1): measured on B200 it is
  // slower than reading the table through L1/L2 (the per-step partial-sum
  // exchange between the ranks is latency-bound).
  const char* env = getenv("MPV_CLUSTER_SPLIT");
  const int max_cs = (env && env[0] == '1') ? 4 : 1;
  for (int cs : {1, 2, 4}) {
    if (cs > max_cs) break;
    if (plan_layout(n_visible, (n_hidden + cs - 1) / cs, kfmt, var, min_lanes, &G, &U)) return MPV_ERR_ARGS;
    const size_t need = rank_block_bytes(n_visible, G * U, eb) + vis16(n_visible, vb) +
                        (cs > 1 ? xchg_bytes(cs, kFlipThreads / 32, sum_bytes(kfmt)) : 0) + 1024;
    const bool instantiated = cs == 1 || (G == 8 && (U == 8 || U == 13 || U == 25));  // tools/gen_sweep_instances.py
    if (need <= kSmemPlan && instantiated && (cs == 1 || n_hidden > 1)) {
      *cluster = cs;
      *lanes_per_chain = G;
      *units_per_lane = U;
      return MPV_OK;
    }
  }
  // nothing fits on chip: one CTA per chain group, table read through L1/L2
  if (plan_layout(n_visible, n_hidden, kfmt, var, min_lanes, &G, &U)) return MPV_ERR_ARGS;
  *cluster = 1;
  *lanes_per_chain = G;
  *units_per_lane = U;
  return MPV_OK;
}

int mpv_snapshot_round(int N, int M, int fmt, const double* params, double* rounded, double* plan, void* stream) {
  if (N < 1 || M < 1 || fmt < MPV_FMT_F64 || fmt > MPV_FMT_BF16 || !params || !rounded || !plan)
    return fail(MPV_ERR_ARGS, "snapshot_round: bad args");
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(plan, 0, 8 * sizeof(double), st) != cudaSuccess) return check_launch("snapshot_round");
  const int64_t n = 2 * ((int64_t)N + M + (int64_t)N * M);
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
  snapshot_round_kernel<<<grid, 256, 0, st>>>(N, M, fmt, params, rounded, plan);
  snapshot_bound_kernel<<<(M + 127) / 128, 128, 0, st>>>(N, M, rounded, plan);
  return check_launch("snapshot_round");
}

int mpv_snapshot_fill(const mpv_snapshot* snap, const double* rounded, double split, void* stream) {
  if (!snap || !rounded || !snap->table || !snap->bias || !snap->vis || snap->n_visible < 1 ||
      snap->hidden_pad < snap->n_hidden || snap->n_hidden < 1)
    return fail(MPV_ERR_ARGS, "snapshot_fill: bad args");
  // XI: the quantum is applied in f32 (bf16: folded into the log cosh, exact for q >= 2^-100)
  if (snap->variant == MPV_ACC_XI && !(snap->quantum >= 0x1p-100)) return fail(MPV_ERR_ARGS, "snapshot_fill: XI quantum");
  if (snap->variant == MPV_ACC_X2 && snap->mode == MPV_MODE_NATIVE && !(split > 0.0))
    return fail(MPV_ERR_ARGS, "snapshot_fill: X2 split");
  const int64_t n = (int64_t)(snap->n_visible + 1) * snap->hidden_pad + snap->n_visible;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
  const bool f64a = snap->fmt == MPV_FMT_F64 || snap->mode == MPV_MODE_STORAGE_ONLY;
  const size_t eb = entry_bytes(f64a ? MPV_FMT_F64 : snap->fmt, f64a ? MPV_ACC_F64 : snap->variant);
  snapshot_fill_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(*snap, rounded, split, eb);
  return check_launch("snapshot_fill");
}

int mpv_table_sweep(const double* table, const mpv_chains* ch, uint64_t key, int proposal, int64_t init_draws,
                    int64_t step_index, int64_t n_steps, int64_t thin, uint32_t* samples, int64_t n_samples_total,
                    int64_t n_chains_total, int64_t round_offset, int64_t row0, void* stream) {
  if (!table || !ch || ch->n_sites < 1 || ch->n_sites > 30 || ch->words != 1 || n_steps < 0 || thin < 0 ||
      (proposal != MPV_PROPOSAL_FLIP && proposal != MPV_PROPOSAL_EXCHANGE) ||
      (proposal == MPV_PROPOSAL_EXCHANGE && ch->n_sites < 2))
    return fail(MPV_ERR_ARGS, "table_sweep: bad args (table evaluators need 1 <= n_sites <= 30)");
  if (ch->n_chains == 0) return MPV_OK;
  int64_t base = 0, extra = 0;
  if (samples) {
    if (n_chains_total < 1 || thin < 1) return fail(MPV_ERR_ARGS, "table_sweep: sample layout");
    base = n_samples_total / n_chains_total;
    extra = n_samples_total % n_chains_total;
  }
  table_sweep_kernel<<<(unsigned)((ch->n_chains + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      table, ch->n_sites, *ch, key, proposal, init_draws, step_index, n_steps, thin, samples, base, extra,
      round_offset, row0);
  return check_launch("table_sweep");
}

int mpv_chains_init(const mpv_chains* ch, uint64_t key, int proposal, int sector_weight, void* stream) {
  if (!ch || ch->n_chains < 0 || ch->n_sites < 1 || ch->words != (ch->n_sites + 31) / 32 || !ch->bits)
    return fail(MPV_ERR_ARGS, "chains_init: bad chain descriptor");
  if (ch->words > MAX_WORDS_INIT) return fail(MPV_ERR_ARGS, "chains_init: n_sites too large");
  if (proposal == MPV_PROPOSAL_EXCHANGE && (sector_weight < 0 || sector_weight > ch->n_sites))
    return fail(MPV_ERR_ARGS, "sector weight out of range");
  if (ch->status) {
    const int64_t init[2] = {0, (int64_t)0x7FFFFFFFFFFFFFFFll};
    cudaMemcpyAsync(ch->status, init, sizeof init, cudaMemcpyHostToDevice, (cudaStream_t)stream);
  }
  if (ch->n_chains == 0) return MPV_OK;
  chains_init_kernel<<<(unsigned)((ch->n_chains + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      *ch, key, proposal, sector_weight);
  return check_launch("chains_init");
}

int mpv_mh_sweep(const mpv_snapshot* snap, const mpv_chains* ch, uint64_t key, int proposal,
                 int64_t init_draws, int64_t step_index, int64_t n_steps, int64_t thin,
                 uint32_t* samples, int64_t n_samples_total, int64_t n_chains_total,
                 int64_t round_offset, int64_t row0, void* stream) {
  if (!snap || !ch || !snap->table || !snap->bias || !ch->bits || !ch->log_probs)
    return fail(MPV_ERR_ARGS, "mh_sweep: null descriptor");
  if (snap->n_visible != ch->n_sites || ch->words != (ch->n_sites + 31) / 32)
    return fail(MPV_ERR_ARGS, "mh_sweep: snapshot/chain size mismatch");
  if (n_steps < 0 || thin < 0 || (samples && thin < 1)) return fail(MPV_ERR_ARGS, "mh_sweep: bad schedule");
  if (proposal != MPV_PROPOSAL_FLIP && proposal != MPV_PROPOSAL_EXCHANGE)
    return fail(MPV_ERR_ARGS, "mh_sweep: unknown proposal");
  if (proposal == MPV_PROPOSAL_EXCHANGE && ch->n_sites < 2)
    return fail(MPV_ERR_ARGS, "mh_sweep: exchange needs >= 2 sites");
  if (ch->n_sites >= 65536) return fail(MPV_ERR_ARGS, "mh_sweep: n_sites too large");
  if (ch->n_chains == 0) return MPV_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t base = 0, extra = 0;
  if (samples) {
    if (n_chains_total < 1) return fail(MPV_ERR_ARGS, "mh_sweep: n_chains_total");
    base = n_samples_total / n_chains_total;
    extra = n_samples_total % n_chains_total;
  }
  const int fmt = snap->fmt, mode = snap->mode;

  if (mode == MPV_MODE_PER_OPERATION && fmt != MPV_FMT_F64) {
    if (snap->noise_sigma != 0.0) return fail(MPV_ERR_ARGS, "mh_sweep: log-density noise needs f64 arithmetic");
    PerOpSweepArgs a{};
    a.f.N = snap->n_visible; a.f.M = snap->n_hidden; a.f.Mpad = snap->hidden_pad; a.f.words = ch->words;
    a.f.GU = snap->hidden_pad;  // per-op snapshots are never split
    a.f.RB = (int64_t)(rank_block_bytes(snap->n_visible, snap->hidden_pad, entry_bytes(fmt, MPV_ACC_X1)) /
                       entry_bytes(fmt, MPV_ACC_X1));
    a.f.table = snap->table; a.f.bias = snap->bias; a.f.vis = snap->vis; a.f.vis_im = snap->vis_im;
    a.n_chains = ch->n_chains; a.chain_offset = ch->chain_offset; a.bits = ch->bits;
    a.log_probs = ch->log_probs; a.accepted = ch->accepted; a.status = ch->status; a.key = key;
    a.init_draws = init_draws; a.step_index = step_index; a.n_steps = n_steps; a.thin = thin;
    a.samples = samples; a.sample_base = base; a.sample_extra = extra; a.round_offset = round_offset;
    a.row0 = row0;
    const int threads = 128, nw = threads / 32;
    const size_t smem = nw * 64 * sizeof(uint32_t) + (size_t)nw * 2 * snap->n_hidden * sizeof(double);
    const void* fn = nullptr;
    const bool ex = proposal == MPV_PROPOSAL_EXCHANGE;
    if (fmt == MPV_FMT_F16) fn = ex ? (const void*)&perop_sweep_kernel<MPV_FMT_F16, 1> : (const void*)&perop_sweep_kernel<MPV_FMT_F16, 0>;
    else if (fmt == MPV_FMT_BF16) fn = ex ? (const void*)&perop_sweep_kernel<MPV_FMT_BF16, 1> : (const void*)&perop_sweep_kernel<MPV_FMT_BF16, 0>;
    else fn = ex ? (const void*)&perop_sweep_kernel<MPV_FMT_F32, 1> : (const void*)&perop_sweep_kernel<MPV_FMT_F32, 0>;
    if (int rc = ensure_smem(fn, smem)) return rc;
    void* args[] = {&a};
    const cudaError_t e = cudaLaunchKernel(fn, dim3((unsigned)((ch->n_chains + nw - 1) / nw)), dim3(threads), args, smem, st);
    if (e != cudaSuccess) return fail(MPV_ERR_CUDA, std::string("perop sweep: ") + cudaGetErrorString(e));
    return MPV_OK;
  }

  // fused sweep; f64 and storage-only run the f64 arithmetic
  const bool f64arith = (fmt == MPV_FMT_F64) || (mode == MPV_MODE_STORAGE_ONLY);
  if (snap->noise_sigma != 0.0 && (!f64arith || snap->n_visible > 64))
    return fail(MPV_ERR_ARGS, "mh_sweep: log-density noise needs f64 arithmetic and n_visible <= 64");
  const int kfmt = f64arith ? MPV_FMT_F64 : fmt;
  const int variant = f64arith ? MPV_ACC_F64 : snap->variant;
  const int G = snap->lanes_per_chain, U = snap->units_per_lane, CS = snap->cluster;
  if (G < 1 || G > 32 || (G & (G - 1)) || (CS != 1 && CS != 2 && CS != 4) || CS * G * U != snap->hidden_pad ||
      snap->hidden_pad < snap->n_hidden)
    return fail(MPV_ERR_ARGS, "mh_sweep: snapshot layout inconsistent");
  if (G < ch->words) return fail(MPV_ERR_ARGS, "mh_sweep: lanes_per_chain < words");
  // [rank blocks | vis], each padded to 16 bytes (the host snapshot layout)
  const size_t eb = entry_bytes(kfmt, variant), vb = vis_bytes(kfmt, variant);
  const size_t rb = rank_block_bytes(snap->n_visible, G * U, eb);
  if ((const char*)snap->vis != (const char*)snap->table + CS * rb)
    return fail(MPV_ERR_ARGS, "mh_sweep: vis must follow the rank blocks at the next 16-byte boundary");
  // flip kernels: 512-thread blocks (one staged table per 16 warps, <= 128 regs);
  // exchange kernels need more registers: 256-thread blocks
  const int threads = (proposal == MPV_PROPOSAL_FLIP) ? kFlipThreads : kExchangeThreads;
  const size_t xoff = rb + vis16(snap->n_visible, vb);
  size_t smem = 0;
  int sm = 0;
  if (CS > 1) {
    smem = xoff + xchg_bytes(CS, threads / 32, sum_bytes(kfmt));
    if (smem + 1024 > (size_t)max_smem_optin()) return fail(MPV_ERR_ARGS, "mh_sweep: rank block exceeds shared memory");
    sm = 1;
  } else if (xoff + 1024 <= (size_t)max_smem_optin()) {  // static smem: mbarrier
    smem = xoff;
    sm = 1;
  }
  void* fn = sweep_kernel_ptr(kfmt, variant, G, U, proposal, sm, CS);
  if (!fn) return fail(MPV_ERR_ARGS, "mh_sweep: no kernel for this (format, variant, layout)");
  const int64_t cpw = 32 / G;
  const int64_t n_groups = (ch->n_chains + cpw - 1) / cpw;
  // segment length: a multiple of G (draw batches never straddle segments),
  // >= 32 steps, <= 16 segments per launch
  int64_t seg_len = std::max<int64_t>(32, (n_steps + 15) / 16);
  seg_len = (seg_len + G - 1) / G * G;
  const int64_t n_segments = n_steps == 0 ? 1 : (n_steps + seg_len - 1) / seg_len;
  const size_t need = mpv_sweep_scratch_bytes(snap, ch->n_chains);
  if (!ch->scratch || ch->scratch_bytes < need) return fail(MPV_ERR_ARGS, "mh_sweep: scratch too small (mpv_sweep_scratch_bytes)");
  char* sp = (char*)ch->scratch;
  const size_t done_bytes = ((CS * n_groups * 4 + 255) / 256) * 256;
  int* queue = (int*)sp;
  int* done = (int*)(sp + 256);
  float* save = (float*)(sp + 256 + done_bytes);
  void* vsave = (char*)save + ((size_t)CS * n_groups * U * acc_bytes(kfmt, variant) * 32 + 255) / 256 * 256;
  if (cudaMemsetAsync(sp, 0, 256 + CS * n_groups * 4, st) != cudaSuccess) return check_launch("mh_sweep memset");
  SweepArgs a{};
  a.N = snap->n_visible; a.M = snap->n_hidden; a.Mpad = snap->hidden_pad; a.G = G; a.words = ch->words;
  a.table = snap->table; a.bias = snap->bias; a.vis = snap->vis; a.table_bytes = xoff;
  a.table_in_smem = sm;
  a.rank_block_bytes = rb; a.vis_bytes = (size_t)snap->n_visible * vb; a.xchg_off = xoff;
  a.n_chains = ch->n_chains; a.chain_offset = ch->chain_offset; a.bits = ch->bits;
  a.log_probs = ch->log_probs; a.accepted = ch->accepted; a.status = ch->status; a.key = key;
  a.init_draws = init_draws; a.step_index = step_index; a.n_steps = n_steps; a.thin = thin;
  a.samples = samples; a.sample_base = base; a.sample_extra = extra; a.round_offset = round_offset;
  a.row0 = row0;
  a.seg_len = seg_len; a.n_groups = n_groups; a.n_items = n_groups * n_segments;
  a.queue = queue; a.done = done; a.save = save; a.vis_save = vsave;
  a.xi_scale = (float)snap->quantum;
  a.noise_key = snap->noise_key;
  a.noise_sigma = snap->noise_sigma;
  if (variant == MPV_ACC_XI && !(snap->quantum >= 0x1p-100))
    return fail(MPV_ERR_ARGS, "mh_sweep: XI needs quantum >= 2^-100");
  if (int rc = ensure_smem(fn, smem)) return rc;
  int dev = 0, n_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  void* args[] = {&a};
  if (CS == 1) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess || per_sm < 1)
      return fail(MPV_ERR_CUDA, "mh_sweep: kernel does not fit on an SM");
    const int64_t warps_needed = a.n_items;
    const int64_t blocks = std::min<int64_t>((int64_t)n_sm * per_sm, (warps_needed + threads / 32 - 1) / (threads / 32));
    const cudaError_t e = cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(threads), args, smem, st);
    if (e != cudaSuccess) return fail(MPV_ERR_CUDA, std::string("mh_sweep: ") + cudaGetErrorString(e));
    return MPV_OK;
  }
  // cluster split: as many co-resident clusters as the device holds (persistent)
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)(n_sm / CS * CS));
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, fn, &cfg) != cudaSuccess || clusters < 1)
    return fail(MPV_ERR_CUDA, "mh_sweep: cluster does not fit on the device");
  const int64_t warps_needed = a.n_items;
  const int64_t want = (warps_needed + threads / 32 - 1) / (threads / 32);
  cfg.gridDim = dim3((unsigned)(std::min<int64_t>(clusters, want) * CS));
  const cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess) return fail(MPV_ERR_CUDA, std::string("mh_sweep (cluster): ") + cudaGetErrorString(e));
  return MPV_OK;
}

size_t mpv_sweep_scratch_bytes(const mpv_snapshot* snap, int64_t n_chains) {
  if (!snap) return 0;
  const bool f64arith = (snap->fmt == MPV_FMT_F64) || (snap->mode == MPV_MODE_STORAGE_ONLY);
  const int kfmt = f64arith ? MPV_FMT_F64 : snap->fmt;
  const int variant = f64arith ? MPV_ACC_F64 : snap->variant;
  const int G = std::max(1, (int)snap->lanes_per_chain), U = std::max(1, (int)snap->units_per_lane);
  const int CS = std::max(1, (int)snap->cluster);
  const int64_t n_groups = (n_chains + 32 / G - 1) / (32 / G);
  return 256 + ((CS * n_groups * 4 + 255) / 256) * 256 +
         ((size_t)CS * n_groups * U * acc_bytes(kfmt, variant) * 32 + 255) / 256 * 256 +
         (size_t)(n_chains + 1) * 16 + 256;
}

int mpv_snapshot_forward(const mpv_snapshot* snap, const uint32_t* bits, int64_t B, double* out_lp,
                         double* out_re, double* out_im, int64_t* status, void* scratch,
                         size_t scratch_bytes, void* stream) {
  if (!snap || !bits || !out_lp || B < 0) return fail(MPV_ERR_ARGS, "snapshot_forward: bad args");
  if (B == 0) return MPV_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int words = (snap->n_visible + 31) / 32;
  const int fmt = snap->fmt, mode = snap->mode;
  if (mode == MPV_MODE_NATIVE && fmt != MPV_FMT_F64) {
    if (out_re || out_im) return fail(MPV_ERR_ARGS, "snapshot_forward: NATIVE mode has no log psi output");
    // the fused sweep with zero steps: refresh theta from the bits and write log p
    mpv_chains ch{};
    ch.n_chains = B; ch.chain_offset = 0; ch.n_sites = snap->n_visible; ch.words = words;
    ch.bits = const_cast<uint32_t*>(bits);  // read-only with n_steps == 0 (bits written back unchanged)
    ch.log_probs = out_lp; ch.accepted = nullptr; ch.status = status;
    ch.scratch = scratch; ch.scratch_bytes = scratch_bytes;
    return mpv_mh_sweep(snap, &ch, 0, MPV_PROPOSAL_FLIP, 0, 0, 0, 0, nullptr, 0, 1, 0, 0, stream);
  }
  FwdArgs a{};
  a.N = snap->n_visible; a.M = snap->n_hidden; a.Mpad = snap->hidden_pad; a.words = words;
  {
    const int cs = std::max(1, (int)snap->cluster);
    const bool f64a = fmt == MPV_FMT_F64 || mode == MPV_MODE_STORAGE_ONLY;
    const size_t eb = entry_bytes(f64a ? MPV_FMT_F64 : fmt, f64a ? MPV_ACC_F64 : snap->variant);
    a.GU = snap->hidden_pad / cs;
    a.RB = (int64_t)(rank_block_bytes(snap->n_visible, a.GU, eb) / eb);
  }
  a.table = snap->table; a.bias = snap->bias; a.vis = snap->vis; a.vis_im = snap->vis_im;
  a.bits = bits; a.B = B; a.out_lp = out_lp; a.out_re = out_re; a.out_im = out_im; a.status = status;
  const bool want_im = out_re || out_im;
  if (want_im && !snap->vis_im) return fail(MPV_ERR_ARGS, "snapshot_forward: log psi needs vis_im");
  const int threads = 256, nw = threads / 32;
  const size_t smem = nw * 32 * sizeof(uint32_t) + (size_t)nw * 2 * snap->n_hidden * sizeof(double);
  const void* fn;
  if (fmt == MPV_FMT_F64 || mode == MPV_MODE_STORAGE_ONLY) fn = (const void*)&forward_kernel<MPV_FMT_F64>;
  else if (fmt == MPV_FMT_F16) fn = (const void*)&forward_kernel<MPV_FMT_F16>;
  else if (fmt == MPV_FMT_BF16) fn = (const void*)&forward_kernel<MPV_FMT_BF16>;
  else fn = (const void*)&forward_kernel<MPV_FMT_F32>;
  if (int rc = ensure_smem(fn, smem)) return rc;
  int wi = want_im ? 1 : 0;
  void* args[] = {&a, &wi};
  const unsigned grid = (unsigned)std::min<int64_t>((B + nw - 1) / nw, 148 * 32);
  const cudaError_t e = cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, smem, st);
  if (e != cudaSuccess) return fail(MPV_ERR_CUDA, std::string("snapshot_forward: ") + cudaGetErrorString(e));
  if (snap->noise_sigma != 0.0) {
    if (snap->n_visible > 64 || !(fmt == MPV_FMT_F64 || mode == MPV_MODE_STORAGE_ONLY))
      return fail(MPV_ERR_ARGS, "snapshot_forward: log-density noise needs f64 arithmetic and n_visible <= 64");
    noise_add_kernel<<<(unsigned)std::min<int64_t>((B + 255) / 256, 148 * 8), 256, 0, st>>>(
        bits, B, words, snap->noise_key, snap->noise_sigma, out_lp);
    return check_launch("snapshot_forward noise");
  }
  return MPV_OK;
}

static size_t rup(size_t x) { return (x + 255) / 256 * 256; }

size_t mpv_rounded_scratch_bytes(int64_t B, int N, int M, int fmt) {
  const size_t pair = fmt == MPV_FMT_F32 ? 8 : 4;
  return rup((size_t)N * M * pair) + rup((size_t)M * pair) + rup((size_t)N * 4) +
         rup((size_t)B * ((N + 31) / 32) * 4);
}

int mpv_rounded_log_prob(const uint8_t* bits, int64_t B, int N, int M, const double* a_re,
                         const double* b_re, const double* b_im, const double* w_re,
                         const double* w_im, int fmt, double* out_lp, void* scratch, void* stream) {
  if (fmt != MPV_FMT_F32 && fmt != MPV_FMT_F16 && fmt != MPV_FMT_BF16)
    return fail(MPV_ERR_ARGS, "rounded_log_prob: fmt must be f32, f16 or bf16");
  if (!bits || !a_re || !b_re || !b_im || !w_re || !w_im || !out_lp || !scratch || N < 1 || M < 1 || B < 0)
    return fail(MPV_ERR_ARGS, "rounded_log_prob: bad args");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t pair = fmt == MPV_FMT_F32 ? 8 : 4;
  char* p = (char*)scratch;
  void* table = p;
  p += rup((size_t)N * M * pair);
  void* bias = p;
  p += rup((size_t)M * pair);
  float* vis = (float*)p;
  p += rup((size_t)N * 4);
  uint32_t* packed = (uint32_t*)p;
  const int64_t n = (int64_t)N * M + M + N;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
  if (fmt == MPV_FMT_F16) perop_table_kernel<MPV_FMT_F16><<<grid, 256, 0, st>>>(N, M, a_re, b_re, b_im, w_re, w_im, table, bias, vis);
  else if (fmt == MPV_FMT_BF16) perop_table_kernel<MPV_FMT_BF16><<<grid, 256, 0, st>>>(N, M, a_re, b_re, b_im, w_re, w_im, table, bias, vis);
  else perop_table_kernel<MPV_FMT_F32><<<grid, 256, 0, st>>>(N, M, a_re, b_re, b_im, w_re, w_im, table, bias, vis);
  if (int rc = check_launch("rounded_log_prob table")) return rc;
  if (B == 0) return MPV_OK;
  if (int rc = mpv_pack_bits(bits, B, N, packed, stream)) return rc;
  mpv_snapshot snap{};
  snap.n_visible = N; snap.n_hidden = M; snap.hidden_pad = M;
  snap.fmt = fmt; snap.mode = MPV_MODE_PER_OPERATION; snap.variant = MPV_ACC_X1;
  snap.lanes_per_chain = 1; snap.units_per_lane = M; snap.cluster = 1;
  snap.table = table; snap.bias = bias; snap.vis = vis; snap.vis_im = nullptr;
  return mpv_snapshot_forward(&snap, packed, B, out_lp, nullptr, nullptr, nullptr, nullptr, 0, stream);
}

size_t mpv_energy_tables_bytes(int N, int M, int ham, int n_bonds) {
  const int T = ham == MPV_HAM_TFIM ? N : n_bonds;
  return (size_t)M * T * sizeof(double2) + 2 * (size_t)T * sizeof(double2) + 2 * (size_t)T * sizeof(int32_t) + 128 +
         (size_t)energy_w_rows(N) * energy_w_pitch(M) * sizeof(double);
}

struct EnergyTables {
  double2 *tau, *ea;
  int32_t *ec, *slow;
  double* wp;
};
static EnergyTables energy_layout(int N, int M, int ham, int n_bonds, void* tables) {
  const int T = ham == MPV_HAM_TFIM ? N : n_bonds;
  char* p = (char*)tables;
  EnergyTables e;
  e.tau = (double2*)p;
  p += (size_t)M * T * sizeof(double2);
  e.ea = (double2*)p;
  p += 2 * (size_t)T * sizeof(double2);
  e.ec = (int32_t*)p;
  p += (size_t)T * sizeof(int32_t);
  e.slow = (int32_t*)p;
  p += (size_t)T * sizeof(int32_t);
  e.wp = (double*)(((uintptr_t)p + 127) / 128 * 128);
  return e;
}

int mpv_energy_prepare(int N, int M, const double* a, const double* b, const double* w_t, int ham,
                       const int32_t* bonds, int n_bonds, void* tables, void* stream) {
  if (N < 1 || M < 1 || !a || !b || !w_t || !tables || (ham != MPV_HAM_TFIM && ham != MPV_HAM_HEISENBERG))
    return fail(MPV_ERR_ARGS, "energy_prepare: bad args");
  if (ham == MPV_HAM_HEISENBERG && (n_bonds < 1 || !bonds)) return fail(MPV_ERR_ARGS, "energy_prepare: bonds");
  EnergyArgs e{};
  e.N = N; e.M = M; e.ham = ham; e.n_bonds = n_bonds; e.n_terms = ham == MPV_HAM_TFIM ? N : n_bonds;
  e.a = (const double2*)a; e.b = (const double2*)b; e.w_t = (const double2*)w_t; e.bonds = bonds;
  const EnergyTables tb = energy_layout(N, M, ham, n_bonds, tables);
  const int64_t n = (int64_t)M * e.n_terms;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
  energy_tables_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(e, tb.tau, tb.ea, tb.ec, tb.slow, tb.wp);
  return check_launch("energy_prepare");
}

int mpv_local_energies(int N, int M, const double* a, const double* b, const double* w_t, int ham,
                       const int32_t* bonds, int n_bonds, double J, double h, const void* tables,
                       const uint32_t* bits, int64_t B, double* out_eps, int64_t* status, void* stream) {
  return mpv_local_energies_ex(N, M, a, b, w_t, ham, bonds, n_bonds, J, h, nullptr, nullptr, tables, bits, B,
                               out_eps, status, stream);
}

int mpv_local_energies_ex(int N, int M, const double* a, const double* b, const double* w_t, int ham,
                          const int32_t* bonds, int n_bonds, double J, double h, const double* term_coef,
                          const double* bond_j, const void* tables, const uint32_t* bits, int64_t B,
                          double* out_eps, int64_t* status, void* stream) {
  if (N < 1 || M < 1 || !a || !b || !w_t || !tables || !bits || !out_eps || B < 0)
    return fail(MPV_ERR_ARGS, "local_energies: bad args");
  if (ham != MPV_HAM_TFIM && ham != MPV_HAM_HEISENBERG) return fail(MPV_ERR_ARGS, "local_energies: ham");
  if (n_bonds > 0 && !bonds) return fail(MPV_ERR_ARGS, "local_energies: bonds");
  if (B == 0) return MPV_OK;
  EnergyArgs e{};
  e.N = N; e.M = M; e.words = (N + 31) / 32; e.ham = ham; e.n_bonds = n_bonds;
  e.n_terms = ham == MPV_HAM_TFIM ? N : n_bonds;
  e.a = (const double2*)a; e.b = (const double2*)b; e.w_t = (const double2*)w_t; e.bonds = bonds;
  e.J = J; e.h = h; e.term_coef = term_coef; e.bond_j = bond_j;
  const EnergyTables tb = energy_layout(N, M, ham, n_bonds, const_cast<void*>(tables));
  e.tau = tb.tau; e.ea = tb.ea; e.ec = tb.ec; e.slow = tb.slow; e.wp = tb.wp;
  e.bits = bits; e.B = B; e.out = (double2*)out_eps; e.status = status;
  const int T = e.n_terms;
  if (T > 512 || M > 512) return fail(MPV_ERR_ARGS, "local_energies: more than 512 terms or hidden units");
  // (ST samples per thread, SB samples per block): terms x groups flattened
  // over the block; 16 samples per block (two DMMA m-tiles) where it fits.
  // Phase 1 runs in one pass: every warp owns <= KT of the ceil(M/4) n-tiles.
  struct Cfg { int st, sb, kt, tmax; const void* fn; };
  // TFIM: every (sample, term) pair is active; Heisenberg / J1-J2: the active
  // pairs are compacted per block (COMPACT kernels)
  const bool cmp = ham != MPV_HAM_TFIM;
#define MPV_EK(ST, KT, TM, MB) (cmp ? (const void*)&energy_kernel<ST, KT, TM, MB, true> \
                                    : (const void*)&energy_kernel<ST, KT, TM, MB, false>)
  const Cfg cfgs[] = {
      {4, 16, 4, 448, MPV_EK(4, 4, 448, 2)},  // 2 blocks/SM, 72 regs (T <= 112)
      {8, 16, 8, 256, MPV_EK(8, 8, 256, 2)},  // 2 blocks/SM, 128 regs (T <= 128)
      {4, 16, 4, 800, MPV_EK(4, 4, 800, 1)},  // 1 block/SM of up to 25 warps, 80 regs (T <= 200)
      {4, 8, 4, 800, MPV_EK(4, 4, 800, 1)},   // 8 samples per block (T <= 400: J1-J2)
      {8, 16, 4, 512, MPV_EK(8, 4, 512, 1)},
      {8, 16, 8, 512, MPV_EK(8, 8, 512, 1)},
      {8, 8, 4, 512, MPV_EK(8, 4, 512, 1)},
      {8, 8, 8, 512, MPV_EK(8, 8, 512, 1)},
  };
#undef MPV_EK
  const size_t optin = (size_t)max_smem_optin();
  const int NT = (M + 3) / 4;
  // profiling only: MPV_ENERGY_CFG=ci[,nbt,rows] forces a configuration
  static const char* force = getenv("MPV_ENERGY_CFG");
  int f_ci = -1, f_nbt = 0, f_rows = 0;
  if (force) sscanf(force, "%d,%d,%d", &f_ci, &f_nbt, &f_rows);
  for (int ci = 0; ci < (int)(sizeof(cfgs) / sizeof(cfgs[0])); ++ci) {
    const Cfg& cf = cfgs[ci];
    if (f_ci >= 0 && ci != f_ci) continue;
    const int threads = std::max(std::max(32, ((cf.sb / cf.st) * T + 31) / 32 * 32), 32 * ((NT + cf.kt - 1) / cf.kt));
    if (threads > cf.tmax) continue;
    for (int nbt = f_nbt ? f_nbt : 3; nbt >= 2; --nbt)
      for (int rows = f_rows ? f_rows : 12; rows >= 2; rows -= 2) {
        EnergyPlan pl;
        const size_t smem = energy_plan(N, M, T, cf.sb, rows, nbt, &pl);
        // profiling only: MPV_ENERGY_SKIP bit mask drops kernel phases (profiles/r01/README.md)
        static const int skip = getenv("MPV_ENERGY_SKIP") ? atoi(getenv("MPV_ENERGY_SKIP")) : 0;
        pl.skip = skip;
        if (smem > optin) continue;
        if (int rc = ensure_smem(cf.fn, smem)) return rc;
        const unsigned grid = (unsigned)((B + cf.sb - 1) / cf.sb);
        void* args[] = {&e, &pl};
        if (cudaLaunchKernel(cf.fn, grid, threads, args, smem, (cudaStream_t)stream) != cudaSuccess)
          return check_launch("local_energies");
        return check_launch("local_energies");
      }
  }
  return fail(MPV_ERR_ARGS, "local_energies: n_hidden / terms too large for shared memory");
}

static size_t ld_ov_bytes(int N, int M) {
  // the DMMA kernel's padded vW^T, or the tcgen05 kernel's limb matrix (ov_tc.cu)
  return std::max(((size_t)ld_rows(N) * ld_pitch(M) * sizeof(double) + 255) / 256 * 256, ov_tc_blob_bytes(N, M));
}

size_t mpv_logderiv_scratch_bytes(int64_t U, int N, int M) {
  const int64_t chunk = ld_chunk(std::max<int64_t>(U, 1), N, M), chunks = (U + chunk - 1) / chunk;
  return ld_ov_bytes(N, M) + (size_t)std::max<int64_t>(chunks, 1) * ld_rows_a(M) * ld_cols(N) * sizeof(double);
}

// O v (MODE 0, weights fused) or T = tanh(b + W x) (MODE 1, v = parameters)
static int launch_ov(int mode, const double* t, const uint32_t* bits, int64_t U, int N, int M, const double* v,
                     const double* w, double* q, double* t_out, void* scratch, cudaStream_t st,
                     const double* skip = nullptr) {
  double* vwt = (double*)scratch;
  // O v on tcgen05 (exact f16 limbs, ov_tc.cu) unless MPV_OV_TC=0 (the DMMA kernel below)
  if (mode == 0) {
    const char* tc = getenv("MPV_OV_TC");
    if (!(tc && atoi(tc) == 0)) {
      const int rc = ov_tc_launch(t, bits, U, N, M, v, w, q, scratch, st, skip);
      if (rc == 0) return check_launch("logderiv_ov_tc");
      if (rc < 0) return check_launch("logderiv_ov_tc");
    }
  }
  const int64_t n = (int64_t)ld_rows(N) * ld_pitch(M);
  ld_transpose_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 4), 256, 0, st>>>(
      (const double2*)v, N, M, vwt, skip);
  const int NT = (M + 3) / 4;
  // O v (MODE 0): 16 warps per block, two blocks per SM; tanh (MODE 1): 8 warps
  static const char* ovw = getenv("MPV_LD_OV_WARPS");  // experiments: 8 or 16
  const int nw = (mode == 0 && !(ovw && atoi(ovw) == 8)) ? 16 : 8;
  const int kt = (NT + nw - 1) / nw;
  const unsigned grid = (unsigned)((U + kLdSB - 1) / kLdSB);
  const int words = (N + 31) / 32;
  const double2* T = (const double2*)t;
  const double2* V = (const double2*)v;
  double2* Q = (double2*)q;
  double2* TO = (double2*)t_out;
  const size_t tbytes = (size_t)kLdSB * M * 16;  // MODE 0: the block's T rows in shared memory
#define MPV_OV(K)                                                                                             \
  if (mode == 0 && nw == 16) {                                                                                \
    if (int rc = ensure_smem((const void*)&ld_ov_kernel<K, 0, 16>, tbytes)) return rc;                       \
    ld_ov_kernel<K, 0, 16><<<grid, 512, tbytes, st>>>(T, bits, U, N, M, words, V, vwt, Q, w, TO, skip);     \
  } else if (mode == 0) {                                                                                     \
    if (int rc = ensure_smem((const void*)&ld_ov_kernel<K, 0>, tbytes)) return rc;                           \
    ld_ov_kernel<K, 0><<<grid, 256, tbytes, st>>>(T, bits, U, N, M, words, V, vwt, Q, w, TO, skip);         \
  } else {                                                                                                    \
    ld_ov_kernel<K, 1><<<grid, 256, 0, st>>>(T, bits, U, N, M, words, V, vwt, Q, w, TO);                    \
  }
  if (kt <= 2) { MPV_OV(2) }
  else if (kt <= 4) { MPV_OV(4) }
  else if (kt <= 8) { MPV_OV(8) }
  else { MPV_OV(16) }
#undef MPV_OV
  return check_launch(mode == 0 ? "logderiv_ov" : "logderiv_tanh");
}

int mpv_logderiv_ov(const double* t, const uint32_t* bits, int64_t U, int N, int M, const double* v, const double* w,
                    double* q, void* scratch, void* stream) {
  if (!t || !bits || !v || !q || !scratch || U < 0 || N < 1 || N > 256 || M < 1 || M > 512)
    return fail(MPV_ERR_ARGS, "logderiv_ov: bad args (N <= 256, M <= 512)");
  if (U == 0) return MPV_OK;
  return launch_ov(0, t, bits, U, N, M, v, w, q, nullptr, scratch, (cudaStream_t)stream);
}

int mpv_logderiv_tanh(const double* params, const uint32_t* bits, int64_t U, int N, int M, double* t, void* scratch,
                      void* stream) {
  if (!params || !bits || !t || !scratch || U < 0 || N < 1 || N > 256 || M < 1 || M > 512)
    return fail(MPV_ERR_ARGS, "logderiv_tanh: bad args (N <= 256, M <= 512)");
  if (U == 0) return MPV_OK;
  return launch_ov(1, nullptr, bits, U, N, M, params, nullptr, nullptr, t, scratch, (cudaStream_t)stream);
}

static int launch_ohu(const double* t, const uint32_t* bits, int64_t U, int N, int M, const double* u,
                      const double* w, double* out, double* sum_out, void* scratch, cudaStream_t st,
                      const double* skip);

int mpv_logderiv_ohu(const double* t, const uint32_t* bits, int64_t U, int N, int M, const double* u, const double* w,
                     double* out, double* sum_out, void* scratch, void* stream) {
  if (!t || !bits || !u || !out || !scratch || U < 0 || N < 1 || N > 256 || M < 1)
    return fail(MPV_ERR_ARGS, "logderiv_ohu: bad args (N <= 256)");
  return launch_ohu(t, bits, U, N, M, u, w, out, sum_out, scratch, (cudaStream_t)stream, nullptr);
}

static int launch_ohu(const double* t, const uint32_t* bits, int64_t U, int N, int M, const double* u,
                      const double* w, double* out, double* sum_out, void* scratch, cudaStream_t st,
                      const double* skip) {
  const int P = N + M + M * N;
  if (U == 0) {
    if (cudaMemsetAsync(out, 0, (size_t)P * 2 * sizeof(double), st) != cudaSuccess) return check_launch("logderiv_ohu");
    if (sum_out && cudaMemsetAsync(sum_out, 0, 2 * sizeof(double), st) != cudaSuccess)
      return check_launch("logderiv_ohu");
    return MPV_OK;
  }
  double* partial = (double*)((char*)scratch + ld_ov_bytes(N, M));
  const int64_t chunk = ld_chunk(U, N, M);
  const int chunks = (int)((U + chunk - 1) / chunk);
  const int ntc = ld_ntc(N);
  const dim3 grid((unsigned)(ld_rows_a(M) / 64), (unsigned)chunks, (unsigned)(ld_cols(N) / (8 * ntc)));
  const int words = (N + 31) / 32;
  const double2* T = (const double2*)t;
  const double2* Uv = (const double2*)u;
  if (ntc == 16) ld_ohu_kernel<16><<<grid, 256, 0, st>>>(T, bits, U, N, M, words, Uv, partial, chunk, w, skip);
  else if (ntc == 13) ld_ohu_kernel<13><<<grid, 256, 0, st>>>(T, bits, U, N, M, words, Uv, partial, chunk, w, skip);
  else if (ntc == 8) ld_ohu_kernel<8><<<grid, 256, 0, st>>>(T, bits, U, N, M, words, Uv, partial, chunk, w, skip);
  else ld_ohu_kernel<4><<<grid, 256, 0, st>>>(T, bits, U, N, M, words, Uv, partial, chunk, w, skip);
  ld_ohu_reduce_kernel<<<(unsigned)std::min(148 * 8, (P + 256) / 256), 256, 0, st>>>(partial, chunks, N, M,
                                                                                      (double2*)out,
                                                                                      (double2*)sum_out, skip);
  return check_launch("logderiv_ohu");
}

int mpv_logderiv_dense(const double* t, const uint32_t* bits, int64_t U, int N, int M, const double* obar, double* o,
                       void* stream) {
  if (!t || !bits || !o || U < 0 || N < 1 || M < 1) return fail(MPV_ERR_ARGS, "logderiv_dense: bad args");
  if (U == 0) return MPV_OK;
  const int64_t n = U * ((int64_t)N + M + (int64_t)M * N);
  ld_dense_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(
      (const double2*)t, bits, U, N, M, (N + 31) / 32, (const double2*)obar, (double2*)o);
  return check_launch("logderiv_dense");
}

int mpv_sr_smatrix(const double* c, const double* w, int64_t U, int P, double* s, void* stream) {
  if (!c || !s || U < 0 || P < 1) return fail(MPV_ERR_ARGS, "sr_smatrix: bad args");
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned tiles = (unsigned)((P + kSmT - 1) / kSmT);
  sr_smatrix_kernel<<<dim3(tiles, tiles), 256, 0, st>>>((const double2*)c, w, U, P, (double2*)s);
  sr_real_diag_kernel<<<(unsigned)std::min(148 * 4, (P + 255) / 256), 256, 0, st>>>(P, (double2*)s);
  return check_launch("sr_smatrix");
}

// ---- device-resident conjugate gradients (sr.cuh) ----
static int cg_blocks(int P) { return std::max(1, std::min(kCgMaxBlocks, (P + kCgThreads - 1) / kCgThreads)); }
static int cg_check(const mpv_cg* cg) {
  if (!cg || !cg->t || !cg->bits || !cg->obar || !cg->g || !cg->r || !cg->p || !cg->ap || !cg->y || !cg->ysum ||
      !cg->q || !cg->partials || !cg->scalars || !cg->scratch || cg->n_visible < 1 || cg->n_visible > 256 ||
      cg->n_hidden < 1 || cg->n_hidden > 512 || cg->n_samples < 0)
    return fail(MPV_ERR_ARGS, "cg: bad descriptor");
  if (cg->scratch_bytes < mpv_logderiv_scratch_bytes(cg->n_samples, cg->n_visible, cg->n_hidden))
    return fail(MPV_ERR_ARGS, "cg: scratch too small (mpv_logderiv_scratch_bytes)");
  return MPV_OK;
}
static int cg_P(const mpv_cg* cg) { return cg->n_visible + cg->n_hidden + cg->n_hidden * cg->n_visible; }

size_t mpv_cg_partials_len(void) { return 3 * (size_t)kCgMaxBlocks; }

int mpv_cg_init(const mpv_cg* cg, const double* f, double tol, int64_t maxiter, void* stream) {
  if (int rc = cg_check(cg)) return rc;
  if (!f || tol < 0) return fail(MPV_ERR_ARGS, "cg_init: bad args");
  cudaStream_t st = (cudaStream_t)stream;
  const int P = cg_P(cg), nb = cg_blocks(P);
  cg_init_kernel<<<nb, kCgThreads, 0, st>>>(P, (const double2*)f, (double2*)cg->g, (double2*)cg->r, (double2*)cg->p,
                                            cg->partials);
  cg_init_scalars_kernel<<<1, 32, 0, st>>>(cg->partials, nb, tol, (double)maxiter, cg->scalars);
  return check_launch("cg_init");
}

static int cg_apply(const mpv_cg* cg, const double* v, double* y, double* ysum, void* stream, const double* skip) {
  const int N = cg->n_visible, M = cg->n_hidden;
  if (cg->n_samples == 0) {
    return mpv_logderiv_ohu(cg->t, cg->bits, 0, N, M, cg->q, nullptr, y, ysum, cg->scratch, stream);
  }
  if (int rc = launch_ov(0, cg->t, cg->bits, cg->n_samples, N, M, v, cg->w, cg->q, nullptr, cg->scratch,
                         (cudaStream_t)stream, skip))
    return rc;
  return launch_ohu(cg->t, cg->bits, cg->n_samples, N, M, cg->q, nullptr, y, ysum, cg->scratch, (cudaStream_t)stream,
                    skip);
}

int mpv_cg_apply(const mpv_cg* cg, const double* v, double* y, double* ysum, void* stream) {
  if (int rc = cg_check(cg)) return rc;
  if (!v || !y || !ysum) return fail(MPV_ERR_ARGS, "cg_apply: bad args");
  return cg_apply(cg, v, y, ysum, stream, nullptr);
}

int mpv_cg_apply_finish(const mpv_cg* cg, const double* v, const double* y, const double* ysum, double* out,
                        void* stream) {
  if (int rc = cg_check(cg)) return rc;
  if (!v || !y || !ysum || !out) return fail(MPV_ERR_ARGS, "cg_apply_finish: bad args");
  const int P = cg_P(cg);
  cg_ap_kernel<<<cg_blocks(P), kCgThreads, 0, (cudaStream_t)stream>>>(
      P, (const double2*)y, (const double2*)ysum, (const double2*)cg->obar, cg->lambda, (const double2*)v,
      (double2*)out, nullptr);
  return check_launch("cg_apply_finish");
}

int mpv_cg_step(const mpv_cg* cg, void* stream) {
  if (int rc = cg_check(cg)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int P = cg_P(cg), nb = cg_blocks(P);
  double* pap = cg->partials;
  double* rr = cg->partials + kCgMaxBlocks;
  cg_ap_kernel<<<nb, kCgThreads, 0, st>>>(P, (const double2*)cg->y, (const double2*)cg->ysum,
                                          (const double2*)cg->obar, cg->lambda, (const double2*)cg->p,
                                          (double2*)cg->ap, pap);
  cg_update_kernel<<<nb, kCgThreads, 0, st>>>(P, (const double2*)cg->p, (const double2*)cg->ap, (double2*)cg->g,
                                              (double2*)cg->r, pap, nb, rr, cg->scalars);
  cg_direction_kernel<<<nb, kCgThreads, 0, st>>>(P, (const double2*)cg->r, (double2*)cg->p, rr, nb, cg->scalars);
  cg_commit_kernel<<<1, 32, 0, st>>>(rr, nb, cg->scalars);
  return check_launch("cg_step");
}

int mpv_cg_run(const mpv_cg* cg, int n_iter, void* stream) {
  if (n_iter < 0) return fail(MPV_ERR_ARGS, "cg_run: n_iter < 0");
  if (int rc = cg_check(cg)) return rc;
  // once the device flag reports convergence the products of the batch's
  // remaining iterations return at once (the updates are no-ops anyway)
  const double* done = cg->scalars + kCgDone;
  for (int it = 0; it < n_iter; ++it) {
    if (int rc = cg_apply(cg, cg->p, cg->y, cg->ysum, stream, done)) return rc;
    if (int rc = mpv_cg_step(cg, stream)) return rc;
  }
  return MPV_OK;
}

int mpv_minsr_gram(const double* t_rows, const uint32_t* bits_rows, int64_t U_rows, int64_t row0,
                   const double* t_all, const uint32_t* bits_all, int64_t U_all, int N, int M, const double* d_all,
                   const double* w_all, double obar2, double lambda, int out_f32, void* out, void* stream) {
  if (!t_rows || !bits_rows || !t_all || !bits_all || !d_all || !w_all || !out || U_rows < 0 || U_all < 1 ||
      row0 < 0 || row0 + U_rows > U_all || N < 1 || M < 1)
    return fail(MPV_ERR_ARGS, "minsr_gram: bad args");
  if (U_rows == 0) return MPV_OK;
  const dim3 grid((unsigned)((U_all + kSmT - 1) / kSmT), (unsigned)((U_rows + kSmT - 1) / kSmT));
  const int words = (N + 31) / 32;
  cudaStream_t st = (cudaStream_t)stream;
  if (out_f32)
    minsr_gram_kernel<float2><<<grid, 256, 0, st>>>((const double2*)t_rows, bits_rows, U_rows, row0,
                                                    (const double2*)t_all, bits_all, U_all, M, words,
                                                    (const double2*)d_all, w_all, obar2, lambda, (float2*)out);
  else
    minsr_gram_kernel<double2><<<grid, 256, 0, st>>>((const double2*)t_rows, bits_rows, U_rows, row0,
                                                     (const double2*)t_all, bits_all, U_all, M, words,
                                                     (const double2*)d_all, w_all, obar2, lambda, (double2*)out);
  return check_launch("minsr_gram");
}

int mpv_chain_stats(const double* eps_u, const int64_t* inverse, int64_t n_chains, int64_t chain_offset,
                    int64_t base, int64_t extra, int64_t row0, double* means, double* partials, double* out,
                    void* stream) {
  if (!eps_u || !means || !partials || !out || n_chains < 1 || base < 0 || extra < 0 || (base == 0 && extra == 0))
    return fail(MPV_ERR_ARGS, "chain_stats: bad args");
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = (int)std::min<int64_t>(kCgMaxBlocks, (n_chains + kCgThreads - 1) / kCgThreads);
  chain_means_kernel<<<nb, kCgThreads, 0, st>>>((const double2*)eps_u, inverse, n_chains, chain_offset, base, extra,
                                                row0, means, partials);
  moments_pass2_kernel<<<nb, kCgThreads, 0, st>>>(means, n_chains, partials, nb, partials + kCgMaxBlocks);
  moments_finish_kernel<<<1, 32, 0, st>>>(partials, nb, partials + kCgMaxBlocks, n_chains, out);
  return check_launch("chain_stats");
}

int mpv_moments(const double* x, int64_t n, double* partials, double* out, void* stream) {
  if (!x || !partials || !out || n < 1) return fail(MPV_ERR_ARGS, "moments: bad args");
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = (int)std::min<int64_t>(kCgMaxBlocks, (n + kCgThreads - 1) / kCgThreads);
  moments_pass1_kernel<<<nb, kCgThreads, 0, st>>>(x, n, partials);
  moments_pass2_kernel<<<nb, kCgThreads, 0, st>>>(x, n, partials, nb, partials + kCgMaxBlocks);
  moments_finish_kernel<<<1, 32, 0, st>>>(partials, nb, partials + kCgMaxBlocks, n, out);
  return check_launch("moments");
}

// ---- batched forward on tcgen05 (forward_tc.cu) ----
size_t mpv_forward_tc_weights_bytes(int N, int M) { return forward_tc_weights_bytes(N, M); }

int mpv_forward_tc_prepare(int N, int M, int fmt, const double* params, void* weights, void* stream) {
  if (!params || !weights) return fail(MPV_ERR_ARGS, "forward_tc_prepare: null pointer");
  if (fmt != MPV_FMT_F16 && fmt != MPV_FMT_BF16)
    return fail(MPV_ERR_ARGS, "forward_tc_prepare: the tensor-core forward takes f16 or bf16 parameters");
  if (!forward_tc_weights_bytes(N, M)) return fail(MPV_ERR_ARGS, "forward_tc_prepare: unsupported N/M");
  const cudaError_t e = forward_tc_prepare(N, M, fmt, params, weights, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(MPV_ERR_CUDA, std::string("forward_tc_prepare: ") + cudaGetErrorString(e));
  return MPV_OK;
}

int mpv_forward_tc(int N, int M, int fmt, const void* weights, const uint32_t* bits, int64_t B, double* out_lp,
                   double* out_re, double* out_im, int max_ctas, void* stream) {
  if (B == 0 && weights) return MPV_OK;
  if (!weights || !bits || B < 0 || !(out_lp || out_re || out_im)) return fail(MPV_ERR_ARGS, "forward_tc: bad args");
  if (fmt != MPV_FMT_F16 && fmt != MPV_FMT_BF16)
    return fail(MPV_ERR_ARGS, "forward_tc: the tensor-core forward takes f16 or bf16 parameters");
  if (!forward_tc_weights_bytes(N, M)) return fail(MPV_ERR_ARGS, "forward_tc: unsupported N/M");
  const cudaError_t e =
      forward_tc_launch(N, M, fmt, weights, bits, B, out_lp, out_re, out_im, max_ctas, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(MPV_ERR_CUDA, std::string("forward_tc: ") + cudaGetErrorString(e));
  return MPV_OK;
}

// ---- ResCNN (rescnn.cu) ----
size_t mpv_rescnn_blob_bytes(int L, int n_res) { return rescnn_blob_bytes(L, n_res); }

int mpv_rescnn_forward(int L, int n_res, int fmt, const void* blob, const uint32_t* bits, int64_t B, double* out_lp,
                       int64_t* status, void* stream) {
  if (!blob || !bits || !out_lp || B < 0 || (fmt != MPV_FMT_F16 && fmt != MPV_FMT_BF16) || !rescnn_blob_bytes(L, n_res))
    return fail(MPV_ERR_ARGS, "rescnn_forward: bad args (f16/bf16, 3 <= L <= 30, n_res <= 8)");
  if (B == 0) return MPV_OK;
  const cudaError_t e = rescnn_launch(L, n_res, fmt, blob, const_cast<uint32_t*>(bits), B, (L * L + 31) / 32, out_lp,
                                      nullptr, status, 0, 0, 0, 0, 0, 0, nullptr, 0, 0, 0, 0, 0, 0, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(MPV_ERR_CUDA, std::string("rescnn_forward: ") + cudaGetErrorString(e));
  return MPV_OK;
}

int mpv_rescnn_forward_f64(const double* theta, int L, int n_res, const uint32_t* bits, int64_t B, double* out,
                           void* stream) {
  if (!theta || !bits || !out || B < 0 || L < 3 || L > 30 || n_res < 0 || n_res > 8)
    return fail(MPV_ERR_ARGS, "rescnn_forward_f64: bad args");
  if (B == 0) return MPV_OK;
  const cudaError_t e = rescnn_f64_launch(theta, L, n_res, bits, B, (L * L + 31) / 32, out, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(MPV_ERR_CUDA, std::string("rescnn_forward_f64: ") + cudaGetErrorString(e));
  return MPV_OK;
}

size_t mpv_rescnn_mh_scratch_bytes(int64_t n_chains) { return 16 + 4 * (size_t)std::max<int64_t>(n_chains, 0); }

int mpv_rescnn_mh_sweep(int L, int n_res, int fmt, const void* blob, const mpv_chains* ch, uint64_t key, int proposal,
                        int64_t init_draws, int64_t step_index, int64_t n_steps, int64_t thin, uint32_t* samples,
                        int64_t n_samples_total, int64_t n_chains_total, int64_t round_offset, int64_t row0,
                        void* stream) {
  if (!blob || !ch || !ch->bits || !ch->log_probs || ch->n_sites != L * L || ch->words != (L * L + 31) / 32 ||
      n_steps < 0 || thin < 0 || (samples && thin < 1) || (fmt != MPV_FMT_F16 && fmt != MPV_FMT_BF16) ||
      !rescnn_blob_bytes(L, n_res) || (proposal != MPV_PROPOSAL_FLIP && proposal != MPV_PROPOSAL_EXCHANGE))
    return fail(MPV_ERR_ARGS, "rescnn_mh_sweep: bad args");
  if (ch->n_chains == 0) return MPV_OK;
  int64_t base = 0, extra = 0;
  if (samples) {
    if (n_chains_total < 1) return fail(MPV_ERR_ARGS, "rescnn_mh_sweep: n_chains_total");
    base = n_samples_total / n_chains_total;
    extra = n_samples_total % n_chains_total;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // exchange steps evaluate only the chains whose swap changes the configuration
  // (list + two step counters in the chains' scratch, mpv_rescnn_mh_scratch_bytes)
  int32_t *list = nullptr, *count = nullptr;
  if (proposal == MPV_PROPOSAL_EXCHANGE && ch->scratch &&
      ch->scratch_bytes >= mpv_rescnn_mh_scratch_bytes(ch->n_chains)) {
    count = (int32_t*)ch->scratch;
    list = count + 4;
    if (cudaMemsetAsync(count, 0, 4 * sizeof(int32_t), st) != cudaSuccess) return check_launch("rescnn_mh_sweep");
  }
  // the cached log p of the current configurations (set_evaluator semantics)
  cudaError_t e = rescnn_launch(L, n_res, fmt, blob, ch->bits, ch->n_chains, ch->words, ch->log_probs, nullptr,
                                ch->status, 0, 0, 0, 0, 0, 0, nullptr, 0, 0, 0, 0, 0, 0, st);
  for (int64_t s = 0; e == cudaSuccess && s < n_steps; ++s)
    e = rescnn_launch(L, n_res, fmt, blob, ch->bits, ch->n_chains, ch->words, ch->log_probs, ch->accepted,
                      ch->status, 1, key, ch->chain_offset, init_draws, step_index + s, proposal, samples, thin, base,
                      extra, round_offset, row0, s + 1, st, list, count);
  if (e != cudaSuccess) return fail(MPV_ERR_CUDA, std::string("rescnn_mh_sweep: ") + cudaGetErrorString(e));
  return MPV_OK;
}

int mpv_unpack_bits(const uint32_t* words, int64_t B, int N, uint8_t* out, void* stream) {
  if (!words || !out || B < 0 || N < 1) return fail(MPV_ERR_ARGS, "unpack_bits: bad args");
  if (B == 0) return MPV_OK;
  const int64_t n = B * N;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  unpack_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(words, B, N, (N + 31) / 32, out);
  return check_launch("unpack_bits");
}

int mpv_pack_bits(const uint8_t* bits, int64_t B, int N, uint32_t* out, void* stream) {
  if (!bits || !out || B < 0 || N < 1) return fail(MPV_ERR_ARGS, "pack_bits: bad args");
  if (B == 0) return MPV_OK;
  const int nw = (N + 31) / 32;
  const int64_t n = B * nw;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  pack_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(bits, B, N, nw, out);
  return check_launch("pack_bits");
}

int mpv_sum_i64(const int64_t* x, int64_t n, int64_t* out, void* stream) {
  if (!x || !out || n < 0) return fail(MPV_ERR_ARGS, "sum_i64: bad args");
  sum_i64_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(x, n, out);
  return check_launch("sum_i64");
}

#pragma GCC visibility pop
}  // extern "C"
