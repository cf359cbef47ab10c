// Batched RBM forward on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// North-star subsystem (2): "the batched proposal and forward pass is a
// tcgen05 tensor-core GEMM in f16/bf16, since that path really is a dense
// contraction".  For B configurations x in {0,1}^N (packed words, the layout
// of mpv_chains.bits) it evaluates the reference's forward
// (ref: rbm.py:130-150 _fast_forward / _logcosh_pair; oracle/c/oracle_port.c
// f64_row) with the parameters rounded to f16/bf16:
//
//   theta_i = b_i + sum_k w_ik x_k                       (GEMM, f32 accumulate)
//   log psi = sum_k a_k x_k + sum_i [u - log 2 + log|(1+t)cos v + i(1-t)sin v|]
//             + i (... + sum_i atan2((1-t) sin v, (1+t) cos v)),
//   u = |Re theta|, v = sign(Re theta) Im theta, t = exp(-2u).
//
// GEMM per CTA tile: D[128 configurations x (HC hidden + 16)] for the re and
// the im block = A[128 x Kp] * B[Kp x (HC+16)], Kp = N + 1 rounded up to 16:
// column N of A is the constant 1 and row N of B the hidden bias, so theta =
// W x + b leaves the tensor core complete (row HC of the first chunk's blocks
// holds a, giving a . x).  A is decoded from the packed bits straight into
// shared memory (x in {0,1} is exact in f16/bf16, so the products are exact
// and only the f32 accumulation order differs from the f64 reference); B (the
// rounded weights) is staged once per CTA by the bulk copy engine.  Both
// operands use the K-major no-swizzle canonical layout: 8x16-byte core
// matrices, K-adjacent core matrices 128 B apart (LBO), 8-row groups Kp*16 B
// apart (SBO).  forward_tc_pipe_kernel: 4 producer warps build A and one of
// their threads issues tcgen05.mma (M=128, K=16 per instruction) into one of
// two TMEM buffers and commits to an mbarrier; 16 epilogue warps drain the
// other buffer with tcgen05.ld and run the f32 log-cosh epilogue, which is the
// kernel's bound (3 MUFU ops per hidden unit for log p, + sin and a minimax atan2 for
// the phase, against 4*Kp tensor flops per hidden unit).  forward_tc_kernel is
// the unpipelined fallback for weights beyond shared memory (B re-staged per
// chunk from L2, visible term from a bit loop).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <stdint.h>

#include "../../include/mpvmc_b200.h"

namespace mpv {
namespace tc {

constexpr int kRows = 128;     // MMA M (configurations per tile)
constexpr int kThreads = 512;  // 16 epilogue warps: 4 TMEM lane quarters x 4 column slices
constexpr int kSlices = kThreads / 128;
constexpr int kProducers = 4;  // producer warps of the pipelined kernel (A build, MMA issue)
constexpr int kRowsPerLane = kRows / (32 * kProducers);
constexpr int kMaxHC = 256;    // MMA N limit / TMEM block
constexpr size_t kSmemBudget = 200 * 1024;
constexpr size_t kSmemFloor = 116 * 1024;  // one CTA per SM (512 TMEM columns each)

struct Layout {
  int N, M, Kp, HC, HCB, nchunks, words;  // HCB: B rows (MMA N) per re/im block
  int pipe;            // 1: B resident, A and TMEM double-buffered (forward_tc_pipe_kernel)
  int cols_proc;       // hidden columns the pipelined epilogue evaluates (8-column groups)
  size_t a_bytes;      // A tile bytes
  size_t chunk_bytes;  // B chunk bytes (re + im rows)
  size_t smem;         // dynamic smem
  // weights blob: [chunks of B (weights, bias in column N)][a re/im f32 (N each)]
  size_t off_vis, blob_bytes;
};

__host__ __device__ inline size_t rup(size_t x, size_t a) { return (x + a - 1) / a * a; }

inline bool make_layout(int N, int M, Layout* L) {
  if (N < 1 || N > 1024 || M < 1) return false;
  L->N = N; L->M = M; L->words = (N + 31) / 32;
  L->Kp = (int)rup(N + 1, 16);  // column N of A is the constant 1 (bias row of B)
  L->a_bytes = (size_t)kRows * L->Kp * 2;
  if (L->a_bytes + 2ull * 16 * L->Kp * 2 + 4096 > kSmemBudget) return false;
  const size_t hc_cap = (kSmemBudget - L->a_bytes - 4096) / (4ull * L->Kp);
  const int hcmax = (int)std::min<size_t>(kMaxHC, hc_cap / 16 * 16);
  if (hcmax < 16) return false;
  {  // pipelined variant: HC <= 112 hidden + 16 rows (row HC = visible biases) per
     // re/im block, two TMEM buffers of re|im (2 x 128 columns), all chunks resident
    const int nch = (M + 111) / 112;
    const int hc = (int)rup((M + nch - 1) / nch, 16);
    const size_t bytes = 2 * L->a_bytes + (size_t)nch * 4 * (hc + 16) * L->Kp +
                         3ull * kSlices * kRows * 3 * 4 + 2ull * kRows * 2 * 4 + 1024;
    if (bytes <= kSmemBudget) {
      L->pipe = 1;
      L->nchunks = nch;
      L->HC = hc;
      L->HCB = hc + 16;
      L->chunk_bytes = 4ull * L->HCB * L->Kp;
      L->smem = std::max(bytes, kSmemFloor);
      L->cols_proc = 0;
      for (int c = 0; c < nch; ++c) L->cols_proc += (int)rup(std::min(hc, M - c * hc), 4);
      L->off_vis = L->chunk_bytes * nch;
      L->blob_bytes = rup(L->off_vis + 2ull * N * 4, 256);
      return true;
    }
  }
  L->pipe = 0;
  L->cols_proc = 0;
  L->nchunks = (M + hcmax - 1) / hcmax;
  L->HC = (int)rup((M + L->nchunks - 1) / L->nchunks, 16);
  L->HCB = L->HC;
  L->chunk_bytes = 4ull * L->HC * L->Kp;
  const size_t used = L->a_bytes + L->chunk_bytes + 2ull * N * 4 + 3ull * kRows * kSlices * 4 + 1024;
  L->smem = std::max(used, kSmemFloor);
  L->off_vis = L->chunk_bytes * L->nchunks;
  L->blob_bytes = rup(L->off_vis + 2ull * N * 4, 256);
  return true;
}

// byte offset of element (row r, k) in a K-major no-swizzle tile with Kp columns
__host__ __device__ inline size_t kmajor_off(int r, int k, int Kp) {
  return (size_t)(r & 7) * 16 + (size_t)(r >> 3) * Kp * 16 + (size_t)(k >> 3) * 128 + (size_t)(k & 7) * 2;
}

template <int FMT>
__device__ inline uint16_t to_bits16(double v) {
  if (FMT == MPV_FMT_F16) return __half_as_ushort(__double2half(v));
  return __bfloat16_as_ushort(__double2bfloat16(v));
}
template <int FMT>
__device__ inline float from_bits16(uint16_t h) {
  if (FMT == MPV_FMT_F16) return __half2float(__ushort_as_half(h));
  return __bfloat162float(__ushort_as_bfloat16(h));
}

// params = [a (N) | b (M) | w_t (N x M)] complex (re, im) f64, as mpv_snapshot_round.
template <int FMT>
__global__ void prepare_kernel(Layout L, const double* __restrict__ params, uint8_t* __restrict__ blob) {
  const int N = L.N, M = L.M, HC = L.HC, HCB = L.HCB, Kp = L.Kp;
  const double* a = params;
  const double* b = params + 2 * (size_t)N;
  const double* wt = params + 2 * (size_t)(N + M);
  const int64_t nb = (int64_t)L.nchunks * 2 * HCB * Kp;  // B elements
  float* vis = reinterpret_cast<float*>(blob + L.off_vis);
  const int64_t total = nb + 2LL * N;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    if (idx < nb) {
      const int64_t per_chunk = 2LL * HCB * Kp;
      const int c = (int)(idx / per_chunk);
      const int rem = (int)(idx % per_chunk);
      const int r = rem / Kp, k = rem % Kp;  // r in [0, 2HCB): re rows then im rows
      const int part = r / HCB, rr = r % HCB, i = c * HC + rr;
      uint16_t h = 0;
      if (rr < HC) {
        if (i < M && k < N) h = to_bits16<FMT>(wt[2 * ((size_t)k * M + i) + part]);
        if (i < M && k == N) h = to_bits16<FMT>(b[2 * (size_t)i + part]);
      } else if (rr == HC && c == 0 && k < N) {  // pipelined layout: a . x from the tensor core
        h = to_bits16<FMT>(a[2 * (size_t)k + part]);
      }
      *reinterpret_cast<uint16_t*>(blob + (size_t)c * L.chunk_bytes + (size_t)part * 2 * HCB * Kp +
                                   kmajor_off(rr, k, Kp)) = h;
    } else {
      const int j = (int)(idx - nb);  // [re: N][im: N]
      const int part = j / N, k = j % N;
      vis[j] = from_bits16<FMT>(to_bits16<FMT>(a[2 * (size_t)k + part]));
    }
  }
}

// 1 - e^{-2u} for 0 <= u < 1/16 without cancellation: the series of
// -expm1(-2u) through u^5 (truncation < 5e-8 relative at u = 1/16).
__device__ __forceinline__ float omt_series(float u) {
  return u * fmaf(u, fmaf(u, fmaf(u, fmaf(u, 0.266666667f, -0.666666667f), 1.333333333f), -2.0f), 2.0f);
}
__device__ inline uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ inline uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100)
  return d;         // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__device__ inline void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ inline void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{.reg .pred p;\nWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          bar),
      "r"(phase)
      : "memory");
}

// Stage one B chunk (bytes multiple of 16) global -> smem with the bulk copy engine.
__device__ inline void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  const uint32_t step = 65536;  // keep each bulk copy well inside the size field
  for (uint32_t off = 0; off < bytes; off += step) {
    const uint32_t n = bytes - off < step ? bytes - off : step;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst + off),
                 "l"((const uint8_t*)src + off), "r"(n), "r"(bar)
                 : "memory");
  }
}

// MUFU approximations without the denormal fix-ups of the non-ftz intrinsics
// (arguments are kept >= FLT_MIN where it matters: the lg2 input is clamped).
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_ftz(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float cos_ftz(float x) {
  float y;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sin_ftz(float x) {
  float y;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// atan2(y, x) for finite arguments: a = min/max through MUFU rcp, atan(a) as
// a * p(a^2), p the degree-7 f32 minimax fit (max |error| 1.3e-7 on [0,1],
// evaluated in f32 Horner, the f32 rounding floor; fit by tools/fit_atan.py),
// then the octant/quadrant fix-ups.  The result takes y's sign, so signed
// zeros give +-0 / +-pi as libm's atan2f does.
__device__ __forceinline__ float atan2_fast(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  const float a = mx > 0.0f ? mn * rcp_ftz(mx) : 0.0f;
  const float s = a * a;
  float p = -0.004054425284266472f;
  p = fmaf(p, s, 0.02186243049800396f);
  p = fmaf(p, s, -0.05591154471039772f);
  p = fmaf(p, s, 0.09642138332128525f);
  p = fmaf(p, s, -0.139086052775383f);
  p = fmaf(p, s, 0.19946560263633728f);
  p = fmaf(p, s, -0.33329859375953674f);
  p = fmaf(p, s, 0.9999993443489075f);
  float r = p * a;
  if (ay > ax) r = 1.57079632679489662f - r;
  if (x < 0.0f || (x == 0.0f && __float_as_uint(x) != 0u)) r = 3.14159265358979324f - r;
  return copysignf(r, y);
}

// cos(x) with a two-constant Cody-Waite reduction to [-pi, pi] ahead of the
// MUFU approximation (cos.approx is accurate to ~2^-21 absolute only there).
__device__ __forceinline__ float reduce_2pi(float x) {
  const float k = rintf(x * 0.159154943091895336f);
  x = fmaf(-k, 6.28318548202514648f, x);
  return fmaf(-k, -1.74845553e-7f, x);
}

// Per hidden unit (theta = x + i y), with u = |x|, v = sign(x) y, t = e^{-2u}:
//   |(1+t) cos v + i (1-t) sin v|^2 = (1-t)^2 + 4 t cos^2 v,
// so Re log cosh theta = u - log 2 + 0.5 log((1-t)^2 + 4t cos^2 v): three MUFU
// ops (ex2, cos, lg2).  The phase atan2((1-t) sin v, (1+t) cos v) is computed
// only when Im log psi is requested (IM), from sin v / cos v.
template <int FMT>
__device__ inline void build_a(uint8_t* sA, const uint32_t* __restrict__ bits, int64_t row0, int64_t B, int N,
                               int Kp, int words, int tid);
template <bool IM>
__device__ inline void epilogue_unit(uint32_t t_re, uint32_t t_im, int nquads, int slice, int rot, float& su,
                                     float& sl, float& si);

template <int FMT, bool IM>
__global__ void __launch_bounds__(kThreads, 1)
    forward_tc_kernel(Layout L, const uint8_t* __restrict__ blob, const uint32_t* __restrict__ bits, int64_t B,
                      double* __restrict__ out_lp, double* __restrict__ out_re, double* __restrict__ out_im) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bars[2];  // [0] MMA done, [1] B staged

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = L.N, Kp = L.Kp, HC = L.HC, nchunks = L.nchunks, words = L.words;
  uint8_t* sA = smem;
  uint8_t* sB = smem + L.a_bytes;
  float* sVis = reinterpret_cast<float*>(sB + L.chunk_bytes);  // [re N][im N]
  float* sRed = sVis + 2 * N;                                   // [slice][128][3]
  const uint32_t aA = smem_u32(sA), aB = smem_u32(sB);
  const uint32_t bar_mma = smem_u32(&bars[0]), bar_b = smem_u32(&bars[1]);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_mma));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const float* gvis = reinterpret_cast<const float*>(blob + L.off_vis);
  for (int j = tid; j < 2 * N; j += kThreads) sVis[j] = gvis[j];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  // instruction descriptor: f32 accumulate, A/B format, K-major both, N = HC, M = 128
  const uint32_t fmtbits = FMT == MPV_FMT_BF16 ? 1u : 0u;
  const uint32_t idesc = (1u << 4) | (fmtbits << 7) | (fmtbits << 10) | ((uint32_t)(HC >> 3) << 17) |
                         ((uint32_t)(kRows >> 4) << 24);
  const uint32_t sbo = (uint32_t)Kp * 16, lbo = 128;
  uint32_t ph_mma = 0, ph_b = 0;

  const int q = warp & 3, slice = warp >> 2;
  const int row = q * 32 + lane;  // TMEM lane = tile row
  const uint32_t t_lane = (uint32_t)(q * 32) << 16;
  const int64_t ntiles = (B + kRows - 1) / kRows;
  // every column (padding included) contributes -log 2; padded columns (theta = 0) add log 2 back
  const float ln2 = 0.693147180559945309f;

  if (nchunks == 1 && tid == 0) bulk_load(aB, blob, (uint32_t)L.chunk_bytes, bar_b);
  bool b_resident = false;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kRows;
    build_a<FMT>(sA, bits, row0, B, N, Kp, words, tid);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();

    float su = 0.0f, sl = 0.0f, si = 0.0f;  // sum u, sum log2(q), sum phase
    for (int c = 0; c < nchunks; ++c) {
      if (tid == 0) {
        if (nchunks > 1) bulk_load(aB, blob + (size_t)c * L.chunk_bytes, (uint32_t)L.chunk_bytes, bar_b);
        if (!b_resident) {
          mbar_wait(bar_b, ph_b);
          ph_b ^= 1;
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int ks = 0; ks < Kp / 16; ++ks) {
          const uint64_t da = make_desc(aA + ks * 256, lbo, sbo);
          const uint64_t dre = make_desc(aB + ks * 256, lbo, sbo);
          const uint64_t dim = make_desc(aB + (uint32_t)HC * Kp * 2 + ks * 256, lbo, sbo);
          mma_f16(tmem, da, dre, idesc, ks > 0);
          mma_f16(tmem + 256, da, dim, idesc, ks > 0);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_mma)
                     : "memory");
      }
      b_resident = nchunks == 1;
      mbar_wait(bar_mma, ph_mma);
      ph_mma ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      epilogue_unit<IM>(tmem + t_lane, tmem + t_lane + 256, HC / 4, slice, 0, su, sl, si);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();  // TMEM and the B buffer are free for the next chunk / tile
    }
    if (slice > 0) {
      float* r = sRed + 3 * ((slice - 1) * kRows + row);
      r[0] = su;
      r[1] = sl;
      r[2] = si;
    }
    __syncthreads();
    if (slice == 0) {
      const int64_t s = row0 + row;
#pragma unroll
      for (int k = 1; k < kSlices; ++k) {
        const float* r = sRed + 3 * ((k - 1) * kRows + row);
        su += r[0];
        sl += r[1];
        si += r[2];
      }
      if (s < B) {
        float vr = 0.0f, vi = 0.0f;
        for (int w = 0; w < words; ++w) {
          uint32_t m = bits[s * words + w];
          if (w == words - 1 && (N & 31)) m &= (1u << (N & 31)) - 1u;
          while (m) {
            const int k = w * 32 + __ffs(m) - 1;
            m &= m - 1;
            vr += sVis[k];
            if (IM) vi += sVis[N + k];
          }
        }
        const double re = (double)vr + (double)su + 0.5 * (double)ln2 * (double)sl -
                          (double)ln2 * (double)(nchunks * HC);
        if (out_lp) out_lp[s] = 2.0 * re;
        if (out_re) out_re[s] = re;
        if (IM && out_im) out_im[s] = (double)vi + (double)si;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// A tile (configurations row0 .. row0+127) from packed bits: 8 bits -> 8
// f16/bf16 values per 16-byte store; column N is the constant 1.
template <int FMT>
__device__ inline void build_a(uint8_t* sA, const uint32_t* __restrict__ bits, int64_t row0, int64_t B, int N,
                               int Kp, int words, int tid) {
  const uint16_t one = FMT == MPV_FMT_BF16 ? 0x3F80 : 0x3C00;
  const int kgroups = Kp / 8;
  for (int idx = tid; idx < kRows * kgroups; idx += kThreads) {
    const int r = idx / kgroups, g = idx % kgroups;
    const int64_t s = row0 + r;
    uint32_t byte = 0;
    if (s < B && g * 8 < N) {
      byte = (bits[s * words + (g >> 2)] >> ((g & 3) * 8)) & 0xFFu;
      const int valid = N - g * 8;
      if (valid < 8) byte &= (1u << valid) - 1u;
    }
    if (g * 8 <= N && N < g * 8 + 8) byte |= 1u << (N - g * 8);
    uint32_t p[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      p[j] = ((byte >> (2 * j)) & 1u ? (uint32_t)one : 0u) | ((byte >> (2 * j + 1)) & 1u ? (uint32_t)one << 16 : 0u);
    *reinterpret_cast<uint4*>(sA + kmajor_off(r, g * 8, Kp)) = make_uint4(p[0], p[1], p[2], p[3]);
  }
}

// A tile built by the producer warps of the pipelined kernel: lane l of
// producer warp pw owns rows l + 32 (pw + kProducers rr); their packed words are loaded first (up to 4 per
// row in registers), then expanded into 16-byte stores (each 8-lane group
// writes one 128-byte core matrix: conflict-free).
template <int FMT>
__device__ inline void build_a_warp(uint8_t* sA, const uint32_t* __restrict__ bits, int64_t row0, int64_t B, int N,
                                    int Kp, int words, int lane, int pw) {
  const uint32_t one = FMT == MPV_FMT_BF16 ? 0x3F80u : 0x3C00u;
  const int kgroups = Kp / 8, nw = (kgroups + 3) / 4;
  uint32_t wv[kRowsPerLane][4];
#pragma unroll
  for (int rr = 0; rr < kRowsPerLane; ++rr) {
    const int64_t s = row0 + lane + 32 * (pw + kProducers * rr);
#pragma unroll
    for (int w = 0; w < 4; ++w) wv[rr][w] = (s < B && w < words) ? __ldg(bits + s * words + w) : 0u;
  }
  auto expand = [&](int r, uint32_t word, int w) {
    if (w == words - 1 && (N & 31)) word &= (1u << (N & 31)) - 1u;
#pragma unroll
    for (int g4 = 0; g4 < 4; ++g4) {
      const int g = w * 4 + g4;
      if (g < kgroups) {
        uint32_t byte = (word >> (8 * g4)) & 0xFFu;
        if (g * 8 <= N && N < g * 8 + 8) byte |= 1u << (N - g * 8);
        uint32_t p[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          p[j] = ((byte >> (2 * j)) & 1u ? one : 0u) | ((byte >> (2 * j + 1)) & 1u ? one << 16 : 0u);
        *reinterpret_cast<uint4*>(sA + kmajor_off(r, g * 8, Kp)) = make_uint4(p[0], p[1], p[2], p[3]);
      }
    }
  };
#pragma unroll
  for (int rr = 0; rr < kRowsPerLane; ++rr) {
    const int r = lane + 32 * (pw + kProducers * rr);
    const int64_t s = row0 + r;
#pragma unroll
    for (int w = 0; w < 4; ++w)
      if (w < nw) expand(r, wv[rr][w], w);
    for (int w = 4; w < nw; ++w) expand(r, (s < B && w < words) ? __ldg(bits + s * words + w) : 0u, w);
  }
}

// Log-cosh epilogue over this thread's row and its slice's 8-column groups
// (see forward_tc_kernel for the formulas).
__device__ inline void tmem_ld4(uint32_t taddr, float* v) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = __uint_as_float(r[j]);
}

__device__ inline void tmem_ld4_pair(uint32_t a0, uint32_t a1, float* v0, float* v1) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a0));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(a1));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    v0[j] = __uint_as_float(r[j]);
    v1[j] = __uint_as_float(r[4 + j]);
  }
}

// Floor of a unit's |cosh|^2 factor.  The smallest factor finite f32 theta can
// give is ~4e-14 (u = 0, v one f32 ulp from pi/2), so the floor never binds
// short of an exact zero of cosh; it keeps the product of two factors normal.
constexpr float kFactorFloor = 2.16840434e-19f;  // 2^-62

// 4-column groups, group j to slice (j - rot) mod 4: the rotation (tile index +
// chunk) evens out the remainder groups across slices over consecutive units.
template <bool IM>
__device__ inline void epilogue_unit(uint32_t t_re, uint32_t t_im, int nquads, int slice, int rot, float& su,
                                     float& sl, float& si) {
  for (int cq = (slice + rot) % kSlices; cq < nquads; cq += kSlices) {
    float tr[4], ti[4], f[4];
    tmem_ld4_pair(t_re + cq * 4, t_im + cq * 4, tr, ti);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float x = tr[j], y = ti[j];
      const float u = fabsf(x);
      su += u;
      if (IM) {
        const float t = ex2_ftz(-2.885390081777926815f * u);  // e^{-2u}
        // 1 - t without cancellation for small u (series of -expm1(-2u))
        const float omt = u < 0.0625f ? omt_series(u) : 1.0f - t;
        const float vr = reduce_2pi(x < 0.0f ? -y : y);  // v = sign(x) y
        const float sv = sin_ftz(vr), cv = cos_ftz(vr);
        const float wr = (1.0f + t) * cv, wi = omt * sv;
        f[j] = fmaxf(fmaf(wr, wr, wi * wi), kFactorFloor);
        si += atan2_fast(wi, wr);
      } else {
        // |.|^2 = (1-t)^2 + 4t cos^2 v: no cancellation near the zeros of cosh; cos is even, so v -> y.
        // The 4 rides in the exponent: t4 = 4t = 2^(2 - 2u log2 e).
        const float t4 = ex2_ftz(fmaf(-2.885390081777926815f, u, 2.0f));
        const float omt = u < 0.0625f ? omt_series(u) : fmaf(t4, -0.25f, 1.0f);
        const float cv = cos_ftz(reduce_2pi(y));
        f[j] = fmaxf(fmaf(t4 * cv, cv, omt * omt), kFactorFloor);
      }
    }
    // one lg2 per pair of units: each factor lies in [2^-62, 4], so the product stays normal
    sl += lg2_ftz(f[0] * f[1]) + lg2_ftz(f[2] * f[3]);
  }
}

__device__ inline void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ inline void commit_to(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// Software-pipelined variant (Layout.pipe): all B chunks resident in shared
// memory, A double-buffered, two TMEM accumulator buffers (re | im, 2*HC <= 256
// columns each).  Work units are (tile, chunk) pairs; while the 16 warps run
// the epilogue of unit u, the tensor core computes unit u+1 into the other
// TMEM buffer.  No CTA-wide barrier inside the loop: mbarriers hand off
//   full[b]       MMA of the unit in TMEM buffer b done (tcgen05.commit),
//   tmem_empty[b] all 512 epilogue threads drained buffer b (the issuer waits
//                 on it before MMA(u+2) reuses the buffer),
//   a_empty[b]    the MMAs of the tile in A buffer b done (A(t+2) may be built),
//   red_full[k]   slices 1..3 wrote their per-tile partial sums into sRed[k]
//                 (k = tile mod 3; slice 0 reduces tile i at the start of tile
//                 i+1, and a writer of tile i+3 is held back by tmem_empty until
//                 slice 0 has drained tile i+1, so three buffers never collide),
// so a slow epilogue warp only stalls the issuer two units later, not its peers.
template <int FMT, bool IM>
__global__ void __launch_bounds__(kThreads + 32 * kProducers, 1)
    forward_tc_pipe_kernel(Layout L, const uint8_t* __restrict__ blob, const uint32_t* __restrict__ bits, int64_t B,
                           double* __restrict__ out_lp, double* __restrict__ out_re, double* __restrict__ out_im) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  // [0,1] full, [2,3] tmem_empty, [4,5] a_empty, [6,7,8] red_full, [9] B staged
  __shared__ __align__(8) uint64_t bars[10];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = L.N, M = L.M, Kp = L.Kp, HC = L.HC, HCB = L.HCB, nchunks = L.nchunks;
  uint8_t* sA = smem;                          // 2 x a_bytes
  uint8_t* sB = smem + 2 * L.a_bytes;          // nchunks x chunk_bytes
  float* sRed = reinterpret_cast<float*>(sB + (size_t)nchunks * L.chunk_bytes);  // [tile % 3][slice][128][3]
  float* sAx = sRed + 3 * kSlices * kRows * 3; // [tile parity][128][2]: a . x (re, im)
  const bool producer = warp >= kThreads / 32;  // build A tiles; producer warp 0 issues the MMAs
  const int pw = warp - kThreads / 32;
  const bool issuer = pw == 0 && lane == 0;
  const uint32_t aA = smem_u32(sA), aB = smem_u32(sB);
  const uint32_t bar0 = smem_u32(&bars[0]);
  const uint32_t bar_full = bar0, bar_tempty = bar0 + 16, bar_aempty = bar0 + 32, bar_red = bar0 + 48,
                 bar_b = bar0 + 72;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int k = 0; k < 10; ++k) {
      const uint32_t count = (k == 2 || k == 3) ? kThreads : (k >= 6 && k <= 8) ? kThreads - 128 : 1;
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar0 + 8 * k), "r"(count));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  const uint32_t fmtbits = FMT == MPV_FMT_BF16 ? 1u : 0u;
  const uint32_t idesc = (1u << 4) | (fmtbits << 7) | (fmtbits << 10) | ((uint32_t)(HCB >> 3) << 17) |
                         ((uint32_t)(kRows >> 4) << 24);
  const uint32_t sbo = (uint32_t)Kp * 16, lbo = 128;
  const int q = warp & 3, slice = warp >> 2;
  const int row = q * 32 + lane;
  const int words = L.words;
  const uint32_t t_lane = (uint32_t)(q * 32) << 16;
  const int64_t ntiles = (B + kRows - 1) / kRows;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t units = my_tiles * nchunks;
  const float ln2 = 0.693147180559945309f;

  auto tile_row0 = [&](int64_t t) { return (blockIdx.x + t * gridDim.x) * (int64_t)kRows; };
  if (producer) {
    // per tile t: wait until the MMAs of tile t-2 released A buffer t&1, build
    // A(t) (4 warps), then the issuer issues the tile's units, each once the
    // epilogue has drained the TMEM buffer it overwrites (unit u-2)
    for (int64_t t = 0; t < my_tiles; ++t) {
      if (t >= 2) mbar_wait(bar_aempty + 8 * (uint32_t)(t & 1), (uint32_t)(((t - 2) >> 1) & 1));
      build_a_warp<FMT>(sA + (size_t)(t & 1) * L.a_bytes, bits, tile_row0(t), B, N, Kp, words, lane, pw);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kProducers) : "memory");
      if (issuer) {
        if (t == 0) {
          bulk_load(aB, blob, (uint32_t)(nchunks * L.chunk_bytes), bar_b);
          mbar_wait(bar_b, 0);
        }
        for (int c = 0; c < nchunks; ++c) {
          const int64_t u = t * nchunks + c;
          const uint32_t b = (uint32_t)(u & 1);
          if (u >= 2) mbar_wait(bar_tempty + 8 * b, (uint32_t)(((u >> 1) + 1) & 1));
          const uint32_t a0 = aA + (uint32_t)(t & 1) * (uint32_t)L.a_bytes;
          const uint32_t b0 = aB + (uint32_t)c * (uint32_t)L.chunk_bytes;
          const uint32_t d0 = tmem + b * 256;
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          for (int ks = 0; ks < Kp / 16; ++ks) {
            const uint64_t da = make_desc(a0 + ks * 256, lbo, sbo);
            mma_f16(d0, da, make_desc(b0 + ks * 256, lbo, sbo), idesc, ks > 0);
            mma_f16(d0 + HCB, da, make_desc(b0 + (uint32_t)HCB * Kp * 2 + ks * 256, lbo, sbo), idesc, ks > 0);
          }
          commit_to(bar_full + 8 * b);
          if (c == nchunks - 1) commit_to(bar_aempty + 8 * (uint32_t)(t & 1));
        }
      }
      __syncwarp();
    }
  } else {
    auto finish_tile = [&](int64_t i) {  // slice 0: reduce the four slices (+ a . x), store
      if (slice != 0) return;
      mbar_wait(bar_red + 8 * (uint32_t)(i % 3), (uint32_t)((i / 3) & 1));
      const int64_t s = (blockIdx.x + i * gridDim.x) * kRows + row;
      if (s >= B) return;
      const float* r = sRed + (size_t)(i % 3) * kSlices * kRows * 3;
      float su = 0.0f, sl = 0.0f, si = 0.0f;
#pragma unroll
      for (int k = 0; k < kSlices; ++k) {
        su += r[3 * (k * kRows + row)];
        sl += r[3 * (k * kRows + row) + 1];
        si += r[3 * (k * kRows + row) + 2];
      }
      const float vr = sAx[2 * ((i & 1) * kRows + row)], vi = sAx[2 * ((i & 1) * kRows + row) + 1];
      const double re =
          (double)vr + (double)su + 0.5 * (double)ln2 * (double)sl - (double)ln2 * (double)L.cols_proc;
      if (out_lp) out_lp[s] = 2.0 * re;
      if (out_re) out_re[s] = re;
      if (IM && out_im) out_im[s] = (double)vi + (double)si;
    };
    uint32_t ph0 = 0, ph1 = 0;
    float su = 0.0f, sl = 0.0f, si = 0.0f;
    for (int64_t u = 0; u < units; ++u) {
      const int64_t i = u / nchunks;
      const int c = (int)(u % nchunks);
      if (c == 0 && i > 0) finish_tile(i - 1);
      if (u & 1) {
        mbar_wait(bar_full + 8, ph1);
        ph1 ^= 1;
      } else {
        mbar_wait(bar_full, ph0);
        ph0 ^= 1;
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tb = tmem + t_lane + (uint32_t)(u & 1) * 256;
      const int nquads = (min(HC, M - c * HC) + 3) / 4;
      // rotation keyed by the global tile index: each row's summation order is grid-independent
      const int rot = (int)((blockIdx.x + i * gridDim.x + c) % kSlices);
      epilogue_unit<IM>(tb, tb + HCB, nquads, slice, rot, su, sl, si);
      if (c == 0 && slice == 0) {  // column HC of chunk 0: the visible term a . x
        float ar[4], ai[4];
        tmem_ld4(tb + HC, ar);
        tmem_ld4(tb + HCB + HC, ai);
        sAx[2 * ((i & 1) * kRows + row)] = ar[0];
        sAx[2 * ((i & 1) * kRows + row) + 1] = ai[0];
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(bar_tempty + 8 * (uint32_t)(u & 1));
      if (c == nchunks - 1) {
        float* r = sRed + (size_t)(i % 3) * kSlices * kRows * 3 + 3 * (slice * kRows + row);
        r[0] = su;
        r[1] = sl;
        r[2] = si;
        su = sl = si = 0.0f;
        if (slice != 0) mbar_arrive(bar_red + 8 * (uint32_t)(i % 3));
      }
    }
    if (units > 0) finish_tile(my_tiles - 1);
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace tc

// -------- launchers (C ABI wrappers live in capi.cu) --------
size_t forward_tc_weights_bytes(int N, int M) {
  tc::Layout L;
  return tc::make_layout(N, M, &L) ? L.blob_bytes : 0;
}

cudaError_t forward_tc_prepare(int N, int M, int fmt, const double* params, void* weights, cudaStream_t st) {
  tc::Layout L;
  if (!tc::make_layout(N, M, &L)) return cudaErrorInvalidValue;
  const int64_t total = (int64_t)L.nchunks * 2 * L.HCB * L.Kp + 2LL * N;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (fmt == MPV_FMT_F16)
    tc::prepare_kernel<MPV_FMT_F16><<<grid, 256, 0, st>>>(L, params, (uint8_t*)weights);
  else
    tc::prepare_kernel<MPV_FMT_BF16><<<grid, 256, 0, st>>>(L, params, (uint8_t*)weights);
  return cudaGetLastError();
}

cudaError_t forward_tc_launch(int N, int M, int fmt, const void* weights, const uint32_t* bits, int64_t B,
                              double* out_lp, double* out_re, double* out_im, int max_ctas, cudaStream_t st) {
  tc::Layout L;
  if (!tc::make_layout(N, M, &L)) return cudaErrorInvalidValue;
  const bool im = out_im != nullptr;
  const void* fn;
  if (L.pipe)
    fn = fmt == MPV_FMT_F16 ? (im ? (const void*)&tc::forward_tc_pipe_kernel<MPV_FMT_F16, true>
                                  : (const void*)&tc::forward_tc_pipe_kernel<MPV_FMT_F16, false>)
                            : (im ? (const void*)&tc::forward_tc_pipe_kernel<MPV_FMT_BF16, true>
                                  : (const void*)&tc::forward_tc_pipe_kernel<MPV_FMT_BF16, false>);
  else
    fn = fmt == MPV_FMT_F16 ? (im ? (const void*)&tc::forward_tc_kernel<MPV_FMT_F16, true>
                                  : (const void*)&tc::forward_tc_kernel<MPV_FMT_F16, false>)
                            : (im ? (const void*)&tc::forward_tc_kernel<MPV_FMT_BF16, true>
                                  : (const void*)&tc::forward_tc_kernel<MPV_FMT_BF16, false>);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = (B + tc::kRows - 1) / tc::kRows;
  int64_t grid = std::min<int64_t>(ntiles, sms);
  if (max_ctas > 0) grid = std::min<int64_t>(grid, max_ctas);
  const uint8_t* blob = (const uint8_t*)weights;
  void* args[] = {&L, &blob, &bits, &B, &out_lp, &out_re, &out_im};
  const unsigned block = L.pipe ? tc::kThreads + 32 * tc::kProducers : tc::kThreads;  // + the producer warps
  return cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(block), args, L.smem, st);
}

}  // namespace mpv
