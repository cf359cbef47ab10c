// ResCNN neural quantum state on the 5th-generation tensor cores.
//
// North-star subsystem (2) for the convolutional ansatz of BASELINE configs[3]
// ("CNN/ResNet NQS, J1-J2 Heisenberg 10x10, tensor-core forward"): the model of
// /root/reference/PAPER.md:876-890 (oracle/rescnn.py is its f64 restatement;
// the reference package has no CNN, so parity is pinned by that restatement and
// exact H psi on enumerable lattices):
//   h0 = Conv(s), h_{l+1} = h_l + Conv(GELU(Conv(GELU(LN(h_l))))),
//   log psi = sum LN(h_n);  3x3 periodic convolutions, F = 16 channels.
//
// Tensor-core mapping (no im2col): a CTA holds C configurations as padded
// (L+2) x (L+2) grids, one row per grid position, in two groups of C/2
// configurations (rows back to back within a group, each group starting on an
// MMA tile boundary; <= 2 x 1024 rows = 16 tiles of 128), so one group's
// convolution runs on the tensor core while the other group's epilogue runs.
// Activations are two K planes (channels 0-7, 8-15) of 16 bytes per row, so a
// K-major no-swizzle descriptor with SBO = 128 B (8-row groups contiguous) and
// LBO = the plane stride addresses ANY row offset: the 3x3 neighbour of row r
// is row r + dy (L+2) + dx, so tap (dy, dx) of a convolution is one
//   tcgen05.mma.kind::f16  M=128, N=16 (out channels), K=16 (in channels)
// on the activation planes shifted by a constant, accumulated over the 9 taps
// in TMEM (f32).  The periodic halo rows are rewritten by the epilogue after
// every layer.  TMEM: the residual stream h for 16 tiles (256 columns; the
// second convolution of a block accumulates straight into it) and the
// first convolution's accumulators (256 columns).  Biases enter in the
// epilogues (the residual's biases as a running sum per block).  Epilogues
// (LN, GELU) run in f32 on 16 warps (lane quarter x tile group); layer inputs
// are rounded to the format (f16/bf16), accumulation and the residual stream
// are f32.
//
// Modes: evaluate (packed bits -> log p = 2 log psi), and the fused MH step
// (ref: sampler.py:111-133 with this evaluator): per chain the reference's
// splitmix64 draws pick a flip (or an exchange pair), the proposal is
// evaluated, accepted by the f64 test log u < lp' - lp, state updated in place
// and samples recorded at the thinning rounds (sampler.py:142-167 layout).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <stdint.h>

#include "common.cuh"

namespace mpv {
namespace cnn {

constexpr int kF = 16;           // channels (the paper's 16 filters)
constexpr int kTaps = 9;         // 3x3
constexpr int kRowsMax = 2048;   // 16 MMA tiles
constexpr int kThreads = 512;    // 16 warps: TMEM lane quarter x tile group
constexpr int kTapBytes = kF * kF * 2;  // one B block (16 x 16 f16)
constexpr int kMaxC = 96;        // configurations per CTA (L >= 3: <= 81)
constexpr int kIssuers = 4;      // threads issuing a convolution's MMAs

struct Shape {
  int L, Lp, R, n_res, C, tiles, margin;  // R = Lp^2 rows per configuration
  int Cg, GT;                             // configurations and MMA tiles per group (two groups)
  int n_conv;                             // 1 + 2 n_res
  size_t off_vec;                         // byte offset of the f32 vectors in the blob
  size_t blob_bytes;
  size_t smem;
};

__host__ __device__ inline int plane_rows(const Shape& s) { return s.tiles * 128 + 2 * s.margin; }

inline bool make_shape(int L, int n_res, Shape* s) {
  if (L < 3 || L > 30 || n_res < 0 || n_res > 8) return false;
  s->L = L;
  s->Lp = L + 2;
  s->R = s->Lp * s->Lp;
  s->n_res = n_res;
  // two groups of Cg configurations, each starting on a tile boundary, so the
  // tensor core runs one group's convolution under the other's epilogue
  s->Cg = (kRowsMax / 2) / s->R;
  s->C = 2 * s->Cg;
  if (s->Cg < 1 || s->C > kMaxC) return false;
  s->GT = (s->Cg * s->R + 127) / 128;
  s->tiles = 2 * s->GT;
  s->margin = (s->Lp + 1 + 7) / 8 * 8;
  s->n_conv = 1 + 2 * n_res;
  s->off_vec = (size_t)s->n_conv * kTaps * kTapBytes;
  // vectors: per LN i (n_res + 1): cumulative residual bias, gain, shift; per block: first conv bias
  s->blob_bytes = s->off_vec + ((size_t)(n_res + 1) * 3 * kF + (size_t)n_res * kF) * 4;
  s->blob_bytes = (s->blob_bytes + 255) / 256 * 256;
  const size_t planes = 2ull * plane_rows(*s) * 16;
  s->smem = planes + s->blob_bytes + (size_t)s->tiles * 128 * 4 + 1024;
  return s->smem <= 220 * 1024;
}

// ---- tcgen05 helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // sm_100 descriptor version; base offset 0, SWIZZLE_NONE
  return d;
}
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{.reg .pred p;\nWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// tanh-form GELU: u = z (c + c 0.044715 z^2), 0.5 z (1 + tanh u) = z (0.5 + 0.5 tanh u)
// (6 f32 ops + one MUFU per activation)
__device__ __forceinline__ float gelu(float z) {
  const float u = z * fmaf(0.035677408136300125f, z * z, 0.7978845608028654f);
  return z * fmaf(0.5f, tanh_approx(u), 0.5f);
}

template <int FMT>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  uint32_t r;
  if (FMT == MPV_FMT_BF16) asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  else asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// Write one grid position's 16 channels (rounded to FMT) to the activation
// planes at row `row` and at the periodic halo images of an interior position.
template <int FMT>
__device__ __forceinline__ void store_row(uint8_t* plane0, size_t plane_stride, int row, int pr, int pc, int Lp,
                                          const float* v) {
  uint4 a, b;
  a.x = pack2<FMT>(v[0], v[1]); a.y = pack2<FMT>(v[2], v[3]); a.z = pack2<FMT>(v[4], v[5]); a.w = pack2<FMT>(v[6], v[7]);
  b.x = pack2<FMT>(v[8], v[9]); b.y = pack2<FMT>(v[10], v[11]); b.z = pack2<FMT>(v[12], v[13]);
  b.w = pack2<FMT>(v[14], v[15]);
  const int L = Lp - 2;
  const int dr = pr == 1 ? L : (pr == L ? -L : 0);
  const int dc = pc == 1 ? L : (pc == L ? -L : 0);
  const int offs[4] = {0, dr * Lp, dc, dr * Lp + dc};
  const bool use[4] = {true, dr != 0, dc != 0, dr != 0 && dc != 0};
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (use[k]) {
      const int r = row + offs[k];
      *reinterpret_cast<uint4*>(plane0 + (size_t)r * 16) = a;
      *reinterpret_cast<uint4*>(plane0 + plane_stride + (size_t)r * 16) = b;
    }
}

struct Args {
  Shape S;
  const uint8_t* blob;
  // configurations / chains
  int64_t B;                 // configurations (evaluate) or chains (MH)
  int N, words;
  uint32_t* bits;            // packed [B][words] (MH: updated in place)
  double* out_lp;            // evaluate: log p; MH: cached log p (updated)
  int64_t* accepted;         // MH (may be NULL)
  int64_t* status;           // first non-finite (step, chain)
  // MH schedule
  int mh;
  uint64_t key;
  int64_t chain_offset, init_draws, step_index;
  int proposal;
  uint32_t* samples;
  int64_t thin, sample_base, sample_extra, round_offset, row0;
  int64_t local_step1;       // 1-based step within the recording launch
  // compacted MH step (exchange): the chains to evaluate, list[0 .. *count)
  const int32_t* list;
  const int32_t* count;
  int cpc;  // configurations per CTA group (<= S.C; fewer spread small batches over more SMs)
};

template <int FMT>
__global__ void __launch_bounds__(kThreads, 1) rescnn_kernel(const Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar_mma[2];  // MMA completion, one per group
  __shared__ int s_site[kMaxC];    // per configuration: flipped sites (MH), -1 none
  __shared__ int s_site2[kMaxC];
  __shared__ double s_logu[kMaxC];
  const Shape& S = a.S;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Lp = S.Lp, R = S.R, C = S.C, N = a.N, words = a.words;
  const int prow = plane_rows(S);
  const size_t pstride = (size_t)prow * 16;
  uint8_t* planes = smem;                                // [2][prow][16 B]
  uint8_t* sblob = smem + 2 * pstride;                   // B blocks + vectors
  float* vec = reinterpret_cast<float*>(sblob + S.off_vec);
  float* rowsum = reinterpret_cast<float*>(sblob + S.blob_bytes);  // [tiles * 128]
  uint8_t* plane0 = planes + (size_t)S.margin * 16;      // row 0 of the grid rows
  const uint32_t aPlanes = smem_u32(plane0), aBlob = smem_u32(sblob);
  const uint32_t sbar[2] = {smem_u32(&bar_mma[0]), smem_u32(&bar_mma[1])};

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sbar[0]), "r"(kIssuers));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sbar[1]), "r"(kIssuers));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (size_t i = tid * 16; i < S.blob_bytes; i += kThreads * 16)
    *reinterpret_cast<uint4*>(sblob + i) = *reinterpret_cast<const uint4*>(a.blob + i);
  for (size_t i = tid * 16; i < 2 * pstride; i += kThreads * 16) *reinterpret_cast<uint4*>(planes + i) = make_uint4(0, 0, 0, 0);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  uint32_t phase[2] = {0u, 0u};

  const uint32_t fmtbits = FMT == MPV_FMT_BF16 ? 1u : 0u;
  const uint32_t idesc = (1u << 4) | (fmtbits << 7) | (fmtbits << 10) | ((uint32_t)(kF >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const int q = warp & 3, tg = warp >> 2;  // TMEM lane quarter, tile group
  const uint32_t t_lane = (uint32_t)(q * 32) << 16;
  const int L = S.L;
  const float* cb = vec;                          // [(n_res+1)][3][16]: cumulative bias, gain, shift
  const float* b1 = vec + (S.n_res + 1) * 3 * kF;  // [n_res][16]

  const int GT = S.GT, Cg = S.Cg, gb = GT * 128;  // tiles and first row of group 1
  int ntile[2] = {GT, GT};                        // tiles of each group in use (set per CTA group)
  // one convolution of group g: 9 taps x GT tile MMAs into dst columns (the
  // first tap overwrites unless keep); every warp's epilogue writes must be done
  auto issue = [&](int g, int ci, uint32_t dst_col, bool keep) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    // kIssuers threads (lane 0 of warps 0..kIssuers-1, one per SM sub-partition)
    // issue the group's tiles round-robin; each commits its own MMAs to the barrier
    if (lane == 0 && warp < kIssuers) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int t = g * GT + warp; t < g * GT + ntile[g]; t += kIssuers)
        for (int d = 0; d < kTaps; ++d) {
          const int off = (d / 3 - 1) * Lp + (d % 3 - 1);
          const uint32_t aaddr = aPlanes + (uint32_t)((t * 128 + off) * 16);
          const uint64_t da = make_desc(aaddr, (uint32_t)pstride, 128);
          const uint64_t db = make_desc(aBlob + (uint32_t)((ci * kTaps + d) * kTapBytes), 128, 256);
          mma_f16(tmem + dst_col + t * kF, da, db, idesc, (keep || d > 0) ? 1u : 0u);
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sbar[g])
                   : "memory");
    }
  };
  auto wait = [&](int g) {
    mbar_wait(sbar[g], phase[g]);
    phase[g] ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  };
  // convolution k of the network: 0 embedding -> h; odd: first conv of block
  // (k-1)/2 -> acc; even >= 2: second conv of block (k-2)/2 accumulated into h
  auto issue_conv = [&](int g, int k) {
    if (k == 0) issue(g, 0, 0, false);
    else if (k & 1) issue(g, k, 256, false);
    else issue(g, k, 0, true);
  };
  const int64_t B = a.list ? (int64_t)*a.count : a.B;  // compacted: only the chains that move
  auto chain_of = [&](int64_t idx) -> int64_t { return a.list ? (int64_t)a.list[idx] : idx; };
  // per-lane epilogue rows (tile slot m of group g: t = g GT + tg + 4 m): the
  // configuration within the group and the grid position, computed once
  // (integer divisions by runtime sizes stay out of the epilogues)
  uint32_t rinfo[2][2];
#pragma unroll
  for (int g = 0; g < 2; ++g)
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int rr = (tg + 4 * m) * 128 + q * 32 + lane;  // row within the group
      const int jj = rr / R, pos = rr - jj * R;
      rinfo[g][m] = jj < Cg ? ((uint32_t)jj << 16) | ((uint32_t)(pos / Lp) << 8) | (uint32_t)(pos % Lp) : 0xFFFF0000u;
    }
  const int cpc = a.cpc > 0 ? min(a.cpc, C) : C;
  for (int64_t grp = blockIdx.x; grp < (B + cpc - 1) / cpc; grp += gridDim.x) {
    const int64_t c0 = grp * cpc;
    const int nc = (int)min((int64_t)cpc, B - c0);
    // MMA tiles holding this group's configurations (an empty second group is skipped)
    const int used0 = (min(nc, Cg) * R + 127) / 128, used1 = (max(0, nc - Cg) * R + 127) / 128;
    // ---- proposals (MH) ----
    if (a.mh && tid < nc) {
      const int64_t c = chain_of(c0 + tid), gchain = a.chain_offset + c;
      const uint64_t s0 = stream_state(a.key, (uint64_t)gchain);
      const uint64_t t = (uint64_t)(a.init_draws + 2 * a.step_index);
      const double us = stream_draw(s0, t), ua = stream_draw(s0, t + 1);
      int k1, k2 = -1;
      if (a.proposal == MPV_PROPOSAL_FLIP) {
        k1 = (int)floor_scaled(us, (double)N);
      } else {
        int i, j;
        pair_of(floor_scaled(us, 0.5 * (double)N * (double)(N - 1)), N, i, j);
        const uint32_t bi = (a.bits[c * words + (i >> 5)] >> (i & 31)) & 1u;
        const uint32_t bj = (a.bits[c * words + (j >> 5)] >> (j & 31)) & 1u;
        k1 = bi != bj ? i : -1;  // an exchange of equal bits is the identity (always accepted)
        k2 = bi != bj ? j : -1;
      }
      s_site[tid] = k1;
      s_site2[tid] = k2;
      s_logu[tid] = log(ua);
    }
    __syncthreads();
    // row r -> (configuration j, grid position pos); false for padding rows
    auto rowmap = [&](int r, int& j, int& pos) -> bool {
      const int g = r >= gb ? 1 : 0;
      const int rr = r - g * gb, jj = rr / R;
      pos = rr - jj * R;
      j = g * Cg + jj;
      return jj < Cg && j < nc;
    };
    // ---- input plane of group g: s = 1 - 2x in channel 0 (all grid rows incl. halo) ----
    auto epi_in = [&](int g) {
      for (int r = g * gb + tid; r < g * gb + ntile[g] * 128; r += kThreads) {
        int j, pos;
        float v0 = 0.0f;
        if (rowmap(r, j, pos)) {
          int pr = pos / Lp, pc = pos % Lp;
          pr = pr == 0 ? L : (pr == L + 1 ? 1 : pr);
          pc = pc == 0 ? L : (pc == L + 1 ? 1 : pc);
          const int site = (pr - 1) * L + (pc - 1);
          uint32_t x = (a.bits[chain_of(c0 + j) * words + (site >> 5)] >> (site & 31)) & 1u;
          if (a.mh && (site == s_site[j] || site == s_site2[j])) x ^= 1u;
          v0 = x ? -1.0f : 1.0f;
        }
        uint4 lo, hi = make_uint4(0, 0, 0, 0);
        lo.x = pack2<FMT>(v0, 0.0f);
        lo.y = lo.z = lo.w = 0;
        *reinterpret_cast<uint4*>(plane0 + (size_t)r * 16) = lo;
        *reinterpret_cast<uint4*>(plane0 + pstride + (size_t)r * 16) = hi;
      }
    };
    // ---- epilogue m (1 .. n_conv) of group g: odd m = LayerNorm of h (+ the running
    // bias) for block (m-1)/2 -> GELU -> next input, or the final per-row sums;
    // even m = GELU of the first convolution of block (m-2)/2 (+ its bias) ----
    auto epi = [&](int g, int m) {
      if (m & 1) {
        const int l = (m - 1) / 2;
        const float* cbl = cb + l * 3 * kF;
#pragma unroll
        for (int m2 = 0; m2 < 2; ++m2) {
          const int t = g * GT + tg + 4 * m2;
          if (t >= g * GT + ntile[g]) break;
          float h[16];
          tmem_ld16(tmem + t_lane + t * kF, h);
          const int r = t * 128 + q * 32 + lane;
          const uint32_t ri = g ? rinfo[1][m2] : rinfo[0][m2];
          const int jj = (int)(ri >> 16), pr = (int)((ri >> 8) & 0xFF), pc = (int)(ri & 0xFF);
          const bool valid = jj < Cg && g * Cg + jj < nc;
          const bool interior = valid && pr >= 1 && pr <= L && pc >= 1 && pc <= L;
          const float4* c4 = reinterpret_cast<const float4*>(cbl);  // [bias | gain | shift] x 16, LDS.128
          float mu = 0.0f;
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const float4 c = c4[k4];
            h[4 * k4] += c.x; h[4 * k4 + 1] += c.y; h[4 * k4 + 2] += c.z; h[4 * k4 + 3] += c.w;
          }
#pragma unroll
          for (int k = 0; k < 16; ++k) mu += h[k];
          mu *= 1.0f / 16.0f;
          float var = 0.0f;
#pragma unroll
          for (int k = 0; k < 16; ++k) var = fmaf(h[k] - mu, h[k] - mu, var);
          const float rs = rsqrtf(fmaf(var, 1.0f / 16.0f, 1e-6f));
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {  // LN: gain * (h - mu) * rs + shift
            const float4 gk = c4[4 + k4], sk = c4[8 + k4];
            h[4 * k4] = fmaf(gk.x * rs, h[4 * k4] - mu, sk.x);
            h[4 * k4 + 1] = fmaf(gk.y * rs, h[4 * k4 + 1] - mu, sk.y);
            h[4 * k4 + 2] = fmaf(gk.z * rs, h[4 * k4 + 2] - mu, sk.z);
            h[4 * k4 + 3] = fmaf(gk.w * rs, h[4 * k4 + 3] - mu, sk.w);
          }
          if (l < S.n_res) {
#pragma unroll
            for (int k = 0; k < 16; ++k) h[k] = gelu(h[k]);
            if (interior) store_row<FMT>(plane0, pstride, r, pr, pc, Lp, h);
          } else {
            float sum = 0.0f;
#pragma unroll
            for (int k = 0; k < 16; ++k) sum += h[k];
            rowsum[r] = interior ? sum : 0.0f;
          }
        }
      } else {
        const float* b1l = b1 + ((m - 2) / 2) * kF;
#pragma unroll
        for (int m2 = 0; m2 < 2; ++m2) {
          const int t = g * GT + tg + 4 * m2;
          if (t >= g * GT + ntile[g]) break;
          float v[16];
          tmem_ld16(tmem + t_lane + 256 + t * kF, v);
          const int r = t * 128 + q * 32 + lane;
          const uint32_t ri = g ? rinfo[1][m2] : rinfo[0][m2];
          const int jj = (int)(ri >> 16), pr = (int)((ri >> 8) & 0xFF), pc = (int)(ri & 0xFF);
          const bool valid = jj < Cg && g * Cg + jj < nc;
          if (valid && pr >= 1 && pr <= L && pc >= 1 && pc <= L) {
            const float4* b4 = reinterpret_cast<const float4*>(b1l);
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4) {
              const float4 bk = b4[k4];
              v[4 * k4] = gelu(v[4 * k4] + bk.x);
              v[4 * k4 + 1] = gelu(v[4 * k4 + 1] + bk.y);
              v[4 * k4 + 2] = gelu(v[4 * k4 + 2] + bk.z);
              v[4 * k4 + 3] = gelu(v[4 * k4 + 3] + bk.w);
            }
            store_row<FMT>(plane0, pstride, r, pr, pc, Lp, v);
          }
        }
      }
    };
    // ---- two-group software pipeline: group 1's convolution k runs on the
    // tensor core under group 0's epilogue k+1, group 0's convolution k+1 under
    // group 1's epilogue k+1 ----
    const int K = S.n_conv;
    ntile[0] = used0;
    ntile[1] = used1;
    const bool two = used1 > 0;  // block-uniform
    epi_in(0);
    if (two) epi_in(1);
    issue_conv(0, 0);
    for (int k = 0; k < K; ++k) {
      if (two) issue_conv(1, k);
      wait(0);
      epi(0, k + 1);
      if (k + 1 < K) issue_conv(0, k + 1);
      if (two) {
        wait(1);
        epi(1, k + 1);
      }
    }
    __syncthreads();
    // ---- per-configuration sums (fixed order), accept / write ----
    if (tid < nc) {
      const int j = tid;
      float sum = 0.0f;
      const int base = (j / Cg) * gb + (j % Cg) * R;  // the configuration's first row
      for (int pos = 0; pos < R; ++pos) sum += rowsum[base + pos];
      const double lp_new = 2.0 * (double)sum;
      const int64_t c = chain_of(c0 + j);
      if (!a.mh) {
        a.out_lp[c] = lp_new;
        if (!isfinite(lp_new) && a.status) {
          atomicMin((unsigned long long*)&a.status[1], (unsigned long long)c);
          atomicExch((unsigned long long*)&a.status[0], (unsigned long long)MPV_ERR_NONFINITE);
        }
      } else {
        const double lp_old = a.out_lp[c];
        const bool identity = s_site[j] < 0;  // exchange of equal bits
        const bool accept = identity || s_logu[j] < lp_new - lp_old;  // NaN -> reject
        if (!identity && !isfinite(lp_new) && a.status) {
          atomicMin((unsigned long long*)&a.status[1],
                    (unsigned long long)(((a.step_index + 1) << 32) | (unsigned long long)c));
          atomicExch((unsigned long long*)&a.status[0], (unsigned long long)MPV_ERR_NONFINITE);
        }
        if (accept && !identity) {
          const int k1 = s_site[j], k2 = s_site2[j];
          a.bits[c * words + (k1 >> 5)] ^= 1u << (k1 & 31);
          if (k2 >= 0) a.bits[c * words + (k2 >> 5)] ^= 1u << (k2 & 31);
          a.out_lp[c] = lp_new;
        }
        if (accept && a.accepted) a.accepted[c] += 1;
        const int64_t s1 = a.local_step1;
        if (a.samples && a.thin > 0 && s1 % a.thin == 0) {
          const int64_t gchain = a.chain_offset + c;
          const int64_t count_c = a.sample_base + (gchain < a.sample_extra ? 1 : 0);
          const int64_t offset_c =
              gchain * a.sample_base + (gchain < a.sample_extra ? gchain : a.sample_extra) - a.row0;
          const int64_t rr = a.round_offset + s1 / a.thin - 1;
          if (rr < count_c)
            for (int w = 0; w < words; ++w) a.samples[(offset_c + rr) * words + w] = a.bits[c * words + w];
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---- f64 forward on the CUDA cores (local energies, parity).  A CTA holds G
// configurations; thread = (configuration, site) keeps its site's residual
// stream h[16] in registers and computes all 16 output channels of a
// convolution (16 FMA per activation load; the weights of the current
// convolution are staged in shared memory and read warp-uniformly).  Two
// activation buffers per configuration (layer input / first-convolution
// output) hold the neighbours' values.
// e^x for the GELU (a few ulp): x = n ln2 + r with |r| <= ln2/2 (Cody-Waite,
// two-constant ln2), e^r by a degree-11 Taylor polynomial (truncation < 1e-16
// relative), times 2^n by exponent arithmetic; saturates outside [-708, 708]
// (the GELU only needs e^x -> 0 or -> inf there).
__device__ __forceinline__ double exp_gelu(double x) {
  x = fmin(fmax(x, -708.0), 708.0);
  const double n = rint(x * 1.4426950408889634);
  const double r = fma(n, -1.90821492927058770002e-10, fma(n, -6.93147180369123816490e-01, x));  // fdlibm ln2 hi/lo
  double p = 2.5052108385441720e-08;  // 1/11!
  p = fma(p, r, 2.7557319223985893e-07);
  p = fma(p, r, 2.7557319223985888e-06);
  p = fma(p, r, 2.4801587301587302e-05);
  p = fma(p, r, 1.9841269841269841e-04);
  p = fma(p, r, 1.3888888888888889e-03);
  p = fma(p, r, 8.3333333333333332e-03);
  p = fma(p, r, 4.1666666666666664e-02);
  p = fma(p, r, 1.6666666666666666e-01);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  return __hiloint2double(__double2hiint(p) + ((int)n << 20), __double2loint(p));
}
// tanh-form GELU, 0.5 z (1 + tanh u) = z / (1 + e^{-2u}): one exp and one
// reciprocal (MUFU seed + Newton steps, rounding of a few ulp)
__device__ __forceinline__ double gelu64(double z) {
  const double u = 0.7978845608028654 * fma(0.044715 * z, z * z, z);
  const double d = 1.0 + exp_gelu(-2.0 * u);
  double y = __drcp_rn(d);
  return z * y;
}

constexpr int kF64Threads = 512;
constexpr int kFS = kF + 1;  // doubles per site in the activation buffers (odd: conflict-free LDS.64 across sites)

__global__ void __launch_bounds__(kF64Threads) rescnn_f64_kernel(const double* __restrict__ theta, int L, int n_res,
                                                                  const uint32_t* __restrict__ bits, int64_t B,
                                                                  int words, int G, double* __restrict__ out) {
  extern __shared__ double sm64[];
  const int N = L * L;
  double* wsm = sm64;                 // [9 taps][16 cin][16 cout]: a (tap, cin)'s 16 weights are 8 LDS.128
  double* bufA = wsm + kF * kF * kTaps;  // [G][N][kFS]
  double* bufB = bufA + (size_t)G * N * kFS;
  __shared__ double red[kF64Threads];
  const int tid = threadIdx.x;
  const int g = tid / N, p = tid % N;  // configuration slot, site
  const bool active = g < G;
  const int pr = p / L, pc = p % L;
  int nb[kTaps];
#pragma unroll
  for (int d = 0; d < kTaps; ++d) nb[d] = ((pr + d / 3 - 1 + L) % L) * L + (pc + d % 3 - 1 + L) % L;
  // parameter offsets (oracle/rescnn.py order)
  const size_t blk = 2 * kF + 2 * (kF * kF * kTaps + kF);

  auto stage = [&](const double* w) {  // one 16x16x9 convolution's weights
    __syncthreads();
    for (int i = tid; i < kF * kF * kTaps; i += blockDim.x) {  // w: [cout][cin][tap] (oracle/rescnn.py)
      const int c = i / (kF * kTaps), ci = (i / kTaps) % kF, d = i % kTaps;
      wsm[(d * kF + ci) * kF + c] = w[i];
    }
    __syncthreads();
  };
  // out[c] = bias[c] + sum_{tap, cin} w[c][cin][tap] src[nb(tap)][cin]
  auto conv = [&](const double* src, const double* bias, double* o) {
#pragma unroll
    for (int c = 0; c < kF; ++c) o[c] = bias[c];
    for (int d = 0; d < kTaps; ++d) {
      const double* sq = src + (size_t)nb[d] * kFS;
      const double2* wd = reinterpret_cast<const double2*>(wsm + d * kF * kF);
#pragma unroll 2
      for (int ci = 0; ci < kF; ++ci) {
        const double a = sq[ci];
#pragma unroll
        for (int c2 = 0; c2 < kF / 2; ++c2) {
          const double2 w2 = wd[ci * (kF / 2) + c2];
          o[2 * c2] = fma(w2.x, a, o[2 * c2]);
          o[2 * c2 + 1] = fma(w2.y, a, o[2 * c2 + 1]);
        }
      }
    }
  };
  auto ln = [&](const double* h, const double* gm, const double* be, double* z) {
    double mu = 0.0, var = 0.0;
#pragma unroll
    for (int c = 0; c < kF; ++c) mu += h[c];
    mu /= kF;
#pragma unroll
    for (int c = 0; c < kF; ++c) var += (h[c] - mu) * (h[c] - mu);
    const double rs = 1.0 / sqrt(var / kF + 1e-6);
#pragma unroll
    for (int c = 0; c < kF; ++c) z[c] = gm[c] * (h[c] - mu) * rs + be[c];
  };

  for (int64_t cfg0 = (int64_t)blockIdx.x * G; cfg0 < B; cfg0 += (int64_t)gridDim.x * G) {
    const int64_t cfg = cfg0 + g;
    const bool live = active && cfg < B;
    double* A = bufA + (size_t)g * N * kFS;
    double* Bv = bufB + (size_t)g * N * kFS;
    double h[kF], t[kF];
    if (live) A[p * kFS] = ((bits[cfg * words + (p >> 5)] >> (p & 31)) & 1u) ? -1.0 : 1.0;
    __syncthreads();
    // embedding (one input channel)
    if (live) {
      const double* w0 = theta;
      const double* b0 = theta + kF * kTaps;
#pragma unroll
      for (int c = 0; c < kF; ++c) h[c] = b0[c];
      for (int d = 0; d < kTaps; ++d) {
        const double sv = A[nb[d] * kFS];
#pragma unroll
        for (int c = 0; c < kF; ++c) h[c] = fma(w0[c * kTaps + d], sv, h[c]);
      }
    }
    const double* pp = theta + kF * kTaps + kF;
    for (int l = 0; l < n_res; ++l, pp += blk) {
      const double* gm = pp;
      const double* be = pp + kF;
      const double* wa = pp + 2 * kF;
      const double* ba = wa + kF * kF * kTaps;
      const double* wb = ba + kF;
      const double* bb = wb + kF * kF * kTaps;
      stage(wa);  // (also orders the previous block's reads of A before the writes below)
      if (live) {
        ln(h, gm, be, t);
#pragma unroll
        for (int c = 0; c < kF; ++c) A[p * kFS + c] = gelu64(t[c]);
      }
      __syncthreads();
      if (live) {
        conv(A, ba, t);
#pragma unroll
        for (int c = 0; c < kF; ++c) Bv[p * kFS + c] = gelu64(t[c]);
      }
      stage(wb);
      if (live) {
        conv(Bv, bb, t);
#pragma unroll
        for (int c = 0; c < kF; ++c) h[c] += t[c];
      }
    }
    double sum = 0.0;
    if (live) {
      ln(h, pp, pp + kF, t);
#pragma unroll
      for (int c = 0; c < kF; ++c) sum += t[c];
    }
    red[tid] = sum;
    __syncthreads();
    if (live && p == 0) {
      double acc = 0.0;
      for (int i = 0; i < N; ++i) acc += red[g * N + i];
      out[cfg] = acc;
    }
    __syncthreads();
  }
}


// ---- f64 forward on the FP64 tensor cores (DMMA m8n8k4): the production f64
// path (local energies, sigma-hat, parity).  A convolution is the GEMM
//   out[site][cout] = b[cout] + sum_{tap, cin} act[nb(site, tap)][cin] W[cout][cin][tap]
// with M = sites (m-tiles of 8), N = 16 output channels (two n-tiles of 8),
// K = 9 taps x 16 input channels (36 k-steps of 4): the A fragment of lane
// (row = lane / 4, k = lane % 4) is one gathered LDS.64 of the neighbour's
// channel (activation rows padded to 20 doubles: the 8 x 4 gather hits
// disjoint bank pairs), the B fragments come pre-arranged per (k-step,
// n-tile, lane) from shared memory.  Warp w owns m-tile w of each of the CTA's
// G configurations (MP = G tiles); the residual stream h stays in registers in
// the D-fragment layout (lane: site row lane / 4, channels 2 (lane % 4) + {0, 1}
// of each n-tile), LayerNorm reduces over the 4 lanes of a row by shuffles.
constexpr int kRow = 20;        // doubles per site row in the activation buffers
constexpr int kMP = 4;          // m-tiles per warp (configurations per CTA when a warp owns one tile per config)
constexpr int kWFrag = 36 * 2 * 32;  // one convolution's B fragments (doubles)

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

struct F64Plan {
  int N, L, n_res, words, mtc, tpc, warps, G;  // m-tiles per config, tiles per config per warp, warps, configs per CTA
  size_t smem;
};

__host__ __device__ inline size_t f64_dmma_smem(int N, int G, int mtc) {
  return (2 * (size_t)G * mtc * 8 * kRow + 2 * (size_t)kWFrag + (size_t)G * mtc) * sizeof(double) +
         (size_t)N * kTaps * sizeof(int) + (size_t)G * 32 * sizeof(uint32_t);
}

template <int TPC, int MP>
__global__ void __launch_bounds__(MP == 2 ? 448 : 512, MP == 2 ? 2 : 1) rescnn_f64_dmma_kernel(const double* __restrict__ theta, const F64Plan P,
                                                                  const uint32_t* __restrict__ bits, int64_t B,
                                                                  double* __restrict__ out) {
  extern __shared__ __align__(16) double sm[];
  constexpr int G = MP / TPC, tpc = TPC;
  const int N = P.N, L = P.L, mtc = P.mtc, W = P.warps, words = P.words;
  const int rows = mtc * 8;
  double* actA = sm;                                   // [G][rows][kRow]
  double* actB = actA + (size_t)G * rows * kRow;
  double* wf = actB + (size_t)G * rows * kRow;         // [2][36][2][32] B fragments of two convolutions
  double* part = wf + 2 * kWFrag;                      // [G][mtc] per-tile partial sums
  int* nbt = reinterpret_cast<int*>(part + (size_t)G * mtc);  // [N][9] neighbour sites
  uint32_t* sbits = reinterpret_cast<uint32_t*>(nbt + (size_t)N * kTaps);  // [G][32]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qr = lane >> 2, qc = lane & 3;
  for (int i = tid; i < N * kTaps; i += blockDim.x) {
    const int site = i / kTaps, d = i % kTaps, r = site / L, c = site % L;
    nbt[i] = ((r + d / 3 - 1 + L) % L) * L + (c + d % 3 - 1 + L) % L;
  }
  const size_t blk = 2 * kF + 2 * (kF * kF * kTaps + kF);  // parameters per residual block (oracle/rescnn.py order)
  // B fragments of a [cout][cin][tap] weight: (k-step kk, n-tile nt, lane) ->
  // W[nt 8 + lane / 4][(kk % 4) 4 + lane % 4][kk / 4]
  auto stage = [&](const double* w, double* dst) {
    for (int i = tid; i < kWFrag; i += blockDim.x) {
      const int kk = i / 64, nt = (i / 32) & 1, l = i & 31;
      dst[i] = w[((nt * 8 + (l >> 2)) * kF + (kk & 3) * 4 + (l & 3)) * kTaps + kk / 4];
    }
  };
  // this warp's tiles: (config g, tile t) for k = 0 .. MP-1 -> g = k / tpc, t = warp + (k % tpc) W
  auto tile_of = [&](int k, int& g, int& t) {
    g = k / tpc;
    t = warp + (k % tpc) * W;
  };
  constexpr int MPw = MP;  // tiles per warp
  // one convolution over `src` with fragments `wfr`: acc (per tile, n-tile) = bias + GEMM
  auto conv = [&](const double* src, const double* wfr, const double* bias, double (&acc)[MP][2][2]) {
    int nbrow[MP];
#pragma unroll
    for (int k = 0; k < MP; ++k) {
      if (k < MPw) {
        int g, t;
        tile_of(k, g, t);
        const double2 bv0 = make_double2(bias[2 * qc], bias[2 * qc + 1]);
        const double2 bv1 = make_double2(bias[8 + 2 * qc], bias[8 + 2 * qc + 1]);
        acc[k][0][0] = bv0.x; acc[k][0][1] = bv0.y; acc[k][1][0] = bv1.x; acc[k][1][1] = bv1.y;
        (void)g; (void)t;
      }
    }
#pragma unroll 3
    for (int d = 0; d < kTaps; ++d) {
#pragma unroll
      for (int k = 0; k < MP; ++k) {
        if (k < MPw) {
          int g, t;
          tile_of(k, g, t);
          const int site = min(t * 8 + qr, N - 1);  // padded rows gather a valid site (results dropped)
          nbrow[k] = (g * rows + nbt[site * kTaps + d]) * kRow;
        }
      }
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        const int kk = d * 4 + cb;
        const double b0 = wfr[(kk * 2 + 0) * 32 + lane], b1 = wfr[(kk * 2 + 1) * 32 + lane];
#pragma unroll
        for (int k = 0; k < MP; ++k) {
          if (k < MPw) {
            const double av = src[nbrow[k] + cb * 4 + qc];
            dmma884(acc[k][0][0], acc[k][0][1], av, b0);
            dmma884(acc[k][1][0], acc[k][1][1], av, b1);
          }
        }
      }
    }
  };
  // LayerNorm over the 16 channels of the lane's row (4 lanes hold a row)
  auto layernorm = [&](const double (&h)[2][2], const double* gm, const double* be, double (&z)[2][2]) {
    double s = h[0][0] + h[0][1] + h[1][0] + h[1][1];
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    const double mu = s / kF;
    double v = 0.0;
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) v += (h[n][e] - mu) * (h[n][e] - mu);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    const double rs = 1.0 / sqrt(v / kF + 1e-6);
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = n * 8 + 2 * qc + e;
        z[n][e] = gm[c] * (h[n][e] - mu) * rs + be[c];
      }
  };
  auto store = [&](double* dst, int g, int t, const double (&v)[2][2]) {
    const int row = t * 8 + qr;
    if (row < N) {
      double* r = dst + (size_t)(g * rows + row) * kRow;
      *reinterpret_cast<double2*>(r + 2 * qc) = make_double2(v[0][0], v[0][1]);
      *reinterpret_cast<double2*>(r + 8 + 2 * qc) = make_double2(v[1][0], v[1][1]);
    }
  };

  const int64_t groups = (B + G - 1) / G;
  for (int64_t grp = blockIdx.x; grp < groups; grp += gridDim.x) {
    const int64_t cfg0 = grp * G;
    __syncthreads();  // previous group's reads of the buffers / partials done
    for (int i = tid; i < G * 32; i += blockDim.x) {
      const int g = i / 32, w = i % 32;
      sbits[i] = (w < words && cfg0 + g < B) ? bits[(cfg0 + g) * words + w] : 0u;
    }
    __syncthreads();
    double h[MP][2][2];
    // embedding: one input channel s = 1 - 2x, 9 taps
    {
      const double* w0 = theta;             // [16][1][9]
      const double* b0 = theta + kF * kTaps;
#pragma unroll
      for (int k = 0; k < MP; ++k) {
        if (k < MPw) {
          int g, t;
          tile_of(k, g, t);
          const int site = min(t * 8 + qr, N - 1);
#pragma unroll
          for (int n = 0; n < 2; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e) h[k][n][e] = b0[n * 8 + 2 * qc + e];
          for (int d = 0; d < kTaps; ++d) {
            const int nbs = nbt[site * kTaps + d];
            const double sv = ((sbits[g * 32 + (nbs >> 5)] >> (nbs & 31)) & 1u) ? -1.0 : 1.0;
#pragma unroll
            for (int n = 0; n < 2; ++n)
#pragma unroll
              for (int e = 0; e < 2; ++e) h[k][n][e] = fma(w0[(n * 8 + 2 * qc + e) * kTaps + d], sv, h[k][n][e]);
          }
        }
      }
    }
    const double* pp = theta + kF * kTaps + kF;
    for (int l = 0; l < P.n_res; ++l, pp += blk) {
      const double *gm = pp, *be = pp + kF, *wa = pp + 2 * kF, *ba = wa + kF * kF * kTaps;
      const double *wb = ba + kF, *bb = wb + kF * kF * kTaps;
      stage(wa, wf);
      stage(wb, wf + kWFrag);
#pragma unroll
      for (int k = 0; k < MP; ++k) {
        if (k < MPw) {
          int g, t;
          tile_of(k, g, t);
          double z[2][2];
          layernorm(h[k], gm, be, z);
#pragma unroll
          for (int n = 0; n < 2; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e) z[n][e] = gelu64(z[n][e]);
          store(actA, g, t, z);
        }
      }
      __syncthreads();
      double acc[MP][2][2];
      conv(actA, wf, ba, acc);
#pragma unroll
      for (int k = 0; k < MP; ++k) {
        if (k < MPw) {
          int g, t;
          tile_of(k, g, t);
#pragma unroll
          for (int n = 0; n < 2; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e) acc[k][n][e] = gelu64(acc[k][n][e]);
          store(actB, g, t, acc[k]);
        }
      }
      __syncthreads();
      conv(actB, wf + kWFrag, bb, acc);
#pragma unroll
      for (int k = 0; k < MP; ++k)
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
          for (int e = 0; e < 2; ++e) h[k][n][e] += acc[k][n][e];
      __syncthreads();  // conv2's reads of actB and the fragments done before the next staging
    }
    // final LayerNorm, summed over channels and sites (fixed order: lanes, rows, tiles)
    const double* gf = pp;
    const double* bef = pp + kF;
#pragma unroll
    for (int k = 0; k < MP; ++k) {
      if (k < MPw) {
        int g, t;
        tile_of(k, g, t);
        double z[2][2];
        layernorm(h[k], gf, bef, z);
        double sum = (t * 8 + qr < N) ? (z[0][0] + z[0][1]) + (z[1][0] + z[1][1]) : 0.0;
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        sum += __shfl_xor_sync(0xffffffffu, sum, 4);
        sum += __shfl_xor_sync(0xffffffffu, sum, 8);
        sum += __shfl_xor_sync(0xffffffffu, sum, 16);
        if (lane == 0 && t < mtc) part[g * mtc + t] = sum;
      }
    }
    __syncthreads();
    if (tid < G && cfg0 + tid < B) {
      double acc = 0.0;
      for (int t = 0; t < mtc; ++t) acc += part[tid * mtc + t];
      out[cfg0 + tid] = acc;
    }
  }
}

}  // namespace cnn

using namespace cnn;

size_t rescnn_blob_bytes(int L, int n_res) {
  Shape s;
  return make_shape(L, n_res, &s) ? s.blob_bytes : 0;
}

// Exchange MH step, part 1: the reference's draws of every chain; a swap of
// equal bits is the identity (always accepted, sampler.py:119-131): its
// counter and sample record are written here, and only the other chains are
// appended to the list the tensor-core step evaluates (their order does not
// matter: each configuration's log p is independent of its tile slot).
// count[step & 1] collects this step; count[(step + 1) & 1] is cleared for the next.
__global__ void rescnn_propose_kernel(const Args a, int32_t* list, int32_t* count) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (threadIdx.x == 0 && blockIdx.x == 0) count[(a.step_index + 1) & 1] = 0;
  if (c >= a.B) return;
  const int64_t gchain = a.chain_offset + c;
  const uint64_t s0 = stream_state(a.key, (uint64_t)gchain);
  const double us = stream_draw(s0, (uint64_t)(a.init_draws + 2 * a.step_index));
  int i, j;
  pair_of(floor_scaled(us, 0.5 * (double)a.N * (double)(a.N - 1)), a.N, i, j);
  const uint32_t bi = (a.bits[c * a.words + (i >> 5)] >> (i & 31)) & 1u;
  const uint32_t bj = (a.bits[c * a.words + (j >> 5)] >> (j & 31)) & 1u;
  if (bi != bj) {
    list[atomicAdd(&count[a.step_index & 1], 1)] = (int32_t)c;
    return;
  }
  if (a.accepted) a.accepted[c] += 1;
  const int64_t s1 = a.local_step1;
  if (a.samples && a.thin > 0 && s1 % a.thin == 0) {
    const int64_t count_c = a.sample_base + (gchain < a.sample_extra ? 1 : 0);
    const int64_t offset_c = gchain * a.sample_base + (gchain < a.sample_extra ? gchain : a.sample_extra) - a.row0;
    const int64_t rr = a.round_offset + s1 / a.thin - 1;
    if (rr < count_c)
      for (int w = 0; w < a.words; ++w) a.samples[(offset_c + rr) * a.words + w] = a.bits[c * a.words + w];
  }
}

cudaError_t rescnn_launch(int L, int n_res, int fmt, const void* blob, uint32_t* bits, int64_t B, int words,
                          double* lp, int64_t* accepted, int64_t* status, int mh, uint64_t key, int64_t chain_offset,
                          int64_t init_draws, int64_t step_index, int proposal, uint32_t* samples, int64_t thin,
                          int64_t sample_base, int64_t sample_extra, int64_t round_offset, int64_t row0,
                          int64_t local_step1, cudaStream_t st, int32_t* list, int32_t* count) {
  Args a{};
  if (!make_shape(L, n_res, &a.S)) return cudaErrorInvalidValue;
  a.blob = (const uint8_t*)blob;
  a.B = B; a.N = L * L; a.words = words; a.bits = bits; a.out_lp = lp; a.accepted = accepted; a.status = status;
  a.mh = mh; a.key = key; a.chain_offset = chain_offset; a.init_draws = init_draws; a.step_index = step_index;
  a.proposal = proposal; a.samples = samples; a.thin = thin; a.sample_base = sample_base;
  a.sample_extra = sample_extra; a.round_offset = round_offset; a.row0 = row0; a.local_step1 = local_step1;
  const void* fn = fmt == MPV_FMT_BF16 ? (const void*)&rescnn_kernel<MPV_FMT_BF16> : (const void*)&rescnn_kernel<MPV_FMT_F16>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a.S.smem);
  if (e != cudaSuccess) return e;
  int dev = 0, n_sm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  // small batches: fewer configurations per CTA so that every SM gets work (a
  // compacted exchange step evaluates about half of the chains)
  const bool compacted = mh && proposal == MPV_PROPOSAL_EXCHANGE && list && count;
  const int64_t expect = compacted ? (B + 1) / 2 : B;
  a.cpc = (int)std::max<int64_t>(1, std::min<int64_t>(a.S.C, (expect + n_sm - 1) / n_sm));
  const int64_t groups = (B + a.cpc - 1) / a.cpc;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(groups, n_sm));
  if (mh && proposal == MPV_PROPOSAL_EXCHANGE && list && count) {
    rescnn_propose_kernel<<<(unsigned)((B + 255) / 256), 256, 0, st>>>(a, list, count);
    a.list = list;
    a.count = count + (step_index & 1);
  }
  void* args[] = {&a};
  return cudaLaunchKernel(fn, dim3(grid), dim3(kThreads), args, a.S.smem, st);
}

cudaError_t rescnn_f64_launch(const double* theta, int L, int n_res, const uint32_t* bits, int64_t B, int words,
                              double* out, cudaStream_t st) {
  const int N = L * L;
  {  // FP64 tensor cores: warps own one m-tile of each configuration (tpc tiles per config when > 32 tiles)
    F64Plan P{};
    P.N = N; P.L = L; P.n_res = n_res; P.words = words;
    P.mtc = (N + 7) / 8;
    P.tpc = 1;
    while ((P.mtc + P.tpc - 1) / P.tpc > 16) P.tpc *= 2;  // <= 16 warps (launch bounds 512)
    P.warps = (P.mtc + P.tpc - 1) / P.tpc;
    P.G = kMP / P.tpc;
    // two CTAs per SM (two configurations each) when one m-tile per config per warp
    static const char* two = getenv("MPV_CNN64_G2");
    if (P.tpc == 1 && P.warps <= 14 && (!two || two[0] != '0')) P.G = 2;
    if (P.tpc <= 4 && words <= 32) {
      P.smem = f64_dmma_smem(N, P.G, P.mtc);
      if (P.smem <= 227 * 1024) {
        for (const void* fn : {(const void*)&rescnn_f64_dmma_kernel<1, 2>, (const void*)&rescnn_f64_dmma_kernel<1, 4>,
                               (const void*)&rescnn_f64_dmma_kernel<2, 4>, (const void*)&rescnn_f64_dmma_kernel<4, 4>}) {
          cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem);
          if (e != cudaSuccess) return e;
        }
        const int64_t groups = (B + P.G - 1) / P.G;
        const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(groups, 148 * (P.G == 2 ? 4 : 2)));
        if (P.tpc == 1 && P.G == 2) rescnn_f64_dmma_kernel<1, 2><<<grid, 32 * P.warps, P.smem, st>>>(theta, P, bits, B, out);
        else if (P.tpc == 1) rescnn_f64_dmma_kernel<1, 4><<<grid, 32 * P.warps, P.smem, st>>>(theta, P, bits, B, out);
        else if (P.tpc == 2) rescnn_f64_dmma_kernel<2, 4><<<grid, 32 * P.warps, P.smem, st>>>(theta, P, bits, B, out);
        else rescnn_f64_dmma_kernel<4, 4><<<grid, 32 * P.warps, P.smem, st>>>(theta, P, bits, B, out);
        return cudaGetLastError();
      }
    }
  }
  if (N > kF64Threads) return cudaErrorInvalidValue;
  const int G = kF64Threads / N;
  const size_t smem = ((size_t)kF * kF * kTaps + 2ull * G * N * kFS) * sizeof(double);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute((const void*)&rescnn_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t groups = (B + G - 1) / G;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(groups, 148 * 4));
  rescnn_f64_kernel<<<grid, kF64Threads, smem, st>>>(theta, L, n_res, bits, B, words, G, out);
  return cudaGetLastError();
}

}  // namespace mpv
