// q = w (O v) of the SR solve on the 5th-generation tensor cores (tcgen05 +
// TMEM), exact in f64 through f16 limbs.
//
// The DMMA kernel (logderiv.cuh ld_ov_kernel) evaluates
//   q_s = w_s [ sum_k x_sk va_k + sum_i t_si (vb_i + (X vW^T)_si) ]
// with the GEMM X vW^T on the FP64 tensor cores (64 FMA/clk/SM on B200, the
// same rate as the FP64 pipe).  Here the GEMM runs in f16 with f32
// accumulation, which is exact: x in {0,1}, and every column i (re / im part
// separately) of [vW^T ; vb] is scaled by a power of two sigma >= its largest
// magnitude and split into L = 5 integer limbs,
//   v / sigma = d0 2^-10 + d1 2^-21 + d2 2^-32 + d3 2^-43 + d4 2^-54 (+ < 2^-55),
// |d| <= 1024 (exact in f16), so each limb's dot product over K <= 272 terms
// is an integer below 2^24 (exact in f32).  The epilogue rebuilds
// Y_si + vb_i = sigma (sum_l S_l 2^-e_l) in f64 (the only rounding: the f64
// sum of the five exact limb sums and the dropped 2^-55 sigma residual,
// against the DMMA kernel's 100 f64 roundings), multiplies by t_si and reduces
// over units in a fixed order.
//
// Tile = 128 samples (MMA M) x (L x HC) limb columns per re/im block (MMA N =
// 5 HC <= 240), K = N + 1 rounded up to 16 (column N of A is the constant 1,
// row N of B carries vb).  A is expanded from the packed sample bits, B (the
// limb matrix, rebuilt per call: v changes every CG iteration) is staged one
// chunk of HC units at a time and reused by all the CTA's tiles (chunk-outer
// loop, per-sample partial sums in shared memory), so B crosses L2 -> SMEM
// once per CTA.  Operand layout and descriptors as forward_tc.cu (K-major,
// no swizzle: 8x16-byte core matrices, LBO 128 B, SBO Kp*16 B).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <stdint.h>

#include "../../include/mpvmc_b200.h"
#include "ov_tc.h"

namespace mpv {
namespace ovtc {

constexpr int kRows = 128;      // MMA M: samples per tile
constexpr int kThreads = 512;   // 4 TMEM lane quarters x 4 column slices
constexpr int kSlices = 4;
constexpr int kLimbs = 5;
constexpr int kMaxTiles = 4;    // tiles per CTA (per-sample partials in shared memory)
constexpr size_t kSmemMax = 225 * 1024;

struct Layout {
  int N, M, Kp, HC, NB, nch, words;
  size_t a_bytes, chunk_bytes, t_bytes, off_sigma, blob_bytes, part_bytes, smem;
};

__host__ __device__ inline size_t rup(size_t x, size_t a) { return (x + a - 1) / a * a; }

inline bool make_layout(int N, int M, Layout* L) {
  if (N < 1 || M < 1 || N > 1024) return false;
  L->N = N; L->M = M; L->words = (N + 31) / 32;
  L->Kp = (int)rup(N + 1, 16);
  L->a_bytes = (size_t)kRows * L->Kp * 2;
  L->part_bytes = (size_t)kMaxTiles * kSlices * kRows * 16;
  for (int hc = 48; hc >= 16; hc -= 16) {
    const size_t chunk = 2ull * kLimbs * hc * L->Kp * 2;
    const size_t tb = (size_t)kRows * (hc + 1) * 16;  // the tile's t rows of the chunk, padded rows
    const size_t smem = L->a_bytes + chunk + tb + L->part_bytes + rup((size_t)N * 16, 16) + 2 * hc * 8 +
                        (size_t)kMaxTiles * kRows * L->words * 4 + 1024;
    if (smem <= kSmemMax) {
      L->HC = hc;
      L->NB = kLimbs * hc;
      L->nch = (M + hc - 1) / hc;
      L->chunk_bytes = chunk;
      L->t_bytes = tb;
      L->off_sigma = chunk * L->nch;
      L->blob_bytes = rup(L->off_sigma + (size_t)L->nch * hc * 2 * sizeof(double), 256);
      L->smem = smem;
      return true;
    }
  }
  return false;
}

// byte offset of element (row r, k) in a K-major no-swizzle tile with Kp columns
__host__ __device__ inline size_t kmajor_off(int r, int k, int Kp) {
  return (size_t)(r & 7) * 16 + (size_t)(r >> 3) * Kp * 16 + (size_t)(k >> 3) * 128 + (size_t)(k & 7) * 2;
}

// One warp per (unit i, part): sigma (warp max) and the five limbs of rows
// k = 0..Kp-1 of column i (k < N: vW[i][k], k = N: vb_i, beyond: 0).
__global__ void prepare_kernel(Layout L, const double2* __restrict__ v, uint8_t* __restrict__ blob,
                               const double* __restrict__ skip) {
  if (skip && *skip != 0.0) return;
  const int N = L.N, M = L.M, Kp = L.Kp, HC = L.HC, NB = L.NB;
  const int ncol = L.nch * HC, lane = threadIdx.x & 31;
  double* sigma = reinterpret_cast<double*>(blob + L.off_sigma);
  for (int idx = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; idx < 2 * ncol; idx += (gridDim.x * blockDim.x) >> 5) {
    const int i = idx >> 1, part = idx & 1;
    const double2* vw = v + N + M + (size_t)i * N;
    auto val = [&](int k) -> double {
      if (i >= M || k > N) return 0.0;
      const double2 z = k < N ? vw[k] : v[N + i];
      return part ? z.y : z.x;
    };
    double mx = 0.0;
    for (int k = lane; k <= N; k += 32) mx = fmax(mx, fabs(val(k)));
    for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
    const double inv = ldexp(1.0, -e);
    if (lane == 0) sigma[(size_t)i * 2 + part] = ldexp(1.0, e);
    const int c = i / HC, jj = i - c * HC;
    uint8_t* base = blob + (size_t)c * L.chunk_bytes + (size_t)part * NB * Kp * 2;
    for (int k = lane; k < Kp; k += 32) {
      double r = val(k) * inv * 1024.0;  // |r| < 1024, exact
#pragma unroll
      for (int l = 0; l < kLimbs; ++l) {
        const double d = rint(r);  // |d| <= 1024
        r = (r - d) * 2048.0;      // exact
        *reinterpret_cast<uint16_t*>(base + kmajor_off(l * HC + jj, k, Kp)) = __half_as_ushort(__double2half(d));
      }
    }
  }
}

__device__ inline uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ inline uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100); base offset 0, SWIZZLE_NONE
  return d;
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

__device__ inline void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  for (uint32_t off = 0; off < bytes; off += 65536u) {
    const uint32_t n = bytes - off < 65536u ? bytes - off : 65536u;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst + off),
                 "l"((const uint8_t*)src + off), "r"(n), "r"(bar)
                 : "memory");
  }
}

__device__ inline void tmem_ld4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}

// A tile (samples row0 .. row0+127) from packed bits, column N = 1 (f16).
__device__ inline void build_a(uint8_t* sA, const uint32_t* __restrict__ bits, int64_t row0, int64_t U, int N,
                               int Kp, int words, int tid) {
  const uint16_t one = 0x3C00;
  const int kgroups = Kp / 8;
  for (int idx = tid; idx < kRows * kgroups; idx += kThreads) {
    const int r = idx / kgroups, g = idx % kgroups;
    const int64_t s = row0 + r;
    uint32_t byte = 0;
    if (s < U && g * 8 < N) {
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

__device__ __forceinline__ double limb_sum(const float* s) {
  return fma((double)s[0], 0x1p-10,
             fma((double)s[1], 0x1p-21, fma((double)s[2], 0x1p-32, fma((double)s[3], 0x1p-43, (double)s[4] * 0x1p-54))));
}

__global__ void __launch_bounds__(kThreads, 1)
    ov_tc_kernel(Layout L, const uint8_t* __restrict__ blob, const double2* __restrict__ t,
                 const uint32_t* __restrict__ bits, int64_t U, const double2* __restrict__ v,
                 const double* __restrict__ w, double2* __restrict__ q, const double* __restrict__ skip) {
  if (skip && *skip != 0.0) return;
  const int64_t ntiles = (U + kRows - 1) / kRows;
  const int64_t tpc = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * tpc, t1 = min(ntiles, t0 + tpc);
  if (t0 >= t1) return;  // block-uniform, before any TMEM allocation
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bars[3];  // [0] MMA done, [1] B staged, [2] t rows staged

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = L.N, M = L.M, Kp = L.Kp, HC = L.HC, NB = L.NB, words = L.words;
  const int tstride = HC + 1;  // double2 per staged t row (padded: conflict-free per-lane rows)
  uint8_t* sA = smem;
  uint8_t* sB = smem + L.a_bytes;
  double2* sT = reinterpret_cast<double2*>(sB + L.chunk_bytes);                       // [row][HC + 1]
  double2* sPart = reinterpret_cast<double2*>(reinterpret_cast<uint8_t*>(sT) + L.t_bytes);  // [tile][slice][row]
  double2* sVa = reinterpret_cast<double2*>(reinterpret_cast<uint8_t*>(sPart) + L.part_bytes);  // [N]
  double* sSig = reinterpret_cast<double*>(sVa + N);                                   // [HC][2] of the chunk
  uint32_t* sBits = reinterpret_cast<uint32_t*>(sSig + 2 * HC);  // [tile][row][words]: the CTA's samples
  const uint32_t aA = smem_u32(sA), aB = smem_u32(sB), aT = smem_u32(sT);
  const uint32_t bar_mma = smem_u32(&bars[0]), bar_b = smem_u32(&bars[1]), bar_t = smem_u32(&bars[2]);
  const double* sigma = reinterpret_cast<const double*>(blob + L.off_sigma);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_mma));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_b));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_t));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int k = tid; k < N; k += kThreads) sVa[k] = v[k];
  for (int i = tid; i < kMaxTiles * kSlices * kRows; i += kThreads) sPart[i] = make_double2(0.0, 0.0);
  const int64_t u_cta = U - t0 * kRows;  // samples from the CTA's first row on
  for (int i = tid; i < (int)(t1 - t0) * kRows * words; i += kThreads)
    sBits[i] = i / words < u_cta ? bits[t0 * kRows * words + i] : 0u;  // the A tiles are rebuilt per chunk
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  // f32 accumulate (bit 4), f16 A and B (0), K-major both, N = NB, M = 128
  const uint32_t idesc = (1u << 4) | ((uint32_t)(NB >> 3) << 17) | ((uint32_t)(kRows >> 4) << 24);
  const uint32_t sbo = (uint32_t)Kp * 16, lbo = 128;
  uint32_t ph_mma = 0, ph_b = 0, ph_t = 0;
  const int qd = warp & 3, slice = warp >> 2;
  const int row = qd * 32 + lane;  // TMEM lane = tile row
  const uint32_t t_lane = (uint32_t)(qd * 32) << 16;
  const int per_slice = HC / kSlices;  // 4, 8 or 12 units (multiples of 4)

  for (int c = 0; c < L.nch; ++c) {
    if (tid == 0) bulk_load(aB, blob + (size_t)c * L.chunk_bytes, (uint32_t)L.chunk_bytes, bar_b);
    const int ncols = min(HC, M - c * HC);  // units of this chunk
    for (int j = tid; j < 2 * HC; j += kThreads) sSig[j] = sigma[2 * (size_t)c * HC + j];
    for (int64_t tile = t0; tile < t1; ++tile) {
      const int64_t row0 = tile * kRows;
      // the tile's t rows of this chunk (one bulk copy per sample row, under A build and MMA);
      // a copy may complete before the expect_tx arrival (tx-count is signed)
      if (tid < kRows && row0 + tid < U)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         aT + (uint32_t)(tid * tstride * 16)),
                     "l"(t + (row0 + tid) * M + (int64_t)c * HC), "r"((uint32_t)ncols * 16u), "r"(bar_t)
                     : "memory");
      if (tid == 0) {
        const uint32_t rows = (uint32_t)(U - row0 < kRows ? U - row0 : kRows);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_t), "r"(rows * ncols * 16u)
                     : "memory");
      }
      build_a(sA, sBits, (tile - t0) * kRows, u_cta, N, Kp, words, tid);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        if (tile == t0) {
          mbar_wait(bar_b, ph_b);
          ph_b ^= 1;
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int ks = 0; ks < Kp / 16; ++ks) {
          const uint64_t da = make_desc(aA + ks * 256, lbo, sbo);
          const uint64_t dre = make_desc(aB + ks * 256, lbo, sbo);
          const uint64_t dim = make_desc(aB + (uint32_t)NB * Kp * 2 + ks * 256, lbo, sbo);
          mma_f16(tmem, da, dre, idesc, ks > 0);
          mma_f16(tmem + 256, da, dim, idesc, ks > 0);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_mma)
                     : "memory");
      }
      mbar_wait(bar_mma, ph_mma);
      ph_mma ^= 1;
      mbar_wait(bar_t, ph_t);
      ph_t ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // epilogue: this thread's sample row, units slice*per_slice .. +per_slice of the chunk
      const int64_t s = row0 + row;
      double2 acc = make_double2(0.0, 0.0);
      for (int j0 = slice * per_slice; j0 < (slice + 1) * per_slice; j0 += 4) {
        float re[4][kLimbs], im[4][kLimbs];
#pragma unroll
        for (int l = 0; l < kLimbs; ++l) {
          uint32_t a[4], b[4];
          tmem_ld4(tmem + t_lane + (uint32_t)(l * HC + j0), a);
          tmem_ld4(tmem + t_lane + 256u + (uint32_t)(l * HC + j0), b);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            re[j][l] = __uint_as_float(a[j]);
            im[j][l] = __uint_as_float(b[j]);
          }
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int jj = j0 + j;
          if (jj < ncols && s < U) {
            const double yr = sSig[2 * jj] * limb_sum(re[j]);
            const double yi = sSig[2 * jj + 1] * limb_sum(im[j]);
            const double2 ts = sT[row * tstride + jj];
            acc.x = fma(ts.x, yr, fma(-ts.y, yi, acc.x));
            acc.y = fma(ts.x, yi, fma(ts.y, yr, acc.y));
          }
        }
      }
      double2& p = sPart[((tile - t0) * kSlices + slice) * kRows + row];
      p.x += acc.x;
      p.y += acc.y;
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();  // TMEM and the A tile are free; after the last tile, B is too
    }
  }
  // q_s = w_s (sum_k x_sk va_k + sum over slices), fixed order
  if (slice == 0) {
    for (int64_t tile = t0; tile < t1; ++tile) {
      const int64_t s = tile * kRows + row;
      if (s >= U) continue;
      double2 a2 = make_double2(0.0, 0.0);
      for (int wd = 0; wd < words; ++wd) {
        uint32_t m = bits[s * words + wd];
        if (wd == words - 1 && (N & 31)) m &= (1u << (N & 31)) - 1u;
        while (m) {
          const int k = wd * 32 + __ffs(m) - 1;
          m &= m - 1;
          a2.x += sVa[k].x;
          a2.y += sVa[k].y;
        }
      }
#pragma unroll
      for (int sl = 0; sl < kSlices; ++sl) {
        const double2 p = sPart[((tile - t0) * kSlices + sl) * kRows + row];
        a2.x += p.x;
        a2.y += p.y;
      }
      if (w) {
        a2.x *= w[s];
        a2.y *= w[s];
      }
      q[s] = a2;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace ovtc

size_t ov_tc_blob_bytes(int N, int M) {
  ovtc::Layout L;
  return ovtc::make_layout(N, M, &L) ? L.blob_bytes : 0;
}

// 0: launched; 1: shape not supported (caller uses the DMMA kernel); < 0: CUDA error
int ov_tc_launch(const double* t, const uint32_t* bits, int64_t U, int N, int M, const double* v, const double* w,
                 double* q, void* blob, cudaStream_t st, const double* skip) {
  ovtc::Layout L;
  if (U <= 0) return 0;
  if (!ovtc::make_layout(N, M, &L)) return 1;
  static int optin = -1;
  if (optin < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  if ((int)L.smem > optin) return 1;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(ovtc::ov_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ovtc::kSmemMax) !=
        cudaSuccess)
      return -1;
    attr = true;
  }
  const int ncol2 = 2 * L.nch * L.HC;
  ovtc::prepare_kernel<<<(ncol2 + 7) / 8, 256, 0, st>>>(L, (const double2*)v, (uint8_t*)blob, skip);
  int n_sm = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t ntiles = (U + ovtc::kRows - 1) / ovtc::kRows;
  int64_t grid = std::max<int64_t>(n_sm, (ntiles + ovtc::kMaxTiles - 1) / ovtc::kMaxTiles);
  grid = std::min<int64_t>(grid, ntiles);
  const int64_t tpc = (ntiles + grid - 1) / grid;
  grid = (ntiles + tpc - 1) / tpc;  // every CTA owns >= 1 tile
  ovtc::ov_tc_kernel<<<(unsigned)grid, ovtc::kThreads, L.smem, st>>>(L, (const uint8_t*)blob, (const double2*)t,
                                                                     bits, U, (const double2*)v, w, (double2*)q, skip);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;  // the caller's check_launch reports it
}

}  // namespace mpv
