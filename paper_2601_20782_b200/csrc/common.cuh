// Shared device helpers of the sm_100a hot path: splitmix64 streams, packed
// configuration bits, reduced-format packing and MUFU wrappers.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mpvmc_b200.h"

namespace mpv {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr unsigned kFull = 0xffffffffu;

// splitmix64 finalizer (ref: rng.py:21-27).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// (z >> 12) * 2^-52 + 2^-53 (ref: rng.py:50-53), exactly, without the slow
// 64-bit integer->double conversion: 1 + m 2^-52 is built from bits, the
// subtraction of 1 and the addition of 2^-53 are exact.
__device__ __forceinline__ double uniform_from_bits(uint64_t z) {
  const double one_m = __longlong_as_double((long long)(0x3FF0000000000000ull | (z >> 12)));
  return __dadd_rn(__dadd_rn(one_m, -1.0), 0x1p-53);
}

// Stream state of chain c (ref: rng.py:71-73): s0 = mix64(key ^ (c+1) G).
__device__ __forceinline__ uint64_t stream_state(uint64_t key, uint64_t chain) {
  return mix64(key ^ ((chain + 1) * kGolden));
}
// Draw t (0-based, counted from stream creation) of a stream (ref: rng.py:75-77).
__device__ __forceinline__ double stream_draw(uint64_t s0, uint64_t t) {
  return uniform_from_bits(mix64(s0 + (t + 1) * kGolden));
}

// floor(u * n) for 0 < u < 1 computed as the reference does,
// (u_select * n).astype(int64) (ref: sampler.py:117, 120): a RN product and a
// truncation; the truncation uses add.rz with 2^52 (exact for r < 2^52).
__device__ __forceinline__ int64_t floor_scaled(double u, double n) {
  const double r = __dmul_rn(u, n);
  const double t = __dadd_rz(r, 4503599627370496.0);  // 2^52
  return (int64_t)(__double_as_longlong(t) & 0x000FFFFFFFFFFFFFll);
}

// Lexicographic (i<j) pair of index idx (ref: sampler.py:42-45 pair_table).
__device__ __forceinline__ void pair_of(int64_t idx, int n, int& i, int& j) {
  // row i starts at S(i) = i*(2n-i-1)/2; invert with a double estimate then fix.
  const double nn = 2.0 * n - 1.0;
  int r = (int)floor((nn - sqrt(nn * nn - 8.0 * (double)idx)) * 0.5);
  if (r < 0) r = 0;
  if (r > n - 2) r = n - 2;
  while (r > 0 && (int64_t)r * (2 * n - r - 1) / 2 > idx) --r;
  while (r < n - 2 && (int64_t)(r + 1) * (2 * n - r - 2) / 2 <= idx) ++r;
  i = r;
  j = (int)(idx - (int64_t)r * (2 * n - r - 1) / 2) + r + 1;
}

// ---- MUFU wrappers (ftz variants: one SASS MUFU each, no range fix-ups) ----
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float cos_approx(float x) {
  float y;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- reduced formats ----
// Packed pair (re in low half, im in high half) of f16 / bf16.
template <int FMT> struct Half;
template <> struct Half<MPV_FMT_F16> {
  static constexpr uint16_t kOne = 0x3C00, kMinusOne = 0xBC00;
  // RN of two f32 to a packed pair (cvt.rn.f16x2.f32: one F2FP).
  __device__ static __forceinline__ uint32_t pack(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
  }
  // acc + a*b with f16 a, b and f32 acc (sm_100 mixed-precision FMA, exact products).
  __device__ static __forceinline__ float fma_lo(uint32_t a, uint16_t b, float acc) {
    float d;
    asm("{.reg .b16 l, h;\n mov.b32 {l, h}, %1;\n fma.rn.f32.f16 %0, l, %2, %3;}"
        : "=f"(d) : "r"(a), "h"(b), "f"(acc));
    return d;
  }
  __device__ static __forceinline__ float fma_hi(uint32_t a, uint16_t b, float acc) {
    float d;
    asm("{.reg .b16 l, h;\n mov.b32 {l, h}, %1;\n fma.rn.f32.f16 %0, h, %2, %3;}"
        : "=f"(d) : "r"(a), "h"(b), "f"(acc));
    return d;
  }
  __device__ static __forceinline__ float lo(uint32_t a) { return fma_lo(a, kOne, -0.0f); }
  __device__ static __forceinline__ float hi(uint32_t a) { return fma_hi(a, kOne, -0.0f); }
  // 2 * (high half), exact
  __device__ static __forceinline__ float hi2(uint32_t a) { return fma_hi(a, 0x4000, -0.0f); }
  // acc + half (f32 accumulate of an f16 value, one mixed-precision add)
  __device__ static __forceinline__ float acc_lo(uint32_t a, float acc) {
    float d;
    asm("{.reg .b16 l, h;\n mov.b32 {l, h}, %1;\n add.rn.f32.f16 %0, l, %2;}" : "=f"(d) : "r"(a), "f"(acc));
    return d;
  }
  __device__ static __forceinline__ float acc_hi(uint32_t a, float acc) {
    float d;
    asm("{.reg .b16 l, h;\n mov.b32 {l, h}, %1;\n add.rn.f32.f16 %0, h, %2;}" : "=f"(d) : "r"(a), "f"(acc));
    return d;
  }
  // per-op emulation: RN(a + b) in f16 (exact-sum rounding == ref _quantize(a+b))
  __device__ static __forceinline__ uint16_t add(uint16_t a, uint16_t b) {
    return __half_as_ushort(__hadd(__ushort_as_half(a), __ushort_as_half(b)));
  }
  __device__ static __forceinline__ double to_f64(uint16_t a) {
    return (double)__half2float(__ushort_as_half(a));
  }
  __device__ static __forceinline__ uint16_t from_f64(double v) {
    return __half_as_ushort(__double2half(v));
  }
};
template <> struct Half<MPV_FMT_BF16> {
  static constexpr uint16_t kOne = 0x3F80, kMinusOne = 0xBF80;
  __device__ static __forceinline__ uint32_t pack(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
  }
  __device__ static __forceinline__ float fma_lo(uint32_t a, uint16_t b, float acc) {
    float d;
    asm("{.reg .b16 l, h;\n mov.b32 {l, h}, %1;\n fma.rn.f32.bf16 %0, l, %2, %3;}"
        : "=f"(d) : "r"(a), "h"(b), "f"(acc));
    return d;
  }
  __device__ static __forceinline__ float fma_hi(uint32_t a, uint16_t b, float acc) {
    float d;
    asm("{.reg .b16 l, h;\n mov.b32 {l, h}, %1;\n fma.rn.f32.bf16 %0, h, %2, %3;}"
        : "=f"(d) : "r"(a), "h"(b), "f"(acc));
    return d;
  }
  // bf16 -> f32 is a shift: exact and on the ALU pipe.
  __device__ static __forceinline__ float lo(uint32_t a) { return __uint_as_float(a << 16); }
  __device__ static __forceinline__ float hi(uint32_t a) { return __uint_as_float(a & 0xFFFF0000u); }
  __device__ static __forceinline__ float hi2(uint32_t a) { return fma_hi(a, 0x4000, -0.0f); }
  __device__ static __forceinline__ float acc_lo(uint32_t a, float acc) {
    float d;
    asm("{.reg .b16 l, h;\n mov.b32 {l, h}, %1;\n add.rn.f32.bf16 %0, l, %2;}" : "=f"(d) : "r"(a), "f"(acc));
    return d;
  }
  __device__ static __forceinline__ float acc_hi(uint32_t a, float acc) {
    float d;
    asm("{.reg .b16 l, h;\n mov.b32 {l, h}, %1;\n add.rn.f32.bf16 %0, h, %2;}" : "=f"(d) : "r"(a), "f"(acc));
    return d;
  }
  __device__ static __forceinline__ uint16_t add(uint16_t a, uint16_t b) {
    return __bfloat16_as_ushort(__hadd(__ushort_as_bfloat16(a), __ushort_as_bfloat16(b)));
  }
  __device__ static __forceinline__ double to_f64(uint16_t a) {
    return (double)__uint_as_float(((uint32_t)a) << 16);
  }
  __device__ static __forceinline__ uint16_t from_f64(double v) {
    return __bfloat16_as_ushort(__double2bfloat16(v));
  }
};

// Warp-segment (width G) xor-butterfly sum.  Commutativity of IEEE addition
// makes every lane of the segment end with the identical value.
// Frozen Gaussian log-density noise of a configuration code (ref: rng.py:56-60
// counter_uniform, rng.py:86-96 gaussian_field): sigma * ndtri(u), u =
// uniform_from_bits(mix64((code + 1) * G ^ key)).
__device__ __forceinline__ double noise_zeta(uint64_t key, uint64_t code, double sigma) {
  const double u = uniform_from_bits(mix64(((code + 1ull) * 0x9E3779B97F4A7C15ull) ^ key));
  return sigma * normcdfinv(u);
}

template <typename T>
__device__ __forceinline__ T segment_sum(T v, int G) {
  for (int off = G >> 1; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off, G);
  return v;
}

}  // namespace mpv
