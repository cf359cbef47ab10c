// Parameter snapshot built on the device (ref: rbm.py:91-101 round_parameters,
// rbm.py:161-200 _PreparedRounded): the f64 master parameters are uploaded
// once, rounded RNE to the storage format here, and written into the kernel
// layout of mpv_snapshot (include/mpvmc_b200.h) after the host planner has
// picked the accumulator variant from the four plan numbers computed here.
#pragma once
#include "common.cuh"

namespace mpv {

// RNE rounding of an f64 value to fmt, returned as f64 (overflow -> inf, like
// the reference's quantizer under errstate(over="ignore")).
__device__ __forceinline__ double round_to(int fmt, double x) {
  switch (fmt) {
    case MPV_FMT_F32: return (double)__double2float_rn(x);
    case MPV_FMT_F16: return (double)__half2float(__double2half(x));
    case MPV_FMT_BF16: return (double)__bfloat162float(__double2bfloat16(x));
    default: return x;
  }
}

// Exponent of the lowest set bit of a nonzero finite double (value = odd * 2^e).
__device__ __forceinline__ int lowest_bit_exp(double v) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffull;
  const int e = (int)(bits >> 52);
  const unsigned long long m = bits & 0xfffffffffffffull;
  if (e == 0) return __ffsll((long long)m) - 1 - 1074;
  return __ffsll((long long)(m | (1ull << 52))) - 1 + e - 1075;
}

// plan scratch (8 doubles): [0] quantum, [1] bound_re, [2] bound_im, [3] bound_a,
// [4] (as int) 4096 - min lowest-bit exponent (0: no nonzero value)
__global__ void snapshot_round_kernel(int N, int M, int fmt, const double* __restrict__ src,
                                      double* __restrict__ dst, double* plan) {
  const int64_t n = 2 * ((int64_t)N + M + (int64_t)N * M);  // doubles
  int lo = 0;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const double r = round_to(fmt, src[idx]);
    dst[idx] = r;
    // quantum over a_re, b, w (ref planner: a_im is not an accumulated value)
    const bool a_im = idx < 2 * (int64_t)N && (idx & 1);
    if (!a_im && r != 0.0 && isfinite(r)) lo = max(lo, 4096 - lowest_bit_exp(r));
  }
  for (int off = 16; off > 0; off >>= 1) lo = max(lo, __shfl_xor_sync(kFull, lo, off));
  if ((threadIdx.x & 31) == 0 && lo > 0) atomicMax(reinterpret_cast<int*>(plan + 4), lo);
}

// bound_re/im = max_i |b_i| + sum_k |w_ki| (per component), bound_a = sum_k |a_re_k|.
// Every term is a multiple of the quantum, so the sums are exact below 2^53 q
// (the planner's thresholds are 2^24 q and 2^30 q): order does not matter.
__global__ void snapshot_bound_kernel(int N, int M, const double* __restrict__ r, double* plan) {
  const double2* a = reinterpret_cast<const double2*>(r);
  const double2* b = a + N;
  const double2* w = b + M;  // [N][M]
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M) {
    double sr = fabs(b[i].x), si = fabs(b[i].y);
    for (int k = 0; k < N; ++k) {
      sr += fabs(w[(size_t)k * M + i].x);
      si += fabs(w[(size_t)k * M + i].y);
    }
    atomicMax(reinterpret_cast<unsigned long long*>(plan + 1), (unsigned long long)__double_as_longlong(sr));
    atomicMax(reinterpret_cast<unsigned long long*>(plan + 2), (unsigned long long)__double_as_longlong(si));
  }
  if (i == 0) {
    double s = 0.0;
    for (int k = 0; k < N; ++k) s += fabs(a[k].x);
    plan[3] = s;
    const int lo = *reinterpret_cast<const int*>(plan + 4);
    plan[0] = lo > 0 ? ldexp(1.0, 4096 - lo) : 1.0;
  }
}

__device__ __forceinline__ uint32_t half_bits(int fmt, double x) {
  if (fmt == MPV_FMT_F16) return (uint32_t)__half_as_ushort(__double2half(x));
  return (uint32_t)__bfloat16_as_ushort(__double2bfloat16(x));
}

// One (re, im) entry of the table/bias in the snapshot's layout.
__device__ __forceinline__ void put_entry(const mpv_snapshot& s, void* base, size_t e, double2 z, double split) {
  const bool f64 = s.variant == MPV_ACC_F64;
  if (f64) {
    reinterpret_cast<double2*>(base)[e] = z;
  } else if (s.variant == MPV_ACC_XI) {
    reinterpret_cast<int2*>(base)[e] = make_int2(__double2int_rn(z.x / s.quantum), __double2int_rn(z.y / s.quantum));
  } else if (s.variant == MPV_ACC_X2 && s.mode == MPV_MODE_NATIVE) {
    const double hr = rint(z.x / split) * split, hi = rint(z.y / split) * split;
    const double lr = z.x - hr, li = z.y - hi;
    if (s.fmt == MPV_FMT_F32) {
      reinterpret_cast<float4*>(base)[e] = make_float4((float)hr, (float)hi, (float)lr, (float)li);
    } else {
      reinterpret_cast<uint2*>(base)[e] = make_uint2(half_bits(s.fmt, hr) | (half_bits(s.fmt, hi) << 16),
                                                     half_bits(s.fmt, lr) | (half_bits(s.fmt, li) << 16));
    }
  } else if (s.fmt == MPV_FMT_F32) {
    reinterpret_cast<float2*>(base)[e] = make_float2((float)z.x, (float)z.y);
  } else {
    reinterpret_cast<uint32_t*>(base)[e] = half_bits(s.fmt, z.x) | (half_bits(s.fmt, z.y) << 16);
  }
}

__global__ void snapshot_fill_kernel(const mpv_snapshot s, const double* __restrict__ r, double split, size_t eb) {
  const int N = s.n_visible, M = s.n_hidden, P = s.hidden_pad;
  const double2* a = reinterpret_cast<const double2*>(r);
  const double2* b = a + N;
  const double2* w = b + M;  // [N][M]
  // rank blocks (include/mpvmc_b200.h): unit i of block r = i / GU at element r RB + k GU + i % GU
  const int CS = s.cluster > 1 ? s.cluster : 1, GU = P / CS;
  const int64_t RB = (int64_t)((((size_t)N * GU * eb + 15) & ~(size_t)15) / eb);
  const int64_t n_tab = (int64_t)N * P, n = n_tab + P + N;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    if (idx < n_tab) {
      const int k = (int)(idx / P), i = (int)(idx % P);
      const double2 z = i < M ? w[(size_t)k * M + i] : make_double2(0.0, 0.0);
      put_entry(s, const_cast<void*>(s.table), (size_t)((i / GU) * RB + (int64_t)k * GU + i % GU), z, split);
    } else if (idx < n_tab + P) {
      const int i = (int)(idx - n_tab);
      put_entry(s, const_cast<void*>(s.bias), (size_t)i, i < M ? b[i] : make_double2(0.0, 0.0), split);
    } else {
      const int k = (int)(idx - n_tab - P);
      const double ar = a[k].x;
      void* vis = const_cast<void*>(s.vis);
      if (s.variant == MPV_ACC_F64) {
        reinterpret_cast<double*>(vis)[k] = ar;
      } else if (s.variant == MPV_ACC_XI) {
        reinterpret_cast<int*>(vis)[k] = __double2int_rn(ar / s.quantum);
      } else if (s.variant == MPV_ACC_X2 && s.mode == MPV_MODE_NATIVE) {
        const double h = rint(ar / split) * split;
        reinterpret_cast<float2*>(vis)[k] = make_float2((float)h, (float)(ar - h));
      } else {
        reinterpret_cast<float*>(vis)[k] = (float)ar;
      }
      if (s.vis_im) const_cast<double*>(s.vis_im)[k] = a[k].y;
    }
  }
}

}  // namespace mpv
