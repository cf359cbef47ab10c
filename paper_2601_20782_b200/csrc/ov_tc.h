// q = w (O v) on tcgen05 with exact f16 limbs (ov_tc.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace mpv {
// bytes of the per-call limb matrix (0: shape not supported)
size_t ov_tc_blob_bytes(int N, int M);
// 0: launched; 1: shape not supported (use the DMMA kernel); < 0: CUDA error
int ov_tc_launch(const double* t, const uint32_t* bits, int64_t U, int N, int M, const double* v, const double* w,
                 double* q, void* blob, cudaStream_t st, const double* skip);
}  // namespace mpv
