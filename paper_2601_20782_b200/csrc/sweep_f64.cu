// Instantiations of the fused sweep for MPV_FMT_F64 (generated layout; see sweep.cuh).
#include "sweep.cuh"
namespace mpv {
void* sweep_kernel_ptr_f64(int variant, int U, int prop, int smem) {
  if (variant == MPV_ACC_F64 && U == 4 && prop == MPV_PROPOSAL_FLIP && smem == 1) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 4, MPV_PROPOSAL_FLIP, true>;
  if (variant == MPV_ACC_F64 && U == 4 && prop == MPV_PROPOSAL_FLIP && smem == 0) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 4, MPV_PROPOSAL_FLIP, false>;
  if (variant == MPV_ACC_F64 && U == 4 && prop == MPV_PROPOSAL_EXCHANGE && smem == 1) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 4, MPV_PROPOSAL_EXCHANGE, true>;
  if (variant == MPV_ACC_F64 && U == 4 && prop == MPV_PROPOSAL_EXCHANGE && smem == 0) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 4, MPV_PROPOSAL_EXCHANGE, false>;
  if (variant == MPV_ACC_F64 && U == 8 && prop == MPV_PROPOSAL_FLIP && smem == 1) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 8, MPV_PROPOSAL_FLIP, true>;
  if (variant == MPV_ACC_F64 && U == 8 && prop == MPV_PROPOSAL_FLIP && smem == 0) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 8, MPV_PROPOSAL_FLIP, false>;
  if (variant == MPV_ACC_F64 && U == 8 && prop == MPV_PROPOSAL_EXCHANGE && smem == 1) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 8, MPV_PROPOSAL_EXCHANGE, true>;
  if (variant == MPV_ACC_F64 && U == 8 && prop == MPV_PROPOSAL_EXCHANGE && smem == 0) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 8, MPV_PROPOSAL_EXCHANGE, false>;
  if (variant == MPV_ACC_F64 && U == 10 && prop == MPV_PROPOSAL_FLIP && smem == 1) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 10, MPV_PROPOSAL_FLIP, true>;
  if (variant == MPV_ACC_F64 && U == 10 && prop == MPV_PROPOSAL_FLIP && smem == 0) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 10, MPV_PROPOSAL_FLIP, false>;
  if (variant == MPV_ACC_F64 && U == 10 && prop == MPV_PROPOSAL_EXCHANGE && smem == 1) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 10, MPV_PROPOSAL_EXCHANGE, true>;
  if (variant == MPV_ACC_F64 && U == 10 && prop == MPV_PROPOSAL_EXCHANGE && smem == 0) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 10, MPV_PROPOSAL_EXCHANGE, false>;
  if (variant == MPV_ACC_F64 && U == 13 && prop == MPV_PROPOSAL_FLIP && smem == 1) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 13, MPV_PROPOSAL_FLIP, true>;
  if (variant == MPV_ACC_F64 && U == 13 && prop == MPV_PROPOSAL_FLIP && smem == 0) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 13, MPV_PROPOSAL_FLIP, false>;
  if (variant == MPV_ACC_F64 && U == 13 && prop == MPV_PROPOSAL_EXCHANGE && smem == 1) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 13, MPV_PROPOSAL_EXCHANGE, true>;
  if (variant == MPV_ACC_F64 && U == 13 && prop == MPV_PROPOSAL_EXCHANGE && smem == 0) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 13, MPV_PROPOSAL_EXCHANGE, false>;
  if (variant == MPV_ACC_F64 && U == 16 && prop == MPV_PROPOSAL_FLIP && smem == 1) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 16, MPV_PROPOSAL_FLIP, true>;
  if (variant == MPV_ACC_F64 && U == 16 && prop == MPV_PROPOSAL_FLIP && smem == 0) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 16, MPV_PROPOSAL_FLIP, false>;
  if (variant == MPV_ACC_F64 && U == 16 && prop == MPV_PROPOSAL_EXCHANGE && smem == 1) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 16, MPV_PROPOSAL_EXCHANGE, true>;
  if (variant == MPV_ACC_F64 && U == 16 && prop == MPV_PROPOSAL_EXCHANGE && smem == 0) return (void*)&sweep_kernel<MPV_FMT_F64, MPV_ACC_F64, 16, MPV_PROPOSAL_EXCHANGE, false>;
  return nullptr;
}
}  // namespace mpv
