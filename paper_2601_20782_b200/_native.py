"""ctypes binding of the sm_100a library ``lib/libmpvmc_b200.so`` (C ABI in
include/mpvmc_b200.h).  There is no CPU fallback: if the library or a CUDA
device is missing, every device entry point raises NativeLibraryError.

torch provides device memory and the stream; pointers and the stream handle
are passed as plain integers.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import EvaluationFailureError, NativeLibraryError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libmpvmc_b200.so")

MPV_OK, MPV_ERR_ARGS, MPV_ERR_CUDA, MPV_ERR_NONFINITE = 0, 1, 2, 3
FMT_F64, FMT_F32, FMT_F16, FMT_BF16 = 0, 1, 2, 3
MODE_NATIVE, MODE_PER_OPERATION, MODE_STORAGE_ONLY = 0, 1, 2
ACC_X1, ACC_X2, ACC_F64, ACC_XI = 0, 1, 2, 3
PROPOSAL_FLIP, PROPOSAL_EXCHANGE = 0, 1
HAM_TFIM, HAM_HEISENBERG = 0, 1

_vp = ctypes.c_void_p
_i32, _i64, _u64, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double


class Snapshot(ctypes.Structure):
    _fields_ = [
        ("n_visible", _i32), ("n_hidden", _i32), ("hidden_pad", _i32),
        ("fmt", _i32), ("mode", _i32), ("variant", _i32),
        ("lanes_per_chain", _i32), ("units_per_lane", _i32), ("cluster", _i32),
        ("table", _vp), ("bias", _vp), ("vis", _vp), ("vis_im", _vp), ("quantum", _f64),
        ("noise_key", _u64), ("noise_sigma", _f64),
    ]


class Chains(ctypes.Structure):
    _fields_ = [
        ("n_chains", _i64), ("chain_offset", _i64), ("n_sites", _i32), ("words", _i32),
        ("bits", _vp), ("log_probs", _vp), ("accepted", _vp), ("status", _vp),
        ("scratch", _vp), ("scratch_bytes", ctypes.c_size_t),
    ]


class CG(ctypes.Structure):
    _fields_ = [
        ("n_visible", _i32), ("n_hidden", _i32), ("n_samples", _i64),
        ("t", _vp), ("bits", _vp), ("w", _vp), ("obar", _vp), ("lam", _f64),
        ("g", _vp), ("r", _vp), ("p", _vp), ("ap", _vp), ("y", _vp), ("ysum", _vp), ("q", _vp),
        ("partials", _vp), ("scalars", _vp), ("scratch", _vp), ("scratch_bytes", ctypes.c_size_t),
    ]


_SIGNATURES = {
    "mpv_stream_uniforms": (ctypes.c_int, [_u64, _i64, _i64, _i64, _i64, _vp, _vp]),
    "mpv_snapshot_bytes": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]),
    "mpv_plan_cluster": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "mpv_plan_cluster_ex": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                                           ctypes.POINTER(_i32)]),
    "mpv_snapshot_round": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp]),
    "mpv_snapshot_fill": (ctypes.c_int, [ctypes.POINTER(Snapshot), _vp, ctypes.c_double, _vp]),
    "mpv_table_sweep": (ctypes.c_int, [_vp, ctypes.POINTER(Chains), _u64, ctypes.c_int, _i64, _i64, _i64, _i64, _vp,
                                       _i64, _i64, _i64, _i64, _vp]),
    "mpv_logderiv_scratch_bytes": (ctypes.c_size_t, [_i64, ctypes.c_int, ctypes.c_int]),
    "mpv_logderiv_ov": (ctypes.c_int, [_vp, _vp, _i64, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp, _vp]),
    "mpv_logderiv_ohu": (ctypes.c_int, [_vp, _vp, _i64, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mpv_logderiv_tanh": (ctypes.c_int, [_vp, _vp, _i64, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]),
    "mpv_logderiv_dense": (ctypes.c_int, [_vp, _vp, _i64, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]),
    "mpv_sr_smatrix": (ctypes.c_int, [_vp, _vp, _i64, ctypes.c_int, _vp, _vp]),
    "mpv_cg_partials_len": (ctypes.c_size_t, []),
    "mpv_cg_init": (ctypes.c_int, [ctypes.POINTER(CG), _vp, _f64, _i64, _vp]),
    "mpv_cg_apply": (ctypes.c_int, [ctypes.POINTER(CG), _vp, _vp, _vp, _vp]),
    "mpv_cg_apply_finish": (ctypes.c_int, [ctypes.POINTER(CG), _vp, _vp, _vp, _vp, _vp]),
    "mpv_cg_step": (ctypes.c_int, [ctypes.POINTER(CG), _vp]),
    "mpv_cg_run": (ctypes.c_int, [ctypes.POINTER(CG), ctypes.c_int, _vp]),
    "mpv_chain_stats": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp]),
    "mpv_moments": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp]),
    "mpv_minsr_gram": (ctypes.c_int, [_vp, _vp, _i64, _i64, _vp, _vp, _i64, ctypes.c_int, ctypes.c_int, _vp, _vp,
                                      _f64, _f64, ctypes.c_int, _vp, _vp]),
    "mpv_chains_init": (ctypes.c_int, [ctypes.POINTER(Chains), _u64, ctypes.c_int, ctypes.c_int, _vp]),
    "mpv_mh_sweep": (ctypes.c_int, [ctypes.POINTER(Snapshot), ctypes.POINTER(Chains), _u64, ctypes.c_int,
                                    _i64, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _vp]),
    "mpv_snapshot_forward": (ctypes.c_int, [ctypes.POINTER(Snapshot), _vp, _i64, _vp, _vp, _vp, _vp, _vp,
                                            ctypes.c_size_t, _vp]),
    "mpv_sweep_scratch_bytes": (ctypes.c_size_t, [ctypes.POINTER(Snapshot), _i64]),
    "mpv_rounded_scratch_bytes": (ctypes.c_size_t, [_i64, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "mpv_rounded_log_prob": (ctypes.c_int, [_vp, _i64, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp, _vp,
                                            ctypes.c_int, _vp, _vp, _vp]),
    "mpv_energy_tables_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "mpv_energy_prepare": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, ctypes.c_int, _vp,
                                          ctypes.c_int, _vp, _vp]),
    "mpv_local_energies": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, ctypes.c_int, _vp,
                                          ctypes.c_int, _f64, _f64, _vp, _vp, _i64, _vp, _vp, _vp]),
    "mpv_local_energies_ex": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, ctypes.c_int, _vp,
                                             ctypes.c_int, _f64, _f64, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp]),
    "mpv_forward_tc_weights_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int]),
    "mpv_forward_tc_prepare": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]),
    "mpv_forward_tc": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp, _i64, _vp, _vp, _vp,
                                      ctypes.c_int, _vp]),
    "mpv_rescnn_blob_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int]),
    "mpv_rescnn_mh_scratch_bytes": (ctypes.c_size_t, [_i64]),
    "mpv_rescnn_forward": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp, _i64, _vp, _vp, _vp]),
    "mpv_rescnn_forward_f64": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _i64, _vp, _vp]),
    "mpv_rescnn_mh_sweep": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, ctypes.POINTER(Chains), _u64,
                                           ctypes.c_int, _i64, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _vp]),
    "mpv_unpack_bits": (ctypes.c_int, [_vp, _i64, ctypes.c_int, _vp, _vp]),
    "mpv_pack_bits": (ctypes.c_int, [_vp, _i64, ctypes.c_int, _vp, _vp]),
    "mpv_sum_i64": (ctypes.c_int, [_vp, _i64, _vp, _vp]),
    "mpv_plan_layout": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_i32),
                                       ctypes.POINTER(_i32)]),
    "mpv_last_error": (ctypes.c_char_p, []),
    "mpv_version": (ctypes.c_char_p, []),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None
_lock = threading.Lock()


def load():
    """Load the library (no CUDA context is created by loading)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device: the B200 path has no CPU fallback")


def check(rc: int, what: str):
    if rc == MPV_OK:
        return
    msg = load().mpv_last_error().decode(errors="replace")
    if rc == MPV_ERR_NONFINITE:
        raise EvaluationFailureError(f"{what}: non-finite value ({msg})")
    if rc == MPV_ERR_ARGS:
        raise ValueError(f"{what}: {msg}")
    raise NativeLibraryError(f"{what}: {msg}")


def call(name: str, *args):
    rc = getattr(load(), name)(*args)
    check(rc, name)
    return rc


def stream_handle(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def plan_cluster(n_visible: int, n_hidden: int, fmt: int, mode: int, variant: int, min_lanes: int = 1):
    """(cluster, G, U) of the fused sweep's layout (mpv_plan_cluster_ex)."""
    c, g, u = _i32(), _i32(), _i32()
    call("mpv_plan_cluster_ex", n_visible, n_hidden, fmt, mode, variant, min_lanes, ctypes.byref(c), ctypes.byref(g),
         ctypes.byref(u))
    return c.value, g.value, u.value


def plan_layout(n_visible: int, n_hidden: int, fmt: int = FMT_F16, variant: int = ACC_X1):
    g, u = _i32(), _i32()
    call("mpv_plan_layout", n_visible, n_hidden, fmt, variant, ctypes.byref(g), ctypes.byref(u))
    return g.value, u.value
