"""ctypes binding of the C ABI in include/rl_cddt.h.

The library is the only compute path: if librl_cddt.so is missing the import
fails loudly (there is no CPU fallback). Build it with
``python -m paper_1705_01167_b200.build`` or ``__graft_entry__.build()``.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

_PKG = Path(__file__).resolve().parent
# RL_CDDT_LIB selects an alternative in-tree build (kernel variants for A/B timing)
LIB_PATH = Path(os.environ.get("RL_CDDT_LIB", str(_PKG / "librl_cddt.so")))

RL_OK, RL_EINVAL, RL_ELOGIC, RL_ERANGE, RL_ECUDA, RL_ENOMEM, RL_EDEGENERATE, RL_EPARSE = range(8)


class ParseError(ValueError):
    """rangelib::ParseError (proj/include/rangelib/grid.hpp:81-90)."""


class LogicError(RuntimeError):
    """std::logic_error (edits after prune, proj/src/cddt.cpp:333)."""


class CudaError(RuntimeError):
    pass


class rl_cddt_info_t(C.Structure):
    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32), ("theta_disc", C.c_int32),
        ("slice_count", C.c_int32), ("pruned", C.c_int32), ("device", C.c_int32),
        ("max_range", C.c_double), ("resolution", C.c_double), ("rows", C.c_uint64),
        ("zero_points", C.c_uint64), ("memory_bytes", C.c_uint64), ("device_bytes", C.c_uint64),
        ("init_seconds", C.c_double),
    ]


class rl_beam_params_t(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("w_hit", "w_short", "w_max", "w_rand", "sigma_hit", "lambda_short", "z_max")]


class rl_motion_noise_t(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("trans_per_trans", "trans_per_rot", "rot_per_rot", "rot_per_trans")]


_P = C.c_void_p
_SIG = {
    "rl_last_error": (C.c_char_p, []),
    "rl_cddt_create": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_double,
                                 C.c_int32, C.c_int32, C.POINTER(_P)]),
    "rl_cddt_destroy": (C.c_int, [_P]),
    "rl_cddt_prune": (C.c_int, [_P]),
    "rl_cddt_info": (C.c_int, [_P, C.POINTER(rl_cddt_info_t)]),
    "rl_cddt_cast": (C.c_int, [_P, C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]),
    "rl_cddt_cast_pair": (C.c_int, [_P, C.c_double, C.c_double, C.c_double,
                                    C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "rl_cddt_cast_batch": (C.c_int, [_P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "rl_cddt_cast_batch_f64": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "rl_cddt_directional_batch": (C.c_int, [_P, _P, _P, _P, _P, C.c_size_t, _P]),
    "rl_cddt_cast_batch_host": (C.c_int, [_P, _P, _P, _P, _P, C.c_size_t]),
    "rl_cddt_cast_queries_host": (C.c_int, [_P, _P, _P, C.c_size_t]),
    "rl_cddt_set_occupancy": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32]),
    "rl_cddt_set_occupancy_batch": (C.c_int, [_P, _P, _P, C.c_size_t]),
    "rl_cddt_export": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "rl_cddt_serialize": (C.c_int, [_P, _P, C.c_size_t, C.POINTER(C.c_size_t)]),
    "rl_cddt_deserialize": (C.c_int, [_P, C.c_size_t, C.c_int32, C.POINTER(_P)]),
    "rl_cddt_sync": (C.c_int, [_P]),
    "rl_diag_gather": (C.c_int, [_P, C.c_size_t, C.c_size_t, _P, C.POINTER(C.c_double),
                                 C.POINTER(C.c_uint64)]),
    "rl_debug_checks": (C.c_int, [C.c_int32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]),
    "rl_beam_likelihood": (C.c_double, [C.POINTER(rl_beam_params_t), C.c_double, C.c_double]),
    "rl_beam_table": (C.c_int, [C.POINTER(rl_beam_params_t), C.c_int32, C.c_double, _P]),
    "rl_sensor_update": (C.c_int, [_P, _P, _P, _P, C.c_size_t, _P, C.c_int32, C.c_double,
                                   C.POINTER(rl_beam_params_t), _P, C.c_int32, C.c_double, _P,
                                   _P, _P]),
    "rl_exact_cast_batch": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "rl_lut_build": (C.c_int, [_P, C.c_int32, _P, _P]),
    "rl_simulate_scans": (C.c_int, [_P, _P, _P, _P, C.c_size_t, C.c_int32, C.c_double, C.c_double,
                                    C.c_double, C.c_uint64, C.c_uint64, _P, _P, _P, _P]),
    "rl_sensor_logw": (C.c_int, [_P, _P, _P, _P, C.c_size_t, _P, C.c_int32, C.c_double,
                                 C.POINTER(rl_beam_params_t), _P, C.c_int32, C.c_double, _P, _P]),
    "rl_motion_update": (C.c_int, [_P, _P, _P, C.c_size_t, C.c_uint64, C.c_double, C.c_double,
                                   C.c_double, C.POINTER(rl_motion_noise_t), C.c_uint64,
                                   C.c_uint64, _P]),
    "rl_pf_max": (C.c_int, [_P, C.c_size_t, _P, _P]),
    "rl_pf_weights": (C.c_int, [_P, _P, _P, _P, _P, C.c_size_t, _P, _P, _P]),
    "rl_pf_normalize": (C.c_int, [_P, C.c_size_t, _P, C.c_uint64, _P, _P]),
    "rl_resample_low_variance": (C.c_int, [_P, _P, _P, _P, C.c_size_t, C.c_size_t, C.c_size_t,
                                           _P, _P, _P, _P, C.c_uint64, C.c_uint64, _P]),
    "rl_mcl_step": (C.c_int, [_P, _P, _P, _P, _P, C.c_size_t, C.c_double, C.c_double, C.c_double,
                              _P, C.c_int32, C.c_double, C.POINTER(rl_motion_noise_t),
                              C.POINTER(rl_beam_params_t), _P, C.c_int32, C.c_double,
                              C.c_uint64, C.c_uint64, _P, _P]),
    "rl_mcl_step_async": (C.c_int, [_P, _P, _P, _P, _P, C.c_size_t, C.c_double, C.c_double,
                                    C.c_double, _P, C.c_int32, C.c_double,
                                    C.POINTER(rl_motion_noise_t), C.POINTER(rl_beam_params_t), _P,
                                    C.c_int32, C.c_double, C.c_uint64, C.c_uint64, _P, _P]),
    "rl_sensor_update_async": (C.c_int, [_P, _P, _P, _P, C.c_size_t, _P, C.c_int32, C.c_double,
                                         C.POINTER(rl_beam_params_t), _P, C.c_int32, C.c_double,
                                         _P, _P, _P, _P]),
    "rl_pf_estimate": (C.c_int, [_P, _P, C.c_uint64, _P, _P]),
    "rl_resample_gathered": (C.c_int, [_P, C.c_size_t, C.c_int32, C.c_size_t, C.c_size_t, _P, _P,
                                       _P, _P, C.c_uint64, C.c_uint64, _P]),
    "rl_pf_shard_sensor": (C.c_int, [_P, _P, _P, _P, C.c_size_t, C.c_uint64, C.c_double,
                                     C.c_double, C.c_double, C.POINTER(rl_motion_noise_t),
                                     C.c_uint64, C.c_uint64, _P, C.c_int32, C.c_double,
                                     C.POINTER(rl_beam_params_t), _P, C.c_int32, C.c_double, _P,
                                     _P, _P]),
}

_lib = None


def lib() -> C.CDLL:
    """Load librl_cddt.so (once). Raises ImportError when it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -m paper_1705_01167_b200.build); there is no CPU fallback")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIG.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib


# cudaStreamLegacy: the legacy default stream named explicitly. A NULL stream
# means "the handle's own stream, synchronous" in the C ABI, so torch's
# default stream (pointer 0) must be passed as this handle to keep the ops
# ordered with torch's work.
CUDA_STREAM_LEGACY = 1


def torch_stream(device) -> C.c_void_p:
    """The C-ABI stream argument for torch's current stream on `device`."""
    import torch
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream or CUDA_STREAM_LEGACY)


def check(status: int) -> int:
    """Map a status code to the reference's exception types."""
    if status in (RL_OK, RL_EDEGENERATE):
        return status
    msg = lib().rl_last_error().decode(errors="replace")
    if status == RL_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if status == RL_ELOGIC:
        raise LogicError(msg)
    if status == RL_ERANGE:
        raise IndexError(msg)  # std::out_of_range
    if status == RL_EPARSE:
        raise ParseError(msg)
    if status == RL_ENOMEM:
        raise MemoryError(msg)
    raise CudaError(msg or f"status {status}")
