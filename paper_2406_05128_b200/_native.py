"""ctypes binding of the C ABI in include/tvlp.h (libtvlp_b200.so).

The product path has exactly one implementation: the sm_100a kernels behind
this library.  There is no CPU fallback; if the library or a CUDA device is
missing, every call raises.
"""
from __future__ import annotations

import contextlib
import ctypes
import functools
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libtvlp_b200.so")

F32, F64 = 0, 1
CARRY_F64, CARRY_F32, CARRY_AUTO = 0, 1, 2
CARRY_REUSE = 16  # OR-ed: the carry tape is already filled for the same (e, A)
(OP_FWD_TV, OP_BWD_TV, OP_FWD_TI, OP_BWD_TI, OP_FW_FWD, OP_FW_BWD, OP_FWD_TV_FRAMES,
 OP_BWD_TV_FRAMES, OP_BWD_TV_EX, OP_SEGMENT_TRANSITION) = range(10)

_lib = None


class FwdGroup(ctypes.Structure):
    """tvlp_lp_fwd_group (include/tvlp.h)."""
    _fields_ = [("e", ctypes.c_void_p), ("A", ctypes.c_void_p), ("zi", ctypes.c_void_p),
                ("s", ctypes.c_void_p), ("B", ctypes.c_int64)]


class BwdGroup(ctypes.Structure):
    """tvlp_lp_bwd_group (include/tvlp.h)."""
    _fields_ = [("grad_s", ctypes.c_void_p), ("A", ctypes.c_void_p), ("s", ctypes.c_void_p),
                ("zi", ctypes.c_void_p), ("grad_e", ctypes.c_void_p), ("grad_A", ctypes.c_void_p),
                ("B", ctypes.c_int64)]


MAX_GROUPS = 4

# (name, restype, argtypes)
_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_SZ = ctypes.c_size_t
_D = ctypes.c_double
_SIGS = [
    ("tvlp_abi_version", ctypes.c_int, []),
    ("tvlp_status_string", ctypes.c_char_p, [ctypes.c_int]),
    ("tvlp_last_cuda_error", ctypes.c_int, []),
    ("tvlp_max_order", _I32, []),
    ("tvlp_carry_elems", _I64, [_I64, _I64, _I32]),
    ("tvlp_carry_elems_frames", _I64, [_I64, _I64, _I32]),
    ("tvlp_subchunk_len", _I64, [_I64, _I64, _I32]),
    ("tvlp_workspace_bytes", _SZ, [_I32, _I32, _I64, _I64, _I32, _I64, _I32, _I32]),
    ("tvlp_framewise_nframes", _I64, [_I64, _I64, _I32, _I32]),
    ("tvlp_lp_forward_tv", ctypes.c_int,
     [_I32, _P, _P, _P, _P, _I64, _I64, _I32, _P, _I32, _P, _SZ, _P, _P]),
    ("tvlp_lp_backward_tv", ctypes.c_int,
     [_I32, _P, _P, _P, _P, _P, _P, _I64, _I64, _I32, _P, _I32, _P, _SZ, _P]),
    ("tvlp_lp_forward_tv_frames", ctypes.c_int,
     [_I32, _P, _P, _P, _P, _I64, _I64, _I32, _I64, _I32, _P, _I32, _P, _SZ, _P, _P]),
    ("tvlp_lp_backward_tv_frames", ctypes.c_int,
     [_I32, _P, _P, _P, _P, _P, _P, _I64, _I64, _I32, _I64, _I32, _P, _I32, _P, _SZ, _P]),
    ("tvlp_reflection_to_lpc", ctypes.c_int, [_I32, _P, _P, _I64, _I32, _P, _P]),
    ("tvlp_reflection_to_lpc_vjp", ctypes.c_int, [_I32, _P, _P, _P, _I64, _I32, _P]),
    ("tvlp_lp_backward_tv_ex", ctypes.c_int,
     [_I32, _P, _P, _P, _P, _P, _P, _I64, _I64, _I32, _P, _I32, _P, _P, _P, _SZ, _P]),
    ("tvlp_segment_transition", ctypes.c_int, [_I32, _P, _I64, _I64, _I32, _P, _P, _SZ, _P]),
    ("tvlp_lp_forward_tv_grouped", ctypes.c_int,
     [_I32, _I32, ctypes.POINTER(FwdGroup), _I64, _I32, _P, _I32, _P, _SZ, _P, _P]),
    ("tvlp_lp_backward_tv_grouped", ctypes.c_int,
     [_I32, _I32, ctypes.POINTER(BwdGroup), _I64, _I32, _P, _I32, _P, _SZ, _P]),
    ("tvlp_workspace_bytes_grouped", _SZ, [_I32, _I32, _I32, ctypes.POINTER(_I64), _I64, _I32]),
    ("tvlp_lp_forward_ti", ctypes.c_int,
     [_I32, _P, _P, _P, _P, _I64, _I64, _I32, _P, _I32, _P, _SZ, _P, _P]),
    ("tvlp_lp_backward_ti", ctypes.c_int,
     [_I32, _P, _P, _P, _P, _P, _P, _I64, _I64, _I32, _P, _I32, _P, _SZ, _P]),
    ("tvlp_shift_coeffs", ctypes.c_int, [_I32, _P, _P, _I64, _I64, _I32, _P]),
    ("tvlp_lagged_signal_matrix", ctypes.c_int, [_I32, _P, _P, _P, _I64, _I64, _I32, _P]),
    ("tvlp_framewise_forward", ctypes.c_int,
     [_I32, _P, _P, _P, _D, _P, _P, _I64, _I64, _I64, _I32, _I32, _I32, _P, _SZ, _P]),
    ("tvlp_framewise_backward", ctypes.c_int,
     [_I32, _P, _P, _P, _D, _P, _P, _P, _I64, _I64, _I64, _I32, _I32, _I32, _P, _SZ, _P]),
    ("tvlp_framewise_aux_elems", _I64, [_I64, _I64, _I64, _I32, _I32, _I32]),
    ("tvlp_framewise_forward_ex", ctypes.c_int,
     [_I32, _P, _P, _P, _D, _P, _P, _P, _I64, _I64, _I64, _I32, _I32, _I32, _P, _SZ, _P]),
    ("tvlp_framewise_backward_ex", ctypes.c_int,
     [_I32, _P, _P, _P, _D, _P, _P, _P, _P, _I64, _I64, _I64, _I32, _I32, _I32, _P, _SZ, _P]),
    ("tvlp_wavetable_osc", ctypes.c_int,
     [_P, _P, _P, _I32, _I32, _P, _I32, _P, _I64, _I64, _I64, _I32, _I32, _D, _P]),
    ("tvlp_wavetable_osc_vjp", ctypes.c_int,
     [_P, _P, _P, _I32, _I32, _P, _I32, _P, _P, _P, _I64, _I64, _I64, _I32, _I32, _D, _P]),
    ("tvlp_global_fir", ctypes.c_int, [_P, _P, _P, _I64, _I64, _I32, _P]),
    ("tvlp_global_fir_workspace", _SZ, [_I64, _I64, _I32]),
    ("tvlp_global_fir_vjp", ctypes.c_int, [_P, _P, _P, _P, _P, _P, _SZ, _I64, _I64, _I32, _P]),
    ("tvlp_noise_frames", ctypes.c_int, [_P, _P, _P, _I64, _I64, _I64, _I32, _I32, _I64, _I32, _P]),
    ("tvlp_frame_ola", ctypes.c_int,
     [_P, _P, _I64, _I64, _I64, _I32, _I32, _I32, _I64, _I32, ctypes.c_float, _I32, _P]),
    ("tvlp_spectra_mul", ctypes.c_int, [_P, _P, _P, _P, _I64, _I64, _I64, _I32, _P]),
    ("tvlp_spectra_mul_vjp", ctypes.c_int, [_P, _P, _P, _P, _I64, _I64, _I64, _I32, _P]),
    ("tvlp_source_pair", ctypes.c_int, [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I32, _I64, _P]),
    ("tvlp_source_pair_vjp", ctypes.c_int,
     [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I32, _I64, _P]),
    ("tvlp_stft_nframes", _I64, [_I64, _I32, _I32]),
    ("tvlp_stft_frames", ctypes.c_int, [_P, _P, _P, _I64, _I64, _I32, _I32, _P]),
    ("tvlp_stft_frames_vjp", ctypes.c_int,
     [_P, _P, _P, _I64, _I64, _I32, _I32, ctypes.c_float, _P, _I64, ctypes.c_float, _P]),
    ("tvlp_mss_terms_workspace", _SZ, [_I64, _I64]),
    ("tvlp_mss_terms", ctypes.c_int, [_P, _P, _I64, _I64, ctypes.c_float, _P, _P, _P, _SZ, _P]),
    ("tvlp_mss_terms_vjp", ctypes.c_int, [_P, _P, _P, _P, _P, _I64, _I64, ctypes.c_float, _P]),
    ("tvlp_launch_count", _I64, []),
    ("tvlp_refined_sequences", _I64, []),
    ("tvlp_profile_enable", None, [_I32]),
    ("tvlp_chain_trace", None, [_P, _SZ]),
    ("tvlp_profile_dump", _I32, [ctypes.c_char_p, _I32]),
]
EXPORTS = [name for name, _, _ in _SIGS]


class TVLPError(RuntimeError):
    """A C-ABI call failed (launch error, bad workspace, unsupported order)."""


def load(path=None):
    """Load libtvlp_b200.so and declare its signatures (no GPU needed).

    $TVLP_LIB selects a tuning variant built with ``build --define ... --out``."""
    global _lib
    if _lib is None:
        path = path or os.environ.get("TVLP_LIB") or LIB_PATH
        if not os.path.exists(path):
            raise TVLPError(
                f"{path} is missing: build the B200 kernels with "
                "`python -m paper_2406_05128_b200.build` (there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, res, args in _SIGS:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        # size queries are pure functions of their arguments (the plan is
        # deterministic): memoised, so a training step's calls skip the
        # ctypes round trips
        for name in _PURE:
            setattr(lib, name, functools.lru_cache(maxsize=256)(getattr(lib, name)))
        _lib = lib
    return _lib


_PURE = ("tvlp_workspace_bytes", "tvlp_carry_elems", "tvlp_max_order",
         "tvlp_framewise_aux_elems", "tvlp_framewise_nframes", "tvlp_subchunk_len",
         "tvlp_global_fir_workspace", "tvlp_mss_terms_workspace", "tvlp_stft_nframes")


def on_device(device):
    """``torch.cuda.device(device)`` only when it is not already current."""
    if device.index is None or device.index == torch.cuda.current_device():
        return contextlib.nullcontext()
    return torch.cuda.device(device)


def profile_dump():
    """{kernel family: (launches, total_ms)} since the last dump."""
    buf = ctypes.create_string_buffer(1 << 16)
    load().tvlp_profile_dump(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, n, ms = line.split()
        out[name] = (int(n), float(ms))
    return out


def check(rc):
    if rc != 0:
        msg = load().tvlp_status_string(rc).decode()
        raise TVLPError(f"tvlp C ABI call failed ({rc}): {msg}")


def dtype_code(dtype):
    if dtype == torch.float32:
        return F32
    if dtype == torch.float64:
        return F64
    raise TypeError(f"B200 LP kernels support float32 and float64, got {dtype}")


def stream_ptr(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def workspace(nbytes, device):
    if nbytes <= 0:
        return None, 0
    return torch.empty(int(nbytes), dtype=torch.uint8, device=device), int(nbytes)
