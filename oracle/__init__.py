"""CPU oracle for the B200 LP kernels -- TEST INFRASTRUCTURE ONLY.

This package is the parity checker and the CPU baseline ("port") for the
product in ``paper_2406_05128_b200``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It never runs on the product path.

It restates the reference ``tvlp`` 0.1.0 LP path (``pkg/src/tvlp/lpc.py`` and
the frame-wise part of ``pkg/src/tvlp/params.py``) in plain C
(``oracle/tvlp_oracle.c``, built by ``oracle/Makefile`` into
``oracle/_ref/liboracle.so``) with the reference's exact arithmetic order.
Parity is PINNED: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by the reference itself
(``tests/golden/make_golden.py``), bit-exact in float64 and float32.

The numpy-level wrappers below mirror the reference signatures (1-D signals,
``(T, M)`` tracks) and validation messages; ``*_batch`` helpers loop over a
leading batch axis (the reference has no batch axis).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_ref", "liboracle.so")
_lib = None

__all__ = [
    "build",
    "lp_forward_tv",
    "lp_forward_ti",
    "lp_backward_tv",
    "lp_backward_ti",
    "shift_coeffs",
    "lagged_signal_matrix",
    "raised_cosine_window",
    "framewise_forward",
    "framewise_backward",
    "gradcheck_error",
    "batch_fwd_bwd",
]


def build(force=False):
    """Compile the C oracle (``make -C oracle``)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "tvlp_oracle.c"))
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        I = ctypes.c_int
        D = ctypes.c_double
        for sfx in ("f32", "f64"):
            getattr(_lib, f"oracle_lp_forward_tv_{sfx}").argtypes = [P, P, P, P, I64, I]
            getattr(_lib, f"oracle_lp_forward_ti_{sfx}").argtypes = [P, P, P, P, I64, I]
            getattr(_lib, f"oracle_shift_coeffs_{sfx}").argtypes = [P, P, I64, I]
            getattr(_lib, f"oracle_lagged_signal_matrix_{sfx}").argtypes = [P, P, P, I64, I]
            getattr(_lib, f"oracle_lp_backward_tv_{sfx}").argtypes = [P, P, P, P, P, P, I64, I]
            getattr(_lib, f"oracle_lp_backward_ti_{sfx}").argtypes = [P, P, P, P, P, P, I64, I]
            getattr(_lib, f"oracle_framewise_forward_{sfx}").argtypes = [
                P, P, P, D, P, P, I64, I64, I, I64, I64]
            getattr(_lib, f"oracle_framewise_backward_{sfx}").argtypes = [
                P, P, P, D, P, P, P, I64, I64, I, I64, I64]
        _lib.oracle_batch_fwd_bwd_f32.argtypes = [
            I, I, I64, I64, I64, I64, I64, I64, P, P, P, P, D, P, P, P, P]
        _lib.oracle_batch_fwd_bwd_f32.restype = I
    return _lib


def _sfx(dtype):
    if dtype == np.float32:
        return "f32"
    if dtype == np.float64:
        return "f64"
    raise TypeError(f"oracle supports float32/float64, got {dtype}")


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# lpc.py restatement (validation mirrors lpc.py:64-117, 152-195)
# ---------------------------------------------------------------------------

def _check_signal(x, name):
    x = np.ascontiguousarray(x)
    if x.ndim != 1 or x.shape[0] < 1:
        raise ValueError(f"{name} must be a 1-d signal of length >= 1")
    if not np.all(np.isfinite(x)):
        raise ValueError(f"{name} contains non-finite values")
    return x


def _zi(zi, M, dtype):
    if zi is None:
        return None
    zi = np.ascontiguousarray(zi, dtype=dtype)
    if zi.shape != (M,):
        raise ValueError(f"zi must have shape ({M},), got {zi.shape}")
    return zi


def lp_forward_tv(e, A, zi=None):
    """lpc.py:101-117."""
    e = _check_signal(e, "e")
    A = np.ascontiguousarray(A)
    if A.ndim != 2:
        raise ValueError("A must be a (T+1, M) coefficient track")
    if A.shape[0] != e.shape[0]:
        raise ValueError(
            f"coefficient track has {A.shape[0]} rows but the signal has {e.shape[0]} samples")
    if not np.all(np.isfinite(A)):
        raise ValueError("A contains non-finite values")
    A = np.ascontiguousarray(A.astype(e.dtype, copy=False))
    zi = _zi(zi, A.shape[1], e.dtype)
    out = np.empty_like(e)
    getattr(_load(), f"oracle_lp_forward_tv_{_sfx(e.dtype)}")(
        _ptr(e), _ptr(A), _ptr(zi), _ptr(out), e.shape[0], A.shape[1])
    return out


def lp_forward_ti(e, a, zi=None):
    """lpc.py:82-98."""
    e = _check_signal(e, "e")
    a = np.ascontiguousarray(a)
    if a.ndim != 1 or a.shape[0] < 1:
        raise ValueError("a must be a 1-d coefficient row of order >= 1")
    if not np.all(np.isfinite(a)):
        raise ValueError("a contains non-finite values")
    a = np.ascontiguousarray(a.astype(e.dtype, copy=False))
    zi = _zi(zi, a.shape[0], e.dtype)
    out = np.empty_like(e)
    getattr(_load(), f"oracle_lp_forward_ti_{_sfx(e.dtype)}")(
        _ptr(e), _ptr(a), _ptr(zi), _ptr(out), e.shape[0], a.shape[0])
    return out


def shift_coeffs(A):
    """lpc.py:120-135."""
    A = np.ascontiguousarray(A)
    if A.ndim != 2:
        raise ValueError("A must be a (T+1, M) coefficient track")
    out = np.empty_like(A)
    getattr(_load(), f"oracle_shift_coeffs_{_sfx(A.dtype)}")(
        _ptr(A), _ptr(out), A.shape[0], A.shape[1])
    return out


def lagged_signal_matrix(s, M, zi=None):
    """lpc.py:138-149."""
    s = np.ascontiguousarray(s)
    out = np.empty((s.shape[0], M), dtype=s.dtype)
    zi = None if zi is None else np.ascontiguousarray(zi, dtype=s.dtype)
    getattr(_load(), f"oracle_lagged_signal_matrix_{_sfx(s.dtype)}")(
        _ptr(s), _ptr(zi), _ptr(out), s.shape[0], M)
    return out


def lp_backward_tv(grad_s, A, s, zi=None):
    """lpc.py:152-173."""
    grad_s = np.ascontiguousarray(grad_s)
    A = np.ascontiguousarray(A)
    s = np.ascontiguousarray(s)
    if not (grad_s.shape[0] == A.shape[0] == s.shape[0]):
        raise ValueError("grad_s, A and s must share the same length")
    dt = grad_s.dtype
    A = np.ascontiguousarray(A.astype(dt, copy=False))
    s = np.ascontiguousarray(s.astype(dt, copy=False))
    zi = None if zi is None else np.ascontiguousarray(zi, dtype=dt)
    ge = np.empty_like(grad_s)
    gA = np.empty_like(A)
    getattr(_load(), f"oracle_lp_backward_tv_{_sfx(dt)}")(
        _ptr(grad_s), _ptr(A), _ptr(s), _ptr(zi), _ptr(ge), _ptr(gA), A.shape[0], A.shape[1])
    return ge, gA


def lp_backward_ti(grad_s, a, s, zi=None):
    """lpc.py:176-195."""
    grad_s = np.ascontiguousarray(grad_s)
    s = np.ascontiguousarray(s)
    if grad_s.shape[0] != s.shape[0]:
        raise ValueError("grad_s and s must share the same length")
    dt = grad_s.dtype
    a = np.ascontiguousarray(np.asarray(a).astype(dt, copy=False))
    s = np.ascontiguousarray(s.astype(dt, copy=False))
    zi = None if zi is None else np.ascontiguousarray(zi, dtype=dt)
    ge = np.empty_like(grad_s)
    ga = np.empty_like(a)
    getattr(_load(), f"oracle_lp_backward_ti_{_sfx(dt)}")(
        _ptr(grad_s), _ptr(a), _ptr(s), _ptr(zi), _ptr(ge), _ptr(ga), s.shape[0], a.shape[0])
    return ge, ga


# ---------------------------------------------------------------------------
# params.py frame-wise restatement (params.py:152-273)
# ---------------------------------------------------------------------------

def raised_cosine_window(n):
    """params.py:152-154 (float64)."""
    return 0.5 - 0.5 * np.cos(2.0 * np.pi * np.arange(n) / n)


def _frame_args(frame_size, hop, window):
    if window is None:
        window = raised_cosine_window(frame_size)
    window = np.asarray(window, dtype=np.float64)
    cola = float(window.sum() / hop)  # params.py:199-201
    return window, cola


def n_frames_total(T1, F, frame_size, hop):
    n_lead = (frame_size - 1) // hop
    count = 0
    for f in range(-n_lead, F):
        start = f * hop
        if min(start + frame_size, T1) > max(start, 0):
            count += 1
    return count


def framewise_forward(e, frames, hop, frame_size=None, window=None):
    """params.py:220-239.  Returns (out, seg_outputs[n_frames, frame_size])."""
    e = np.ascontiguousarray(e)
    frame_size = 4 * hop if frame_size is None else frame_size
    window, cola = _frame_args(frame_size, hop, window)
    dt = e.dtype
    frames = np.ascontiguousarray(np.asarray(frames).astype(dt, copy=False))
    T1 = e.shape[0]
    F, M = frames.shape
    if F != (T1 - 1) // hop + 1:
        raise ValueError(f"got {F} coefficient frames but length {T1} at hop {hop} "
                         f"requires {(T1 - 1) // hop + 1}")
    w = np.ascontiguousarray(window.astype(dt))
    out = np.empty(T1, dtype=dt)
    seg = np.empty((n_frames_total(T1, F, frame_size, hop), frame_size), dtype=dt)
    getattr(_load(), f"oracle_framewise_forward_{_sfx(dt)}")(
        _ptr(e), _ptr(frames), _ptr(w), cola, _ptr(out), _ptr(seg), T1, F, M, frame_size, hop)
    return out, seg


def framewise_backward(grad_out, frames, seg_outputs, hop, frame_size=None, window=None):
    """params.py:259-273.  Returns (grad_e, grad_frames)."""
    grad_out = np.ascontiguousarray(grad_out)
    frame_size = 4 * hop if frame_size is None else frame_size
    window, cola = _frame_args(frame_size, hop, window)
    dt = grad_out.dtype
    frames = np.ascontiguousarray(np.asarray(frames).astype(dt, copy=False))
    seg_outputs = np.ascontiguousarray(np.asarray(seg_outputs).astype(dt, copy=False))
    T1 = grad_out.shape[0]
    F, M = frames.shape
    w = np.ascontiguousarray(window.astype(dt))
    ge = np.empty(T1, dtype=dt)
    gf = np.empty((F, M), dtype=dt)
    getattr(_load(), f"oracle_framewise_backward_{_sfx(dt)}")(
        _ptr(grad_out), _ptr(frames), _ptr(w), cola, _ptr(seg_outputs), _ptr(ge), _ptr(gf),
        T1, F, M, frame_size, hop)
    return ge, gf


# ---------------------------------------------------------------------------
# oracle.py:228-234
# ---------------------------------------------------------------------------

# ---------------------------------------------------------------------------
# upsample_linear (params.py:102-145): restated for the frame-rate LP path
# ---------------------------------------------------------------------------

def expected_frame_count(T, hop):
    """params.py:102-104."""
    return T // hop + 1


def _upsample_weights(F, hop, T):
    """params.py:107-117: frame f anchored at sample f*hop, held after the last."""
    if F != expected_frame_count(T, hop):
        raise ValueError(
            f"got {F} frames but T={T} at hop={hop} requires {expected_frame_count(T, hop)}")
    t = np.arange(T + 1)
    f0 = t // hop
    w = (t - f0 * hop) / float(hop)
    f1 = np.minimum(f0 + 1, F - 1)
    w[f0 == F - 1] = 0.0
    return f0, f1, w


def upsample_linear(frames, hop, T):
    """params.py:120-132: (F, D) frames -> (T+1, D) samples."""
    frames = np.asarray(frames)
    f0, f1, w = _upsample_weights(frames.shape[0], hop, T)
    if frames.ndim == 1:
        return (1.0 - w) * frames[f0] + w * frames[f1]
    wcol = w[:, None]
    return (1.0 - wcol) * frames[f0] + wcol * frames[f1]


def upsample_linear_vjp(grad_out, F, hop, T):
    """params.py:135-145 (np.add.at: f0 contributions, then f1, in t order)."""
    f0, f1, w = _upsample_weights(F, hop, T)
    grad_frames = np.zeros((F,) + grad_out.shape[1:], dtype=grad_out.dtype)
    wcol = w if grad_out.ndim == 1 else w[:, None]
    np.add.at(grad_frames, f0, (1.0 - wcol) * grad_out)
    np.add.at(grad_frames, f1, wcol * grad_out)
    return grad_frames


def lp_tv_frames_fwd_bwd(e, frames, hop, grad_s, zi=None):
    """The composed reference path the fused frame-rate kernels replace:
    s = lp_forward_tv(e, upsample_linear(frames)); (grad_e, grad_frames) by
    the VJP chain (lp_backward_tv, then the upsample VJP)."""
    T = e.shape[-1] - 1
    A = upsample_linear(frames, hop, T)
    s = lp_forward_tv(e, A, zi)
    ge, gA = lp_backward_tv(grad_s, A, s, zi)
    return s, ge, upsample_linear_vjp(gA, frames.shape[0], hop, T)


# ---------------------------------------------------------------------------
# step-up recursion (params.py:43-84), restated for the frame-rate path
# ---------------------------------------------------------------------------

def step_up(k):
    """params.py:43-53: rows plus the per-stage intermediates."""
    k = np.asarray(k, dtype=np.float64)
    M = k.shape[-1]
    stages = []
    a = k[..., :1].copy()
    for m in range(2, M + 1):
        stages.append(a)
        km = k[..., m - 1: m]
        a = np.concatenate([a + km * a[..., ::-1], km], axis=-1)
    return a, stages


def reflection_to_lpc(k):
    """params.py:56-71."""
    k = np.asarray(k, dtype=np.float64)
    if k.shape[-1] < 1:
        raise ValueError("reflection rows need order >= 1")
    if np.any(np.abs(k) >= 1.0):
        raise ValueError("reflection coefficients must satisfy |k| < 1")
    return step_up(k)[0]


def reflection_to_lpc_vjp(grad_a, k):
    """params.py:74-84."""
    k = np.asarray(k, dtype=np.float64)
    _, stages = step_up(k)
    g = np.array(grad_a, dtype=np.float64, copy=True)
    grad_k = np.zeros_like(k)
    M = k.shape[-1]
    for m in range(M, 1, -1):
        prev = stages[m - 2]
        g_new = g[..., : m - 1]
        grad_k[..., m - 1] = g[..., m - 1] + np.sum(g_new * prev[..., ::-1], axis=-1)
        g = g_new + k[..., m - 1: m] * g_new[..., ::-1]
    grad_k[..., 0] = g[..., 0]
    return grad_k


def gradcheck_error(analytic, numeric):
    """Max elementwise deviation normalised by the largest entry (oracle.py:228-234)."""
    analytic = np.asarray(analytic, dtype=np.float64)
    numeric = np.asarray(numeric, dtype=np.float64)
    scale = max(np.max(np.abs(analytic), initial=0.0),
                np.max(np.abs(numeric), initial=0.0), 1e-8)
    return float(np.max(np.abs(analytic - numeric), initial=0.0) / scale)


# ---------------------------------------------------------------------------
# batched helpers (loop over the leading batch axis)
# ---------------------------------------------------------------------------

def tv_fwd_bwd_batch(e, A, grad_s, zi=None):
    """Per-item lp_forward_tv + lp_backward_tv over a leading batch axis."""
    B = e.shape[0]
    s = np.empty_like(e)
    ge = np.empty_like(e)
    gA = np.empty_like(A)
    for b in range(B):
        z = None if zi is None else zi[b]
        s[b] = lp_forward_tv(e[b], A[b], z)
        ge[b], gA[b] = lp_backward_tv(grad_s[b], A[b], s[b], z)
    return s, ge, gA


def batch_fwd_bwd(kind, e, A, grad_s, nthreads, hop=240, frame_size=None):
    """Threaded float32 fwd+bwd over independent items (the CPU baseline leg).

    kind "tv": A is [B, T, M]; kind "framewise": A is the frame track [B, F, M].
    Returns the outputs so callers can also use it as a checker.
    """
    lib = _load()
    e = np.ascontiguousarray(e, dtype=np.float32)
    A = np.ascontiguousarray(A, dtype=np.float32)
    grad_s = np.ascontiguousarray(grad_s, dtype=np.float32)
    B, T1 = e.shape
    M = A.shape[-1]
    s = np.empty_like(e)
    ge = np.empty_like(e)
    gA = np.empty_like(A)
    if kind == "tv":
        lib.oracle_batch_fwd_bwd_f32(0, nthreads, B, T1, M, 0, 0, 0, _ptr(e), _ptr(A),
                                     _ptr(grad_s), None, 0.0, _ptr(s), _ptr(ge), _ptr(gA),
                                     None)
        return s, ge, gA
    frame_size = 4 * hop if frame_size is None else frame_size
    window, cola = _frame_args(frame_size, hop, None)
    w = np.ascontiguousarray(window.astype(np.float32))
    F = A.shape[1]
    nfr = n_frames_total(T1, F, frame_size, hop)
    seg = np.empty((B, nfr, frame_size), dtype=np.float32)
    lib.oracle_batch_fwd_bwd_f32(1, nthreads, B, T1, M, F, frame_size, hop, _ptr(e), _ptr(A),
                                 _ptr(grad_s), _ptr(w), cola, _ptr(s), _ptr(ge), _ptr(gA),
                                 _ptr(seg))
    return s, ge, gA
