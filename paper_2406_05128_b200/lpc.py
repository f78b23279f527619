"""Sample-wise all-pole filtering on B200 -- the reference ``tvlp.lpc`` API.

Drop-in for pkg/src/tvlp/lpc.py (reference tvlp 0.1.0): same function names,
argument order, validation messages and return values, with an optional
leading batch axis.  Arrays may be CUDA tensors (results stay on the device)
or numpy arrays (moved to ``cuda:0`` and returned as numpy).  All arithmetic
runs in the sm_100a kernels of libtvlp_b200.so; there is no CPU path.

    s(t) = e(t) - sum_{i=1..M} A[t, i-1] s(t-i)          (lpc.py:1-13)

Shapes: e [T] or [B, T]; A [T, M] or [B, T, M]; a [M] or [B, M]; zi [M] or
[B, M] with zi[i-1] = s(-i).  dtype float32 (production) or float64
(gradient checking); A is cast to e's dtype (lpc.py:113).

Non-finite e/A raise ``ValueError`` like lpc.py:68-69/111-112.  The check is
fused into the forward kernel (a device flag); ``set_validation("eager")``
(default) reads the flag after each forward (one 4-byte device->host read),
``"lazy"`` accumulates it until :func:`check_nonfinite`, ``"off"`` skips it.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _native as N

__all__ = [
    "lp_forward_ti",
    "lp_forward_tv",
    "lp_backward_ti",
    "lp_backward_tv",
    "lp_forward_tv_frames",
    "lp_backward_tv_frames",
    "lp_forward_tv_grouped",
    "lp_backward_tv_grouped",
    "shift_coeffs",
    "lagged_signal_matrix",
    "set_validation",
    "check_nonfinite",
    "set_carry_precision",
    "carry_precision",
]

_VALIDATION = os.environ.get("TVLP_VALIDATION", "auto")
_CARRY = os.environ.get("TVLP_CARRY", "auto")
_pending_flags = {}


def set_validation(mode):
    """Non-finite input checks: 'eager' (the reference's semantics: the call
    raises ValueError, one host sync per forward), 'lazy' (a device flag,
    reported by check_nonfinite()), 'off', or 'auto' (default): eager for
    numpy callers -- the reference API, whose result returns to the host
    anyway -- and lazy for CUDA-tensor callers, so a training step's
    forwards never stall the host."""
    global _VALIDATION
    if mode not in ("eager", "lazy", "off", "auto"):
        raise ValueError(f"unknown validation mode {mode!r}")
    _VALIDATION = mode


def set_carry_precision(p):
    """Precision of the sub-chunk transition matrices ("carries"):
    'auto' (default) -- fp32 chains, then an a-posteriori boundary-defect check
    and a device-side refinement pass for the sequences that fail it;
    'fp64' -- float64 chains (no check needed); 'fp32' -- fp32 chains without
    the check (~1e-3 relative error on near-unit-circle poles)."""
    global _CARRY
    if p not in ("fp64", "fp32", "auto"):
        raise ValueError(f"unknown carry precision {p!r}")
    _CARRY = p


def carry_precision():
    return _CARRY


def _carry_code(p=None):
    return {"fp32": N.CARRY_F32, "fp64": N.CARRY_F64, "auto": N.CARRY_AUTO}[p or _CARRY]


def check_nonfinite(device=None):
    """Lazy mode: returns True if a forward since the last call produced a
    non-finite output (non-finite input or overflow; re-run eagerly to tell)."""
    devs = list(_pending_flags) if device is None else [torch.device(device)]
    seen = False
    for d in devs:
        flag = _pending_flags.get(d)
        if flag is not None and int(flag.item()) != 0:
            flag.zero_()
            seen = True
    return seen


# ---------------------------------------------------------------------------
# argument handling
# ---------------------------------------------------------------------------

class _Conv:
    """numpy <-> CUDA tensor bridge: numpy in, numpy out."""

    def __init__(self, *xs):
        self.numpy = any(isinstance(x, np.ndarray) for x in xs if x is not None)
        dev = None
        for x in xs:
            if isinstance(x, torch.Tensor):
                dev = x.device
                break
        if dev is None:
            dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
                else torch.device("cuda")
        if dev.type != "cuda":
            raise RuntimeError(
                "the B200 LP kernels run on CUDA tensors only (no CPU fallback); "
                f"got a tensor on {dev}")
        self.device = dev

    def t(self, x, dtype=None):
        if x is None:
            return None
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x))
        elif not isinstance(x, torch.Tensor):
            x = torch.as_tensor(np.asarray(x))
        if x.device != self.device:
            x = x.to(self.device)
        if dtype is not None and x.dtype != dtype:
            x = x.to(dtype)
        return x.contiguous()

    def out(self, x):
        return x.cpu().numpy() if self.numpy else x


def _signal(x, name):
    if x.dim() not in (1, 2) or x.shape[-1] < 1 or x.numel() == 0:
        raise ValueError(f"{name} must be a 1-d signal of length >= 1")
    if x.dtype not in (torch.float32, torch.float64):
        x = x.to(torch.float64 if x.dtype == torch.float64 else torch.float32)
    return x


def _zi(zi, M, B, batched, dtype, conv):
    if zi is None:
        return None
    zi = conv.t(zi, dtype)
    want = (B, M) if batched else (M,)
    if tuple(zi.shape) != want:
        if batched and tuple(zi.shape) == (M,):
            zi = zi.expand(B, M)
        else:
            raise ValueError(f"zi must have shape ({M},), got {tuple(zi.shape)}")
    return zi.reshape(B, M).contiguous()


def _mode(numpy_io=True):
    """The effective validation mode of a call (numpy_io: host arrays in/out)."""
    if _VALIDATION == "auto":
        return "eager" if numpy_io else "lazy"
    return _VALIDATION


def _flag(device, mode=None):
    mode = mode or _mode()
    if mode == "off":
        return None
    if mode == "lazy":
        f = _pending_flags.get(device)
        if f is None:
            f = torch.zeros(1, dtype=torch.int32, device=device)
            _pending_flags[device] = f
        return f
    return torch.zeros(1, dtype=torch.int32, device=device)


def _raise_nonfinite(flag, e, A, a_name="A", mode=None):
    """The kernel flags a non-finite OUTPUT: either non-finite input (an error,
    lpc.py:68-69/111-112) or overflow of an unstable filter (legitimate,
    lpc.py:86-87).  Only then are the inputs scanned to tell them apart."""
    if flag is None or (mode or _mode()) != "eager":
        return
    if int(flag.item()) != 0:
        if not bool(torch.isfinite(e).all()):
            raise ValueError("e contains non-finite values")
        if not bool(torch.isfinite(A).all()):
            raise ValueError(f"{a_name} contains non-finite values")


# ---------------------------------------------------------------------------
# forward
# ---------------------------------------------------------------------------

def _forward(ti, e, A, zi, carry_prec=None, return_carry=False):
    conv = _Conv(e, A, zi)
    e = _signal(conv.t(e), "e")
    A = conv.t(A)
    batched = e.dim() == 2
    B = e.shape[0] if batched else 1
    T = e.shape[-1]
    if ti:
        if A.dim() not in (1, 2) or A.shape[-1] < 1:
            raise ValueError("a must be a 1-d coefficient row of order >= 1")
        if A.dim() == 2 and not batched:
            raise ValueError("a must be a 1-d coefficient row of order >= 1")
        M = A.shape[-1]
        A = A.to(e.dtype).expand(B, M).contiguous() if A.dim() == 1 else A.to(e.dtype)
        if batched and A.shape[0] != B:
            raise ValueError(f"a has {A.shape[0]} rows but the batch has {B} signals")
        if _mode(conv.numpy) == "eager" and not bool(torch.isfinite(A).all()):  # lpc.py:92-93
            raise ValueError("a contains non-finite values")
    else:
        if A.dim() != e.dim() + 1:
            raise ValueError("A must be a (T+1, M) coefficient track")
        if A.shape[-2] != T or (batched and A.shape[0] != B):
            raise ValueError(
                f"coefficient track has {A.shape[-2]} rows but the signal has {T} samples")
        M = A.shape[-1]
        A = A.to(e.dtype).contiguous()
    if M > N.load().tvlp_max_order():
        raise ValueError(f"order M={M} exceeds the kernels' maximum {N.load().tvlp_max_order()}")
    zi = _zi(zi, M, B, batched, e.dtype, conv)
    e = e.contiguous()
    dt = N.dtype_code(e.dtype)
    lib = N.load()
    s = torch.empty_like(e)
    ncarry = lib.tvlp_carry_elems(B, T, M)
    carry = torch.empty(ncarry, dtype=e.dtype, device=conv.device)
    op = N.OP_FWD_TI if ti else N.OP_FWD_TV
    ws, nws = N.workspace(lib.tvlp_workspace_bytes(op, dt, B, T, M, 0, 0, 0), conv.device)
    vmode = _mode(conv.numpy)
    flag = _flag(conv.device, vmode)
    fn = lib.tvlp_lp_forward_ti if ti else lib.tvlp_lp_forward_tv
    cp = _carry_code(carry_prec)
    with N.on_device(conv.device):
        N.check(fn(dt, N.ptr(e), N.ptr(A), N.ptr(zi), N.ptr(s), B, T, M, N.ptr(carry), cp,
                   N.ptr(ws), nws, N.ptr(flag), N.stream_ptr(conv.device)))
    _raise_nonfinite(flag, e, A, "a" if ti else "A", vmode)
    out = conv.out(s)
    if return_carry:
        return out, carry
    return out


def lp_forward_tv(e, A, zi=None, *, carry_precision=None):
    """Sample-wise all-pole filter ``s(t) = e(t) - sum_i A[t, i-1] s(t-i)``
    (lpc.py:101-117)."""
    return _forward(False, e, A, zi, carry_precision)


def lp_forward_ti(e, a, zi=None, *, carry_precision=None):
    """Time-invariant all-pole filter (lpc.py:82-98).  Unstable ``a`` is not
    rejected; overflow is a legitimate outcome."""
    return _forward(True, e, a, zi, carry_precision)


# ---------------------------------------------------------------------------
# backward
# ---------------------------------------------------------------------------

def _backward(ti, grad_s, A, s, zi, carry=None, carry_prec=None):
    conv = _Conv(grad_s, A, s, zi)
    grad_s = conv.t(grad_s)
    if grad_s.dtype not in (torch.float32, torch.float64):
        grad_s = grad_s.to(torch.float32)
    dtype = grad_s.dtype
    A = conv.t(A, dtype)
    s = conv.t(s, dtype)
    batched = grad_s.dim() == 2
    B = grad_s.shape[0] if batched else 1
    T = grad_s.shape[-1]
    shared_row = ti and batched and A.dim() == 1  # one row for the whole batch
    if ti:
        M = A.shape[-1]
        if s.shape[-1] != T:
            raise ValueError("grad_s and s must share the same length")
        A = A.expand(B, M).contiguous() if A.dim() == 1 else A
    else:
        if not (T == A.shape[-2] == s.shape[-1]):
            raise ValueError("grad_s, A and s must share the same length")
        M = A.shape[-1]
    zi = _zi(zi, M, B, batched, dtype, conv)
    dt = N.dtype_code(dtype)
    lib = N.load()
    ge = torch.empty_like(grad_s)
    gA = torch.empty((B, M) if ti else A.shape, dtype=dtype, device=conv.device)
    if ti and not batched:
        gA = gA.reshape(M)
    op = N.OP_BWD_TI if ti else N.OP_BWD_TV
    ws, nws = N.workspace(lib.tvlp_workspace_bytes(op, dt, B, T, M, 0, 0, 0), conv.device)
    if carry is not None and carry.numel() != lib.tvlp_carry_elems(B, T, M):
        carry = None
    fn = lib.tvlp_lp_backward_ti if ti else lib.tvlp_lp_backward_tv
    with N.on_device(conv.device):
        N.check(fn(dt, N.ptr(grad_s), N.ptr(A), N.ptr(s), N.ptr(zi), N.ptr(ge), N.ptr(gA), B, T,
                   M, N.ptr(carry), _carry_code(carry_prec), N.ptr(ws), nws,
                   N.stream_ptr(conv.device)))
    if shared_row:
        # a shared [M] row fans out to every sequence: its adjoint is the sum
        # over the batch (lpc.py:176-195 per sequence, summed like a tape fan-out)
        gA = gA.sum(0)
    return conv.out(ge), conv.out(gA)


def lp_backward_tv(grad_s, A, s, zi=None, *, carry=None, carry_precision=None):
    """Adjoints of :func:`lp_forward_tv` given the saved output ``s``
    (lpc.py:152-173): returns ``(grad_e, grad_A)`` with
    ``grad_A[t, i-1] = -grad_e(t) s(t-i)``.  No gradient for ``zi``.
    ``carry`` is the optional tape of the forward (skips recomputing it)."""
    return _backward(False, grad_s, A, s, zi, carry, carry_precision)


def lp_backward_ti(grad_s, a, s, zi=None, *, carry=None, carry_precision=None):
    """Adjoints of :func:`lp_forward_ti` (lpc.py:176-195):
    ``grad_a[i-1] = -sum_t grad_e(t) s(t-i)``."""
    return _backward(True, grad_s, a, s, zi, carry, carry_precision)


# ---------------------------------------------------------------------------
# frame-rate coefficients: upsample_linear fused into the filter
# ---------------------------------------------------------------------------

def _frames_args(e_or_g, frames, hop, conv):
    batched = e_or_g.dim() == 2
    B = e_or_g.shape[0] if batched else 1
    T = e_or_g.shape[-1]
    if frames.dim() != e_or_g.dim() + 1 or (batched and frames.shape[0] != B):
        raise ValueError("frames must be a (F, M) track ((B, F, M) with a batch axis)")
    F, M = frames.shape[-2], frames.shape[-1]
    hop = int(hop)
    if hop < 1 or F != (T - 1) // hop + 1:
        raise ValueError(
            f"got {F} frames but T={T - 1} at hop={hop} requires {(T - 1) // max(hop, 1) + 1}")
    if M > N.load().tvlp_max_order():
        raise ValueError(f"order M={M} exceeds the kernels' maximum {N.load().tvlp_max_order()}")
    return B, T, F, M, hop, batched


def lp_forward_tv_frames(e, frames, hop, zi=None, *, carry_precision=None, return_carry=False):
    """``lp_forward_tv(e, upsample_linear(frames, hop, T - 1))`` without
    materialising the (T, M) track (params.py:120-132 + lpc.py:101-117; the
    synthesiser's H(z) call site synth.py:268-273).  ``frames`` [F, M] or
    [B, F, M] with F = (T - 1) // hop + 1; rows are interpolated inside the
    scan kernels."""
    conv = _Conv(e, frames, zi)
    e = _signal(conv.t(e), "e").contiguous()
    frames = conv.t(frames, e.dtype)
    B, T, F, M, hop, batched = _frames_args(e, frames, hop, conv)
    if _mode(conv.numpy) == "eager" and not bool(torch.isfinite(frames).all()):
        raise ValueError("frames contains non-finite values")
    zi = _zi(zi, M, B, batched, e.dtype, conv)
    dt = N.dtype_code(e.dtype)
    lib = N.load()
    s = torch.empty_like(e)
    carry = torch.empty(lib.tvlp_carry_elems_frames(B, T, M), dtype=e.dtype, device=conv.device)
    ws, nws = N.workspace(lib.tvlp_workspace_bytes(N.OP_FWD_TV_FRAMES, dt, B, T, M, F, 0, hop),
                          conv.device)
    vmode = _mode(conv.numpy)
    flag = _flag(conv.device, vmode)
    with N.on_device(conv.device):
        N.check(lib.tvlp_lp_forward_tv_frames(
            dt, N.ptr(e), N.ptr(frames), N.ptr(zi), N.ptr(s), B, T, M, F, hop, N.ptr(carry),
            _carry_code(carry_precision), N.ptr(ws), nws, N.ptr(flag), N.stream_ptr(conv.device)))
    _raise_nonfinite(flag, e, frames, "frames", vmode)
    out = conv.out(s)
    return (out, carry) if return_carry else out


def lp_backward_tv_frames(grad_s, frames, hop, s, zi=None, *, carry=None, carry_precision=None):
    """(grad_e, grad_frames) of :func:`lp_forward_tv_frames`: the reference's
    VJP chain lpc.py:152-173 -> params.py:135-145, with grad_A never
    written."""
    conv = _Conv(grad_s, frames, s, zi)
    grad_s = conv.t(grad_s)
    if grad_s.dtype not in (torch.float32, torch.float64):
        grad_s = grad_s.to(torch.float32)
    dtype = grad_s.dtype
    frames = conv.t(frames, dtype)
    s = conv.t(s, dtype)
    B, T, F, M, hop, batched = _frames_args(grad_s, frames, hop, conv)
    if s.shape != grad_s.shape:
        raise ValueError("grad_s and s must share the same length")
    zi = _zi(zi, M, B, batched, dtype, conv)
    dt = N.dtype_code(dtype)
    lib = N.load()
    ge = torch.empty_like(grad_s)
    gF = torch.empty(frames.shape, dtype=dtype, device=conv.device)
    if carry is not None and carry.numel() != lib.tvlp_carry_elems_frames(B, T, M):
        carry = None
    ws, nws = N.workspace(lib.tvlp_workspace_bytes(N.OP_BWD_TV_FRAMES, dt, B, T, M, F, 0, hop),
                          conv.device)
    with N.on_device(conv.device):
        N.check(lib.tvlp_lp_backward_tv_frames(
            dt, N.ptr(grad_s), N.ptr(frames), N.ptr(s), N.ptr(zi), N.ptr(ge), N.ptr(gF), B, T, M,
            F, hop, N.ptr(carry), _carry_code(carry_precision), N.ptr(ws), nws,
            N.stream_ptr(conv.device)))
    return conv.out(ge), conv.out(gF)


# ---------------------------------------------------------------------------
# grouped: several independent batches (own buffers, same T and M) per launch
# ---------------------------------------------------------------------------

def _group_args(pairs, what):
    if not 1 <= len(pairs) <= N.MAX_GROUPS:
        raise ValueError(f"1..{N.MAX_GROUPS} groups, got {len(pairs)}")
    conv = _Conv(*[x for p in pairs for x in p])
    return conv


def lp_forward_tv_grouped(groups, *, carry_precision=None, return_carry=False):
    """``[lp_forward_tv(e, A, zi) for (e, A[, zi]) in groups]`` in ONE launch
    sequence, each group on its own buffers: the HpN synthesiser's H(z) on the
    glottal source and C(z) on the noise (synth.py:264-273 records them as two
    lp_tv tape ops).  Every group is [B_g, T] / [B_g, T, M] with the same T
    and M; returns the list of outputs (and the shared carry tape)."""
    conv = _group_args(groups, "groups")
    es, As, zis = [], [], []
    for gspec in groups:
        e, A = gspec[0], gspec[1]
        zi = gspec[2] if len(gspec) > 2 else None
        e = _signal(conv.t(e), "e").contiguous()
        if e.dim() == 1:
            raise ValueError("grouped calls take batched signals [B, T]")
        A = conv.t(A, e.dtype)
        if A.dim() != 3 or A.shape[:2] != e.shape:
            raise ValueError("A must be a (B, T, M) coefficient track per group")
        es.append(e)
        As.append(A.contiguous())
        zis.append(_zi(zi, A.shape[-1], e.shape[0], True, e.dtype, conv))
    T, M, dtype = es[0].shape[-1], As[0].shape[-1], es[0].dtype
    if any(e.shape[-1] != T or A.shape[-1] != M or e.dtype != dtype for e, A in zip(es, As)):
        raise ValueError("grouped batches must share T, M and dtype")
    lib = N.load()
    dt = N.dtype_code(dtype)
    Bs = (ctypes.c_int64 * len(es))(*[e.shape[0] for e in es])
    outs = [torch.empty_like(e) for e in es]
    carry = torch.empty(lib.tvlp_carry_elems(sum(Bs), T, M), dtype=dtype, device=conv.device)
    ws, nws = N.workspace(lib.tvlp_workspace_bytes_grouped(N.OP_FWD_TV, dt, len(es), Bs, T, M),
                          conv.device)
    arr = (N.FwdGroup * len(es))(*[N.FwdGroup(e.data_ptr(), A.data_ptr(),
                                              0 if z is None else z.data_ptr(), s.data_ptr(),
                                              e.shape[0])
                                   for e, A, z, s in zip(es, As, zis, outs)])
    vmode = _mode(conv.numpy)
    flag = _flag(conv.device, vmode)
    with N.on_device(conv.device):
        N.check(lib.tvlp_lp_forward_tv_grouped(dt, len(es), arr, T, M, N.ptr(carry),
                                               _carry_code(carry_precision), N.ptr(ws), nws,
                                               N.ptr(flag), N.stream_ptr(conv.device)))
    if flag is not None and vmode == "eager" and int(flag.item()) != 0:
        for e, A in zip(es, As):
            _raise_nonfinite(flag, e, A, "A", vmode)
    res = [conv.out(s) for s in outs]
    return (res, carry) if return_carry else res


def lp_backward_tv_grouped(groups, *, carry=None, carry_precision=None):
    """Adjoints of :func:`lp_forward_tv_grouped`: ``groups`` holds
    (grad_s, A, s[, zi]) per group; returns [(grad_e, grad_A), ...]."""
    conv = _group_args(groups, "groups")
    gs_, As, ss, zis = [], [], [], []
    for gspec in groups:
        g = conv.t(gspec[0]).contiguous()
        if g.dtype not in (torch.float32, torch.float64):
            g = g.to(torch.float32)
        A = conv.t(gspec[1], g.dtype).contiguous()
        s = conv.t(gspec[2], g.dtype).contiguous()
        zi = gspec[3] if len(gspec) > 3 else None
        if g.dim() != 2 or A.dim() != 3 or A.shape[:2] != g.shape or s.shape != g.shape:
            raise ValueError("grad_s, A and s must share the same length")
        gs_.append(g)
        As.append(A)
        ss.append(s)
        zis.append(_zi(zi, A.shape[-1], g.shape[0], True, g.dtype, conv))
    T, M, dtype = gs_[0].shape[-1], As[0].shape[-1], gs_[0].dtype
    if any(g.shape[-1] != T or A.shape[-1] != M or g.dtype != dtype for g, A in zip(gs_, As)):
        raise ValueError("grouped batches must share T, M and dtype")
    lib = N.load()
    dt = N.dtype_code(dtype)
    Bs = (ctypes.c_int64 * len(gs_))(*[g.shape[0] for g in gs_])
    if carry is not None and carry.numel() != lib.tvlp_carry_elems(sum(Bs), T, M):
        carry = None
    ges = [torch.empty_like(g) for g in gs_]
    gAs = [torch.empty_like(A) for A in As]
    ws, nws = N.workspace(lib.tvlp_workspace_bytes_grouped(N.OP_BWD_TV, dt, len(gs_), Bs, T, M),
                          conv.device)
    arr = (N.BwdGroup * len(gs_))(*[N.BwdGroup(g.data_ptr(), A.data_ptr(), s.data_ptr(),
                                               0 if z is None else z.data_ptr(), ge.data_ptr(),
                                               gA.data_ptr(), g.shape[0])
                                    for g, A, s, z, ge, gA in zip(gs_, As, ss, zis, ges, gAs)])
    with N.on_device(conv.device):
        N.check(lib.tvlp_lp_backward_tv_grouped(dt, len(gs_), arr, T, M, N.ptr(carry),
                                                _carry_code(carry_precision), N.ptr(ws), nws,
                                                N.stream_ptr(conv.device)))
    return [(conv.out(ge), conv.out(gA)) for ge, gA in zip(ges, gAs)]


# ---------------------------------------------------------------------------
# helpers of the reference API
# ---------------------------------------------------------------------------

def shift_coeffs(A):
    """``A_hat[t, i-1] = A[t+i, i-1]``, zero past the end (lpc.py:120-135)."""
    conv = _Conv(A)
    A = conv.t(A)
    if A.dim() not in (2, 3):
        raise ValueError("A must be a (T+1, M) coefficient track")
    if A.dtype not in (torch.float32, torch.float64):
        A = A.to(torch.float64)
    B = A.shape[0] if A.dim() == 3 else 1
    T, M = A.shape[-2], A.shape[-1]
    out = torch.empty_like(A)
    with N.on_device(conv.device):
        N.check(N.load().tvlp_shift_coeffs(N.dtype_code(A.dtype), N.ptr(A), N.ptr(out), B, T, M,
                                           N.stream_ptr(conv.device)))
    return conv.out(out)


def lagged_signal_matrix(s, M, zi=None):
    """``L[t, i-1] = s(t-i)`` with ``s(-i)`` from ``zi`` (lpc.py:138-149)."""
    conv = _Conv(s, zi)
    s = conv.t(s)
    if s.dtype not in (torch.float32, torch.float64):
        s = s.to(torch.float64)
    batched = s.dim() == 2
    B = s.shape[0] if batched else 1
    T = s.shape[-1]
    zi = None if zi is None else conv.t(zi, s.dtype).expand(B, M).contiguous()
    out = torch.empty(s.shape + (M,), dtype=s.dtype, device=conv.device)
    with N.on_device(conv.device):
        N.check(N.load().tvlp_lagged_signal_matrix(N.dtype_code(s.dtype), N.ptr(s), N.ptr(zi),
                                                   N.ptr(out), B, T, M,
                                                   N.stream_ptr(conv.device)))
    return conv.out(out)
