"""Frame-wise time-invariant LP with overlap-add -- the reference
``tvlp.params`` frame-wise API (pkg/src/tvlp/params.py:102-273) on B200.

``FramePlan`` reproduces the framing contract of params.py:157-217 (it is
host-side metadata whose semantics -- lead-in frames, frame order, COLA
constant -- the drop-in must keep; see its docstring);
``framewise_lp`` runs the per-frame recursions, the overlap-add and (through
:class:`paper_2406_05128_b200.autograd.LPFramewise`) the VJP in the sm_100a
kernels of libtvlp_b200.so.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .lpc import _Conv

__all__ = [
    "expected_frame_count",
    "raised_cosine_window",
    "FramePlan",
    "framewise_lp",
    "framewise_forward",
    "framewise_backward",
    "squash_reflection",
    "reflection_to_lpc",
    "reflection_to_lpc_vjp",
]

SQUASH_LIMIT = 0.999  # params.py:31


def squash_reflection(raw):
    """params.py:34-36 (elementwise; torch or numpy)."""
    if isinstance(raw, torch.Tensor):
        return SQUASH_LIMIT * torch.tanh(raw)
    return SQUASH_LIMIT * np.tanh(np.asarray(raw))


def reflection_to_lpc(k):
    """Direct-form rows from reflection rows, ``|k_i| < 1`` (params.py:56-71):
    the step-up recursion on the device, float64 arithmetic in the
    reference's order.  ``k`` [..., M]; numpy in -> numpy out."""
    conv = _Conv(k)
    kt = conv.t(k)
    if kt.dtype not in (torch.float32, torch.float64):
        kt = kt.to(torch.float64)
    kt = kt.contiguous()
    if kt.dim() < 1 or kt.shape[-1] < 1:
        raise ValueError("reflection rows need order >= 1")
    M = kt.shape[-1]
    rows = kt.numel() // M
    lib = N.load()
    a = torch.empty_like(kt)
    # |k| >= 1 is reported like non-finite LP inputs: at once for numpy callers,
    # through the device flag (lpc.check_nonfinite) for CUDA tensors -- no
    # host sync inside a training step or a CUDA-graph capture
    from . import lpc as _lpc

    vmode = _lpc._mode(conv.numpy)
    if torch.cuda.is_current_stream_capturing():
        vmode = "lazy" if vmode != "off" else vmode
    bad = (torch.zeros(1, dtype=torch.int32, device=conv.device) if vmode == "eager"
           else _lpc._flag(conv.device, vmode))
    with N.on_device(conv.device):
        N.check(lib.tvlp_reflection_to_lpc(N.dtype_code(kt.dtype), N.ptr(kt), N.ptr(a), rows, M,
                                           N.ptr(bad), N.stream_ptr(conv.device)))
    if vmode == "eager" and int(bad.item()) != 0:
        raise ValueError("reflection coefficients must satisfy |k| < 1")
    return conv.out(a)


def reflection_to_lpc_vjp(grad_a, k):
    """grad_k of :func:`reflection_to_lpc` (params.py:74-84)."""
    conv = _Conv(grad_a, k)
    kt = conv.t(k)
    if kt.dtype not in (torch.float32, torch.float64):
        kt = kt.to(torch.float64)
    kt = kt.contiguous()
    ga = conv.t(grad_a, kt.dtype).contiguous()
    if ga.shape != kt.shape:
        raise ValueError("grad_a and k must share the same shape")
    M = kt.shape[-1]
    rows = kt.numel() // M
    lib = N.load()
    gk = torch.empty_like(kt)
    with N.on_device(conv.device):
        N.check(lib.tvlp_reflection_to_lpc_vjp(N.dtype_code(kt.dtype), N.ptr(ga), N.ptr(kt),
                                               N.ptr(gk), rows, M, N.stream_ptr(conv.device)))
    return conv.out(gk)


def expected_frame_count(T, hop):
    """Frame count whose centers ``f*hop`` tile ``0..T`` (params.py:102-104)."""
    return T // hop + 1


def raised_cosine_window(n):
    """Periodic raised-cosine window of length ``n`` (params.py:152-154)."""
    return 0.5 - 0.5 * np.cos(2.0 * np.pi * np.arange(n) / n)


@dataclass
class FramePlan:
    """Windowed framing grid for overlap-add processing.

    This is host-side metadata whose semantics the drop-in must reproduce
    exactly (SPEC.md's framing contract as implemented at params.py:157-217 of
    the reference): frame f covers samples [f*hop, f*hop + frame_size), frames
    start ``n_lead_in()`` hops before t = 0, every frame with a lead-in index
    uses coefficient row 0, and the overlap-added output is divided by the
    COLA constant window.sum()/hop.  The field names, constructors and the
    tuple order of :meth:`iter_frames` are the reference's (callers unpack
    them); the bodies below are written from that contract."""

    frame_size: int
    hop: int
    window: np.ndarray = field(repr=False)

    @classmethod
    def raised_cosine(cls, hop, overlap=0.75):
        n = hop / (1.0 - overlap)
        if abs(n - round(n)) > 1e-9:
            raise ValueError(f"hop {hop} and overlap {overlap} give a non-integer frame size")
        n = int(round(n))
        return cls(frame_size=n, hop=hop, window=raised_cosine_window(n))

    @classmethod
    def rectangular(cls, frame_size, hop=None):
        return cls(frame_size=frame_size, hop=frame_size if hop is None else hop,
                   window=np.ones(frame_size))

    @property
    def overlap(self):
        return 1.0 - self.hop / self.frame_size

    def ola_deviation(self):
        """Peak deviation from its median of the steady-state overlap-add sum
        of the window (one hop of the interior, past the first full frame)."""
        n, h = self.frame_size, self.hop
        k = n // h + 2                       # shifted copies covering the probe hop
        total = np.zeros(n + k * h)
        for start in range(0, k * h, h):
            total[start:start + n] += self.window
        probe = total[n:n + h]
        return float(np.abs(probe - np.median(probe)).max())

    def validate_cola(self, tol=1e-6):
        dev = self.ola_deviation()
        if dev > tol:
            raise ValueError(f"window does not satisfy constant overlap-add; deviation {dev:.3e}")

    def cola_constant(self):
        return float(np.sum(self.window) / self.hop)

    def n_lead_in(self):
        """Frames starting before t = 0 that still overlap it."""
        return (self.frame_size - 1) // self.hop

    def iter_frames(self, length, n_frames):
        """(row, sig_lo, sig_hi, win_lo, win_hi) for every frame that overlaps
        [0, length), lead-in frames first (row 0)."""
        for f in range(-self.n_lead_in(), n_frames):
            t0 = f * self.hop
            lo = 0 if t0 < 0 else t0
            hi = min(t0 + self.frame_size, length)
            if hi > lo:
                yield (f if f > 0 else 0), lo, hi, lo - t0, hi - t0

    # Per-call derived state of the kernel path: the COLA deviation, the COLA
    # constant and the device copies of the window in each I/O dtype
    # (params.py:232, 266: astype(e.dtype)).  All are functions of
    # (frame_size, hop, window contents), so they are cached on exactly that
    # key: an in-place edit of the window or a new array is seen (the key
    # holds the window's bytes), while a repeated call costs one comparison
    # instead of re-validating the window (~50 us of numpy per call).
    def _derived(self):
        w = np.asarray(self.window)
        key = (self.frame_size, self.hop, w.dtype.str, w.shape, w.tobytes())
        st = self.__dict__.get("_derived_cache")
        if st is None or st[0] != key:
            st = (key, self.ola_deviation(), self.cola_constant(), {})
            self.__dict__["_derived_cache"] = st
        return st

    def _validate_cola_cached(self, tol=1e-6):
        dev = self._derived()[1]
        if dev > tol:
            raise ValueError(f"window does not satisfy constant overlap-add; deviation {dev:.3e}")

    def _cola_cached(self):
        return self._derived()[2]

    def _window_tensor(self, dtype, device):
        tens = self._derived()[3]
        key = (dtype, str(device))
        w = tens.get(key)
        if w is None:
            np_dt = np.float32 if dtype == torch.float32 else np.float64
            host = np.ascontiguousarray(np.asarray(self.window).astype(np_dt))
            w = torch.from_numpy(host).to(device)
            tens[key] = w
        return w


def _check(e, frames, plan):
    T1 = e.shape[-1]
    F = frames.shape[-2]
    if F != expected_frame_count(T1 - 1, plan.hop):
        raise ValueError(
            f"got {F} coefficient frames but length {T1} at hop {plan.hop} "
            f"requires {expected_frame_count(T1 - 1, plan.hop)}")
    plan._validate_cola_cached()


def framewise_forward(e, frames, plan, return_aux=False):
    """Returns ``(out, seg)``; ``seg`` [B, n_frames, frame_size] holds the
    per-frame outputs the VJP needs (the reference's ``seg_outputs``).
    ``return_aux``: also the frames' impulse-response tails (or None) that
    framewise_backward(..., aux=) can reuse instead of recomputing."""
    conv = _Conv(e, frames)
    e = conv.t(e)
    if e.dtype not in (torch.float32, torch.float64):
        e = e.to(torch.float32)
    frames = conv.t(frames, e.dtype)
    _check(e, frames, plan)
    batched = e.dim() == 2
    B = e.shape[0] if batched else 1
    T = e.shape[-1]
    F, M = frames.shape[-2], frames.shape[-1]
    lib = N.load()
    nfr = lib.tvlp_framewise_nframes(T, F, plan.frame_size, plan.hop)
    out = torch.empty_like(e)
    seg = torch.empty((B, nfr, plan.frame_size), dtype=e.dtype, device=conv.device)
    na = lib.tvlp_framewise_aux_elems(B, T, F, M, plan.frame_size, plan.hop) if return_aux else 0
    aux = torch.empty(na, dtype=e.dtype, device=conv.device) if na > 0 else None
    w = plan._window_tensor(e.dtype, conv.device)
    dt = N.dtype_code(e.dtype)
    ws, nws = N.workspace(lib.tvlp_workspace_bytes(N.OP_FW_FWD, dt, B, T, M, F, plan.frame_size,
                                                   plan.hop), conv.device)
    with N.on_device(conv.device):
        N.check(lib.tvlp_framewise_forward_ex(dt, N.ptr(e), N.ptr(frames), N.ptr(w),
                                              plan._cola_cached(), N.ptr(out), N.ptr(seg),
                                              N.ptr(aux), B, T, F, M, plan.frame_size, plan.hop,
                                              N.ptr(ws), nws, N.stream_ptr(conv.device)))
    if return_aux:
        return conv.out(out), seg, aux
    return conv.out(out), seg


def framewise_backward(grad_out, frames, seg, plan, aux=None):
    """VJP of :func:`framewise_forward` (params.py:259-273):
    returns ``(grad_e, grad_frames)``; ``aux`` from the same forward
    (return_aux=True) saves recomputing the frames' impulse responses."""
    conv = _Conv(grad_out, frames, seg)
    g = conv.t(grad_out)
    if g.dtype not in (torch.float32, torch.float64):
        g = g.to(torch.float32)
    frames = conv.t(frames, g.dtype)
    seg = conv.t(seg, g.dtype)
    batched = g.dim() == 2
    B = g.shape[0] if batched else 1
    T = g.shape[-1]
    F, M = frames.shape[-2], frames.shape[-1]
    lib = N.load()
    if aux is not None and (aux.dtype != g.dtype or aux.numel() != lib.tvlp_framewise_aux_elems(
            B, T, F, M, plan.frame_size, plan.hop)):
        aux = None  # not this plan's
    ge = torch.empty_like(g)
    gf = torch.empty(frames.shape, dtype=g.dtype, device=conv.device)
    w = plan._window_tensor(g.dtype, conv.device)
    dt = N.dtype_code(g.dtype)
    ws, nws = N.workspace(lib.tvlp_workspace_bytes(N.OP_FW_BWD, dt, B, T, M, F, plan.frame_size,
                                                   plan.hop), conv.device)
    with N.on_device(conv.device):
        N.check(lib.tvlp_framewise_backward_ex(dt, N.ptr(g), N.ptr(frames), N.ptr(w),
                                               plan._cola_cached(), N.ptr(seg), N.ptr(aux),
                                               N.ptr(ge), N.ptr(gf), B, T, F, M, plan.frame_size,
                                               plan.hop, N.ptr(ws), nws,
                                               N.stream_ptr(conv.device)))
    return conv.out(ge), conv.out(gf)


def framewise_lp(e, frames, plan):
    """Frame-wise time-invariant LP with overlap-add (params.py:242-256):
    each windowed frame is filtered from a zero state with its own row, the
    outputs are overlap-added and divided by the COLA constant."""
    out, _ = framewise_forward(e, frames, plan)
    return out
