"""Drop-in B200 LP ops for the UNMODIFIED reference tape engine (tvlp 0.1.0).

    import tvlp
    from integration import tvlp_b200_ops
    handle = tvlp_b200_ops.install()     # the LP ops of every tvlp Tape now run on the GPU
    ... tvlp.synth / build_synth_graph / Tape.backward exactly as before ...
    handle.uninstall()                   # back to the numba ops

The reference's plugin table is its op registry: ``register_op(name,
forward, vjp)`` (pkg/src/tvlp/tape.py:54-65) fills ``tape._REGISTRY``, and
``import tvlp`` already registers ``lp_tv``/``lp_ti`` (lpc.py:202-223) and
``framewise_lp`` (params.py:348-360).  ``register_op`` refuses a second
registration of a name (tape.py:63-64), so the shim REPLACES those entries
with ops of the same contract -- ``forward(values, ctx, dtype) -> ndarray``,
``vjp(grad, values, out, ctx) -> tuple`` reading only ctx, the inputs, the
saved output and the adjoint (tape.py:57-61) -- and restores the originals
on ``uninstall()``.  It also registers ``lp_tv_frames`` (upsample_linear ->
lp_tv as one op; record it as ``tape.record("lp_tv_frames", excitation,
a_frames, hop=hop)`` in place of synth.py:268-269).

Each forward keeps what its backward needs on the device in ``ctx`` (the tape
contract allows any stash): the coefficient track, the output and the
per-sub-chunk carry tape, so the VJP neither re-uploads them nor recomputes
the transition matrices.  Arrays cross the host link once per op and
direction.  Validation follows the reference (ValueError for bad shapes and
non-finite e/A, lpc.py:64-117); unstable filters are not rejected.
"""
from __future__ import annotations

import numpy as np
import torch

_STASH = "_b200"
_OPS = ("lp_tv", "lp_ti", "framewise_lp")


def _dev(x, device, dtype):
    t = torch.as_tensor(np.ascontiguousarray(x))
    return t.to(device=device, dtype=dtype, non_blocking=False)


def _torch_dtype(dtype):
    return torch.float64 if np.dtype(dtype) == np.float64 else torch.float32


def make_ops(device=None):
    """The B200 versions of the reference LP ops: {name: (forward, vjp)}."""
    from paper_2406_05128_b200 import lpc, params

    dev = torch.device(device) if device is not None else torch.device("cuda", 0)

    def fw_lp_tv(values, ctx, dtype):
        e, A = values
        td = _torch_dtype(np.asarray(e).dtype)
        et, At = _dev(e, dev, td), _dev(A, dev, td)
        zi = ctx.get("zi")
        zt = None if zi is None else _dev(zi, dev, td)
        s, carry = lpc._forward(False, et, At, zt, return_carry=True)
        ctx[_STASH] = (At, s, zt, carry)
        return s.cpu().numpy()

    def vjp_lp_tv(grad, values, out, ctx):
        At, s, zt, carry = ctx[_STASH]
        g = _dev(grad, dev, At.dtype)
        ge, gA = lpc._backward(False, g, At, s, zt, carry)
        return ge.cpu().numpy(), gA.cpu().numpy()

    def fw_lp_ti(values, ctx, dtype):
        e, a = values
        td = _torch_dtype(np.asarray(e).dtype)
        et, at = _dev(e, dev, td), _dev(a, dev, td)
        zi = ctx.get("zi")
        zt = None if zi is None else _dev(zi, dev, td)
        s, carry = lpc._forward(True, et, at, zt, return_carry=True)
        ctx[_STASH] = (at, s, zt, carry)
        return s.cpu().numpy()

    def vjp_lp_ti(grad, values, out, ctx):
        at, s, zt, carry = ctx[_STASH]
        ge, ga = lpc._backward(True, _dev(grad, dev, at.dtype), at, s, zt, carry)
        return ge.cpu().numpy(), ga.cpu().numpy()

    def fw_framewise(values, ctx, dtype):
        e, frames = values
        plan = ctx["plan"]
        td = _torch_dtype(np.asarray(e).dtype)
        et, ft = _dev(e, dev, td), _dev(frames, dev, td)
        # the reference's plan object carries frame_size, hop and the window
        # (params.py:157-217); the B200 plan restates the same grid
        bplan = params.FramePlan(frame_size=plan.frame_size, hop=plan.hop,
                                 window=np.asarray(plan.window))
        out, seg, aux = params.framewise_forward(et, ft, bplan, return_aux=True)
        ctx[_STASH] = (ft, seg, bplan, aux)
        return out.cpu().numpy()

    def vjp_framewise(grad, values, out, ctx):
        ft, seg, bplan, aux = ctx[_STASH]
        ge, gf = params.framewise_backward(_dev(grad, dev, ft.dtype), ft, seg, bplan, aux=aux)
        return ge.cpu().numpy(), gf.cpu().numpy()

    def fw_lp_tv_frames(values, ctx, dtype):
        e, frames = values
        td = _torch_dtype(np.asarray(e).dtype)
        et, ft = _dev(e, dev, td), _dev(frames, dev, td)
        s, carry = lpc.lp_forward_tv_frames(et, ft, ctx["hop"], return_carry=True)
        ctx[_STASH] = (ft, s, carry)
        return s.cpu().numpy()

    def vjp_lp_tv_frames(grad, values, out, ctx):
        ft, s, carry = ctx[_STASH]
        ge, gf = lpc.lp_backward_tv_frames(_dev(grad, dev, ft.dtype), ft, ctx["hop"], s,
                                           carry=carry)
        return ge.cpu().numpy(), gf.cpu().numpy()

    return {"lp_tv": (fw_lp_tv, vjp_lp_tv), "lp_ti": (fw_lp_ti, vjp_lp_ti),
            "framewise_lp": (fw_framewise, vjp_framewise),
            "lp_tv_frames": (fw_lp_tv_frames, vjp_lp_tv_frames)}


class Handle:
    """Restores the reference's own ops."""

    def __init__(self, tape_mod, saved, added):
        self._tape, self._saved, self._added = tape_mod, saved, added

    def uninstall(self):
        reg = self._tape._REGISTRY
        for name, op in self._saved.items():
            reg[name] = op
        for name in self._added:
            reg.pop(name, None)
        self._saved, self._added = {}, []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.uninstall()


def install(device=None, names=_OPS, tape_module=None):
    """Swap the reference's LP tape ops for the B200 ones (and add
    ``lp_tv_frames``); returns a :class:`Handle` (also a context manager)."""
    if tape_module is None:
        from tvlp import tape as tape_module  # the reference's engine
    import tvlp  # noqa: F401  (its own registrations must exist before the swap)

    ops = make_ops(device)
    reg = tape_module._REGISTRY
    saved, added = {}, []
    for name in list(names) + ["lp_tv_frames"]:
        fw, vjp = ops[name]
        if name in reg:
            saved[name] = reg[name]
            reg[name] = tape_module._Op(name, fw, vjp)
        else:
            tape_module.register_op(name, fw, vjp)
            added.append(name)
    return Handle(tape_module, saved, added)
