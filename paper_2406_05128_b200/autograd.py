"""``torch.autograd.Function``s for the LP operators -- the B200 replacement
of the reference's tape-op registrations (pkg/src/tvlp/lpc.py:202-223 and
params.py:348-360, contract at tape.py:54-65).

The reference contract is kept: the forward saves its OUTPUT ``s`` and the
coefficients ``A`` (not ``e``), the backward returns
``(grad_e, grad_A)`` and nothing for ``zi``.  The forward also
keeps the carry tape (per-sub-chunk transition matrices) in ``ctx`` so the
backward does not recompute it.
"""
from __future__ import annotations

import torch

from . import lpc
from . import params as _params

__all__ = ["LPTV", "LPTI", "LPFramewise", "LPTVGrouped", "lp_tv", "lp_ti", "framewise",
           "lp_tv_grouped"]


class LPTV(torch.autograd.Function):
    """s = LP_A(e) with the analytic adjoint (lpc.py:202-209)."""

    @staticmethod
    def forward(ctx, e, A, zi=None):
        A = A.to(e.dtype)
        s, carry = lpc._forward(False, e.detach(), A.detach(),
                                None if zi is None else zi.detach(), return_carry=True)
        ctx.save_for_backward(A, s, zi)
        ctx.carry = carry
        return s

    @staticmethod
    def backward(ctx, grad_s):
        A, s, zi = ctx.saved_tensors
        ge, gA = lpc._backward(False, grad_s.contiguous(), A, s, zi, ctx.carry)
        return ge, gA, None


class LPTVGrouped(torch.autograd.Function):
    """Several independent lp_tv ops (e.g. the HpN decoder's H(z) on the
    glottal source and C(z) on the noise, synth.py:264-273) in one grouped
    launch: apply(e_1, A_1, e_2, A_2, ...) -> (s_1, s_2, ...), each pair with
    the contract of LPTV (saves A and s, no grad for zi)."""

    @staticmethod
    def forward(ctx, *args):
        pairs = [(args[2 * i].detach(), args[2 * i + 1].detach().to(args[2 * i].dtype))
                 for i in range(len(args) // 2)]
        outs, carry = lpc.lp_forward_tv_grouped(pairs, return_carry=True)
        ctx.save_for_backward(*[p[1] for p in pairs], *outs)
        ctx.n = len(pairs)
        ctx.carry = carry
        return tuple(outs)

    @staticmethod
    def backward(ctx, *grads):
        n = ctx.n
        saved = ctx.saved_tensors
        As, ss = saved[:n], saved[n:]
        gs = [torch.zeros_like(s) if g is None else g.contiguous() for g, s in zip(grads, ss)]
        res = lpc.lp_backward_tv_grouped(list(zip(gs, As, ss)), carry=ctx.carry)
        return tuple(x for ge_gA in res for x in ge_gA)


class LPTVFrames(torch.autograd.Function):
    """s = LP_{upsample(frames)}(e): the tape ops upsample_linear -> lp_tv
    (params.py:337-345, lpc.py:202-209) as one fused op."""

    @staticmethod
    def forward(ctx, e, frames, hop, zi=None):
        frames = frames.to(e.dtype)
        s, carry = lpc.lp_forward_tv_frames(e.detach(), frames.detach(), hop,
                                            None if zi is None else zi.detach(),
                                            return_carry=True)
        ctx.save_for_backward(frames, s, zi)
        ctx.carry = carry
        ctx.hop = hop
        return s

    @staticmethod
    def backward(ctx, grad_s):
        frames, s, zi = ctx.saved_tensors
        ge, gF = lpc.lp_backward_tv_frames(grad_s.contiguous(), frames, ctx.hop, s, zi,
                                           carry=ctx.carry)
        return ge, gF, None, None


class ReflectionToLPC(torch.autograd.Function):
    """a = step_up(k) with the analytic VJP (params.py:56-84, 320-334)."""

    @staticmethod
    def forward(ctx, k):
        a = _params.reflection_to_lpc(k.detach())
        ctx.save_for_backward(k)
        return a

    @staticmethod
    def backward(ctx, grad_a):
        (k,) = ctx.saved_tensors
        return _params.reflection_to_lpc_vjp(grad_a.contiguous(), k)


class LPTI(torch.autograd.Function):
    """Time-invariant filter with the single-filter adjoint (lpc.py:212-219)."""

    @staticmethod
    def forward(ctx, e, a, zi=None):
        a = a.to(e.dtype)
        s, carry = lpc._forward(True, e.detach(), a.detach(),
                                None if zi is None else zi.detach(), return_carry=True)
        ctx.save_for_backward(a, s, zi)
        ctx.carry = carry
        return s

    @staticmethod
    def backward(ctx, grad_s):
        a, s, zi = ctx.saved_tensors
        ge, ga = lpc._backward(True, grad_s.contiguous(), a, s, zi, ctx.carry)
        return ge, ga.reshape(a.shape), None


class LPFramewise(torch.autograd.Function):
    """Frame-wise LP with overlap-add (params.py:348-357); saves the frame
    outputs like the reference's ctx['seg_outputs']."""

    @staticmethod
    def forward(ctx, e, frames, plan):
        frames = frames.to(e.dtype)
        out, seg, aux = _params.framewise_forward(e.detach(), frames.detach(), plan,
                                                  return_aux=True)
        ctx.save_for_backward(frames, seg)
        ctx.aux = aux  # the frames' impulse-response tails (or None)
        ctx.plan = plan
        return out

    @staticmethod
    def backward(ctx, grad_out):
        frames, seg = ctx.saved_tensors
        ge, gf = _params.framewise_backward(grad_out.contiguous(), frames, seg, ctx.plan,
                                            aux=ctx.aux)
        return ge, gf, None


def lp_tv(e, A, zi=None):
    """Differentiable sample-wise LP filter."""
    return LPTV.apply(e, A, zi)


def lp_tv_grouped(*pairs):
    """Differentiable grouped filter: lp_tv_grouped((e1, A1), (e2, A2)) -> (s1, s2)."""
    flat = [x for p in pairs for x in p]
    return LPTVGrouped.apply(*flat)


def lp_tv_frames(e, frames, hop, zi=None):
    return LPTVFrames.apply(e, frames, hop, zi)


def reflection_to_lpc(k):
    return ReflectionToLPC.apply(k)


def lp_ti(e, a, zi=None):
    """Differentiable time-invariant LP filter."""
    return LPTI.apply(e, a, zi)


def framewise(e, frames, plan):
    """Differentiable frame-wise LP with overlap-add."""
    return LPFramewise.apply(e, frames, plan)
