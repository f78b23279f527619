"""One long sequence split in time across ranks (the
exchange step): rank r holds samples [r*Tr, (r+1)*Tr) of every sequence.

The filter is linear in its initial state, so a time segment's output is its
zero-state-entry output plus the response to the state the earlier segments
leave it.  Each rank therefore runs its segment independently and the ranks
exchange only small per-segment summaries:

forward
  1. s0_r, tape_r = LP(e_r, A_r, zi if r == 0 else 0); Phi_r = product of the
     segment's sub-chunk transitions (tvlp_segment_transition), z_r = the end
     state of s0_r.
  2. all_gather (Phi_r, z_r)  -- M*M + M values per sequence per rank.
  3. x_1 = z_0, x_{q+1} = Phi_q x_q + z_q: rank r re-runs the carry and apply
     passes of its segment with zi = x_r (r > 0), reusing its carry tape
     (TVLP_CARRY_REUSE: the tape does not depend on zi).

backward (adjoint flows right to left)
  1. ge0_r, nu_r = VJP of segment r with nothing entering from the right;
     nu_r = dL_r/dzi_r (tvlp_lp_backward_tv_ex's grad_zi).
  2. all_gather nu_r.
  3. mu_{R-1} = 0, mu_{q-1} = nu_q + Phi_q^T mu_q: rank r re-runs its VJP
     with mu_r entering from the right (r < R-1).

The summaries are tiny, so the collective is one all_gather per direction
(NCCL on GPUs, gloo in the CPU tests); the per-rank work is one extra
carry+apply pass and one extra VJP pass over the rank's own segment.  The phases are exposed
separately (``*_local`` / ``*_combine``) so one process can play every rank
(tests) and the CPU tests can swap in a numpy segment engine.
"""
from __future__ import annotations

import torch

from . import _native as N
from . import lpc

__all__ = ["GpuSegmentEngine", "forward_local", "forward_combine", "backward_local",
           "backward_combine", "lp_tv_forward_split", "lp_tv_backward_split"]


class GpuSegmentEngine:
    """Segment primitives on the B200 kernels (the C ABI)."""

    def forward(self, e, A, zi, tape=None):
        """(s, tape); with ``tape`` from a forward over the same (e, A) only the
        carry and apply passes run (the tape does not depend on zi)."""
        if tape is None:
            return lpc._forward(False, e, A, zi, return_carry=True)
        lib = N.load()
        B, T = e.shape
        M = A.shape[-1]
        dt = N.dtype_code(e.dtype)
        s = torch.empty_like(e)
        ws, nws = N.workspace(lib.tvlp_workspace_bytes(N.OP_FWD_TV, dt, B, T, M, 0, 0, 0),
                              e.device)
        flag = lpc._flag(e.device)
        with torch.cuda.device(e.device):
            N.check(lib.tvlp_lp_forward_tv(dt, N.ptr(e), N.ptr(A), N.ptr(zi.contiguous()),
                                           N.ptr(s), B, T, M, N.ptr(tape),
                                           lpc._carry_code() | N.CARRY_REUSE, N.ptr(ws), nws,
                                           N.ptr(flag), N.stream_ptr(e.device)))
        return s, tape

    def transition(self, tape, B, T, M, dtype, device):
        lib = N.load()
        Phi = torch.empty((B, M, M), dtype=dtype, device=device)
        ws, nws = N.workspace(lib.tvlp_workspace_bytes(N.OP_SEGMENT_TRANSITION,
                                                       N.dtype_code(dtype), B, T, M, 0, 0, 0),
                              device)
        with torch.cuda.device(device):
            N.check(lib.tvlp_segment_transition(N.dtype_code(dtype), N.ptr(tape), B, T, M,
                                                N.ptr(Phi), N.ptr(ws), nws,
                                                N.stream_ptr(device)))
        return Phi

    def backward(self, g, A, s, zi, tape, mu_in):
        lib = N.load()
        B, T = g.shape
        M = A.shape[-1]
        dt = N.dtype_code(g.dtype)
        ge = torch.empty_like(g)
        gA = torch.empty_like(A)
        nu = torch.empty((B, M), dtype=g.dtype, device=g.device)
        ws, nws = N.workspace(lib.tvlp_workspace_bytes(N.OP_BWD_TV_EX, dt, B, T, M, 0, 0, 0),
                              g.device)
        with torch.cuda.device(g.device):
            N.check(lib.tvlp_lp_backward_tv_ex(
                dt, N.ptr(g), N.ptr(A), N.ptr(s), N.ptr(zi), N.ptr(ge), N.ptr(gA), B, T, M,
                N.ptr(tape), lpc._carry_code(), N.ptr(mu_in), N.ptr(nu), N.ptr(ws), nws,
                N.stream_ptr(g.device)))
        return ge, gA, nu


def _end_state(s, M):
    """x(T-1) = [s(T-1), ..., s(T-M)] (zero-padded if T < M)."""
    B, T = s.shape
    x = torch.zeros((B, M), dtype=s.dtype, device=s.device)
    k = min(M, T)
    x[:, :k] = s[:, T - k:].flip(-1)
    return x


def forward_local(engine, rank, e, A, zi=None):
    """Phase 1 of rank ``rank``: (s0, tape, Phi, z)."""
    B, T = e.shape
    M = A.shape[-1]
    s0, tape = engine.forward(e, A, zi if rank == 0 else None)
    Phi = engine.transition(tape, B, T, M, e.dtype, e.device)
    return s0, tape, Phi, _end_state(s0, M)


def forward_combine(rank, Phis, zs):
    """State entering segment ``rank`` from the gathered (Phi_q, z_q)."""
    if rank == 0:
        return None
    x = zs[0]
    for q in range(1, rank):
        x = torch.bmm(Phis[q], x.unsqueeze(-1)).squeeze(-1) + zs[q]
    return x


def backward_local(engine, g, A, s, zi, tape):
    """Phase 1 of the VJP: (ge0, gA0, nu) with nothing entering from the right."""
    return engine.backward(g, A, s, zi, tape, None)


def backward_combine(rank, Phis, nus):
    """Adjoint entering segment ``rank`` from the right (None for the last)."""
    R = len(nus)
    if rank == R - 1:
        return None
    mu = nus[R - 1]
    for q in range(R - 2, rank, -1):
        mu = nus[q] + torch.bmm(Phis[q].transpose(1, 2), mu.unsqueeze(-1)).squeeze(-1)
    return mu


def _gather(t, group):
    import torch.distributed as dist

    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t.contiguous(), group=group)
    return out


def lp_tv_forward_split(e, A, zi=None, group=None, engine=None):
    """This rank's time segment of s = LP_A(e) for sequences split across the
    ranks of ``group``; returns (s, ctx) where ctx feeds the backward."""
    import torch.distributed as dist

    engine = engine or GpuSegmentEngine()
    rank = dist.get_rank(group)
    s0, tape, Phi, z = forward_local(engine, rank, e, A, zi)
    Phis, zs = _gather(Phi, group), _gather(z, group)
    x_in = forward_combine(rank, Phis, zs)
    if x_in is None:
        s, zi_r = s0, zi
    else:
        s, tape = engine.forward(e, A, x_in, tape)  # same (e, A): reuse the tape
        zi_r = x_in
    return s, {"tape": tape, "Phis": Phis, "zi": zi_r, "rank": rank}


def lp_tv_backward_split(g, A, s, ctx, group=None, engine=None):
    """This rank's (grad_e, grad_A) for the split sequences."""
    engine = engine or GpuSegmentEngine()
    ge, gA, nu = backward_local(engine, g, A, s, ctx["zi"], ctx["tape"])
    nus = _gather(nu, group)
    mu = backward_combine(ctx["rank"], ctx["Phis"], nus)
    if mu is not None:
        ge, gA, _ = engine.backward(g, A, s, ctx["zi"], ctx["tape"], mu)
    return ge, gA
