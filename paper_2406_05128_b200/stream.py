"""Host-resident batches: forward + VJP of the time-varying LP with the
host<->device copies pipelined against the kernels.

The reference filters numpy arrays in host memory (lpc.py:101-117, 152-173).
For a batch that lives on the host the PCIe/C2C copies (A and grad_A are
4*M bytes per sample each way) dominate the kernels by ~30x, so the batch is
cut into chunks that flow through three CUDA streams (host->device copies,
kernels, device->host copies, ordered by events): chunk i's upload, chunk
i-1's kernels and chunk i-2's download run concurrently, and the two copy
directions use separate copy engines (measured 56 + 57 GB/s concurrently on
the B200 box, tools/copy_bw.py).

    s, grad_e, grad_A = lp_tv_fwd_bwd_host(e, A, grad_s)

``e``/``grad_s`` [B, T] and ``A`` [B, T, M] are host tensors (pinned for
asynchronous copies) or numpy arrays; results are pinned host tensors (or the
``out`` triple).  The arithmetic is the same C-ABI path as
:func:`paper_2406_05128_b200.lpc.lp_forward_tv` / ``lp_backward_tv`` (with the
forward's carry tape reused by the backward).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as N
from . import lpc

_STREAMS = {}
_BUFFERS = {}


def _buffers(dev, B, T, M, dtype, sizes, with_zi):
    """Device buffers of the whole batch plus one chunk's carry tape and
    workspace, kept across calls (the kernels of consecutive chunks run on one
    stream, so one carry/workspace serves every chunk).  The carry tape and
    the workspace are sized for the LARGEST need over the distinct chunk
    sizes: the sub-chunk plan depends on the chunk's batch, and a smaller
    chunk can need a larger tape (shorter sub-chunks below B*T = 4096*512)."""
    sizes = tuple(sorted(set(int(n) for n in sizes)))
    key = (dev.index, B, T, M, dtype, sizes, with_zi)
    if key not in _BUFFERS:
        lib = N.load()
        dt = N.dtype_code(dtype)
        nws = max(lib.tvlp_workspace_bytes(op, dt, nb, T, M, 0, 0, 0)
                  for op in (N.OP_FWD_TV, N.OP_BWD_TV) for nb in sizes)
        ncarry = max(lib.tvlp_carry_elems(nb, T, M) for nb in sizes)
        _BUFFERS.clear()  # one shape at a time
        _BUFFERS[key] = {
            "e": torch.empty((B, T), dtype=dtype, device=dev),
            "g": torch.empty((B, T), dtype=dtype, device=dev),
            "A": torch.empty((B, T, M), dtype=dtype, device=dev),
            "zi": torch.empty((B, M), dtype=dtype, device=dev) if with_zi else None,
            "s": torch.empty((B, T), dtype=dtype, device=dev),
            "ge": torch.empty((B, T), dtype=dtype, device=dev),
            "gA": torch.empty((B, T, M), dtype=dtype, device=dev),
            "carry": torch.empty(ncarry, dtype=dtype, device=dev),
            "ws": torch.empty(nws, dtype=torch.uint8, device=dev),
            "nws": nws,
        }
    return _BUFFERS[key]


def _streams(device, n):
    key = (device.index, n)
    if key not in _STREAMS:
        _STREAMS[key] = [torch.cuda.Stream(device) for _ in range(n)]
    return _STREAMS[key]


def _host(x, dtype=None):
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if x.device.type != "cpu":
        raise ValueError("lp_tv_fwd_bwd_host takes host tensors (use lpc.* for CUDA tensors)")
    return x.contiguous() if dtype is None else x.to(dtype).contiguous()


def schedule(B, n=8):
    """Default chunk sizes: n equal chunks (at least one sequence each)."""
    n = max(1, min(B, n))
    return [B * (i + 1) // n - B * i // n for i in range(n)]


def _bounds(B, chunks):
    sizes = schedule(B) if chunks is None else \
        schedule(B, chunks) if isinstance(chunks, int) else [int(c) for c in chunks]
    if sum(sizes) != B or min(sizes) < 1:
        raise ValueError(f"chunk sizes {sizes} must be positive and sum to B={B}")
    out, lo = [], 0
    for c in sizes:
        out.append((lo, lo + c))
        lo += c
    return out


def lp_tv_fwd_bwd_host(e, A, grad_s, zi=None, *, chunks=None, out=None, device=None,
                       sync=True):
    """s = LP(e, A) and its VJP (grad_e, grad_A) for grad_s, batch-pipelined.

    ``chunks``: number of equal batch chunks, or a sequence of chunk sizes
    (sequences per chunk, summing to B); default :func:`schedule`.
    ``out``: optional (s, grad_e, grad_A) host tensors.  ``sync=False``
    returns once the work is queued on the current stream (the host results
    are complete after that stream synchronises)."""
    e = _host(e)
    A = _host(A, e.dtype)
    grad_s = _host(grad_s, e.dtype)
    if e.dim() != 2 or A.dim() != 3 or grad_s.shape != e.shape or A.shape[:2] != e.shape:
        raise ValueError("expected e, grad_s [B, T] and A [B, T, M]")
    B = e.shape[0]
    dev = torch.device(device) if device is not None else \
        torch.device("cuda", torch.cuda.current_device())
    if out is None:
        pin = torch.cuda.is_available()
        out = (torch.empty_like(e, pin_memory=pin), torch.empty_like(e, pin_memory=pin),
               torch.empty_like(A, pin_memory=pin))
    s_h, ge_h, gA_h = out
    zi_h = None if zi is None else _host(zi, e.dtype)
    bounds = _bounds(B, chunks)
    bufs = _buffers(dev, e.shape[0], e.shape[1], A.shape[2], e.dtype,
                    [h - l for l, h in bounds], zi_h is not None)
    lib = N.load()
    dt = N.dtype_code(e.dtype)
    T, M = e.shape[1], A.shape[2]
    # three streams: host->device copies, kernels, device->host copies; the
    # two copy directions run back to back on their own engines
    h2d, comp, d2h = _streams(dev, 3)
    main = torch.cuda.current_stream(dev)
    for st in (h2d, comp, d2h):
        st.wait_stream(main)
    flag = lpc._flag(dev)
    # Copy order (tools/e2e_order.py, e2e_sched.py: 7.66 -> 7.37 ms on
    # config 3, outputs identical): every chunk ships its A rows; the small
    # per-sequence signals going up (e, grad_s) travel as chunk 0's own, then
    # the rest of the batch in one copy each right behind A_0 -- small
    # host->device copies interleaved with the device->host stream were slow
    # and left idle gaps.  Down, each chunk's s, grad_e, grad_A.
    n = len(bounds)
    for i, (lo, hi) in enumerate(bounds):
        nb = hi - lo
        ed, Ad, gd = bufs["e"][lo:hi], bufs["A"][lo:hi], bufs["g"][lo:hi]
        zd = None if zi_h is None else bufs["zi"][lo:hi]
        sd, ged, gAd = bufs["s"][lo:hi], bufs["ge"][lo:hi], bufs["gA"][lo:hi]
        with torch.cuda.stream(h2d):
            if i == 0:
                ed.copy_(e[lo:hi], non_blocking=True)
                gd.copy_(grad_s[lo:hi], non_blocking=True)
                if zi_h is not None:
                    bufs["zi"].copy_(zi_h, non_blocking=True)
            Ad.copy_(A[lo:hi], non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(h2d)
            if i == 0 and hi < B:  # later chunks' ready events come after these
                bufs["e"][hi:].copy_(e[hi:], non_blocking=True)
                bufs["g"][hi:].copy_(grad_s[hi:], non_blocking=True)
        comp.wait_event(ready)
        ncarry = lib.tvlp_carry_elems(nb, T, M)
        carry = bufs["carry"][:ncarry]
        if carry.numel() != ncarry:
            raise RuntimeError(f"carry tape of {carry.numel()} elements, chunk needs {ncarry}")
        cs = ctypes.c_void_p(comp.cuda_stream)
        with torch.cuda.device(dev):
            N.check(lib.tvlp_lp_forward_tv(dt, N.ptr(ed), N.ptr(Ad), N.ptr(zd), N.ptr(sd), nb, T, M,
                                           N.ptr(carry), lpc._carry_code(), N.ptr(bufs["ws"]),
                                           bufs["nws"], N.ptr(flag), cs))
            N.check(lib.tvlp_lp_backward_tv(dt, N.ptr(gd), N.ptr(Ad), N.ptr(sd), N.ptr(zd),
                                            N.ptr(ged), N.ptr(gAd), nb, T, M, N.ptr(carry),
                                            lpc._carry_code(), N.ptr(bufs["ws"]), bufs["nws"], cs))
        done = torch.cuda.Event()
        done.record(comp)
        d2h.wait_event(done)
        with torch.cuda.stream(d2h):
            for dst, src in ((s_h, sd), (ge_h, ged), (gA_h, gAd)):
                dst[lo:hi].copy_(src, non_blocking=True)
    for st in (h2d, comp, d2h):
        main.wait_stream(st)
    lpc._raise_nonfinite(flag, bufs["e"], bufs["A"])
    if sync:  # the host results are complete on return
        main.synchronize()
    return s_h, ge_h, gA_h
