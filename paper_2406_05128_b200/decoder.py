"""The rest of the GOLF decoder on the GPU.

The reference renders its source-filter (SF) and harmonic-plus-noise (HpN)
decoders on a numpy tape (pkg/src/tvlp/synth.py:217-275) from these pieces:

* wavetable oscillator at ``oversample`` x the output rate, read with
  bilinear interpolation (source.py:224-268) and decimated by a 127-tap
  windowed-sinc lowpass (source.py:215-222, 271-291);
* frame-wise shaped Gaussian noise: linear-phase FIRs from 256 log-magnitude
  bins per frame, overlap-added with the raised-cosine plan (source.py:349-428);
* the trainable 128-tap global FIR at the output (source.py:445-459);
* the multi-resolution spectral loss at prime FFT sizes 509/1021/2053
  (loss.py:25-132; no zero-padding: the transforms run at the native sizes).

Here they are batched torch operations on CUDA tensors (cuFFT/cuDNN
library kernels -- SURVEY.md §8(f): "torch/cuFFT first, fuse only if
profiled hot"), differentiated by torch autograd, except the pieces that
profiled hot in the float32 decoder step, which run on this package's
kernels (csrc/decoder_kernels.cu): the oscillator (phase, table read,
decimation; ``wavetable_osc``), the global FIR (``global_fir``), the noise
shaping's framing and overlap-add (``shape_noise``) and the MSS loss's
framing and loss terms (``mss_loss``; its spectra stay cuFFT); the LP filters
are this package's sm_100a kernels (the fused upsample+LP ``autograd.lp_tv_frames``
and the grouped pair ``autograd.lp_tv_grouped`` for a C(z) LP).
Every op follows the reference's arithmetic order closely enough that the
float64 decoder matches the reference tape to ~1e-12 (tests/test_decoder_gpu.py).
Inputs of shape [B, ...] render B items at once.
"""
from __future__ import annotations

import functools
import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as TF

from . import _native as N
from . import autograd as ag

__all__ = [
    "NOISE_BINS", "FIR_TAPS", "design_lowpass", "oscillator_phase", "upsample_linear",
    "wavetable_read", "decimate_fir", "wavetable_osc", "fir_from_logmag", "shape_noise", "generate_noise",
    "global_fir", "stft_mag", "mss_loss", "Decoder",
]

NOISE_BINS = 256          # source.py:52
FIR_TAPS = 128            # synth.py FIR_TAPS
SQUASH_LIMIT = 0.999      # params.py:31
DEFAULT_FFT_SIZES = (509, 1021, 2053)  # loss.py:22
LOG_EPS = 1e-8            # loss.py:23


@functools.lru_cache(maxsize=16)
def _lowpass_np(num_taps, cutoff, oversample):
    fc = cutoff / (2.0 * oversample)
    n = np.arange(num_taps) - (num_taps - 1) / 2.0
    h = 2.0 * fc * np.sinc(2.0 * fc * n) * np.blackman(num_taps)
    h = h / h.sum()
    h.setflags(write=False)
    return h


_DEV_CACHE = {}


def _on_device(key, build, device, dtype):
    """Host-built constants (taps, windows, frame indices) uploaded once per
    (key, device, dtype): a decoder step makes no host->device copies."""
    k = (key, str(device), dtype)
    t = _DEV_CACHE.get(k)
    if t is None:
        if len(_DEV_CACHE) > 64:
            _DEV_CACHE.clear()
        t = build()
        t = t.to(device=device, dtype=dtype) if dtype is not None else t.to(device=device)
        _DEV_CACHE[k] = t
    return t


def design_lowpass(num_taps=127, cutoff=0.45, oversample=4):
    """Windowed-sinc decimation lowpass (source.py:215-222), float64 numpy."""
    return _lowpass_np(num_taps, cutoff, oversample).copy()


def _block_weights(F, hop, device, dtype):
    """The same weights as [F, hop] blocks (block f covers t = f*hop + j):
    j / hop, and 0 in the last block (params.py:113-115)."""
    w = (torch.arange(hop, device=device).to(dtype) / float(hop))[None].repeat(F, 1)
    w[F - 1] = 0
    return w


def _upsample_w2(hop, device, dtype):
    """[hop, 2]: the interpolation weights (1 - j/hop, j/hop) of one block."""
    return _on_device(("upsample_w2", hop), lambda: torch.stack(
        [1.0 - torch.arange(hop, dtype=torch.float64) / hop,
         torch.arange(hop, dtype=torch.float64) / hop], dim=1), device, dtype)


class _Upsample(torch.autograd.Function):
    """params.py:120-145 as dense block arithmetic: forward
    (1 - w) frames[f] + w frames[f + 1] over [F, hop] blocks (bit-identical to
    the gather form), backward the two weighted block sums (the scatter of
    params.py:135-145 without a sorting index_put)."""

    @staticmethod
    def forward(ctx, frames, hop, T1):
        Bn, F = frames.shape[:2]
        nxt = torch.cat([frames[:, 1:], frames[:, -1:]], dim=1)
        ctx.shape = (F, hop, T1, frames.dim())
        if frames.dim() == 2 and _b200_pieces(frames):
            # float32 CUDA: [a, b] x [(1 - w), w]^T for every block as one thin
            # GEMM (K = 2) writing the track once; the held last block has
            # b = a, so it needs no w = 0 special case (a (1 - w) + a w)
            out = torch.matmul(torch.stack([frames, nxt], dim=-1),
                               _upsample_w2(hop, frames.device, frames.dtype).t())
            return out.reshape(Bn, F * hop)[:, :T1]
        w = _block_weights(F, hop, frames.device, frames.dtype)
        if frames.dim() == 3:
            w = w[..., None]
            out = (1.0 - w) * frames[:, :, None] + w * nxt[:, :, None]   # [B, F, hop, D]
            out = out.reshape(Bn, F * hop, frames.shape[2])[:, :T1]
        else:
            out = (1.0 - w) * frames[:, :, None] + w * nxt[:, :, None]   # [B, F, hop]
            out = out.reshape(Bn, F * hop)[:, :T1]
        ctx.shape = (F, hop, T1, frames.dim())
        return out

    @staticmethod
    def backward(ctx, g):
        F, hop, T1, nd = ctx.shape
        Bn = g.shape[0]
        if nd == 2 and F > 1 and _b200_pieces(g):
            # float32 CUDA: the F-1 full blocks' two weighted sums as ONE thin
            # GEMM over a view of g (no pad copy, no weighted temporaries);
            # the last (held, w = 0) block is a plain sum
            g = g.contiguous()
            ab = torch.matmul(g[:, :(F - 1) * hop].reshape(Bn, F - 1, hop),
                              _upsample_w2(hop, g.device, g.dtype))            # [B, F-1, 2]
            gf = torch.cat([ab[..., 0], g[:, (F - 1) * hop:].sum(dim=1, keepdim=True)], dim=1)
            gf[:, 1:] += ab[..., 1]
            return gf, None, None
        w = _block_weights(F, hop, g.device, g.dtype)
        pad = F * hop - T1
        if nd == 3:
            gp = TF.pad(g, (0, 0, 0, pad)).reshape(Bn, F, hop, g.shape[-1])
            w = w[..., None]
        else:
            gp = TF.pad(g, (0, pad)).reshape(Bn, F, hop)
        ga = ((1.0 - w) * gp).sum(dim=2)        # to frame f
        gb = (w * gp).sum(dim=2)                # to frame f + 1 (zero in the last block)
        gf = ga.clone()
        gf[:, 1:] += gb[:, :-1]
        return gf, None, None


def upsample_linear(frames, hop, T1):
    """params.py:120-132 for [B, F] or [B, F, D] frame controls -> [B, T1(, D)]
    (T1 = T + 1 samples).  Differentiable (the VJP is the scatter of
    params.py:135-145)."""
    F = frames.shape[1]
    if F != (T1 - 1) // hop + 1:
        raise ValueError(f"got {F} frames but T={T1 - 1} at hop={hop} requires "
                         f"{(T1 - 1) // hop + 1}")
    return _Upsample.apply(frames, hop, T1)


def oscillator_phase(f0_frames, hop, n_out, fs, oversample, device=None):
    """Per-sample table phase (periods, mod 1) at the oversampled rate
    (source.py:224-238): float64 cumulative sum, on ``device`` (default: the
    device of ``f0_frames``; host arrays -> CPU)."""
    f0_frames = _checked_f0(f0_frames, fs, device)
    n_os = n_out * oversample
    f0 = upsample_linear(f0_frames, hop * oversample, n_os)
    return torch.remainder(torch.cumsum(f0 / (fs * oversample), dim=-1), 1.0)


def _b200_pieces(t):
    """The float32 CUDA decoder runs the oscillator and the global FIR on
    csrc/decoder_kernels.cu; float64 (the reference-parity runs) and CPU
    tensors compose the torch pieces."""
    return t.is_cuda and t.dtype == torch.float32


def _checked_f0(f0_frames, fs, device=None):
    """f0 frames as float64 [B, F] on ``device``, validated like
    source.py:230-233."""
    f0_frames = torch.as_tensor(f0_frames, dtype=torch.float64, device=device)
    if f0_frames.dim() == 1:
        f0_frames = f0_frames[None]
    bad = ((f0_frames >= fs / 2.0) | (f0_frames < 0)).any()
    # (one host sync; skipped while a CUDA graph is being captured -- the
    # graph's warm-up runs checked the same static inputs)
    if not (f0_frames.is_cuda and torch.cuda.is_current_stream_capturing()) and bool(bad):
        if bool((f0_frames >= fs / 2.0).any()):
            raise ValueError("f0 at or above the output Nyquist frequency")
        raise ValueError("f0 must be nonnegative")
    return f0_frames


class _WavetableOscB200(torch.autograd.Function):
    """The oscillator subgraph of source.py:294-318 (oscillator_phase ->
    upsample_linear(pos) -> wavetable_read -> decimate_fir) as one kernel
    (tvlp_wavetable_osc: the x4 track never leaves shared memory) and its VJP
    to the table-position frames (tvlp_wavetable_osc_vjp).  float32, the phase
    in float64."""

    @staticmethod
    def forward(ctx, pos, f0, tables, taps, hop, n_out, fs):
        lib = N.load()
        B, F = pos.shape
        K, L = tables.shape
        sig = torch.empty((B, n_out), dtype=torch.float32, device=pos.device)
        with N.on_device(pos.device):
            N.check(lib.tvlp_wavetable_osc(N.ptr(f0), N.ptr(pos), N.ptr(tables), K, L, N.ptr(taps),
                                           taps.shape[0], N.ptr(sig), B, n_out, F, hop, 4,
                                           float(fs), N.stream_ptr(pos.device)))
        ctx.save_for_backward(pos, f0, tables, taps)
        ctx.cfg = (hop, n_out, float(fs))
        return sig

    @staticmethod
    def backward(ctx, g):
        pos, f0, tables, taps = ctx.saved_tensors
        hop, n_out, fs = ctx.cfg
        lib = N.load()
        B, F = pos.shape
        K, L = tables.shape
        g = g.contiguous()
        gpos = torch.empty_like(pos)
        ws = torch.empty(2 * B * F, dtype=torch.float32, device=pos.device)
        with N.on_device(pos.device):
            N.check(lib.tvlp_wavetable_osc_vjp(N.ptr(f0), N.ptr(pos), N.ptr(tables), K, L,
                                               N.ptr(taps), taps.shape[0], N.ptr(g), N.ptr(gpos),
                                               N.ptr(ws), B, n_out, F, hop, 4, fs,
                                               N.stream_ptr(pos.device)))
        return gpos, None, None, None, None, None, None


def wavetable_osc(pos, f0_frames, tables, hop, n_out, fs, oversample=4, taps=None):
    """The oscillator's decimated signal [B, n_out] before the gain
    (source.py:294-316) from table-position frames pos [B, F] (already in
    [0, K-1] units) and f0 frames [B, F].  float32 CUDA tensors at the
    reference's oversample 4 run the fused kernels; anything else composes
    the taped pieces (oscillator_phase, upsample_linear, wavetable_read,
    decimate_fir) in torch."""
    if taps is None:
        taps = _on_device(("lowpass", oversample),
                          lambda: torch.as_tensor(_lowpass_np(127, 0.45, oversample).copy()),
                          pos.device, pos.dtype)
    if _b200_pieces(pos) and oversample == 4:
        f0 = _checked_f0(f0_frames, fs, pos.device)
        if f0.shape != pos.shape:
            raise ValueError(f"f0 frames {tuple(f0.shape)} must match positions {tuple(pos.shape)}")
        return _WavetableOscB200.apply(pos.contiguous(), f0.contiguous(),
                                       tables.to(torch.float32).contiguous(),
                                       taps.to(torch.float32).contiguous(), hop, n_out, fs)
    phase = oscillator_phase(f0_frames, hop, n_out, fs, oversample,
                             device=pos.device).to(pos.dtype)
    pos_track = upsample_linear(pos, hop * oversample, n_out * oversample)
    raw = wavetable_read(pos_track, tables.to(pos.dtype), phase)
    return decimate_fir(raw, taps, oversample, n_out) if oversample > 1 else raw


class _WavetableRead(torch.autograd.Function):
    """source.py:241-268: bilinear read; d(out)/d(pos) = the row difference
    (the reference keeps it through the position clip)."""

    @staticmethod
    def forward(ctx, pos, tables, phase):
        K, L = tables.shape
        p = torch.clamp(pos, 0.0, K - 1.0)
        r0 = torch.clamp(torch.floor(p).long(), max=K - 1)
        r1 = torch.clamp(r0 + 1, max=K - 1)
        wr = p - r0.to(p.dtype)
        x = phase * L
        fx = torch.floor(x)
        i0 = torch.remainder(fx.long(), L)
        i1 = torch.remainder(i0 + 1, L)
        wi = x - fx
        low = (1.0 - wi) * tables[r0, i0] + wi * tables[r0, i1]
        high = (1.0 - wi) * tables[r1, i0] + wi * tables[r1, i1]
        ctx.save_for_backward(high - low)
        return (1.0 - wr) * low + wr * high

    @staticmethod
    def backward(ctx, grad):
        (delta,) = ctx.saved_tensors
        return grad * delta, None, None


def wavetable_read(pos, tables, phase):
    return _WavetableRead.apply(pos, tables, phase)


def decimate_fir(x, taps, factor, n_out):
    """source.py:271-291: full convolution with ``taps`` (odd length, group
    delay gd), every ``factor``-th sample from gd.  x [B, N] -> [B, n_out]."""
    nt = taps.shape[0]
    gd = (nt - 1) // 2
    xp = TF.pad(x[:, None], (nt - 1, nt - 1))[:, :, gd:]
    y = TF.conv1d(xp, taps.flip(0)[None, None], stride=factor)
    return y[:, 0, :n_out]


def generate_noise(n, seed):
    """source.py:349-352: unit Gaussian noise from numpy's Philox keyed by the
    seed (a host-side generator: the bits of the reference's noise)."""
    gen = np.random.Generator(np.random.Philox(key=seed))
    return gen.standard_normal(n)


def fir_from_logmag(logmag):
    """source.py:355-364: linear-phase FIR bank [.., 2(B-1)] from log-magnitude
    rows [.., B]: irfft of exp(logmag), centred, Hann-windowed."""
    B = logmag.shape[-1]
    n_fir = 2 * (B - 1)
    zero_phase = torch.fft.irfft(torch.exp(logmag).to(torch.complex128
                                                       if logmag.dtype == torch.float64
                                                       else torch.complex64),
                                 n=n_fir, dim=-1)
    centered = torch.roll(zero_phase, B - 1, dims=-1)
    window = _on_device(("hann", n_fir), lambda: torch.as_tensor(np.hanning(n_fir)),
                        logmag.device, logmag.dtype)
    return centered * window


def _frame_index(plan, n_out, F, device):
    """Per-frame (row, sample index into [0, n_out) or -1) of plan.iter_frames
    (cached per grid and device)."""
    key = ("frames", plan.frame_size, plan.hop, n_out, F)
    rows = _on_device(key + ("rows",), lambda: _frame_index_host(plan, n_out, F)[0], device, None)
    idx = _on_device(key + ("idx",), lambda: _frame_index_host(plan, n_out, F)[1], device, None)
    return rows, idx


def _frame_index_host(plan, n_out, F):
    size = plan.frame_size
    rows, idx = [], []
    for row, sig_lo, sig_hi, win_lo, win_hi in plan.iter_frames(n_out, F):
        ix = np.full(size, -1, dtype=np.int64)
        ix[win_lo:win_hi] = np.arange(sig_lo, sig_hi)
        rows.append(row)
        idx.append(ix)
    return torch.as_tensor(np.array(rows)), torch.as_tensor(np.stack(idx))


def _frame_starts(plan, n_out, F):
    """Sample index of frame 0's window start: plan.iter_frames yields every
    frame from -n_lead_in to F - 1 at hop spacing (params.py:163-171)."""
    return -plan.n_lead_in() * plan.hop


def _row_ranges(plan, n_out, F, device):
    """int32 FIR row of every frame (nondecreasing: lead-in frames share row
    0) and, per row, the first frame using it ([F + 1])."""
    key = ("rowranges", plan.frame_size, plan.hop, n_out, F)

    def build(which):
        rows = np.asarray(_frame_index_host(plan, n_out, F)[0], dtype=np.int64)
        if which == 0:
            return torch.as_tensor(rows.astype(np.int32))
        return torch.as_tensor(np.searchsorted(rows, np.arange(F + 1)).astype(np.int32))
    return (_on_device(key + (0,), lambda: build(0), device, None),
            _on_device(key + (1,), lambda: build(1), device, None))


class _SpecMulB200(torch.autograd.Function):
    """S[b, i] * H[b, rows[i]] (the FFT-convolution product of shape_noise,
    source.py:404-412) on tvlp_spectra_mul without gathering H's rows; the
    VJP to H (the noise spectra S carry no gradient) on tvlp_spectra_mul_vjp."""

    @staticmethod
    def forward(ctx, S, H, rows, first):
        lib = N.load()
        S, H = S.contiguous(), H.contiguous()
        Bn, nfr, K = S.shape
        P = torch.empty_like(S)
        with N.on_device(S.device):
            N.check(lib.tvlp_spectra_mul(N.ptr(S), N.ptr(H), N.ptr(rows), N.ptr(P), Bn, nfr,
                                         H.shape[1], K, N.stream_ptr(S.device)))
        ctx.save_for_backward(S, first)
        ctx.F = H.shape[1]
        return P

    @staticmethod
    def backward(ctx, gP):
        S, first = ctx.saved_tensors
        lib = N.load()
        gP = gP.contiguous()
        Bn, nfr, K = S.shape
        gH = torch.empty((Bn, ctx.F, K), dtype=S.dtype, device=S.device)
        with N.on_device(S.device):
            N.check(lib.tvlp_spectra_mul_vjp(N.ptr(gP), N.ptr(S), N.ptr(first), N.ptr(gH), Bn, nfr,
                                             ctx.F, K, N.stream_ptr(S.device)))
        return None, gH, None, None


class _FrameOLAB200(torch.autograd.Function):
    """shape_noise's overlap-add of the filtered frames, read from the FIR's
    delay on, / COLA (source.py:418-428), as a fixed-order gather
    (tvlp_frame_ola) and its adjoint."""

    @staticmethod
    def forward(ctx, y, n_out, size, delay, start0, hop, scale):
        lib = N.load()
        y = y.contiguous()
        Bn, nfr, ld = y.shape
        out = torch.empty((Bn, n_out), dtype=y.dtype, device=y.device)
        with N.on_device(y.device):
            N.check(lib.tvlp_frame_ola(N.ptr(y), N.ptr(out), Bn, n_out, nfr, size, ld, delay,
                                       start0, hop, scale, 0, N.stream_ptr(y.device)))
        ctx.cfg = (Bn, nfr, ld, n_out, size, delay, start0, hop, scale)
        return out

    @staticmethod
    def backward(ctx, g):
        Bn, nfr, ld, n_out, size, delay, start0, hop, scale = ctx.cfg
        lib = N.load()
        g = g.contiguous()
        gy = torch.empty((Bn, nfr, ld), dtype=g.dtype, device=g.device)
        with N.on_device(g.device):
            N.check(lib.tvlp_frame_ola(N.ptr(g), N.ptr(gy), Bn, n_out, nfr, size, ld, delay,
                                       start0, hop, scale, 1, N.stream_ptr(g.device)))
        return gy, None, None, None, None, None, None


def shape_noise(logmag, noise, plan):
    """source.py:367-428 for [B, F, 256] log-magnitudes and [B, n_out] unit
    noise: each windowed noise frame convolved with its frame's FIR (the
    centred part, delay 255), overlap-added, / COLA constant."""
    Bn, F, nb = logmag.shape
    if nb != NOISE_BINS:
        raise ValueError(f"noise filter frames must be (F, {NOISE_BINS})")
    n_out = noise.shape[-1]
    if F != (n_out - 1) // plan.hop + 1:
        raise ValueError(f"got {F} noise filter frames but length {n_out} at hop {plan.hop}")
    size = plan.frame_size
    delay = NOISE_BINS - 1
    dev, dt = logmag.device, logmag.dtype
    rows, idx = _frame_index(plan, n_out, F, dev)
    fir = fir_from_logmag(logmag)                                 # [B, F, 510]
    win = plan._window_tensor(dt, dev)
    n_fir = fir.shape[-1]
    nfft = 1 << (size + n_fir - 2).bit_length()
    start0 = _frame_starts(plan, n_out, F)
    if (_b200_pieces(logmag) and noise.dtype == dt and not noise.requires_grad
            and rows.shape[0] == plan.n_lead_in() + F):
        # framing (+ zero pad to nfft) and the overlap-add on the kernels of
        # csrc/decoder_kernels.cu; the spectra stay cuFFT
        lib = N.load()
        noise = noise.contiguous()
        nfr = rows.shape[0]
        segs = torch.empty((Bn, nfr, nfft), dtype=dt, device=dev)
        with N.on_device(dev):
            N.check(lib.tvlp_noise_frames(N.ptr(noise), N.ptr(win), N.ptr(segs), Bn, n_out, nfr,
                                          size, nfft, start0, plan.hop, N.stream_ptr(dev)))
        rows32, first32 = _row_ranges(plan, n_out, F, dev)
        spec = _SpecMulB200.apply(torch.fft.rfft(segs), torch.fft.rfft(fir, n=nfft), rows32,
                                  first32)
        y = torch.fft.irfft(spec, n=nfft)                         # [B, nfr, nfft]
        return _FrameOLAB200.apply(y, n_out, size, delay, start0, plan.hop,
                                   1.0 / plan._cola_cached())
    valid = idx >= 0
    segs = torch.where(valid, noise[:, idx.clamp(min=0)], torch.zeros((), dtype=dt, device=dev))
    segs = segs * win                                            # [B, nfr, size]
    spec = torch.fft.rfft(segs, n=nfft) * torch.fft.rfft(fir[:, rows], n=nfft)
    y = torch.fft.irfft(spec, n=nfft)[..., delay:delay + size]   # [B, nfr, size]
    out = torch.zeros((Bn, n_out + 1), dtype=dt, device=dev)     # (slot n_out: padding)
    tgt = torch.where(valid, idx, torch.full_like(idx, n_out))
    # frames f, f + nc, f + 2nc, ... never overlap: nc collision-free (hence
    # deterministic) scatter-adds
    nc = -(-size // plan.hop)
    for j in range(nc):
        out = out.index_add(1, tgt[j::nc].reshape(-1), y[:, j::nc].reshape(Bn, -1))
    return out[:, :n_out] / plan._cola_cached()


class _GlobalFIRB200(torch.autograd.Function):
    """source.py:445-466 on the kernels of csrc/decoder_kernels.cu
    (tvlp_global_fir / tvlp_global_fir_vjp), float32."""

    @staticmethod
    def forward(ctx, x, taps):
        lib = N.load()
        Bn, n = x.shape
        y = torch.empty_like(x)
        with N.on_device(x.device):
            N.check(lib.tvlp_global_fir(N.ptr(x), N.ptr(taps), N.ptr(y), Bn, n, taps.shape[-1],
                                        N.stream_ptr(x.device)))
        ctx.save_for_backward(x, taps)
        return y

    @staticmethod
    def backward(ctx, g):
        x, taps = ctx.saved_tensors
        lib = N.load()
        Bn, n = x.shape
        m = taps.shape[-1]
        g = g.contiguous()
        gx = torch.empty_like(x) if ctx.needs_input_grad[0] else None
        gt = torch.empty_like(taps) if ctx.needs_input_grad[1] else None
        nb = lib.tvlp_global_fir_workspace(Bn, n, m)
        ws = torch.empty(max(nb, 4) // 4, dtype=torch.float32, device=x.device)
        with N.on_device(x.device):
            N.check(lib.tvlp_global_fir_vjp(N.ptr(g), N.ptr(x), N.ptr(taps),
                                            N.ptr(gx) if gx is not None else None,
                                            N.ptr(gt) if gt is not None else None,
                                            N.ptr(ws), nb, Bn, n, m, N.stream_ptr(x.device)))
        return gx, gt


def global_fir(x, taps):
    """source.py:445-459: causal same-length convolution, x [B, n], taps [B, m]
    (float32 CUDA tensors: the kernels of csrc/decoder_kernels.cu)."""
    Bn, n = x.shape
    m = taps.shape[-1]
    if _b200_pieces(x) and taps.dtype == torch.float32 and 1 <= m <= 1024 and taps.shape == (Bn, m):
        return _GlobalFIRB200.apply(x.contiguous(), taps.contiguous())
    xp = TF.pad(x, (m - 1, 0))
    # grouped conv: one filter per item (the taps are per-item parameters)
    y = TF.conv1d(xp[None], taps.flip(-1)[:, None], groups=Bn)
    return y[0, :, :n]


def stft_mag(x, size, hop=None, window=None):
    """loss.py:53-65: reflect-padded centred frames, raised-cosine window,
    |rfft| at the native size (cuFFT handles the prime sizes).  x [B, n]."""
    if hop is None:
        hop = -(-size // 4)
    if x.shape[-1] < size:
        raise ValueError(f"signal of length {x.shape[-1]} is shorter than one {size}-sample frame")
    if window is None:
        window = 0.5 - 0.5 * torch.cos(2.0 * math.pi * torch.arange(size, dtype=x.dtype,
                                                                  device=x.device) / size)
    xp = TF.pad(x[:, None], (size // 2, size // 2), mode="reflect")[:, 0]
    frames = xp.unfold(-1, size, hop) * window
    return torch.abs(torch.fft.rfft(frames, dim=-1))


def _hann_periodic(size, device, dtype):
    return _on_device(("hann_periodic", size),
                      lambda: 0.5 - 0.5 * torch.cos(2.0 * math.pi * torch.arange(
                          size, dtype=torch.float64) / size), device, dtype)


class _SpectrumB200(torch.autograd.Function):
    """One-sided spectra of stft_mag's windowed, reflect-padded frames
    (loss.py:46-63): the framing on tvlp_stft_frames, the DFT on cuFFT; the
    VJP is the reference's adjoint (loss.py:74-86): one c2r inverse FFT of
    the one-sided gradient (bins >= 1 halved: irfft doubles them) and
    tvlp_stft_frames_vjp's windowed overlap-add through the pads."""

    @staticmethod
    def forward(ctx, x, size, hop):
        lib = N.load()
        x = x.contiguous()
        B, n = x.shape
        nfr = lib.tvlp_stft_nframes(n, size, hop)
        win = _hann_periodic(size, x.device, x.dtype)
        fr = torch.empty((B, nfr, size), dtype=x.dtype, device=x.device)
        with N.on_device(x.device):
            N.check(lib.tvlp_stft_frames(N.ptr(x), N.ptr(win), N.ptr(fr), B, n, size, hop,
                                         N.stream_ptr(x.device)))
        ctx.cfg = (B, n, size, hop)
        return torch.fft.rfft(fr, dim=-1)

    @staticmethod
    def backward(ctx, gX):
        B, n, size, hop = ctx.cfg
        lib = N.load()
        gX = gX.contiguous()
        win = _hann_periodic(size, gX.device, torch.float32)
        gx = torch.empty((B, n), dtype=torch.float32, device=gX.device)
        if size % 2:
            # odd N: sum_k Re(g_k e^{i theta}) over the one-sided bins is
            # (N/2) irfft(g) + Re(g_0)/2 (irfft doubles bins >= 1), so the
            # inverse FFT takes the gradient as is and the DC term rides in
            # the overlap-add kernel
            gfr = torch.fft.irfft(gX, n=size, dim=-1).contiguous()
            dc = torch.view_as_real(gX)[..., 0, 0]             # Re(g_0) per frame (view)
            with N.on_device(gX.device):
                N.check(lib.tvlp_stft_frames_vjp(N.ptr(gfr), N.ptr(win), N.ptr(gx), B, n, size,
                                                 hop, 0.5 * size, N.ptr(dc), 2 * gX.shape[-1],
                                                 0.5, N.stream_ptr(gX.device)))
            return gx, None, None
        half = _on_device(("rfft_adjoint_scale", size), lambda: torch.tensor(
            [1.0] + [0.5] * ((size - 1) // 2) + [1.0]), gX.device, torch.float32)
        gfr = torch.fft.irfft(gX * half, n=size, dim=-1).contiguous()
        with N.on_device(gX.device):
            N.check(lib.tvlp_stft_frames_vjp(N.ptr(gfr), N.ptr(win), N.ptr(gx), B, n, size, hop,
                                             float(size), None, 0, 0.0, N.stream_ptr(gX.device)))
        return gx, None, None


class _MSSTermsB200(torch.autograd.Function):
    """One FFT size's loss terms from the spectra (tvlp_mss_terms /
    tvlp_mss_terms_vjp, csrc/decoder_kernels.cu): magnitudes, both norms, the
    log-magnitude mean and their VJP in two passes instead of the ~25
    elementwise ops of the torch graph; the FFTs stay cuFFT."""

    @staticmethod
    def forward(ctx, X, Y, eps):
        lib = N.load()
        X, Y = X.contiguous(), Y.contiguous()
        B = X.shape[0]
        n = X.numel() // B
        term = torch.empty(B, dtype=torch.float32, device=X.device)
        aux = torch.empty(B * 4, dtype=torch.float32, device=X.device)
        nb = lib.tvlp_mss_terms_workspace(B, n)
        ws = torch.empty(max(nb, 4) // 4, dtype=torch.float32, device=X.device)
        with N.on_device(X.device):
            N.check(lib.tvlp_mss_terms(N.ptr(X), N.ptr(Y), B, n, float(eps), N.ptr(term),
                                       N.ptr(aux), N.ptr(ws), nb, N.stream_ptr(X.device)))
        ctx.save_for_backward(X, Y, aux)
        ctx.eps = float(eps)
        return term

    @staticmethod
    def backward(ctx, g):
        X, Y, aux = ctx.saved_tensors
        lib = N.load()
        B = X.shape[0]
        n = X.numel() // B
        g = g.contiguous()
        gX = torch.empty_like(X)
        with N.on_device(X.device):
            N.check(lib.tvlp_mss_terms_vjp(N.ptr(X), N.ptr(Y), N.ptr(aux), N.ptr(g), N.ptr(gX), B,
                                           n, ctx.eps, N.stream_ptr(X.device)))
        return gX, None, None


def mss_loss(x, y, fft_sizes=DEFAULT_FFT_SIZES, eps=LOG_EPS):
    """loss.py:105-126, per item: mean over sizes of spectral convergence +
    mean |log-magnitude difference|; returns [B] losses.  float32 CUDA
    signals compute the terms on tvlp_mss_terms (the spectra on cuFFT)."""
    if _b200_pieces(x) and x.dim() == 2 and y.shape == x.shape:
        total = 0.0
        yd = y.detach().to(x.dtype)
        for size in fft_sizes:
            hop = -(-size // 4)
            if x.shape[-1] < size:
                raise ValueError(f"signal of length {x.shape[-1]} is shorter than one "
                                 f"{size}-sample frame")
            with torch.no_grad():
                Y = _SpectrumB200.apply(yd, size, hop)
            total = total + _MSSTermsB200.apply(_SpectrumB200.apply(x, size, hop), Y, eps)
        return total / len(fft_sizes)
    total = 0.0
    for size in fft_sizes:
        hop = -(-size // 4)
        xm = stft_mag(x, size, hop)
        ym = stft_mag(y, size, hop).detach()
        ynorm = torch.clamp(torch.sqrt(torch.sum(ym * ym, dim=(-2, -1))), min=1e-12)
        sc = torch.sqrt(torch.sum((xm - ym) ** 2, dim=(-2, -1))) / ynorm
        la = torch.mean(torch.abs(torch.log(xm + eps) - torch.log(ym + eps)), dim=(-2, -1))
        total = total + sc + la
    return total / len(fft_sizes)


class _SourcePairB200(torch.autograd.Function):
    """The HpN LP pair's inputs [2B, Tp] -- H (sig V) over N G, zero past T1
    -- in one kernel (tvlp_source_pair) from the gain FRAMES, and the VJP to
    sig, noise and the three gain frame tensors (tvlp_source_pair_vjp)."""

    @staticmethod
    def forward(ctx, sig, noise, vg, ng, hg, hop, Tp):
        lib = N.load()
        sig, noise = sig.contiguous(), noise.contiguous()
        vg, ng, hg = vg.contiguous(), ng.contiguous(), hg.contiguous()
        Bn, T1 = sig.shape
        F = vg.shape[1]
        out = torch.empty((2 * Bn, Tp), dtype=sig.dtype, device=sig.device)
        with N.on_device(sig.device):
            N.check(lib.tvlp_source_pair(N.ptr(sig), N.ptr(noise), N.ptr(vg), N.ptr(ng), N.ptr(hg),
                                         N.ptr(out), Bn, T1, F, hop, Tp,
                                         N.stream_ptr(sig.device)))
        ctx.save_for_backward(sig, noise, vg, ng, hg)
        ctx.cfg = (hop, Tp)
        return out

    @staticmethod
    def backward(ctx, g):
        sig, noise, vg, ng, hg = ctx.saved_tensors
        hop, Tp = ctx.cfg
        lib = N.load()
        g = g.contiguous()
        Bn, T1 = sig.shape
        F = vg.shape[1]
        gs, gn = torch.empty_like(sig), torch.empty_like(noise)
        gv, gng, gh = torch.empty_like(vg), torch.empty_like(ng), torch.empty_like(hg)
        ws = torch.empty(6 * Bn * F, dtype=torch.float32, device=sig.device)
        with N.on_device(sig.device):
            N.check(lib.tvlp_source_pair_vjp(N.ptr(g), N.ptr(sig), N.ptr(noise), N.ptr(vg),
                                             N.ptr(ng), N.ptr(hg), N.ptr(gs), N.ptr(gn), N.ptr(gv),
                                             N.ptr(gng), N.ptr(gh), N.ptr(ws), Bn, T1, F, hop, Tp,
                                             N.stream_ptr(sig.device)))
        return gs, gn, gv, gng, gh, None, None


class _StackPad(torch.autograd.Function):
    """Rows of [B_i, T] tensors stacked into one [sum B_i, Tp] buffer, zero
    past T (one copy, like torch.cat); the VJP slices the gradient back."""

    @staticmethod
    def forward(ctx, Tp, *xs):
        T = xs[0].shape[1]
        out = xs[0].new_empty((sum(x.shape[0] for x in xs), Tp))
        r = 0
        for x in xs:
            out[r:r + x.shape[0], :T].copy_(x)
            r += x.shape[0]
        out[:, T:].zero_()
        ctx.rows = [x.shape[0] for x in xs]
        ctx.T = T
        return out

    @staticmethod
    def backward(ctx, g):
        outs, r = [], 0
        for n in ctx.rows:
            outs.append(g[r:r + n, :ctx.T])
            r += n
        return (None, *outs)


def _lp_frames(xs, frames, hop):
    """The frame-rate LP (autograd.lp_tv_frames) of the rows of ``xs`` stacked
    as one batch.  The signals are laid out at a length Tp >= T that is a
    multiple of the hop with the same frame count (48001 -> 48240 at hop 240,
    zeros after T; the causal filter's first T outputs and, with a zero
    gradient on the tail, their VJP are unchanged), so the C ABI finds a
    sub-chunk plan without its pack/unpack copies; the output is [:, :T]."""
    T = xs[0].shape[1]
    Tp = -(-T // hop) * hop
    if Tp == T or (Tp - 1) // hop != (T - 1) // hop:
        return ag.lp_tv_frames(xs[0] if len(xs) == 1 else torch.cat(xs), frames, hop)
    return ag.lp_tv_frames(_StackPad.apply(Tp, *xs), frames, hop)[:, :T]


@dataclass
class Decoder:
    """The reference decoder graph (synth.py:217-275) in torch on the GPU.

    ``tables`` [K, L] wavetable rows (source.py:57-208 builds them; data here),
    ``mode`` "sf" or "hpn"; ``c_lp=True`` (HpN only) filters the shaped noise
    with an all-pole C(z) too -- the paper's GOLF-v1 form the
    reference does not implement -- with the H(z) and C(z)
    filters in ONE launch sequence (frame rows stacked as 2B sequences)."""

    tables: torch.Tensor
    hop: int = 240
    fs: float = 24000.0
    mode: str = "sf"
    oversample: int = 4
    c_lp: bool = False
    framewise: bool = False   # SF with the frame-wise TI LP (synth.render_framewise)

    def __post_init__(self):
        self.plan = None

    def _plan(self):
        from .params import FramePlan

        if self.plan is None:
            self.plan = FramePlan.raised_cosine(self.hop)
        return self.plan

    def render(self, p, n_out, noise, f0_frames, c_frames=None):
        """p: dict of [B, ...] parameter tensors (reflection_raw, table_pos_raw,
        voiced_gain_raw, noise_gain_raw, h_gain_raw, noise_logmag, fir_taps);
        noise [B, n_out] unit noise; f0_frames [B, F] (no unvoiced zeros).
        Returns the output signal [B, n_out]."""
        hop, T1 = self.hop, n_out
        K = self.tables.shape[0]
        k = SQUASH_LIMIT * torch.tanh(p["reflection_raw"])
        a_frames = ag.reflection_to_lpc(k)
        pos = torch.sigmoid(p["table_pos_raw"]) * (K - 1)
        vgain = torch.exp(p["voiced_gain_raw"])
        # oscillator (source.py:294-314)
        sig = wavetable_osc(pos, f0_frames, self.tables, hop, n_out, self.fs, self.oversample)
        noise_unit = shape_noise(p["noise_logmag"], noise.to(pos.dtype), self._plan())
        if self.mode == "hpn" and self.c_lp and _b200_pieces(sig):
            Tp = -(-T1 // hop) * hop
            if (Tp - 1) // hop == (T1 - 1) // hop:
                # both LP inputs, gains applied, in one kernel (no gain tracks)
                Bn = sig.shape[0]
                e2 = _SourcePairB200.apply(sig, noise_unit, vgain, torch.exp(p["noise_gain_raw"]),
                                           torch.exp(p["h_gain_raw"]), hop, Tp)
                sc = ag.lp_tv_frames(e2, torch.cat([a_frames, c_frames.to(a_frames.dtype)]),
                                     hop)[:, :T1]
                return global_fir(sc[:Bn] + sc[Bn:], p["fir_taps"])
        osc = sig * upsample_linear(vgain, hop, T1)
        noise_s = noise_unit * upsample_linear(torch.exp(p["noise_gain_raw"]), hop, T1)
        hgain = upsample_linear(torch.exp(p["h_gain_raw"]), hop, T1)
        if self.mode == "sf":
            if self.framewise:
                s = ag.framewise(hgain * (osc + noise_s), a_frames, self._plan())
            else:
                s = _lp_frames([hgain * (osc + noise_s)], a_frames, hop)
            return global_fir(s, p["fir_taps"])
        if self.c_lp:
            # H(z) on the glottal source and C(z) on the noise in ONE launch
            # sequence: both filters' frame rows stacked as a batch of 2B
            # (frame rows are small; the rows are interpolated inside the
            # kernels, so no sample-rate track is materialised -- the
            # sample-rate grouped entry point, lp_tv_grouped, serves callers
            # that hold [B, T, M] tracks)
            Bn = osc.shape[0]
            sc = _lp_frames([hgain * osc, noise_s],
                            torch.cat([a_frames, c_frames.to(a_frames.dtype)]), hop)
            return global_fir(sc[:Bn] + sc[Bn:], p["fir_taps"])
        s = _lp_frames([hgain * osc], a_frames, hop)
        return global_fir(s + noise_s, p["fir_taps"])


# ---------------------------------------------------------------- synthetic inputs
FIELDS = ("reflection_raw", "table_pos_raw", "voiced_gain_raw", "noise_gain_raw", "h_gain_raw",
          "noise_logmag", "fir_taps")


def synthetic_tables(K=9, L=512):
    """K smooth one-period waveforms of L samples (harmonic series with a
    spectral tilt growing with the row: a stand-in for the LF wavetable rows
    source.py:57-208 builds; the tables are data here), float64 [K, L]."""
    n = np.arange(L) / L
    rows = []
    for k in range(K):
        tilt = 0.3 + 0.25 * k
        h = np.arange(1, 40)
        amp = h ** (-1.0 - tilt)
        w = (amp[:, None] * np.sin(2 * np.pi * h[:, None] * n[None, :] + 0.1 * h[:, None])).sum(0)
        rows.append(w / np.abs(w).max())
    return np.stack(rows)


def synthetic_inputs(B, n_out, hop=240, seed=0, order=22):
    """Decoder inputs for B items of n_out samples (numpy float64): the
    trainable fields [B, ...] in the ranges of a fitted voice (the golden
    fixtures' generator, tests/golden/make_golden_decoder.py) with the
    reflection frames of distribution D1 (a smooth AR(1)
    walk, as the LP benchmarks use), f0 frames [B, F], the reference's noise
    stream per item [B, n_out] and a target."""
    from .data import d1_reflection_raw

    F = (n_out - 1) // hop + 1
    rng = np.random.default_rng(seed)
    f = {
        "reflection_raw": np.stack([d1_reflection_raw(1000 * seed + b, n_out, order, hop)
                                    for b in range(B)]),
        "table_pos_raw": rng.normal(0.0, 1.0, size=(B, F)),
        "voiced_gain_raw": rng.normal(-1.0, 0.3, size=(B, F)),
        "noise_gain_raw": rng.normal(-2.5, 0.3, size=(B, F)),
        "h_gain_raw": rng.normal(-0.5, 0.2, size=(B, F)),
        "noise_logmag": rng.normal(0.0, 0.5, size=(B, F, NOISE_BINS)),
        "fir_taps": np.concatenate([np.ones((B, 1)), 0.05 * rng.standard_normal((B, FIR_TAPS - 1))],
                                   axis=1),
    }
    f0 = np.linspace(110.0, 190.0, F)[None] * (1 + 0.05 * rng.standard_normal((B, F)))
    noise = np.stack([generate_noise(n_out, seed + b) for b in range(B)])
    target = 0.3 * rng.standard_normal((B, n_out))
    return f, f0, noise, target


def stable_c_frames(B, F, seed=0, order=22):
    """A C(z) all-pole track for the GOLF-v1 noise filter (c_lp=True): step-up
    of squashed small reflection rows (stable), float64 [B, F, order]."""
    from .data import reflection_to_lpc

    rng = np.random.default_rng(seed + 7)
    k = 0.999 * np.tanh(rng.normal(0.0, 0.2, size=(B * F, order)))
    return reflection_to_lpc(k).reshape(B, F, order)


class GraphedStep:
    """One decoder training step -- render, MSS loss, backward to every
    parameter -- captured in a CUDA graph over static device buffers
    (streams and graphs instead of a tracing compiler).
    ``replay()`` re-runs every kernel of the step (the LP kernels, cuFFT, the
    autograd backward) with no host work; write new inputs into
    ``params[k]`` / ``noise`` / ``target`` / ``f0`` in place first.  Outputs:
    ``y``, ``loss`` [B] and ``params[k].grad``."""

    def __init__(self, dec, params, noise, target, f0, c_frames=None, warmup=3):
        self.dec, self.params, self.noise, self.target = dec, params, noise, target
        self.f0 = torch.as_tensor(f0, dtype=torch.float64, device=noise.device)
        self.c_frames = c_frames
        self.n_out = noise.shape[-1]
        side = torch.cuda.Stream(device=noise.device)
        side.wait_stream(torch.cuda.current_stream(noise.device))
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self._run()
        torch.cuda.current_stream(noise.device).wait_stream(side)
        from . import _native

        lib = _native.load()
        n0 = lib.tvlp_launch_count()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.y, self.loss = self._run()
        # this library's kernel launches captured in the graph (each replay
        # runs them all; the host-side counter only sees the capture)
        self.launches = int(lib.tvlp_launch_count() - n0)

    def _run(self):
        for t in self.params.values():
            t.grad = None
        y = self.dec.render(self.params, self.n_out, self.noise, self.f0, self.c_frames)
        L = mss_loss(y, self.target)
        L.sum().backward()
        return y, L

    def replay(self):
        self.graph.replay()
        return self.y, self.loss
