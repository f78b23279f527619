"""Synthetic inputs for parity tests and the benchmark.

Distribution D1 mirrors how the reference synthesiser builds its coefficient
track (synth.py:244-245, 268): a frame-smooth reflection walk (the
``_smooth_track`` of pkg/tests/test_acceptance.py:122-131 with std 0.25 plus
N(0, 0.02) jitter), squashed by ``0.999*tanh`` (params.py:34-36), converted by
the step-up recursion (params.py:43-71) and linearly upsampled to the sample
rate (params.py:107-132).  The stress set is the reference's resonant constant
row, ``oracle.random_stable_track(rng, T, M, n_frames=1)`` (oracle.py:237-249).

The step-up and upsample restatements here are pinned bit-exactly against the
reference by tests/golden/golden_d1.npz.  Inputs are produced in float64 and
cast to float32 once; parity tests feed the SAME float32 values (upcast) to
the float64 oracle.
"""
from __future__ import annotations

import numpy as np

SQUASH_LIMIT = 0.999  # params.py:31


def reflection_to_lpc(k):
    """Step-up recursion, params.py:43-71 (float64, ``(..., M)``)."""
    k = np.asarray(k, dtype=np.float64)
    a = k[..., :1].copy()
    for m in range(2, k.shape[-1] + 1):
        km = k[..., m - 1: m]
        a = np.concatenate([a + km * a[..., ::-1], km], axis=-1)
    return a


def upsample_weights(F, hop, T1):
    """params.py:107-117 for a signal of ``T1`` samples (reference T = T1-1)."""
    t = np.arange(T1)
    f0 = t // hop
    w = (t - f0 * hop) / float(hop)
    f1 = np.minimum(f0 + 1, F - 1)
    w[f0 == F - 1] = 0.0
    return f0, f1, w


def upsample_linear(frames, hop, T1):
    """params.py:120-132: ``(F, D)`` frame controls -> ``(T1, D)`` samples."""
    frames = np.asarray(frames)
    f0, f1, w = upsample_weights(frames.shape[0], hop, T1)
    wcol = w[:, None]
    return (1.0 - wcol) * frames[f0] + wcol * frames[f1]


def frame_count(T1, hop):
    """params.py:102-104 with T = T1-1."""
    return (T1 - 1) // hop + 1


def d1_reflection_raw(seed, T1, M, hop=240, rho=0.95, std=0.25, jitter=0.02):
    """Raw (pre-squash) reflection frames of distribution D1."""
    rng = np.random.default_rng(seed)
    F = frame_count(T1, hop)
    x = np.zeros((F, M))
    x[0] = rng.normal(0, std, M)
    innov = std * np.sqrt(1 - rho ** 2)
    for f in range(1, F):
        x[f] = rho * x[f - 1] + rng.normal(0, innov, M)
    return x + rng.normal(0, jitter, (F, M))


def d1_frames(seed, T1, M, hop=240):
    """Frame-rate LPC rows (float64) of D1 item ``seed``."""
    k = SQUASH_LIMIT * np.tanh(d1_reflection_raw(seed, T1, M, hop))
    return reflection_to_lpc(k)


def d1_item(seed, T1, M=22, hop=240, dtype=np.float32):
    """One D1 item: (e, A, grad_s), A = upsample(step_up(squash(walk)))."""
    a_frames = d1_frames(seed, T1, M, hop)
    A = upsample_linear(a_frames, hop, T1).astype(dtype)
    rng = np.random.default_rng(seed + 1_000_003)
    e = rng.standard_normal(T1).astype(dtype)
    g = rng.standard_normal(T1).astype(dtype)
    return e, A, g


def d1_batch(base_seed, B, T1, M=22, hop=240, dtype=np.float32):
    """D1 batch [B, T1], [B, T1, M], [B, T1]; item b uses seed base+b."""
    e = np.empty((B, T1), dtype=dtype)
    A = np.empty((B, T1, M), dtype=dtype)
    g = np.empty((B, T1), dtype=dtype)
    for b in range(B):
        e[b], A[b], g[b] = d1_item(base_seed + b, T1, M, hop, dtype)
    return e, A, g


def d1_frames_batch(base_seed, B, T1, M=22, hop=240, dtype=np.float32):
    """Frame-wise config inputs: e [B,T1], frames [B,F,M], grad [B,T1]."""
    F = frame_count(T1, hop)
    e = np.empty((B, T1), dtype=dtype)
    fr = np.empty((B, F, M), dtype=dtype)
    g = np.empty((B, T1), dtype=dtype)
    for b in range(B):
        fr[b] = d1_frames(base_seed + b, T1, M, hop).astype(dtype)
        rng = np.random.default_rng(base_seed + b + 1_000_003)
        e[b] = rng.standard_normal(T1).astype(dtype)
        g[b] = rng.standard_normal(T1).astype(dtype)
    return e, fr, g


def stress_row(seed, M=22):
    """oracle.py:246-249 with n_frames=1: one resonant stable row (float64)."""
    rng = np.random.default_rng(seed)
    return reflection_to_lpc(rng.uniform(-0.9, 0.9, size=(1, M)))[0]


def stress_item(seed, T1, M=22, dtype=np.float32):
    """Constant resonant row held over time (the reference bench's track)."""
    row = stress_row(seed, M)
    A = np.repeat(row[None, :].astype(dtype), T1, axis=0)
    rng = np.random.default_rng(seed + 2_000_003)
    e = rng.standard_normal(T1).astype(dtype)
    g = rng.standard_normal(T1).astype(dtype)
    return e, A, g


def d1_batch_torch(base_seed, B, T1, M=22, hop=240, device="cuda", dtype=None):
    """D1 batch built on ``device`` (large configs): frames on the host in
    float64, upsampled on the device with the same separate mul/add ops as
    params.py:120-132 (no contraction), then cast to float32."""
    import torch

    dtype = torch.float32 if dtype is None else dtype
    F = frame_count(T1, hop)
    t = torch.arange(T1, device=device, dtype=torch.int64)
    f0 = torch.div(t, hop, rounding_mode="floor")
    w = (t - f0 * hop).to(torch.float64) / float(hop)
    f1 = torch.clamp(f0 + 1, max=F - 1)
    w = torch.where(f0 == F - 1, torch.zeros_like(w), w)
    wcol = w[:, None]
    A = torch.empty((B, T1, M), device=device, dtype=dtype)
    e = torch.empty((B, T1), device=device, dtype=dtype)
    g = torch.empty((B, T1), device=device, dtype=dtype)
    chunk = 1 << 22
    for b in range(B):
        fr = torch.from_numpy(d1_frames(base_seed + b, T1, M, hop)).to(device)
        for c0 in range(0, T1, chunk):
            c1 = min(T1, c0 + chunk)
            wc = wcol[c0:c1]
            A[b, c0:c1] = ((1.0 - wc) * fr[f0[c0:c1]] + wc * fr[f1[c0:c1]]).to(dtype)
        gen = torch.Generator(device=device)
        gen.manual_seed(base_seed + b + 1_000_003)
        e[b] = torch.randn(T1, generator=gen, device=device, dtype=torch.float32).to(dtype)
        g[b] = torch.randn(T1, generator=gen, device=device, dtype=torch.float32).to(dtype)
    return e, A, g
