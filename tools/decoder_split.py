"""Device time of the decoder step's pieces at B=32 (float32, CUDA events):
the MSS loss fwd+bwd alone, the noise shaping fwd+bwd alone, the LP pair,
the oscillator, and the whole step -- where the config-5 step's time goes."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_05128_b200 import autograd as ag, decoder, lpc  # noqa: E402
from paper_2406_05128_b200.params import FramePlan  # noqa: E402


def timeit(fn, n=20):
    """(eager us, CUDA-graph replay us) per call."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    eager = round(a.elapsed_time(b) / n * 1e3, 1)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return eager, round(a.elapsed_time(b) / n * 1e3, 1)


def main():
    lpc.set_validation("lazy")
    B, n_out, hop = 32, 48001, 240
    F = (n_out - 1) // hop + 1
    dev = torch.device("cuda", 0)
    out = {}
    y = torch.randn(B, n_out, device=dev, requires_grad=True)
    tgt = torch.randn(B, n_out, device=dev)

    def mss():
        y.grad = None
        decoder.mss_loss(y, tgt).sum().backward()
    out["mss_loss_fwd_bwd"] = timeit(mss)
    for size in decoder.DEFAULT_FFT_SIZES:
        def one(size=size):
            y.grad = None
            decoder.mss_loss(y, tgt, fft_sizes=(size,)).sum().backward()
        out[f"mss_{size}"] = timeit(one)
    lm = (0.1 * torch.randn(B, F, 256, device=dev)).requires_grad_(True)
    noise = torch.randn(B, n_out, device=dev)
    plan = FramePlan.raised_cosine(hop)

    def sn():
        lm.grad = None
        decoder.shape_noise(lm, noise, plan).sum().backward()
    out["shape_noise_fwd_bwd"] = timeit(sn)
    x = torch.randn(2 * B, n_out, device=dev, requires_grad=True)
    fr = torch.tensor(decoder.stable_c_frames(2 * B, F), dtype=torch.float32, device=dev)
    fr.requires_grad_(True)

    def lp():
        x.grad = None
        fr.grad = None
        ag.lp_tv_frames(x, fr, hop).sum().backward()
    out["lp_tv_frames_2B_fwd_bwd"] = timeit(lp)
    tabs = torch.tensor(decoder.synthetic_tables(), dtype=torch.float32, device=dev)
    pos = (torch.rand(B, F, device=dev) * 8).requires_grad_(True)
    f0 = torch.tensor(np.linspace(110.0, 180.0, F)[None].repeat(B, 0), device=dev)

    def osc():
        pos.grad = None
        decoder.wavetable_osc(pos, f0, tabs, hop, n_out, 48000.0).sum().backward()
    out["oscillator_fwd_bwd"] = timeit(osc)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
