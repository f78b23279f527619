"""The whole decoder training step on the GPU:
Decoder.render (oscillator x4 + decimator, shaped noise, LP on the B200
kernels, global FIR) + the prime-size MSS loss + backward to every
parameter, for B items of n_out samples (fp32), timed with CUDA events.
Prints one JSON line per mode; compare with the reference's own decoder step
on its Tape (tools/integration_e2e.py: ~0.2 s per 48000-sample item, one core).

    python tools/decoder_bench.py [B] [n_out]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_05128_b200 import decoder, lpc  # noqa: E402

FIELDS = ("reflection_raw", "table_pos_raw", "voiced_gain_raw", "noise_gain_raw", "h_gain_raw",
          "noise_logmag", "fir_taps")


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    n_out = int(sys.argv[2]) if len(sys.argv) > 2 else 48001
    lpc.set_validation("lazy")
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden_decoder.npz"))
    hop = 240
    F = (n_out - 1) // hop + 1
    rng = np.random.default_rng(0)
    dev = torch.device("cuda", 0)
    tables = torch.tensor(g["tables"], dtype=torch.float32, device=dev)
    for mode, fw in (("sf", False), ("hpn", False), ("sf", True)):
        dec = decoder.Decoder(tables, hop=hop, fs=float(g["fs"]), mode=mode, framewise=fw)
        shapes = {"reflection_raw": (B, F, 22), "table_pos_raw": (B, F),
                  "voiced_gain_raw": (B, F), "noise_gain_raw": (B, F), "h_gain_raw": (B, F),
                  "noise_logmag": (B, F, g["sf_noise_logmag"].shape[-1]),
                  "fir_taps": (B, g["sf_fir_taps"].shape[-1])}
        p = {}
        for f in FIELDS:
            base = np.asarray(g["sf_" + f], dtype=np.float64)
            if base.ndim and base.shape[0] == g["sf_f0_frames"].shape[0]:  # frame fields: tile F
                reps = (F + base.shape[0] - 1) // base.shape[0]
                base = np.concatenate([base] * reps)[:F]
            arr = np.broadcast_to(base, shapes[f]) + 0.05 * rng.standard_normal(shapes[f])
            p[f] = torch.tensor(arr, dtype=torch.float32, device=dev, requires_grad=True)
        f0 = np.linspace(110.0, 180.0, F)[None].repeat(B, 0)
        noise = torch.tensor(np.stack([decoder.generate_noise(n_out, 3 + b) for b in range(B)]),
                             dtype=torch.float32, device=dev)
        target = torch.randn(B, n_out, device=dev)

        def step():
            for t in p.values():
                t.grad = None
            y = dec.render(p, n_out, noise, f0)
            L = decoder.mss_loss(y, target)
            L.sum().backward()
            return L

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10
        e0.record()
        for _ in range(n):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(json.dumps({"graph": f"decoder.Decoder mode={mode} framewise={fw} + mss_loss + backward",
                          "B": B, "samples_per_item": n_out - 1, "dtype": "float32",
                          "ms_per_step": round(ms, 3),
                          "samples_per_s": round(B * (n_out - 1) / (ms * 1e-3), 1)}), flush=True)


if __name__ == "__main__":
    main()
