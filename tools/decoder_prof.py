"""torch.profiler table of one GPU decoder step (tools/decoder_bench.py's SF step)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import decoder_bench as db  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    import numpy as np
    from paper_2406_05128_b200 import decoder, lpc
    lpc.set_validation("lazy")
    g = np.load(os.path.join(db.ROOT, "tests", "golden", "golden_decoder.npz"))
    n_out, hop = 48001, 240
    F = (n_out - 1) // hop + 1
    dev = torch.device("cuda", 0)
    dec = decoder.Decoder(torch.tensor(g["tables"], dtype=torch.float32, device=dev), hop=hop,
                          fs=float(g["fs"]), mode=(sys.argv[2] if len(sys.argv) > 2 else "sf"),
                          c_lp=len(sys.argv) > 2 and sys.argv[2] == "hpn")
    rng = np.random.default_rng(0)
    shapes = {"reflection_raw": (B, F, 22), "table_pos_raw": (B, F), "voiced_gain_raw": (B, F),
              "noise_gain_raw": (B, F), "h_gain_raw": (B, F),
              "noise_logmag": (B, F, g["sf_noise_logmag"].shape[-1]),
              "fir_taps": (B, g["sf_fir_taps"].shape[-1])}
    p = {f: torch.tensor(0.1 * rng.standard_normal(s), dtype=torch.float32, device=dev,
                         requires_grad=True) for f, s in shapes.items()}
    f0 = np.linspace(110.0, 180.0, F)[None].repeat(B, 0)
    noise = torch.randn(B, n_out, device=dev)
    target = torch.randn(B, n_out, device=dev)

    cf = (torch.tensor(decoder.stable_c_frames(B, F), dtype=torch.float32, device=dev)
          if dec.c_lp else None)
    f0 = torch.tensor(f0, dtype=torch.float64, device=dev)

    def step():
        y = dec.render(p, n_out, noise, f0, cf)
        decoder.mss_loss(y, target).sum().backward()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                            torch.profiler.ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=30))


if __name__ == "__main__":
    main()
