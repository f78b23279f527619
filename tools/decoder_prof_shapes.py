"""torch profiler of one float32 HpN decoder step grouped by op and input
shape: which torch glue ops (mul, copy_, fill_) remain and on what tensors."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    from paper_2406_05128_b200 import decoder, lpc
    lpc.set_validation("lazy")
    B, n_out, hop = 32, 48001, 240
    F = (n_out - 1) // hop + 1
    dev = torch.device("cuda", 0)
    dec = decoder.Decoder(torch.tensor(decoder.synthetic_tables(), dtype=torch.float32, device=dev),
                          hop=hop, fs=48000.0, mode="hpn", c_lp=True)
    f, f0, noise, target = decoder.synthetic_inputs(B, n_out, hop, seed=0)
    p = {k: torch.tensor(v, dtype=torch.float32, device=dev, requires_grad=True)
         for k, v in f.items()}
    noise = torch.tensor(noise, dtype=torch.float32, device=dev)
    target = torch.tensor(target, dtype=torch.float32, device=dev)
    f0 = torch.tensor(f0, dtype=torch.float64, device=dev)
    cf = torch.tensor(decoder.stable_c_frames(B, F), dtype=torch.float32, device=dev)

    def step():
        for v in p.values():
            v.grad = None
        decoder.mss_loss(dec.render(p, n_out, noise, f0, cf), target).sum().backward()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                            torch.profiler.ProfilerActivity.CUDA],
                                record_shapes=True) as prof:
        step()
        torch.cuda.synchronize()
    print(prof.key_averages(group_by_input_shape=True).table(sort_by="self_cuda_time_total",
                                                             row_limit=40))


if __name__ == "__main__":
    main()
