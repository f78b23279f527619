"""The full decoder step (bench config hpn_full) eager vs captured in a CUDA
graph (decoder.GraphedStep): us per step and the max |difference| of the
outputs and gradients."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_05128_b200 import decoder as dmod  # noqa: E402
from paper_2406_05128_b200 import lpc  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    lpc.set_validation("lazy")
    dev = torch.device("cuda", 0)
    n_out, hop = 48001, 240
    F = (n_out - 1) // hop + 1
    fields, f0, noise, target = dmod.synthetic_inputs(B, n_out, hop, seed=0)
    dec = dmod.Decoder(torch.tensor(dmod.synthetic_tables(), dtype=torch.float32, device=dev),
                       hop=hop, mode="hpn", c_lp=True)
    P = {k: torch.tensor(v, dtype=torch.float32, device=dev, requires_grad=True)
         for k, v in fields.items()}
    nz = torch.tensor(noise, dtype=torch.float32, device=dev)
    tg = torch.tensor(target, dtype=torch.float32, device=dev)
    f0d = torch.tensor(f0, dtype=torch.float64, device=dev)
    cf = torch.tensor(dmod.stable_c_frames(B, F), dtype=torch.float32, device=dev)

    def eager():
        for t in P.values():
            t.grad = None
        y = dec.render(P, n_out, nz, f0d, cf)
        L = dmod.mss_loss(y, tg)
        L.sum().backward()
        return y, L

    y0, L0 = (t.detach() for t in eager())  # (no eager autograd graph may stay alive:
    g0 = {k: v.grad.clone() for k, v in P.items()}  # its AccumulateGrad nodes pin a stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        eager()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        eager()
    e1.record()
    torch.cuda.synchronize()
    t_eager = e0.elapsed_time(e1) / 10
    for t in P.values():
        t.grad = None
    gs = dmod.GraphedStep(dec, P, nz, tg, f0d, cf)
    y1, L1 = gs.replay()
    torch.cuda.synchronize()
    diff = max(float((y1 - y0).abs().max()), float((L1 - L0).abs().max()),
               max(float((P[k].grad - g0[k]).abs().max()) for k in P))
    e0.record()
    for _ in range(10):
        gs.replay()
    e1.record()
    torch.cuda.synchronize()
    t_graph = e0.elapsed_time(e1) / 10
    print(f"B={B}: eager {t_eager:.3f} ms, graph {t_graph:.3f} ms, max|diff| {diff:.3e}",
          flush=True)


if __name__ == "__main__":
    main()
