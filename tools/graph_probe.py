"""Probe: one LP fwd+bwd step captured in a CUDA graph vs eager launches
(small per-GPU batches of config 3's strong split).  Prints us/step both ways
and the max |difference| of the outputs."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_05128_b200 import data, lpc  # noqa: E402


def step(e, A, g):
    s, carry = lpc._forward(False, e, A, None, return_carry=True)
    ge, gA = lpc._backward(False, g, A, s, None, carry)
    return s, ge, gA


def main():
    lpc.set_validation("lazy")
    for B in [int(x) for x in (sys.argv[1:] or ["8", "16", "32", "64"])]:
        e, A, g = data.d1_batch_torch(0, B, 48000, 22, device="cuda")
        ref = step(e, A, g)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            step(e, A, g)
        ev0.record()
        for _ in range(50):
            step(e, A, g)
        ev1.record()
        torch.cuda.synchronize()
        eager = ev0.elapsed_time(ev1) / 50 * 1e3
        s_ = torch.cuda.Stream()
        s_.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_):
            for _ in range(2):
                step(e, A, g)
        torch.cuda.current_stream().wait_stream(s_)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, capture_error_mode="thread_local"):
            outs = step(e, A, g)
        gr.replay()
        torch.cuda.synchronize()
        diff = max(float((o - r).abs().max()) for o, r in zip(outs, ref))
        for _ in range(3):
            gr.replay()
        ev0.record()
        for _ in range(50):
            gr.replay()
        ev1.record()
        torch.cuda.synchronize()
        graph = ev0.elapsed_time(ev1) / 50 * 1e3
        print(f"B={B}: eager {eager:.1f} us  graph {graph:.1f} us  max|diff| {diff:.3e}",
              flush=True)


if __name__ == "__main__":
    main()
