"""Device time of one fwd+bwd (C ABI, tape reuse) per batch-chunk size at T=48000, M=22."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_05128_b200 import data, lpc
lpc.set_validation("lazy")
T, M = 48000, 22
for B in (1, 2, 4, 8, 16, 32, 64):
    e, A, g = data.d1_batch_torch(0, B, T, M, device="cuda")
    def step():
        s, carry = lpc._forward(False, e, A, None, return_carry=True)
        return lpc.lp_backward_tv(g, A, s, None, carry=carry)
    for _ in range(3): step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): step()
    b.record(); torch.cuda.synchronize()
    print("B", B, round(a.elapsed_time(b) / 10 * 1000, 1), "us", flush=True)
