"""Time stream.lp_tv_fwd_bwd_host on config 3 for several chunk schedules."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_05128_b200 import data, lpc, stream
lpc.set_validation("lazy")
B, T, M = 64, 48000, 22
e, A, g = data.d1_batch_torch(0, B, T, M, device="cuda")
eh, Ah, gh = (x.cpu().pin_memory() for x in (e, A, g))
oh = tuple(torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in (e, e, A))
scheds = {
    "u8": 8,
    "h26": [2, 6] + [8] * 7,
    "h134": [1, 3, 4] + [8] * 7,
    "h44": [4, 4] + [8] * 7,
    "h224": [2, 2, 4] + [8] * 7,
    "h26t": [2, 6] + [8] * 6 + [6, 2],
    "h2": [2] * 4 + [8] * 7,
}
for rep in range(2):
    for name, ch in scheds.items():
        for _ in range(2):
            stream.lp_tv_fwd_bwd_host(eh, Ah, gh, out=oh, chunks=ch)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            stream.lp_tv_fwd_bwd_host(eh, Ah, gh, out=oh, chunks=ch)
        b.record(); torch.cuda.synchronize()
        print(name, round(a.elapsed_time(b) / 5, 3), "ms", flush=True)
