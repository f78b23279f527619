"""torch profiler table of decoder.shape_noise fwd+bwd (B=32, float32)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_05128_b200 import decoder  # noqa: E402
from paper_2406_05128_b200.params import FramePlan  # noqa: E402

B, n_out, hop = 32, 48001, 240
F = (n_out - 1) // hop + 1
lm = (0.1 * torch.randn(B, F, 256, device="cuda")).requires_grad_(True)
noise = torch.randn(B, n_out, device="cuda")
plan = FramePlan.raised_cosine(hop)


def step():
    lm.grad = None
    decoder.shape_noise(lm, noise, plan).sum().backward()


for _ in range(3):
    step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=25))
