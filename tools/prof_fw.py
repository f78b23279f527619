"""One framewise fwd+bwd of config 2 (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_05128_b200 import data, params
ev, fr, gv = data.d1_frames_batch(0, 32, 48000, 22, 240)
e, A, g = (torch.from_numpy(x).cuda() for x in (ev, fr, gv))
plan = params.FramePlan.raised_cosine(240)
for _ in range(2):
    y, seg = params.framewise_forward(e, A, plan)
    ge, gf = params.framewise_backward(g, A, seg, plan)
torch.cuda.synchronize()
print("ok")
