"""One frame-rate TV fwd+bwd of config 3 (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_05128_b200 import data, lpc
lpc.set_validation("off")
ev, fr, gv = data.d1_frames_batch(0, 64, 48000, 22, 240)
e, F, g = (torch.from_numpy(x).cuda() for x in (ev, fr, gv))
for _ in range(2):
    s, carry = lpc.lp_forward_tv_frames(e, F, 240, return_carry=True)
    ge, gf = lpc.lp_backward_tv_frames(g, F, 240, s, carry=carry)
torch.cuda.synchronize()
print("ok")
