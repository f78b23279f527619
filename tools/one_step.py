"""One bench step of a bench.py config between cudaProfilerStart/Stop, after
two warm-up steps: the unit an ncu capture with --profile-from-start off
records (tools/r2_profiles.sh).

    python tools/one_step.py CONFIG [--shard-of S]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2406_05128_b200 import data, dist, lpc, params  # noqa: E402


def make_step(cfg, shard_of=0):
    B, T, M, kind = cfg["B"], cfg["T"], cfg["M"], cfg["kind"]
    if shard_of > 1:
        lo, hi = dist.strong_shard(B, 0, shard_of)
        B = hi - lo
    dev = torch.device("cuda", 0)
    if kind in ("tv", "tvsplit"):
        e, A, g = data.d1_batch_torch(0, B, T, M, device=dev)

        def step():
            s, c = lpc._forward(False, e, A, None, return_carry=True)
            lpc._backward(False, g, A, s, None, c)
    elif kind == "hpn":
        eh, Ah, gh = data.d1_batch_torch(0, B, T, M, device=dev)
        ec, Ac, gc = data.d1_batch_torch(B, B, T, M, device=dev)

        def step():
            (sh, sc), c = lpc.lp_forward_tv_grouped([(eh, Ah), (ec, Ac)], return_carry=True)
            lpc.lp_backward_tv_grouped([(gh, Ah, sh), (gc, Ac, sc)], carry=c)
    elif kind == "tvf":
        ev, fr, gv = data.d1_frames_batch(0, B, T, M, cfg["hop"])
        e, f, g = (torch.from_numpy(x).to(dev) for x in (ev, fr, gv))

        def step():
            s, c = lpc.lp_forward_tv_frames(e, f, cfg["hop"], return_carry=True)
            lpc.lp_backward_tv_frames(g, f, cfg["hop"], s, carry=c)
    else:
        ev, fr, gv = data.d1_frames_batch(0, B, T, M, cfg["hop"])
        e, f, g = (torch.from_numpy(x).to(dev) for x in (ev, fr, gv))
        plan = params.FramePlan.raised_cosine(cfg["hop"])

        def step():
            y, seg, aux = params.framewise_forward(e, f, plan, return_aux=True)
            params.framewise_backward(g, f, seg, plan, aux=aux)
    return step


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(bench.CONFIGS))
    ap.add_argument("--shard-of", type=int, default=0)
    a = ap.parse_args()
    lpc.set_validation("lazy")
    torch.cuda.set_device(0)
    step = make_step(bench.CONFIGS[a.config], a.shard_of)
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()


if __name__ == "__main__":
    main()
