"""Experiment: config 3 step variants -- the whole batch on one stream, two
half batches on two streams (per half fwd+bwd, or forward and backward each
split and joined in between), and the carry precisions (the refinement
kernels' share of the step)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_05128_b200 import data, lpc
lpc.set_validation("off")
e, A, g = data.d1_batch_torch(0, 64, 48000, 22, device="cuda")
H = [tuple(x[i * 32:(i + 1) * 32] for x in (e, A, g)) for i in range(2)]
sts = [torch.cuda.Stream() for _ in range(2)]


def full(prec=None):
    def run():
        s, c = lpc._forward(False, e, A, None, carry_prec=prec, return_carry=True)
        lpc._backward(False, g, A, s, None, c, carry_prec=prec)
    return run


def halves_fwdbwd():
    main = torch.cuda.current_stream()
    for st in sts:
        st.wait_stream(main)
    for st, (ee, AA, gg) in zip(sts, H):
        with torch.cuda.stream(st):
            s, c = lpc._forward(False, ee, AA, None, return_carry=True)
            lpc._backward(False, gg, AA, s, None, c)
    for st in sts:
        main.wait_stream(st)


def halves_phase():
    main = torch.cuda.current_stream()
    for st in sts:
        st.wait_stream(main)
    out = []
    for st, (ee, AA, gg) in zip(sts, H):
        with torch.cuda.stream(st):
            out.append(lpc._forward(False, ee, AA, None, return_carry=True))
    for st in sts:
        main.wait_stream(st)
    for st in sts:
        st.wait_stream(main)
    for st, (ee, AA, gg), (s, c) in zip(sts, H, out):
        with torch.cuda.stream(st):
            lpc._backward(False, gg, AA, s, None, c)
    for st in sts:
        main.wait_stream(st)


V = [("full", full()), ("full fp32 carries (no refinement)", full("fp32")),
     ("halves fwd+bwd", halves_fwdbwd), ("halves per phase", halves_phase)]
for rep in range(2):
    for name, fn in V:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(30):
            fn()
        b.record(); torch.cuda.synchronize()
        print(name, round(a.elapsed_time(b) / 30 * 1000, 1), "us", flush=True)
