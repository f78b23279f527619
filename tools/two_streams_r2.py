"""Config 3 (B=64) as two half batches on two streams vs one launch sequence:
can the latency-bound chained kernels of one half overlap the FMA/HBM-bound
kernels of the other?"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_05128_b200 import data, lpc  # noqa: E402


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / n * 1e3, 1)


lpc.set_validation("lazy")
e, A, g = data.d1_batch_torch(0, 64, 48000, 22, device="cuda")
halves = [(e[:32], A[:32], g[:32]), (e[32:], A[32:], g[32:])]
quarters = [(e[i:i + 16], A[i:i + 16], g[i:i + 16]) for i in range(0, 64, 16)]
streams = [torch.cuda.Stream() for _ in range(4)]


def one(x):
    s, c = lpc._forward(False, x[0], x[1], None, return_carry=True)
    lpc._backward(False, x[2], x[1], s, None, c)


def full():
    one((e, A, g))


def seq_halves():
    for h in halves:
        one(h)


def multi(parts):
    def fn():
        main = torch.cuda.current_stream()
        for st in streams[:len(parts)]:
            st.wait_stream(main)
        for st, h in zip(streams, parts):
            with torch.cuda.stream(st):
                one(h)
        for st in streams[:len(parts)]:
            main.wait_stream(st)
    return fn


def staggered():
    """half 2 starts its forward after half 1's forward (so half 1's chained
    kernels meet half 2's basis)"""
    main = torch.cuda.current_stream()
    s1, s2 = streams[0], streams[1]
    s1.wait_stream(main)
    with torch.cuda.stream(s1):
        s_a, c_a = lpc._forward(False, halves[0][0], halves[0][1], None, return_carry=True)
        ev = torch.cuda.Event()
        ev.record(s1)
        lpc._backward(False, halves[0][2], halves[0][1], s_a, None, c_a)
    s2.wait_stream(main)
    with torch.cuda.stream(s2):
        s2.wait_event(ev)
        one(halves[1])
    main.wait_stream(s1)
    main.wait_stream(s2)


print({"full_B64": t(full), "halves_sequential": t(seq_halves), "halves_2_streams": t(multi(halves)),
       "quarters_4_streams": t(multi(quarters)), "halves_staggered": t(staggered)})
