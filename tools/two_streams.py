"""Experiment: config 3 as two half batches on two streams vs one call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_05128_b200 import data, lpc
lpc.set_validation("off")
e, A, g = data.d1_batch_torch(0, 64, 48000, 22, device="cuda")
def parts(n):
    k = 64 // n
    return [tuple(x[i * k:(i + 1) * k].contiguous() for x in (e, A, g)) for i in range(n)]
P = {n: parts(n) for n in (2, 4, 8)}
streams = [torch.cuda.Stream() for _ in range(8)]

def full():
    s, c = lpc._forward(False, e, A, None, return_carry=True)
    lpc._backward(False, g, A, s, None, c)

def split(n):
    def run():
        main = torch.cuda.current_stream()
        sts = streams[:n]
        for st in sts:
            st.wait_stream(main)
        for st, (ee, AA, gg) in zip(sts, P[n]):
            with torch.cuda.stream(st):
                s, c = lpc._forward(False, ee, AA, None, return_carry=True)
                lpc._backward(False, gg, AA, s, None, c)
        for st in sts:
            main.wait_stream(st)
    return run

for name, fn in (("full", full), ("2 streams", split(2)), ("4 streams", split(4)),
                 ("8 streams", split(8)), ("full", full), ("2 streams", split(2)),
                 ("4 streams", split(4))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        fn()
    b.record(); torch.cuda.synchronize()
    print(name, round(a.elapsed_time(b) / 20 * 1000, 1), "us")
