"""Host cost of one bench step (Python + ctypes + launches, no sync) against
its device time, for the frame-wise and config-3 steps: a step whose host
cost approaches its device time is launch-bound."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_05128_b200 import data, lpc, params  # noqa: E402


def measure(name, step, n=50):
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(n):
        step()
    ev1.record()
    torch.cuda.synchronize()
    print(f"{name}: host {1e6 * (t1 - t0) / n:.1f} us/step (enqueue), wall {1e6 * (t2 - t0) / n:.1f},"
          f" device {1e3 * ev0.elapsed_time(ev1) / n:.1f} us/step", flush=True)


def main():
    lpc.set_validation("lazy")
    ev, fr, gv = data.d1_frames_batch(0, 32, 48000, 22, 240)
    e, f, g = (torch.from_numpy(x).cuda() for x in (ev, fr, gv))
    plan = params.FramePlan.raised_cosine(240)

    def fw():
        y, seg = params.framewise_forward(e, f, plan)
        params.framewise_backward(g, f, seg, plan)

    measure("framewise B=32", fw)
    e3, A3, g3 = data.d1_batch_torch(0, 64, 48000, 22, device="cuda")

    def tv():
        s, c = lpc._forward(False, e3, A3, None, return_carry=True)
        lpc._backward(False, g3, A3, s, None, c)

    measure("tv B=64", tv)
    e1, A1, g1 = data.d1_batch_torch(0, 8, 48000, 22, device="cuda")

    def tv8():
        s, c = lpc._forward(False, e1, A1, None, return_carry=True)
        lpc._backward(False, g1, A1, s, None, c)

    measure("tv B=8", tv8)
    e4, A4, g4 = data.d1_batch_torch(0, 4, 24000, 22, device="cuda")

    def tv4():
        s, c = lpc._forward(False, e4, A4, None, return_carry=True)
        lpc._backward(False, g4, A4, s, None, c)

    measure("tv B=4 T=24000 (config 1)", tv4)


if __name__ == "__main__":
    main()
