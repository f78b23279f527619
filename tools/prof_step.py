"""Run a few LP fwd+bwd steps of a bench config (for ncu / nsys-free profiling)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2406_05128_b200 import data, lpc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--T", type=int, default=48000)
    ap.add_argument("--M", type=int, default=22)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--carry", default="fp64")
    a = ap.parse_args()
    lpc.set_validation("off")
    lpc.set_carry_precision(a.carry)
    e, A, g = data.d1_batch_torch(0, a.B, a.T, a.M, device="cuda")
    for _ in range(a.steps):
        s, carry = lpc._forward(False, e, A, None, return_carry=True)
        lpc._backward(False, g, A, s, None, carry)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
