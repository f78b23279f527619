"""Timeline of the chained single-pass kernels (tvlp_chain_trace records).

    python tools/chain_trace.py [--B 64 --T 48000]

Runs warm-up steps, then one traced forward+backward of the bench step, and
prints per-kernel spans and per-phase statistics (microseconds)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2406_05128_b200 import _native as N  # noqa: E402
from paper_2406_05128_b200 import data, lpc  # noqa: E402


def stats(name, v):
    v = np.asarray(v, dtype=np.float64) / 1e3
    if v.size == 0:
        return
    print(f"  {name:22s} n={v.size:5d} mean={v.mean():8.2f} p50={np.median(v):8.2f} "
          f"p90={np.percentile(v, 90):8.2f} max={v.max():8.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--T", type=int, default=48000)
    a = ap.parse_args()
    lpc.set_validation("off")
    lib = N.load()
    e, A, g = data.d1_batch_torch(0, a.B, a.T, 22, device="cuda")
    for _ in range(3):
        s, carry = lpc._forward(False, e, A, None, return_carry=True)
        lpc._backward(False, g, A, s, None, carry)
    torch.cuda.synchronize()
    cap = 1 << 16
    for label, fn in (("fwd", lambda: lpc._forward(False, e, A, None, return_carry=True)),
                      ("bwd", lambda: lpc._backward(False, g, A, s, None, carry))):
        buf = torch.zeros(cap * 8, dtype=torch.int64, device="cuda")
        lib.tvlp_chain_trace(N.ptr(buf), buf.numel() * 8)
        torch.cuda.synchronize()
        fn()
        torch.cuda.synchronize()
        lib.tvlp_chain_trace(None, 0)
        r = buf.view(-1, 8).cpu().numpy().astype(np.uint64)
        r = r[r[:, 1] != 0]
        kind = (r[:, 0] & 0xFF).astype(int)
        sm = ((r[:, 0] >> 8) & 0xFFFFFF).astype(int)
        t = r[:, 1:6].astype(np.int64)
        t0 = t[:, 0].min()
        end = np.where(t[:, 4] > 0, t[:, 4], np.where(t[:, 1] > 0, t[:, 1], t[:, 0]))
        print(f"{label}: {len(r)} records over {len(set(sm))} SMs, span {(end.max() - t0) / 1e3:.1f} us")
        for k, nm in ((1, "basis group"), (2, "apply unit"), (3, "bwd unit")):
            m = kind == k
            if not m.any():
                continue
            tk = t[m]
            print(f" kind {nm}: first start {(tk[:, 0].min() - t0) / 1e3:.1f}, "
                  f"last start {(tk[:, 0].max() - t0) / 1e3:.1f}, "
                  f"last end {((tk[:, 4] if k > 1 else tk[:, 1]).max() - t0) / 1e3:.1f} us")
            if k == 1:
                stats("duration", tk[:, 1] - tk[:, 0])
            elif k == 2:
                stats("wait bases", tk[:, 1] - tk[:, 0])
                stats("wait state+tapes", tk[:, 2] - tk[:, 1])
                stats("carry", tk[:, 3] - tk[:, 2])
                stats("apply pass", tk[:, 4] - tk[:, 3])
            else:
                stats("zero-state pass", tk[:, 1] - tk[:, 0])
                stats("wait state+W", tk[:, 2] - tk[:, 1])
                stats("carry", tk[:, 3] - tk[:, 2])
                stats("apply pass", tk[:, 4] - tk[:, 3])


if __name__ == "__main__":
    main()
