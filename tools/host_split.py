"""Host time of one LP forward/backward call split into the Python wrapper and
the C-ABI call (plan, tensor-map encodes, launches), config 1 and 3 shapes."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_05128_b200 import _native as N  # noqa: E402
from paper_2406_05128_b200 import data, lpc  # noqa: E402


def main():
    lpc.set_validation("lazy")
    lib = N.load()
    for B, T in ((4, 24000), (64, 48000)):
        e, A, g = data.d1_batch_torch(0, B, T, 22, device="cuda")
        for _ in range(5):
            s, c = lpc._forward(False, e, A, None, return_carry=True)
            lpc._backward(False, g, A, s, None, c)
        torch.cuda.synchronize()
        # whole wrapper
        n = 200
        t0 = time.perf_counter()
        for _ in range(n):
            s, c = lpc._forward(False, e, A, None, return_carry=True)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        for _ in range(n):
            lpc._backward(False, g, A, s, None, c)
        t2 = time.perf_counter()
        torch.cuda.synchronize()
        # the bare C call with preallocated buffers
        ws, nws = N.workspace(lib.tvlp_workspace_bytes(N.OP_FWD_TV, N.F32, B, T, 22, 0, 0, 0),
                              e.device)
        st = N.stream_ptr(e.device)
        t3 = time.perf_counter()
        for _ in range(n):
            lib.tvlp_lp_forward_tv(N.F32, N.ptr(e), N.ptr(A), None, N.ptr(s), B, T, 22, N.ptr(c),
                                   N.CARRY_AUTO, N.ptr(ws), nws, None, st)
        t4 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"B={B} T={T}: forward wrapper {1e6 * (t1 - t0) / n:.1f} us, backward wrapper "
              f"{1e6 * (t2 - t1) / n:.1f} us, bare C forward call {1e6 * (t4 - t3) / n:.1f} us",
              flush=True)


if __name__ == "__main__":
    main()
