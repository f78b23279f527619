"""Per-kernel times of one TV and one TI forward at config 3 (tuning aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2406_05128_b200 import _native as N, data, lpc  # noqa: E402

lpc.set_validation("off")
B, T, M = 64, 48000, 22
e, A, g = data.d1_batch_torch(0, B, T, M, device="cuda")
a = A[:, 1000, :].contiguous()
lib = N.load()
for name, fn in (("tv", lambda: lpc.lp_forward_tv(e, A)), ("ti", lambda: lpc.lp_forward_ti(e, a))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    N.profile_dump()
    lib.tvlp_profile_enable(1)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    lib.tvlp_profile_enable(0)
    prof = N.profile_dump()
    print(name, {k: round(v[1] / 5 * 1e3, 1) for k, v in prof.items()})
