"""Per-item parity of the stress rows under each carry precision (diagnostic)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2406_05128_b200 import data, lpc  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 24000
seeds = [4, 11, 28, 31, 52, 35]
items = [data.stress_item(s, T) for s in seeds]
e = np.stack([x[0] for x in items]); A = np.stack([x[1] for x in items]); g = np.stack([x[2] for x in items])
ref = []
for b in range(len(seeds)):
    rs = oracle.lp_forward_tv(e[b].astype(np.float64), A[b].astype(np.float64))
    rge, rgA = oracle.lp_backward_tv(g[b].astype(np.float64), A[b].astype(np.float64), rs)
    rs32 = oracle.lp_forward_tv(e[b], A[b])
    r32 = (rs32,) + oracle.lp_backward_tv(g[b], A[b], rs32)
    ref.append(((rs, rge, rgA), r32))
pad = np.zeros((64 - len(seeds),) + e.shape[1:], np.float32)  # batch to the B*T of config 3's plan
for prec in ("auto", "fp64", "fp32"):
    for B in (len(seeds), 64 if T == 48000 else 128):
        n = B - len(seeds)
        ee = np.concatenate([e, np.repeat(e[:1], n, 0)]) if n else e
        AA = np.concatenate([A, np.repeat(A[:1], n, 0)]) if n else A
        gg = np.concatenate([g, np.repeat(g[:1], n, 0)]) if n else g
        et, At, gt = (torch.from_numpy(x).cuda() for x in (ee, AA, gg))
        s, carry = lpc._forward(False, et, At, None, carry_prec=prec, return_carry=True)
        ge, gA = lpc._backward(False, gt, At, s, None, carry, carry_prec=prec)
        s, ge, gA = (x.cpu().numpy() for x in (s, ge, gA))
        out = []
        for b in range(len(seeds)):
            (rs, rge, rgA), r32 = ref[b]
            mine = max(oracle.gradcheck_error(s[b], rs), oracle.gradcheck_error(ge[b], rge),
                       oracle.gradcheck_error(gA[b], rgA))
            theirs = max(oracle.gradcheck_error(r32[0], rs), oracle.gradcheck_error(r32[1], rge),
                         oracle.gradcheck_error(r32[2], rgA))
            out.append(f"{mine:.1e}/{theirs:.1e}")
        print(f"T={T} prec={prec} B={B} Ls={__import__('paper_2406_05128_b200._native', fromlist=['x']).load().tvlp_subchunk_len(B, T, 22)}: ", " ".join(out), flush=True)
