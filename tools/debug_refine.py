"""Diagnose the 'auto' carry refinement on the resonant stress set."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle
from paper_2406_05128_b200 import data, lpc, _native as N

lib = N.load()
items = [data.stress_item(s, 24000) for s in range(4)]
e = np.stack([x[0] for x in items]); A = np.stack([x[1] for x in items]); g = np.stack([x[2] for x in items])
et, At, gt = (torch.from_numpy(x).cuda() for x in (e, A, g))
res = {}
for prec in ("fp64", "fp32", "auto"):
    r0 = lib.tvlp_refined_sequences()
    s, carry = lpc._forward(False, et, At, None, carry_prec=prec, return_carry=True)
    r1 = lib.tvlp_refined_sequences()
    ge, gA = lpc._backward(False, gt, At, s, None, carry, carry_prec=prec)
    r2 = lib.tvlp_refined_sequences()
    # backward with the fp64 tape but this precision mode
    res[prec] = (s.cpu().numpy(), ge.cpu().numpy(), gA.cpu().numpy(), r1 - r0, r2 - r1)
for b in range(4):
    rs = oracle.lp_forward_tv(e[b].astype(np.float64), A[b].astype(np.float64))
    rge, rgA = oracle.lp_backward_tv(g[b].astype(np.float64), A[b].astype(np.float64), rs)
    for prec, (s, ge, gA, nf, nb) in res.items():
        print(b, prec, 'refined fwd/bwd', nf, nb, 'err s %.2e ge %.2e gA %.2e' % (
            oracle.gradcheck_error(s[b], rs), oracle.gradcheck_error(ge[b], rge), oracle.gradcheck_error(gA[b], rgA)))
# bwd with fp64 tape + auto
s, carry = lpc._forward(False, et, At, None, carry_prec="fp64", return_carry=True)
ge, gA = lpc._backward(False, gt, At, s, None, carry, carry_prec="auto")
for b in range(4):
    rs = oracle.lp_forward_tv(e[b].astype(np.float64), A[b].astype(np.float64))
    rge, rgA = oracle.lp_backward_tv(g[b].astype(np.float64), A[b].astype(np.float64), rs)
    print(b, 'fp64 tape + auto bwd', 'ge %.2e' % oracle.gradcheck_error(ge[b].cpu().numpy(), rge))
