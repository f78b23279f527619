"""One small invocation of every kernel family of libtvlp_b200.so, for
compute-sanitizer (tools/sanitize.sh runs memcheck / racecheck / synccheck /
initcheck over it).  Shapes are small so the instrumented run finishes in
minutes, but each family runs its production code path:

  chain      chained single-pass fwd/bwd (k_basis4, k_fwd_chain, k_adj_zs_units,
             k_bwd_chain, k_grad_A)                     B=3, T=4800
  chain_ref  the same with a resonant stress row (in-kernel refinement)
  grouped    two groups in one launch (H(z) + C(z))
  ti         time-invariant rows through the chain kernels + grad_a
  f64        float64 I/O (separate basis / carry / apply kernels)
  hier       hierarchical carries (TVLP_CARRY_SERIAL_MAX forced small by
             tools/sanitize.sh) -- the config-4 path
  frames     frame-rate rows interpolated in the kernels (+ zi, padded order)
  framewise  frame-wise TI with overlap-add (k_fw_*)
  stepup     reflection -> LPC step-up and its VJP
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_05128_b200 import data, lpc, params  # noqa: E402


def run(fam):
    dev = "cuda"
    if fam in ("chain", "hier"):
        e, A, g = data.d1_batch_torch(0, 3, 4800 if fam == "chain" else 48000, 22, device=dev)
        s, c = lpc._forward(False, e, A, None, return_carry=True)
        lpc._backward(False, g, A, s, None, c)
    elif fam == "chain_ref":
        e, A, g = (torch.from_numpy(np.stack(x)).to(dev) for x in
                   zip(*[data.stress_item(4, 4800)[:3], data.stress_item(5, 4800)[:3]]))
        s, c = lpc._forward(False, e, A, None, return_carry=True)
        lpc._backward(False, g, A, s, None, c)
    elif fam == "grouped":
        eh, Ah, gh = data.d1_batch_torch(0, 2, 4800, 22, device=dev)
        ec, Ac, gc = data.d1_batch_torch(5, 3, 4800, 22, device=dev)
        (sh, sc), c = lpc.lp_forward_tv_grouped([(eh, Ah), (ec, Ac)], return_carry=True)
        lpc.lp_backward_tv_grouped([(gh, Ah, sh), (gc, Ac, sc)], carry=c)
    elif fam == "ti":
        e, A, g = data.d1_batch_torch(0, 3, 4800, 22, device=dev)
        a = A[:, 0].contiguous()
        s, c = lpc._forward(True, e, a, None, return_carry=True)
        lpc._backward(True, g, a, s, None, c)
    elif fam == "f64":
        e, A, g = (x.double() for x in data.d1_batch_torch(0, 2, 4800, 22, device=dev))
        s, c = lpc._forward(False, e, A, None, return_carry=True)
        lpc._backward(False, g, A, s, None, c)
    elif fam == "frames":
        ev, fr, gv = data.d1_frames_batch(0, 2, 4801, 20, 240)
        e, f, g = (torch.from_numpy(x).to(dev) for x in (ev, fr, gv))
        zi = 0.1 * torch.ones(2, 20, device=dev)
        s, c = lpc.lp_forward_tv_frames(e, f, 240, zi, return_carry=True)
        lpc.lp_backward_tv_frames(g, f, 240, s, zi, carry=c)
    elif fam == "framewise":
        ev, fr, gv = data.d1_frames_batch(0, 2, 4800, 22, 240)
        e, f, g = (torch.from_numpy(x).to(dev) for x in (ev, fr, gv))
        plan = params.FramePlan.raised_cosine(240)
        y, seg = params.framewise_forward(e, f, plan)
        params.framewise_backward(g, f, seg, plan)
    elif fam == "stepup":
        k = torch.tanh(torch.randn(3, 50, 22, device=dev, dtype=torch.float64))
        k.requires_grad_(True)
        from paper_2406_05128_b200 import autograd as ag

        ag.ReflectionToLPC.apply(k).sum().backward()
    else:
        raise SystemExit(f"unknown family {fam}")
    torch.cuda.synchronize()
    print(f"{fam}: ok", flush=True)


if __name__ == "__main__":
    lpc.set_validation("lazy")
    for f in sys.argv[1:]:
        run(f)
