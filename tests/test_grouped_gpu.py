"""Grouped launch (north star (3); SURVEY.md §8(b) grouped variant): the HpN
synthesiser's two LPs -- H(z) on the glottal source and C(z) on the noise
(synth.py:264-273) -- on their own buffers in one launch sequence.

Parity: each group against the float64 oracle (two reference lp_forward_tv /
lp_backward_tv calls), and bit-identity with the same
sequences filtered as one concatenated batch (same plan, same arithmetic)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2406_05128_b200 import data

pytestmark = pytest.mark.gpu
lpc = pytest.importorskip("paper_2406_05128_b200.lpc")


def _np(t):
    return t.detach().cpu().numpy()


def _case(BH=5, BC=3, T=24000):
    eh, Ah, gh = data.d1_batch(500, BH, T)
    ec, Ac, gc = data.d1_batch(900, BC, T)
    return (eh, Ah, gh), (ec, Ac, gc)


@pytest.mark.parametrize("BH,BC,T", [(5, 3, 24000), (32, 32, 48000), (2, 1, 4801)])
def test_grouped_matches_concatenated_and_oracle(BH, BC, T):
    (eh, Ah, gh), (ec, Ac, gc) = _case(BH, BC, T)
    t = lambda x: torch.from_numpy(x).cuda()  # noqa: E731
    (sh, sc), carry = lpc.lp_forward_tv_grouped([(t(eh), t(Ah)), (t(ec), t(Ac))],
                                                return_carry=True)
    (geh, gAh), (gec, gAc) = lpc.lp_backward_tv_grouped(
        [(t(gh), t(Ah), sh), (t(gc), t(Ac), sc)], carry=carry)
    # one concatenated batch: same plan (B = BH + BC), same per-sequence arithmetic
    e = t(np.concatenate([eh, ec]))
    A = t(np.concatenate([Ah, Ac]))
    g = t(np.concatenate([gh, gc]))
    s, c2 = lpc._forward(False, e, A, None, return_carry=True)
    ge, gA = lpc._backward(False, g, A, s, None, c2)
    for a, b in ((sh, s[:BH]), (sc, s[BH:]), (geh, ge[:BH]), (gec, ge[BH:]), (gAh, gA[:BH]),
                 (gAc, gA[BH:])):
        torch.testing.assert_close(a, b, rtol=0, atol=0)
    for (e_, A_, g_), (s_, ge_, gA_) in (((eh, Ah, gh), (sh, geh, gAh)),
                                         ((ec, Ac, gc), (sc, gec, gAc))):
        for b in (0, e_.shape[0] - 1):
            rs = oracle.lp_forward_tv(e_[b].astype(np.float64), A_[b].astype(np.float64))
            rge, rgA = oracle.lp_backward_tv(g_[b].astype(np.float64), A_[b].astype(np.float64),
                                             rs)
            errs = (oracle.gradcheck_error(_np(s_)[b], rs), oracle.gradcheck_error(_np(ge_)[b], rge),
                    oracle.gradcheck_error(_np(gA_)[b], rgA))
            assert max(errs) < 1e-4, errs


def test_grouped_with_zi_and_fallback_dtype():
    """Initial states per group; float64 takes the concatenation fallback."""
    rng = np.random.default_rng(4)
    for dt, tol in ((np.float32, 1e-4), (np.float64, 1e-9)):
        (eh, Ah, gh), (ec, Ac, gc) = _case(2, 2, 4800)
        eh, Ah, gh, ec, Ac, gc = (x.astype(dt) for x in (eh, Ah, gh, ec, Ac, gc))
        zh = (0.2 * rng.standard_normal((2, 22))).astype(dt)
        zc = (0.2 * rng.standard_normal((2, 22))).astype(dt)
        t = lambda x: torch.from_numpy(x).cuda()  # noqa: E731
        (sh, sc), carry = lpc.lp_forward_tv_grouped([(t(eh), t(Ah), t(zh)), (t(ec), t(Ac), t(zc))],
                                                    return_carry=True)
        (geh, gAh), (gec, gAc) = lpc.lp_backward_tv_grouped(
            [(t(gh), t(Ah), sh, t(zh)), (t(gc), t(Ac), sc, t(zc))], carry=carry)
        for (e_, A_, g_, z_), (s_, ge_, gA_) in (((eh, Ah, gh, zh), (sh, geh, gAh)),
                                                 ((ec, Ac, gc, zc), (sc, gec, gAc))):
            for b in range(2):
                z64 = z_[b].astype(np.float64)
                rs = oracle.lp_forward_tv(e_[b].astype(np.float64), A_[b].astype(np.float64), z64)
                rge, rgA = oracle.lp_backward_tv(g_[b].astype(np.float64),
                                                 A_[b].astype(np.float64), rs, z64)
                errs = (oracle.gradcheck_error(_np(s_)[b], rs),
                        oracle.gradcheck_error(_np(ge_)[b], rge),
                        oracle.gradcheck_error(_np(gA_)[b], rgA))
                assert max(errs) < tol, (dt, errs)


def test_grouped_autograd_pair():
    """autograd.lp_tv_grouped((e_h, A_h), (e_c, A_c)) == two LPTV ops."""
    from paper_2406_05128_b200 import autograd as ag

    (eh, Ah, gh), (ec, Ac, gc) = _case(3, 2, 4800)
    t = lambda x: torch.from_numpy(x).cuda().requires_grad_()  # noqa: E731
    leaves = [t(x) for x in (eh, Ah, ec, Ac)]
    sh, sc = ag.lp_tv_grouped((leaves[0], leaves[1]), (leaves[2], leaves[3]))
    (sh * torch.from_numpy(gh).cuda()).sum().add((sc * torch.from_numpy(gc).cuda()).sum()).backward()
    ref = [t(x) for x in (eh, Ah, ec, Ac)]
    rh = ag.lp_tv(ref[0], ref[1])
    rc = ag.lp_tv(ref[2], ref[3])
    (rh * torch.from_numpy(gh).cuda()).sum().add((rc * torch.from_numpy(gc).cuda()).sum()).backward()
    for a, b in zip(leaves, ref):
        assert oracle.gradcheck_error(_np(a.grad), _np(b.grad)) < 1e-5
