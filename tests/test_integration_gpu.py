"""The B200 ops inside the UNMODIFIED reference tape engine.

The reference (installed offline into baseline/_ref, which travels with the
repository to the GPU box) builds its own SF / HpN decoder graph
(synth.py:217-275) on its own Tape; integration/tvlp_b200_ops.py swaps the LP
ops of its registry.  Outputs and every parameter gradient must match the
reference's CPU tape (float64 tape: 1e-9; float32 tape: 1e-4 with the
reference's metric)."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def tvlp():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        import tvlp as mod  # noqa: F401
        from tvlp import synth  # noqa: F401
    except Exception as exc:  # the reference is not installed next to the repo
        pytest.skip(f"reference tvlp not importable: {exc}")
    return mod


def _graph(tvlp, mode, dtype, framewise=False):
    from tvlp import synth
    from tvlp.tape import Tape

    hop, fs, n_out = 240, 24000, 4801
    F = (n_out - 1) // hop + 1
    rng = np.random.default_rng(7)
    params = synth.init_params(F, 22, hop, mode=mode, seed=5,
                               f0_frames=np.linspace(110.0, 180.0, F))
    params.reflection_raw = rng.normal(0.0, 0.3, size=(F, 22))   # D1-like spread
    params.h_gain_raw = rng.normal(-1.0, 0.2, size=F)
    params.noise_gain_raw = rng.normal(-2.0, 0.2, size=F)
    tape = Tape(dtype)
    out, leaves = synth.build_synth_graph(tape, params, n_out, fs, seed=3, framewise=framewise)
    loss = tape.mean(tape.mul(out, out))
    tape.backward(loss)
    return out.value.copy(), {k: tape.grad(v).copy() for k, v in leaves.items()}


@pytest.mark.parametrize("mode,dtype,framewise", [("sf", np.float64, False),
                                                  ("hpn", np.float64, False),
                                                  ("sf", np.float64, True),
                                                  ("sf", np.float32, False)])
def test_reference_graph_with_b200_ops(tvlp, mode, dtype, framewise):
    sys.path.insert(0, ROOT)
    from integration import tvlp_b200_ops
    from oracle import gradcheck_error

    ref_out, ref_grads = _graph(tvlp, mode, dtype, framewise)
    with tvlp_b200_ops.install():
        out, grads = _graph(tvlp, mode, dtype, framewise)
    if dtype == np.float64:
        assert gradcheck_error(out, ref_out) < 1e-9
        for k in ref_grads:
            assert gradcheck_error(grads[k], ref_grads[k]) < 1e-9, k
    else:
        # a float32 tape: both runs against the reference's float64 tape; the
        # B200 ops may not add more than the float32 tape's own rounding
        # (the CPU ops of the graph -- oscillator, noise, FIR -- run in fp32 too)
        out64, grads64 = _graph(tvlp, mode, np.float64, framewise)
        assert gradcheck_error(out, out64) <= max(1e-4, 2 * gradcheck_error(ref_out, out64))
        for k in ref_grads:
            mine = gradcheck_error(grads[k], grads64[k])
            theirs = gradcheck_error(ref_grads[k], grads64[k])
            assert mine <= max(1e-4, 2 * theirs), (k, mine, theirs)
    # the original ops are back
    from tvlp import lpc, tape

    assert tape._REGISTRY["lp_tv"].forward is lpc._fw_lp_tv
