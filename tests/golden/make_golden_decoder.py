"""Golden vectors of the reference decoder pieces.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_decoder.py

Records, from the UNMODIFIED reference tvlp 0.1.0: a reduced LF wavetable
(pkg/tests/conftest.py:8-10), seeded SF / HpN / frame-wise parameter sets of
4801 samples (hop 240, M=22), the float64 tape's output of
build_synth_graph (synth.py:217-275), the MSS loss against a seeded target
(loss.py:105-126) and the gradient of that loss for every trainable field,
plus the per-op forward/VJP of wavetable_read, decimate_fir, shape_noise,
global_fir and stft_mag on the same graph's inputs.
tests/test_decoder_gpu.py compares paper_2406_05128_b200.decoder with them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from tvlp import loss, source, synth  # noqa: E402  (the reference)
from tvlp.tape import Tape  # noqa: E402


def params(mode, seed, F):
    rng = np.random.default_rng(seed)
    p = synth.init_params(F, 22, 240, mode=mode, seed=seed,
                          f0_frames=np.linspace(110.0, 190.0, F) * (1 + 0.05 * rng.standard_normal(F)))
    p.reflection_raw = rng.normal(0.0, 0.3, size=(F, 22))
    p.table_pos_raw = rng.normal(0.0, 1.0, size=F)
    p.voiced_gain_raw = rng.normal(-1.0, 0.3, size=F)
    p.noise_gain_raw = rng.normal(-2.5, 0.3, size=F)
    p.h_gain_raw = rng.normal(-0.5, 0.2, size=F)
    p.noise_logmag = rng.normal(0.0, 0.5, size=(F, source.NOISE_BINS))
    p.fir_taps = np.concatenate(([1.0], 0.05 * rng.standard_normal(127)))
    return p


def main():
    n_out, fs, seed = 4801, 24000.0, 11
    F = (n_out - 1) // 240 + 1
    wt = source.build_lf_wavetable(np.linspace(0.3, 2.7, 9), 512)
    out = {"tables": wt.tables, "n_out": n_out, "fs": fs, "seed": seed}
    target = np.random.default_rng(99).standard_normal(n_out) * 0.3
    out["target"] = target
    out["noise"] = source.generate_noise(n_out, seed)
    for mode, fw in (("sf", False), ("hpn", False), ("sf", True)):
        key = f"{mode}{'_fw' if fw else ''}_"
        p = params(mode, 5 if mode == "sf" else 6, F)
        for name in synth.TRAINABLE_FIELDS + ("f0_frames",):
            out[key + name] = getattr(p, name)
        tape = Tape(np.float64)
        y, leaves = synth.build_synth_graph(tape, p, n_out, fs, seed, wavetable=wt, framewise=fw)
        L = loss.mss_loss(tape, y, target)
        tape.backward(L)
        out[key + "y"] = y.value
        out[key + "loss"] = np.float64(L.value)
        for name, node in leaves.items():
            out[key + "grad_" + name] = tape.grad(node)
        # per-op records of this graph (inputs and outputs / VJPs)
        for node in tape.nodes:
            if node.op in ("wavetable_read", "decimate_fir", "shape_noise", "global_fir",
                           "stft_mag") and key + "op_" + node.op + "_out" not in out:
                out[key + "op_" + node.op + "_out"] = node.value
                out[key + "op_" + node.op + "_in0"] = node.inputs[0].value
                if node.adjoint is not None:
                    out[key + "op_" + node.op + "_adj"] = node.adjoint
                    out[key + "op_" + node.op + "_gin0"] = tape.grad(node.inputs[0])
    np.savez_compressed(os.path.join(HERE, "golden_decoder.npz"), **out)
    print("wrote golden_decoder.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
