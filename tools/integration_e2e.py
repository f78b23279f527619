"""End-to-end time of the UNMODIFIED reference's own decoder step (its Tape:
synth.build_synth_graph + Tape.backward, synth.py:217-275, tape.py) with its
numba LP ops and with the B200 ops swapped in by integration/tvlp_b200_ops.py
(host arrays in, host arrays out: the op uploads its inputs and downloads its
outputs, as the tape contract requires).  One item of T = n_out samples;
prints one JSON line per (mode, framewise, dtype).

    python tools/integration_e2e.py [n_out]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tvlp_numba_cache")


def step(mode, dtype, framewise, n_out):
    from tvlp import synth
    from tvlp.tape import Tape

    hop, fs = 240, 24000
    F = (n_out - 1) // hop + 1
    rng = np.random.default_rng(7)
    params = synth.init_params(F, 22, hop, mode=mode, seed=5,
                               f0_frames=np.linspace(110.0, 180.0, F))
    params.reflection_raw = rng.normal(0.0, 0.3, size=(F, 22))
    params.h_gain_raw = rng.normal(-1.0, 0.2, size=F)
    params.noise_gain_raw = rng.normal(-2.0, 0.2, size=F)
    tape = Tape(dtype)
    out, leaves = synth.build_synth_graph(tape, params, n_out, fs, seed=3, framewise=framewise)
    loss = tape.mean(tape.mul(out, out))
    tape.backward(loss)
    return float(loss.value)


def timed(fn, reps):
    fn()
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def main():
    n_out = int(sys.argv[1]) if len(sys.argv) > 1 else 48001
    import tvlp  # noqa: F401

    from integration import tvlp_b200_ops

    for mode, framewise, dtype in (("sf", False, np.float32), ("hpn", False, np.float32),
                                   ("sf", True, np.float32), ("sf", False, np.float64)):
        f = lambda: step(mode, dtype, framewise, n_out)  # noqa: E731
        t_ref = timed(f, 5)
        with tvlp_b200_ops.install():
            t_b200 = timed(f, 5)
        print(json.dumps({"graph": f"synth.build_synth_graph mode={mode} framewise={framewise}",
                          "dtype": np.dtype(dtype).name, "samples": n_out - 1,
                          "reference_ops_s": round(t_ref, 5), "b200_ops_s": round(t_b200, 5),
                          "speedup": round(t_ref / t_b200, 2),
                          "note": "whole decoder step on the reference Tape (numpy CPU ops "
                                  "around the LP ops); only the LP ops differ"}), flush=True)


if __name__ == "__main__":
    main()
