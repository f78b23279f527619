"""Generate the golden vectors that pin the oracle (and the D1 input generator)
to the reference itself.

Run once in the build container, where the read-only reference is importable:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

It imports the UNMODIFIED reference ``tvlp`` 0.1.0 and records inputs and
outputs of its LP path (lpc.py:82-195, params.py:152-273) on seeded inputs:
random small cases in float64 and float32 (with and without ``zi``, M from 1
to 22, T from 1 to 1000), a production-shaped frame-wise case (hop 240,
frame 960, M=22), and the reference's own step-up/upsample applied to the D1
reflection walk (so ``paper_2406_05128_b200.data`` is pinned too).  The
committed ``.npz`` files are what ``tests/test_oracle_golden.py`` and the GPU
parity tests read; ``/root/reference`` is never read at test time.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from tvlp import lpc, oracle, params  # noqa: E402  (the reference)

from paper_2406_05128_b200 import data  # noqa: E402


def lpc_cases():
    rng = np.random.default_rng(20240605)
    out = {}
    shapes = [(1, 3), (2, 3), (3, 1), (5, 2), (17, 4), (32, 6), (64, 5), (100, 1),
              (257, 22), (1000, 22), (24, 22), (40, 7), (333, 12), (96, 16)]
    i = 0
    for T1, M in shapes:
        for dt in (np.float64, np.float32):
            for with_zi in (False, True):
                A = oracle.random_stable_track(rng, T1, M, n_frames=max(1, min(4, T1)))
                e = rng.standard_normal(T1)
                g = rng.standard_normal(T1)
                zi = rng.standard_normal(M) if with_zi else None
                A = A.astype(dt)
                e = e.astype(dt)
                g = g.astype(dt)
                zi = None if zi is None else zi.astype(dt)
                s = lpc.lp_forward_tv(e, A, zi)
                ge, gA = lpc.lp_backward_tv(g, A, s, zi)
                a = A[0].copy()
                s_ti = lpc.lp_forward_ti(e, a, zi)
                ge_ti, ga_ti = lpc.lp_backward_ti(g, a, s_ti, zi)
                key = f"c{i}_"
                out[key + "e"] = e
                out[key + "A"] = A
                out[key + "g"] = g
                if zi is not None:
                    out[key + "zi"] = zi
                out[key + "s"] = s
                out[key + "ge"] = ge
                out[key + "gA"] = gA
                out[key + "s_ti"] = s_ti
                out[key + "ge_ti"] = ge_ti
                out[key + "ga_ti"] = ga_ti
                out[key + "Ahat"] = lpc.shift_coeffs(A)
                out[key + "lag"] = lpc.lagged_signal_matrix(s, M, zi)
                i += 1
    out["n_cases"] = np.array(i)
    return out


def framewise_cases():
    rng = np.random.default_rng(7)
    out = {}
    cfgs = [(640, 64, 4, np.float64), (160, 32, 3, np.float64), (640, 64, 4, np.float32),
            (4800, 240, 22, np.float32), (4801, 240, 22, np.float64), (1000, 100, 6, np.float32)]
    for i, (T1, hop, M, dt) in enumerate(cfgs):
        plan = params.FramePlan.raised_cosine(hop)
        F = params.expected_frame_count(T1 - 1, hop)
        # independent stable rows per frame (each frame is a TI filter); the
        # interpolated tracks of random_stable_track can blow up
        frames = params.reflection_to_lpc(rng.uniform(-0.9, 0.9, size=(F, M))).astype(dt)
        e = rng.standard_normal(T1).astype(dt)
        g = rng.standard_normal(T1).astype(dt)
        y, segs = params._framewise_forward(e, frames, plan)
        ge, gf = params._framewise_vjp(g, e, frames, plan, segs)
        key = f"f{i}_"
        out[key + "cfg"] = np.array([T1, hop, M])
        out[key + "e"] = e
        out[key + "frames"] = frames
        out[key + "g"] = g
        out[key + "y"] = y
        out[key + "segs"] = np.stack(segs)
        out[key + "ge"] = ge
        out[key + "gf"] = gf
    out["n_cases"] = np.array(len(cfgs))
    return out


def d1_cases():
    """The reference's own step-up + upsample on the D1 reflection walk."""
    out = {}
    for i, (T1, seed) in enumerate([(2401, 0), (4800, 1)]):
        raw = data.d1_reflection_raw(seed, T1, 22, hop=240)
        k = params.squash_reflection(raw)
        a_frames = params.reflection_to_lpc(k)
        A = params.upsample_linear(a_frames, 240, T1 - 1)
        out[f"d{i}_cfg"] = np.array([T1, seed])
        out[f"d{i}_raw"] = raw
        out[f"d{i}_A32"] = A.astype(np.float32)
        out[f"d{i}_maxpole"] = np.array(params.max_pole_modulus(a_frames))
    rng = np.random.default_rng(11)
    row = oracle.random_stable_track(rng, 1, 22, n_frames=1)[0]
    out["stress_row"] = row
    out["n_cases"] = np.array(2)
    return out


def upsample_cases():
    """upsample_linear + its VJP (params.py:107-145) and the composed TV LP
    through it (the path the fused frame-rate kernels replace, SURVEY.md
    §8(f) rank 1): lp_forward_tv(e, upsample_linear(frames)) and the VJP
    chain back to the frame rows."""
    rng = np.random.default_rng(7070)
    out = {}
    for i, (T, hop, M) in enumerate([(9, 4, 3), (47, 8, 5), (960, 240, 22), (1200, 80, 22)]):
        F = params.expected_frame_count(T, hop)
        raw = np.clip(rng.normal(0, 0.25, size=(F, M)), -0.9, 0.9)
        frames = params.reflection_to_lpc(params.squash_reflection(raw))
        A = params.upsample_linear(frames, hop, T)
        e = rng.normal(size=T + 1)
        g = rng.normal(size=T + 1)
        s = lpc.lp_forward_tv(e, A)
        ge, gA = lpc.lp_backward_tv(g, A, s)
        gf = params._upsample_linear_vjp(gA, F, hop, T)
        out.update({f"c{i}_frames": frames, f"c{i}_hop": np.array(hop), f"c{i}_A": A,
                    f"c{i}_e": e, f"c{i}_g": g, f"c{i}_s": s, f"c{i}_ge": ge, f"c{i}_gA": gA,
                    f"c{i}_gf": gf})
    out["n"] = np.array(4)
    return out


def stepup_cases():
    """reflection_to_lpc + its VJP (params.py:43-84) on random rows."""
    rng = np.random.default_rng(4343)
    out = {}
    for i, (F, M) in enumerate([(1, 1), (3, 2), (17, 9), (201, 22), (5, 30)]):
        k = params.squash_reflection(rng.normal(0, 0.6, size=(F, M)))
        a, stages = params._step_up(k)
        ga = rng.normal(size=(F, M))
        gk = params._reflection_to_lpc_vjp(ga, k, stages)
        out.update({f"c{i}_k": k, f"c{i}_a": params.reflection_to_lpc(k), f"c{i}_ga": ga,
                    f"c{i}_gk": gk})
    out["n"] = np.array(5)
    return out


def main():
    np.savez_compressed(os.path.join(HERE, "golden_lpc.npz"), **lpc_cases())
    np.savez_compressed(os.path.join(HERE, "golden_framewise.npz"), **framewise_cases())
    np.savez_compressed(os.path.join(HERE, "golden_d1.npz"), **d1_cases())
    np.savez_compressed(os.path.join(HERE, "golden_upsample.npz"), **upsample_cases())
    np.savez_compressed(os.path.join(HERE, "golden_stepup.npz"), **stepup_cases())
    for f in ("golden_lpc.npz", "golden_framewise.npz", "golden_d1.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
