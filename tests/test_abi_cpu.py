"""CPU-side checks of the C ABI and host logic (no GPU, no kernel launches)."""
import os
import re

import numpy as np
import pytest

from paper_2406_05128_b200 import _native as N

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _declared():
    text = open(os.path.join(ROOT, "include", "tvlp.h")).read()
    return sorted(set(re.findall(r"\b(tvlp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = N.load()
    declared = _declared()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(N.EXPORTS) == declared


def test_abi_queries_without_gpu():
    lib = N.load()
    assert lib.tvlp_abi_version() == 1
    assert lib.tvlp_max_order() >= 22
    Ls = lib.tvlp_subchunk_len(64, 48000, 22)
    assert Ls % 8 == 0 and 48000 % Ls == 0 and 256 <= Ls <= 1024
    small = lib.tvlp_subchunk_len(4, 24000, 22)  # small batch: shorter sub-chunks
    assert small % 8 == 0 and 24000 % small == 0 and 128 <= small < Ls
    nsub = -(-48000 // Ls)
    # per-sub-chunk tapes + one forward-refinement flag slot per sequence
    assert lib.tvlp_carry_elems(64, 48000, 22) == 64 * nsub * (2 * 22 + 1) * 24 + 64
    for op in range(4):
        assert lib.tvlp_workspace_bytes(op, 0, 64, 48000, 22, 0, 0, 0) > 0
    assert lib.tvlp_framewise_nframes(48000, 200, 960, 240) == 203
    assert lib.tvlp_workspace_bytes(5, 0, 32, 48000, 22, 200, 960, 240) > 0
    # odd orders pad to a compiled order; too-large orders are rejected
    assert lib.tvlp_carry_elems(1, 100, 5) == 1 * (2 * 6 + 1) * 8 + 1
    assert lib.tvlp_carry_elems(1, 100, 99) == -1
    assert lib.tvlp_workspace_bytes(0, 0, 1, 100, 99, 0, 0, 0) == 0


def test_status_strings():
    lib = N.load()
    assert lib.tvlp_status_string(0) == b"ok"
    assert b"workspace" in lib.tvlp_status_string(3)
    with pytest.raises(N.TVLPError, match="order"):
        N.check(2)


def test_frameplan_host_logic():
    from paper_2406_05128_b200.params import FramePlan, expected_frame_count

    plan = FramePlan.raised_cosine(240)
    assert plan.frame_size == 960 and plan.n_lead_in() == 3
    assert plan.ola_deviation() < 1e-12
    assert plan.cola_constant() == pytest.approx(2.0)
    frames = list(plan.iter_frames(48000, expected_frame_count(47999, 240)))
    assert len(frames) == 203
    assert frames[0] == (0, 0, 240, 720, 960)
    bad = FramePlan(frame_size=256, hop=100, window=np.hanning(256))
    with pytest.raises(ValueError, match="deviation"):
        bad.validate_cola()
    with pytest.raises(ValueError, match="non-integer"):
        FramePlan.raised_cosine(7, overlap=0.7)


def test_abi_queries_frames_and_split():
    """Workspace/carry queries of the frame-rate pair and the time-split
    helpers (no kernel launches)."""
    lib = N.load()
    B, T, M, hop = 64, 48000, 22, 240
    F = (T - 1) // hop + 1
    assert lib.tvlp_workspace_bytes(N.OP_FWD_TV_FRAMES, 0, B, T, M, F, 0, hop) > 0
    assert lib.tvlp_workspace_bytes(N.OP_BWD_TV_FRAMES, 0, B, T, M, F, 0, hop) > 0
    assert lib.tvlp_workspace_bytes(N.OP_FWD_TV_FRAMES, 0, B, T, M, F + 1, 0, hop) == 0  # bad F
    # the frames plan uses shorter sub-chunks: more tapes than the A-track plan
    assert lib.tvlp_carry_elems_frames(B, T, M) > lib.tvlp_carry_elems(B, T, M)
    assert lib.tvlp_workspace_bytes(N.OP_BWD_TV_EX, 0, B, T, M, 0, 0, 0) >= \
        lib.tvlp_workspace_bytes(N.OP_BWD_TV, 0, B, T, M, 0, 0, 0)
    assert lib.tvlp_workspace_bytes(N.OP_SEGMENT_TRANSITION, 0, 1, 14_400_000, M, 0, 0, 0) > 0
    # null pointers are rejected before any launch
    assert lib.tvlp_reflection_to_lpc(0, None, None, 4, 3, None, None) == 1
    assert lib.tvlp_segment_transition(0, None, 1, 100, 3, None, None, 0, None) == 1


def test_abi_decoder_entry_points_validate_before_launch():
    """tvlp_wavetable_osc* / tvlp_global_fir* / tvlp_mss_terms*: argument
    checks and the workspace queries (no kernel launches: B = 0 or rejected
    arguments)."""
    import ctypes
    lib = N.load()
    fake = ctypes.c_void_p(256)          # never dereferenced: rejected or B = 0
    n_out, hop = 48001, 240
    F = (n_out * 4 - 1) // (hop * 4) + 1
    ok = (fake, fake, fake, 9, 512, fake, 127)
    # valid geometry with B = 0: nothing to do
    assert lib.tvlp_wavetable_osc(*ok, fake, 0, n_out, F, hop, 4, 48000.0, None) == 0
    assert lib.tvlp_wavetable_osc_vjp(*ok, fake, fake, fake, 0, n_out, F, hop, 4, 48000.0,
                                      None) == 0
    bad = [
        dict(F=F + 1), dict(os=2), dict(nt=128), dict(fs=0.0), dict(K=0), dict(L=1),
    ]
    for b in bad:
        args = dict(K=9, L=512, nt=127, F=F, os=4, fs=48000.0)
        args.update(b)
        assert lib.tvlp_wavetable_osc(fake, fake, fake, args["K"], args["L"], fake, args["nt"],
                                      fake, 2, n_out, args["F"], hop, args["os"], args["fs"],
                                      None) == 1, b
    assert lib.tvlp_wavetable_osc(None, fake, fake, 9, 512, fake, 127, fake, 2, n_out, F, hop, 4,
                                  48000.0, None) == 1
    assert lib.tvlp_wavetable_osc_vjp(*ok, None, fake, fake, 2, n_out, F, hop, 4, 48000.0,
                                      None) == 1
    # global FIR: taps 1..1024; workspace = B x tiles(n) x m floats
    assert lib.tvlp_global_fir(fake, fake, fake, 2, 5000, 0, None) == 1
    assert lib.tvlp_global_fir(fake, fake, fake, 2, 5000, 1025, None) == 1
    assert lib.tvlp_global_fir(fake, fake, fake, 0, 5000, 128, None) == 0
    assert lib.tvlp_global_fir_workspace(2, 5000, 128) == 2 * 3 * 128 * 4
    assert lib.tvlp_global_fir_workspace(4, 48001, 128) == 4 * 24 * 128 * 4
    assert lib.tvlp_global_fir_vjp(fake, fake, fake, None, fake, None, 0, 2, 5000, 128, None) == 3
    # MSS loss terms: per-item partials (64 chunks at most) of three sums
    assert lib.tvlp_mss_terms_workspace(32, 96000) == 32 * (96000 // 4096) * 3 * 4
    assert lib.tvlp_mss_terms_workspace(2, 10 ** 7) == 2 * 64 * 3 * 4
    assert lib.tvlp_mss_terms(None, fake, 2, 100, 1e-8, fake, fake, fake, 4096, None) == 1
    assert lib.tvlp_mss_terms(fake, fake, 2, 100, 1e-8, fake, fake, None, 0, None) == 3
    assert lib.tvlp_mss_terms(fake, fake, 0, 100, 1e-8, fake, fake, None, 0, None) == 0
    assert lib.tvlp_mss_terms_vjp(fake, fake, fake, None, fake, 2, 100, 1e-8, None) == 1


def test_longseq_combine_algebra():
    """The fold of the time split on small matrices (CPU torch): forward
    states and backward adjoints against a direct composition."""
    import torch

    from paper_2406_05128_b200 import longseq

    g = torch.Generator().manual_seed(0)
    R, B, M = 4, 2, 3
    Phis = [torch.randn(B, M, M, generator=g, dtype=torch.float64) * 0.5 for _ in range(R)]
    zs = [torch.randn(B, M, generator=g, dtype=torch.float64) for _ in range(R)]
    nus = [torch.randn(B, M, generator=g, dtype=torch.float64) for _ in range(R)]
    assert longseq.forward_combine(0, Phis, zs) is None
    x = zs[0]
    for r in range(1, R):
        got = longseq.forward_combine(r, Phis, zs)
        assert torch.allclose(got, x)
        x = torch.bmm(Phis[r], x.unsqueeze(-1)).squeeze(-1) + zs[r]
    assert longseq.backward_combine(R - 1, Phis, nus) is None
    mu = nus[R - 1]
    for r in range(R - 2, -1, -1):
        assert torch.allclose(longseq.backward_combine(r, Phis, nus), mu)
        mu = nus[r] + torch.bmm(Phis[r].transpose(1, 2), mu.unsqueeze(-1)).squeeze(-1)


def test_host_pipeline_chunk_schedule():
    from paper_2406_05128_b200 import stream

    assert stream._bounds(64, None) == [(8 * i, 8 * i + 8) for i in range(8)]
    assert stream._bounds(5, 8) == [(i, i + 1) for i in range(5)]  # at least one sequence each
    assert stream._bounds(10, [2, 8]) == [(0, 2), (2, 10)]
    for bad in ([3, 3], [0, 10], [11, -1]):
        with pytest.raises(ValueError):
            stream._bounds(10, bad)


def test_frameplan_semantics_match_reference_contract():
    """FramePlan (host metadata) reproduces the reference framing contract:
    lead-in frames, (row, sig_lo, sig_hi, win_lo, win_hi) order, COLA constant
    (params.py:152-217).  Against the reference itself when it is importable
    here (the GPU box has no /root/reference), else against hand-derived
    values for hop 240."""
    import os
    import sys

    import numpy as np

    from paper_2406_05128_b200 import params

    p = params.FramePlan.raised_cosine(240)
    assert (p.frame_size, p.n_lead_in(), p.cola_constant()) == (960, 3, 2.0)
    assert p.ola_deviation() < 1e-12
    fr = list(p.iter_frames(48000, 200))
    assert len(fr) == 203 and fr[0] == (0, 0, 240, 720, 960) and fr[3] == (0, 0, 960, 0, 960)
    assert fr[-1] == (199, 47760, 48000, 0, 240)
    ref_src = "/root/reference/pkg/src"
    if not os.path.isdir(ref_src):
        return
    sys.path.insert(0, ref_src)
    try:
        from tvlp import params as R
    except Exception:  # the reference's deps missing: the hand-derived checks stand
        return
    finally:
        sys.path.remove(ref_src)
    for hop in (240, 80, 7):
        try:
            a, b = R.FramePlan.raised_cosine(hop), params.FramePlan.raised_cosine(hop)
        except ValueError:
            continue
        assert a.frame_size == b.frame_size and np.array_equal(a.window, b.window)
        assert a.ola_deviation() == b.ola_deviation() and a.cola_constant() == b.cola_constant()
        for L, F in ((1000, 5), (48000, 201), (5, 1)):
            assert list(a.iter_frames(L, F)) == list(b.iter_frames(L, F))


def test_window_cache_follows_contents():
    """The kernel path's cached window state (COLA check, COLA constant, the
    device copy of the window) is keyed by the window's contents: editing the
    window in place is seen on the next call (no stale copy), and a repeated
    call reuses the cached copy."""
    import numpy as np
    import pytest
    import torch

    from paper_2406_05128_b200 import params

    p = params.FramePlan.raised_cosine(8)
    w1 = p._window_tensor(torch.float32, "cpu")
    assert p._window_tensor(torch.float32, "cpu") is w1  # cached
    np.testing.assert_array_equal(w1.numpy(), p.window.astype(np.float32))
    p._validate_cola_cached()
    assert p._cola_cached() == p.cola_constant()
    p.window[3] = 0.5  # in place: no longer COLA
    w2 = p._window_tensor(torch.float32, "cpu")
    assert float(w2[3]) == 0.5
    with pytest.raises(ValueError, match="constant overlap-add"):
        p._validate_cola_cached()
    assert p._cola_cached() == p.cola_constant()
