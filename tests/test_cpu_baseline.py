"""bench.py's CPU baseline leg (CPU only): the unmodified reference tvlp
(baseline/_ref) on 1 and N worker processes beside the oracle's C port, with
the CPU model -- the shape of the `cpu_baseline` object every bench line
carries (SURVEY.md §8(d) CPU-baseline plan)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline"))


def test_cpu_baseline_reference_and_port():
    import bench
    import tvlp_cpu

    if not tvlp_cpu.available():
        pytest.skip("baseline/_ref (the reference install) is absent")
    cfg = dict(kind="tv", B=2, T=2400, M=22, baseline_cfg=1)
    cb = bench.cpu_baseline(cfg, seconds=0.3)
    assert cb["kind"] == "reference" and cb["unit"] == "samples/s"
    assert cb["cores"] == min(2, len(os.sched_getaffinity(0)))
    assert cb["value"] > 0 and cb["one_core"]["value"] > 0 and cb["one_core"]["cores"] == 1
    assert cb["port"]["kind"] == "port" and cb["port"]["value"] > 0
    assert cb["port"]["one_core"]["cores"] == 1
    assert isinstance(cb["cpu_model"], str) and cb["cpu_model"]


def test_reference_timing_frame_wise_and_frames():
    import tvlp_cpu

    if not tvlp_cpu.available():
        pytest.skip("baseline/_ref (the reference install) is absent")
    for kind in ("framewise", "tvf"):
        r = tvlp_cpu.measure(kind, 4800, 22, hop=240, procs=1, seconds=0.2)
        assert r["one_core"]["value"] > 0 and r["n_core"]["cores"] == 1
