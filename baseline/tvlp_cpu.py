"""CPU timing of the UNMODIFIED reference ``tvlp`` (installed under
``baseline/_ref`` from /root/reference by the offline pip install that
DESIGN.md records) on this host's cores -- the CPU baseline SURVEY.md §8(d)
specifies: the reference's own public functions, 1 process and N processes,
with the CPU model stated.

This is benchmark infrastructure (``bench.py``'s cpu_baseline leg), never a
product path.  The reference is single-threaded numba per sequence
(``lpc.py:36-61`` kernels, ``lpc.py:101-173`` glue), so "N cores" means N
worker processes, each filtering its own share of the batch -- the pattern of
``cli.py:302-338`` (median wall time of the public calls) run in parallel.

Per item the timed work is exactly what the reference's tape op runs for one
forward + backward:
  tv / hpn / tvsplit  lp_forward_tv + lp_backward_tv          (lpc.py:101-173)
  tvf                 upsample_linear -> lp_tv -> _upsample_linear_vjp
                                                              (params.py:120-145)
  framewise           _framewise_forward + _framewise_vjp     (params.py:220-273)
Inputs are the D1 tracks of ``paper_2406_05128_b200.data`` (numpy only),
generated before the timed region.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")
ROOT = os.path.dirname(HERE)


def available():
    return os.path.isdir(os.path.join(REF, "tvlp"))


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def _single_thread_env():
    for k in ("NUMBA_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS",
              "OPENBLAS_NUM_THREADS"):
        os.environ[k] = "1"
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tvlp_numba_cache")


def _import():
    for p in (REF, ROOT):
        if p not in sys.path:
            sys.path.insert(0, p)
    import tvlp.lpc as lpc
    import tvlp.params as params

    return lpc, params


def _items(kind, seeds, T, M, hop):
    from paper_2406_05128_b200 import data

    out = []
    for sd in seeds:
        if kind in ("tvf", "framewise"):
            e, fr, g = data.d1_frames_batch(sd, 1, T, M, hop)
            out.append((e[0], fr[0], g[0]))
        else:
            e, A, g = data.d1_batch(sd, 1, T, M)
            out.append((e[0], A[0], g[0]))
    return out


def _decoder_items(seeds, T, hop):
    from paper_2406_05128_b200 import decoder as dmod

    out = []
    for sd in seeds:
        fields, f0, noise, target = dmod.synthetic_inputs(1, T + 1, hop, seed=sd)
        out.append(({k: v[0] for k, v in fields.items()}, f0[0], sd, target[0]))
    return out, dmod.synthetic_tables()


def _one_decoder(item, tables, hop):
    """The reference HpN decoder step on its Tape (float32 tape): synthesis,
    MSS loss, backward (synth.py:217-275, loss.py:105-126)."""
    from tvlp import loss, source, synth
    from tvlp.tape import Tape
    import numpy as np

    fields, f0, seed, target = item
    n_out = target.shape[0]
    F = (n_out - 1) // hop + 1
    p = synth.init_params(F, 22, hop, mode="hpn", seed=0, f0_frames=f0)
    for k, v in fields.items():
        setattr(p, k, v)
    wt = source.Wavetable(tables=tables, rd_grid=np.linspace(0.3, 2.7, tables.shape[0]))
    tape = Tape(np.float32)
    y, _ = synth.build_synth_graph(tape, p, n_out, 24000.0, seed, wavetable=wt)
    tape.backward(loss.mss_loss(tape, y, target))


def _one(lpc, params, kind, item, hop, plan):
    if kind == "decoder":
        return _one_decoder(item[0], item[1], hop)
    e, A, g = item
    if kind == "tvf":
        T1 = e.shape[0]
        Au = params.upsample_linear(A, hop, T1 - 1)
        s = lpc.lp_forward_tv(e, Au)
        ge, gAu = lpc.lp_backward_tv(g, Au, s)
        params._upsample_linear_vjp(gAu, A.shape[0], hop, T1 - 1)
    elif kind == "framewise":
        y, segs = params._framewise_forward(e, A, plan)
        params._framewise_vjp(g, e, A, plan, segs)
    else:
        s = lpc.lp_forward_tv(e, A)
        lpc.lp_backward_tv(g, A, s)


def _worker(kind, seeds, T, M, hop, seconds, barrier, q):
    _single_thread_env()
    lpc, params = _import()
    plan = params.FramePlan.raised_cosine(hop) if kind == "framewise" else None
    if kind == "decoder":
        its, tables = _decoder_items(seeds, T, hop)
        items = [(it, tables) for it in its]
    else:
        items = _items(kind, seeds, T, M, hop)
    _one(lpc, params, kind, items[0], hop, plan)  # jit compile / cache load
    barrier.wait()
    n = 0
    t0 = time.perf_counter()
    while True:
        for it in items:
            _one(lpc, params, kind, it, hop, plan)
            n += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    q.put((n, el))


def time_reference(kind, T, M, hop=240, procs=1, seconds=6.0, seed=1000):
    """Aggregate samples/s of the reference over ``procs`` worker processes,
    each looping over its own item(s) for ``seconds``; throughput = all items
    finished x T / the slowest worker's wall time."""
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(procs)
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker,
                      args=(kind, [seed + r], T, M, hop, seconds, barrier, q), daemon=True)
          for r in range(procs)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    items = sum(n for n, _ in res)
    wall = max(el for _, el in res)
    return items * T / wall, items, wall


def measure(kind, T, M, hop=240, procs=None, seconds=6.0, lps_per_sample=1):
    """Both legs (1 process, ``procs`` processes) as a dict for bench.py."""
    if procs is None:
        procs = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    one, n1, w1 = time_reference(kind, T, M, hop, 1, seconds)
    many, nn, wn = ((one, n1, w1) if procs == 1 else
                    time_reference(kind, T, M, hop, procs, seconds))
    what = {"tv": "lp_forward_tv + lp_backward_tv (lpc.py:101-173)",
            "hpn": "lp_forward_tv + lp_backward_tv per LP, 2 LPs per audio sample",
            "tvsplit": "lp_forward_tv + lp_backward_tv (lpc.py:101-173)",
            "tvf": "upsample_linear + lp_forward_tv + lp_backward_tv + upsample VJP",
            "framewise": "_framewise_forward + _framewise_vjp (params.py:220-273)",
            "decoder": "the reference's HpN decoder step on its Tape: build_synth_graph + "
                       "mss_loss + backward (synth.py:217-275, loss.py:105-126; no C(z) LP: "
                       "the reference has none)"}[kind]
    return {
        "kind": "reference", "impl": "tvlp (numba, baseline/_ref, unmodified)",
        "unit": "samples/s", "cpu_model": cpu_model(),
        "one_core": {"value": round(one / lps_per_sample, 1), "cores": 1,
                     "items": n1, "wall_s": round(w1, 3)},
        "n_core": {"value": round(many / lps_per_sample, 1), "cores": procs,
                   "items": nn, "wall_s": round(wn, 3)},
        "sample": f"items of T={T}, M={M} (D1), {what}; each worker process loops over its "
                  f"own item for >= {seconds} s after a jit warm-up; aggregate = items x T / "
                  f"slowest worker's wall time",
    }


if __name__ == "__main__":
    import json

    kind = sys.argv[1] if len(sys.argv) > 1 else "tv"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 48000
    print(json.dumps(measure(kind, T, 22, seconds=3.0,
                             procs=int(sys.argv[3]) if len(sys.argv) > 3 else None)))
