#!/usr/bin/env python
"""Benchmark: sample-wise LP forward+backward on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--config NAME] [--impl b200|reference]

A step is one LP forward + backward (lp_forward_tv then lp_backward_tv with
the forward's carry tape, i.e. what ``LPTV`` autograd runs) over one batch of
synthetic D1 input already resident in HBM.  The default
workload is config 3 of BASELINE.json (B=64, T=48000, M=22, fp32); with N
GPUs (torchrun, one process per GPU) the fixed global batch of 64 is split
64/N per rank with no collective in the filter (batch sharding, strong
scaling as the config defines it; ``--scaling weak`` keeps 64 per rank);
the timed region is bracketed by a barrier and synchronisation and the
reported time is the max over ranks.

Besides the device-resident ``value`` the line carries:
  e2e          the same metric through the public API from pinned HOST
               buffers: per step H2D of (e, A, grad_s), forward, backward, D2H
               of (s, grad_e, grad_A), all inside the timed region;
  roofline     the dominant kernel's algorithmic bytes / its CUDA-event
               duration (profiling pass over the same K steps) vs the measured
               HBM copy bandwidth in MEASURED_PEAKS.json, plus the whole step;
  cpu_baseline the reference's own CPU implementation -- the unmodified tvlp
               (numba) installed in baseline/_ref -- on N worker processes
               (N = host threads, capped at the step's sequences) and on one,
               with the oracle's threaded C port (oracle/) beside it, on a
               bounded sample (rank 0, N=1 only; baseline/tvlp_cpu.py).
``--impl reference`` times the same CPU leg alone (the reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LP fwd+bwd audio samples/sec and HBM GB/s vs roofline at 1/2/4/8 B200"
UNIT = "samples/s"

CONFIGS = {
    # name: kind, B (per GPU), T, M[, hop]
    "tv_b64_t48000": dict(kind="tv", B=64, T=48000, M=22, baseline_cfg=3, scaling="strong"),
    "tv_b4_t24000": dict(kind="tv", B=4, T=24000, M=22, baseline_cfg=1),
    "framewise_b32_t48000": dict(kind="framewise", B=32, T=48000, M=22, hop=240, baseline_cfg=2),
    "tv_b1_t14400000": dict(kind="tv", B=1, T=14_400_000, M=22, baseline_cfg=4),
    # config 5: HpN decoder's two LPs (H(z) on the glottal source, C(z) on the
    # noise) grouped into one launch; 256 items over 8 GPUs = 32 items per GPU
    "hpn_b32_t48000": dict(kind="hpn", B=32, T=48000, M=22, baseline_cfg=5,
                           encoder_params=6_100_000),
    # config 5 as BASELINE.json states it: the FULL GOLF HpN synthesiser step
    # on the GPU -- oscillator x4 + decimator, shaped noise, H(z) and the
    # paper's C(z) LP in one frame-rate launch, global FIR, the prime-size MSS
    # loss and the backward to every frame parameter (decoder.py, §8(f)
    # ranks 3-4) -- 32 items per GPU, encoder all-reduce stand-in overlapped
    "hpn_full_b32_t48000": dict(kind="decoder", B=32, T=48000, M=22, hop=240, baseline_cfg=5,
                                encoder_params=6_100_000, mode="hpn", c_lp=True),
    # config 3 with frame-rate coefficients (hop 240)
    # upsampled inside the kernels (the synthesiser's upsample_linear -> lp_tv)
    "tv_frames_b64_t48000": dict(kind="tvf", B=64, T=48000, M=22, hop=240, baseline_cfg=3),
    # config 4 as ONE sequence split in time across the ranks (strong scaling;
    # longseq.py: one all_gather of segment summaries per direction)
    "tv_b1_t14400000_split": dict(kind="tvsplit", B=1, T=14_400_000, M=22, baseline_cfg=4),
}
DEFAULT = "tv_b64_t48000"


def algorithmic_bytes_per_sample(cfg):
    """TV fwd 4(M+2) + bwd 4(2M+3) = 4(3M+5); frame-wise ~21.1;
    HpN: two TV LPs per audio sample (568 B)."""
    M = cfg["M"]
    if cfg["kind"] in ("tv", "tvsplit"):
        return 4 * (3 * M + 5)
    if cfg["kind"] in ("hpn", "decoder"):
        return 2 * 4 * (3 * M + 5)
    if cfg["kind"] == "tvf":
        # e, s (fwd); g_s, s, g_e (bwd); frames in twice and grad_frames out
        # at 1/hop of the sample rate
        return 4 * 5 + 3 * 4 * M / cfg["hop"]
    return 21.1


# per-kernel algorithmic bytes per sample (what each launch must move at least)
def kernel_bytes_per_sample(name, M):
    return {
        "basis": 4 * (M + 1),          # A, e in
        "apply_fwd": 4 * (M + 2),      # A, e in; s out
        "fwd_chain": 4 * (M + 2),      # carries + re-application: A, e in; s out
        "adjoint_zs": 4 * (M + 1),     # A, g_s in
        "adjoint_apply": 4 * (M + 2),  # A, g_s in; g_e out
        "bwd_chain": 4 * (M + 2),      # adjoint carries + re-application: A, g_s in; g_e out
        "grad_A": 4 * (M + 2),         # g_e, s in; g_A out
    }.get(name)


def kernel_bytes_per_sample_frames(name, M):
    """frame-rate path (rows interpolated in the kernels)"""
    return {"basis": 4, "apply_fwd": 8, "adjoint_zs": 4, "adjoint_apply": 8,
            "fwd_chain": 8, "bwd_chain": 8, "grad_frames": 8}.get(name)


def kernel_flops_per_sample_framewise(name, M, overlap=4):
    """frame-wise TI (SURVEY.md §8(d), 536 flop per audio sample at M=22):
    every sample lies in ``overlap`` frames; per frame-sample the forward runs
    M FMAs (+ the window), the backward M FMAs of the adjoint filter and M of
    the coefficient reduction (+ the window); OLA / gather add one each."""
    return {"fw_forward": overlap * (2 * M + 1),
            "fw_backward": overlap * (4 * M + 1)}.get(name)


def fp32_peak_tflops(sm_mhz=1965.0):
    """148 SMs x 128 FP32 lanes x 2 flop per FMA at the SM clock (derived;
    MEASURED_PEAKS.json carries HBM and bf16 only)."""
    return 148 * 128 * 2 * sm_mhz * 1e-6


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class Clocks:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self.go = threading.Event()  # set by the caller when its timed region starts
        self._t = None
        self._nvml = self._nvml_handle(index)

    @staticmethod
    def _nvml_handle(index):
        """In-process NVML sampling: an nvidia-smi child forked from this
        process during the timed region can stall the launching thread long
        enough to drain the GPU queue (step times 345-361 us on one box)."""
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            p = torch.cuda.get_device_properties(index)
            bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            try:
                return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                return pynvml, pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            return None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        flags = ["Active" if r & b else "Not Active" for b in bits]
        self.rows.append([str(self.index), str(sm), str(mx), "", hex(r)] + flags)

    def _run(self):
        self.go.wait(30)
        if self._nvml is not None:
            while not self._stop.is_set():
                try:
                    self._sample_nvml()
                except Exception:
                    self._nvml = None
                    break
                self._stop.wait(0.001)
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.go.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for n, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle (C port of the reference path), threaded
# ---------------------------------------------------------------------------

def cpu_baseline(cfg, seconds=10.0):
    """The reference's own CPU implementation on this host: the unmodified
    ``tvlp`` (numba, baseline/_ref) on N worker processes is the headline
    (kind "reference"), with its 1-process figure; the oracle's threaded C
    port (oracle/tvlp_oracle.c) on N threads and on 1 thread is reported
    beside it (kind "port", the headline only when baseline/_ref is absent).
    N = host threads, capped at the step's independent sequences (the
    reference filters each sequence serially).  Includes the CPU model."""
    nthreads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    # the reference filters each sequence serially: a step's work spreads over
    # at most one core per independent sequence (config 4's one 14.4 M-sample
    # sequence is one core's work whatever the host)
    nthreads = max(1, min(nthreads, cfg["B"] * (2 if cfg["kind"] == "hpn" else 1)))
    if cfg["kind"] == "decoder":
        port = None  # the C port covers the LP path only
    else:
        port = _port_baseline(cfg, nthreads, seconds)
        one = _port_baseline(cfg, 1, max(3.0, seconds / 3), one_core=True)
        port["one_core"] = {"value": one["value"], "cores": 1, "sample": one["sample"]}
    sys.path.insert(0, os.path.join(ROOT, "baseline"))
    import tvlp_cpu

    ref = None
    if tvlp_cpu.available():
        T_ref = min(cfg["T"], 480_000)  # a bounded slice of config 4's one sequence
        try:
            ref = tvlp_cpu.measure(cfg["kind"], T_ref, cfg["M"], cfg.get("hop", 240),
                                   procs=nthreads, seconds=max(3.0, seconds / 2),
                                   lps_per_sample=2 if cfg["kind"] == "hpn" else 1)
        except Exception as ex:  # reported; the port stands in
            if port is not None:
                port["reference_error"] = f"{type(ex).__name__}: {ex}"[:200]
    if ref is None:
        if port is None:
            return {"value": None, "unit": UNIT, "cores": nthreads, "kind": "reference",
                    "unavailable": "baseline/_ref absent",
                    "cpu_model": tvlp_cpu.cpu_model()}
        port["cpu_model"] = tvlp_cpu.cpu_model()
        return port
    return {"value": ref["n_core"]["value"], "unit": UNIT, "cores": ref["n_core"]["cores"],
            "kind": "reference", "impl": ref["impl"], "cpu_model": ref["cpu_model"],
            "sample": ref["sample"], "one_core": ref["one_core"], "port": port}


def _port_baseline(cfg, nthreads, seconds, one_core=False):
    import oracle
    from paper_2406_05128_b200 import data

    T, M = cfg["T"], cfg["M"]
    lps_per_sample = 2 if cfg["kind"] == "hpn" else 1
    if cfg["kind"] == "tvf":
        # the reference chain upsample_linear -> lp_tv fwd+bwd -> upsample VJP
        # (params.py:120-145 in numpy, the LP in the threaded C port)
        hop = cfg["hop"]
        B_s = max(1, min(cfg["B"], nthreads))
        e, fr, g = data.d1_frames_batch(1000, B_s, T, M, hop)

        def run_once():
            A = np.stack([oracle.upsample_linear(fr[b], hop, T - 1) for b in range(B_s)])
            s, ge, gA = oracle.batch_fwd_bwd("tv", e, A.astype(np.float32), g, nthreads=nthreads)
            return [oracle.upsample_linear_vjp(gA[b], fr.shape[1], hop, T - 1) for b in range(B_s)]

        run_once()
        times = []
        t_end = time.perf_counter() + seconds
        while len(times) < 3 or (time.perf_counter() < t_end and len(times) < 50):
            t0 = time.perf_counter()
            run_once()
            times.append(time.perf_counter() - t0)
        med = float(np.median(times))
        return {"value": round(B_s * T / med, 1), "unit": UNIT, "cores": nthreads, "kind": "port",
                "sample": f"{B_s} x {T} samples (M={M}, hop={hop}, D1 frames): upsample_linear "
                          f"(numpy) + LP fwd+bwd (oracle/tvlp_oracle.c, {nthreads} threads) + "
                          f"upsample VJP (numpy) per repeat, median of {len(times)} repeats"}
    if cfg["kind"] in ("tv", "hpn", "tvsplit"):
        T_s = min(T, 480_000)
        B_s = max(1, min(cfg["B"] * lps_per_sample, 4 * nthreads)) if T <= 480_000 else nthreads
        if one_core:
            B_s = min(B_s, 2)
        e, A, g = data.d1_batch(1000, B_s, T_s, M)
        kind = "tv"
    else:
        T_s = T
        B_s = max(1, min(cfg["B"], 4 * nthreads))
        if one_core:
            B_s = min(B_s, 2)
        e, A, g = data.d1_frames_batch(1000, B_s, T_s, M, cfg["hop"])
        kind = "framewise"
    oracle.batch_fwd_bwd(kind, e[:1], A[:1], g[:1], nthreads=1)  # warm (page-in)
    times = []
    t_end = time.perf_counter() + seconds
    while True:
        t0 = time.perf_counter()
        oracle.batch_fwd_bwd(kind, e, A, g, nthreads=nthreads, hop=cfg.get("hop", 240))
        times.append(time.perf_counter() - t0)
        if len(times) >= 3 and time.perf_counter() > t_end:
            break
        if len(times) >= 50:
            break
    med = float(np.median(times))
    return {"value": round(B_s * T_s / med / lps_per_sample, 1), "unit": UNIT, "cores": nthreads,
            "kind": "port",
            "sample": f"{B_s} x {T_s} samples (M={M}, D1) LP fwd+bwd per repeat"
                      f"{' (2 LPs per audio sample)' if lps_per_sample == 2 else ''}, median of "
                      f"{len(times)} repeats, {nthreads} threads, oracle/tvlp_oracle.c"}


def _reference_decoder(item, dtype, fields, f0, noise_seed, target, tables):
    """The reference's own decoder step (synth.build_synth_graph +
    loss.mss_loss + Tape.backward) for one item: (y, loss, grads)."""
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    from tvlp import loss, source, synth
    from tvlp.tape import Tape

    n_out, hop, mode = item["n_out"], item["hop"], item["mode"]
    F = (n_out - 1) // hop + 1
    p = synth.init_params(F, 22, hop, mode=mode, seed=0, f0_frames=f0)
    for k, v in fields.items():
        setattr(p, k, np.asarray(v, dtype=np.float64))
    wt = source.Wavetable(tables=tables, rd_grid=np.linspace(0.3, 2.7, tables.shape[0]))
    tape = Tape(dtype)
    y, leaves = synth.build_synth_graph(tape, p, n_out, 24000.0, noise_seed, wavetable=wt)
    L = loss.mss_loss(tape, y, target)
    tape.backward(L)
    return y.value, float(L.value), {k: tape.grad(v) for k, v in leaves.items()}


def parity_decoder(item):
    """The GPU decoder (float64, c_lp off: the reference has no C(z) LP)
    against the reference's own graph on one item of the bench's generator:
    max gradcheck_error over the output, the loss and every gradient."""
    import torch

    import oracle
    from paper_2406_05128_b200 import decoder as dmod

    n_out, hop = item["n_out"], item["hop"]
    fields, f0, noise, target = dmod.synthetic_inputs(1, n_out, hop, seed=item["seed"])
    tables = dmod.synthetic_tables()
    ry, rL, rg = _reference_decoder(item, np.float64, {k: v[0] for k, v in fields.items()}, f0[0],
                                    item["seed"], target[0], tables)
    dev = torch.device("cuda", 0)
    dec = dmod.Decoder(torch.tensor(tables, device=dev), hop=hop, mode=item["mode"])
    p = {k: torch.tensor(v, device=dev, requires_grad=True) for k, v in fields.items()}
    y = dec.render(p, n_out, torch.tensor(noise, device=dev), f0)
    L = dmod.mss_loss(y, torch.tensor(target, device=dev))
    L.sum().backward()
    errs = [oracle.gradcheck_error(y.detach().cpu().numpy()[0], ry),
            abs(float(L.detach()[0]) - rL) / max(abs(rL), 1e-12)]
    errs += [oracle.gradcheck_error(p[k].grad.cpu().numpy()[0], rg[k]) for k in rg]
    return max(errs)


def parity_check(cfg, sample):
    """Part of the CPU leg (rank 0, outside every timed region): the GPU
    outputs of the LAST timed step, for the first and last item of this
    rank's batch, against the float64 oracle on the same float32 inputs,
    with the reference's metric (oracle.py:228-234).  Returns the max error
    over the items and outputs checked, so the bench line carries parity
    evidence at the exact kernel geometry it timed."""
    import oracle

    kind = cfg["kind"]
    if kind == "decoder":
        try:
            return parity_decoder(sample[0])
        except ImportError:  # the reference install (baseline/_ref) is absent
            return None
    worst = 0.0
    for item in sample:
        x = {k: np.asarray(v, dtype=np.float64) for k, v in item.items()}
        if kind in ("tv", "hpn", "tvsplit"):
            rs = oracle.lp_forward_tv(x["e"], x["A"])
            rge, rgA = oracle.lp_backward_tv(x["g"], x["A"], rs)
            ref = (rs, rge, rgA)
        elif kind == "tvf":
            ref = oracle.lp_tv_frames_fwd_bwd(x["e"], x["A"], cfg["hop"], x["g"])
        else:
            ry, rseg = oracle.framewise_forward(x["e"], x["A"], cfg["hop"])
            ref = (ry,) + tuple(oracle.framewise_backward(x["g"], x["A"], rseg, cfg["hop"]))
        for got, want in zip((x["o0"], x["o1"], x["o2"]), ref):
            worst = max(worst, oracle.gradcheck_error(got, want))
    return worst


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_b200(args, cfg, rank, world, dist):
    import torch

    from paper_2406_05128_b200 import _native as N
    from paper_2406_05128_b200 import data, lpc, params
    from paper_2406_05128_b200 import dist as pdist

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    lpc.set_validation("lazy")
    lib = N.load()
    B, T, M = cfg["B"], cfg["T"], cfg["M"]
    kind = cfg["kind"]
    strong = args.scaling == "strong" and kind != "tvsplit"
    # (strong: a fixed global batch split over the ranks; --shard-of S runs
    # rank 0's share of an S-way split on one GPU, reported as such)
    lo, B, B_glob = pdist.bench_shard(B, "strong" if strong else "weak", rank, world,
                                      args.shard_of)
    allreduce = None
    grad = None
    if kind in ("tv", "hpn"):
        if kind == "tv":
            e, A, g = data.d1_batch_torch(lo, B, T, M, device=dev)

            def step(e=e, A=A, g=g):
                s, carry = lpc._forward(False, e, A, None, return_carry=True)
                ge, gA = lpc._backward(False, g, A, s, None, carry)
                return s, ge, gA
        else:
            # the HpN decoder's two LPs on their OWN buffers -- H(z) on the
            # glottal source, C(z) on the noise (D1 tracks, distinct seeds) --
            # through the grouped launch (tvlp_lp_*_tv_grouped)
            eh, Ah, gh = data.d1_batch_torch(2 * lo, B, T, M, device=dev)
            ec, Ac, gc = data.d1_batch_torch(2 * lo + B, B, T, M, device=dev)
            e, A, g = [eh, ec], [Ah, Ac], [gh, gc]
            if dist is not None:
                grad = torch.randn(cfg["encoder_params"], device=dev)

                def allreduce():
                    return dist.all_reduce(grad, async_op=True)

            def step(e=e, A=A, g=g):
                (sh, sc), carry = lpc.lp_forward_tv_grouped([(e[0], A[0]), (e[1], A[1])],
                                                            return_carry=True)
                # the encoder all-reduce in flight during the LP backward
                (geh, gAh), (gec, gAc) = pdist.overlapped_allreduce(
                    grad, dist, lambda: lpc.lp_backward_tv_grouped(
                        [(g[0], A[0], sh), (g[1], A[1], sc)], carry=carry))
                return [sh, sc], [geh, gec], [gAh, gAc]
    elif kind == "decoder":
        from paper_2406_05128_b200 import decoder as dmod

        n_out = T + 1
        F = (n_out - 1) // cfg["hop"] + 1
        fields, f0, noise, target = dmod.synthetic_inputs(B, n_out, cfg["hop"], seed=lo)
        dec = dmod.Decoder(torch.tensor(dmod.synthetic_tables(), dtype=torch.float32, device=dev),
                           hop=cfg["hop"], mode=cfg["mode"], c_lp=cfg["c_lp"])
        params_d = {k: torch.tensor(v, dtype=torch.float32, device=dev, requires_grad=True)
                    for k, v in fields.items()}
        noise_d = torch.tensor(noise, dtype=torch.float32, device=dev)
        target_d = torch.tensor(target, dtype=torch.float32, device=dev)
        c_frames = torch.tensor(dmod.stable_c_frames(B, F, seed=lo), dtype=torch.float32,
                                device=dev) if cfg["c_lp"] else None
        if dist is not None:
            grad = torch.randn(cfg["encoder_params"], device=dev)
        e, A, g = noise_d, params_d, target_d  # (host copies for e2e: see below)
        # the whole step -- render, loss, backward -- captured once in a CUDA
        # graph over these static buffers (decoder.GraphedStep) and replayed:
        # every kernel of the step runs each replay, with no host work
        gstep = dmod.GraphedStep(dec, params_d, noise_d, target_d,
                                 torch.tensor(f0, dtype=torch.float64, device=dev), c_frames)

        def step(e=noise_d, A=params_d, g=target_d):
            y, L = gstep.replay()
            if dist is not None:  # the encoder all-reduce stand-in (after the graph)
                dist.all_reduce(grad)
            return y, L, A["reflection_raw"].grad

        def eager_step():  # the same step without the graph (per-kernel profiling pass)
            gstep._run()
    elif kind == "tvsplit":
        from paper_2406_05128_b200 import longseq

        Tr = T // world  # this rank's time segment of the one sequence
        e_all, A_all, g_all = data.d1_batch_torch(0, 1, T, M, device=dev)
        e = e_all[:, rank * Tr:(rank + 1) * Tr].contiguous()
        A = A_all[:, rank * Tr:(rank + 1) * Tr].contiguous()
        g = g_all[:, rank * Tr:(rank + 1) * Tr].contiguous()
        del e_all, A_all, g_all

        def step(e=e, A=A, g=g):
            if dist is None:
                s, carry = lpc._forward(False, e, A, None, return_carry=True)
                ge, gA = lpc._backward(False, g, A, s, None, carry)
                return s, ge, gA
            s, ctx = longseq.lp_tv_forward_split(e, A)
            ge, gA = longseq.lp_tv_backward_split(g, A, s, ctx)
            return s, ge, gA
    elif kind == "tvf":
        ev, fr, gv = data.d1_frames_batch(lo, B, T, M, cfg["hop"])
        e = torch.from_numpy(ev).to(dev)
        A = torch.from_numpy(fr).to(dev)  # frame rows [B, F, M]
        g = torch.from_numpy(gv).to(dev)
        hop = cfg["hop"]

        def step(e=e, A=A, g=g):
            s, carry = lpc.lp_forward_tv_frames(e, A, hop, return_carry=True)
            ge, gf = lpc.lp_backward_tv_frames(g, A, hop, s, carry=carry)
            return s, ge, gf
    else:
        ev, fr, gv = data.d1_frames_batch(lo, B, T, M, cfg["hop"])
        e = torch.from_numpy(ev).to(dev)
        A = torch.from_numpy(fr).to(dev)
        g = torch.from_numpy(gv).to(dev)
        plan = params.FramePlan.raised_cosine(cfg["hop"])

        def step(e=e, A=A, g=g):
            y, seg, aux = params.framewise_forward(e, A, plan, return_aux=True)
            ge, gf = params.framewise_backward(g, A, seg, plan, aux=aux)
            return y, ge, gf

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = lib.tvlp_launch_count()
    r0 = lib.tvlp_refined_sequences()
    with Clocks(dev.index) as clk:
        barrier()
        ev0.record(stream)
        clk.go.set()  # the sampler starts with the timed region
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = lib.tvlp_launch_count() - n0
    if kind == "decoder":  # replays: the launches captured in the graph, per step
        launches = gstep.launches * args.steps
    refined = lib.tvlp_refined_sequences() - r0
    ms = pdist.max_over_ranks(ev0.elapsed_time(ev1) / args.steps, dist, dev)
    nonfinite_seen = lpc.check_nonfinite(dev)
    samples = T * (B if kind == "tvsplit" else B_glob)
    value = samples / (ms * 1e-3)

    # outputs of one more step for the parity check of the CPU leg (items 0
    # and B-1 of this rank; the LP rows of an HpN batch are its first items)
    outs = step()
    torch.cuda.synchronize()
    parity_sample = []
    if kind == "decoder":
        # the CPU leg compares the decoder in float64 (c_lp off: the
        # reference has no C(z) LP) with the reference's own graph, item 0
        parity_sample.append({"seed": lo, "n_out": T + 1, "hop": cfg["hop"], "mode": cfg["mode"]})
        outs = None
    # (HpN: item 0 of the H(z) group and the last item of the C(z) group)
    picks = ([] if kind == "decoder" else [(0, 0), (1, B - 1)] if kind == "hpn" else
             [(None, b) for b in sorted({0, e.shape[0] - 1})])
    for grp, b in picks:
        sel = (lambda x: x[b]) if grp is None else (lambda x, grp=grp: x[grp][b])
        parity_sample.append({"e": sel(e).cpu().numpy(), "A": sel(A).cpu().numpy(),
                              "g": sel(g).cpu().numpy(), "o0": sel(outs[0]).cpu().numpy(),
                              "o1": sel(outs[1]).cpu().numpy(), "o2": sel(outs[2]).cpu().numpy()})
    del outs

    # profiling pass: per-kernel CUDA-event durations over K steps
    N.profile_dump()
    lib.tvlp_profile_enable(1)
    for _ in range(args.steps):
        (eager_step if kind == "decoder" else step)()
    torch.cuda.synchronize()
    lib.tvlp_profile_enable(0)
    prof = N.profile_dump()
    hbm, peak_kind = peaks()
    nsteps = max(1, args.steps)
    per_kernel = {}
    tot_all = sum(v[1] for v in prof.values()) or 1.0
    for name, (cnt, tot) in prof.items():
        per_kernel[name] = {"launches_per_step": round(cnt / nsteps, 2),
                            "us_per_step": round(tot / nsteps * 1e3, 2),
                            "share": round(tot / tot_all, 4)}
    dom = max(prof.items(), key=lambda kv: kv[1][1])[0] if prof else None
    if kind == "decoder" and prof:
        # the roofline line is the dominant LP kernel (frame-rate rows); the
        # decoder's other kernels and cuFFT are reported in `kernels`
        lp = {k: v for k, v in prof.items()
              if kernel_bytes_per_sample_frames(k, M) is not None or k in ("carry_fwd", "carry_bwd")}
        dom = max(lp.items(), key=lambda kv: kv[1][1])[0] if lp else dom
    roof = None
    if dom is not None and kind == "framewise":
        cnt, tot = prof[dom]
        t_step = tot / nsteps * 1e-3
        fps = kernel_flops_per_sample_framewise(dom, M, cfg.get("frame_size", 4 * cfg["hop"]) // cfg["hop"])
        ach = fps * B * T / t_step / 1e12
        pk = fp32_peak_tflops()
        roof = {"bound": "fp32", "kernel": dom, "achieved": round(ach, 2), "peak": round(pk, 1),
                "unit": "TFLOP/s", "frac": round(ach / pk, 4), "traffic": None,
                "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 flop x 1965 MHz (max SM "
                               "clock); the path has no tensor-core contraction",
                "flops_per_sample": fps, "us_per_step": round(t_step * 1e6, 2),
                "launches_per_step": cnt / nsteps,
                "step_flops_per_sample": sum(kernel_flops_per_sample_framewise(k, M)
                                             for k in ("fw_forward", "fw_backward"))}
    elif dom is not None:
        bps = (kernel_bytes_per_sample_frames if kind in ("tvf", "decoder")
               else kernel_bytes_per_sample)(dom, M)
        lp_rows = 2 * B if kind in ("hpn", "decoder") else B  # LP sequences per GPU
        T_k = T // world if kind == "tvsplit" else T  # samples per sequence on this GPU
        cnt, tot = prof[dom]
        t_step = tot / nsteps * 1e-3  # seconds of this kernel per step (all its slices)
        ach = (bps * lp_rows * T_k / t_step / 1e9) if bps is not None else None
        traffic = None
        tf = os.path.join(ROOT, "profiles", "r2_traffic.json")
        if (os.path.exists(tf) and kind in ("tv", "hpn") and (lp_rows, T, M) == (64, 48000, 22)
                and world == 1):
            # dram__bytes_read + dram__bytes_write of this phase's kernels in one
            # step, from the ncu capture of the same config
            # (profiles/r2_ncu_tv_b64_t48000.csv via tools/traffic_from_ncu.py)
            with open(tf) as fh:
                traffic = json.load(fh).get("per_step", {}).get(dom, {}).get("dram_bytes")
        roof = {"bound": "hbm", "kernel": dom,
                "achieved": None if ach is None else round(ach, 1), "peak": hbm, "unit": "GB/s",
                "frac": None if ach is None else round(ach / hbm, 4), "traffic": traffic,
                "peak_source": peak_kind,
                "bytes_per_step": None if bps is None else bps * lp_rows * T_k,
                "us_per_step": round(t_step * 1e6, 2), "launches_per_step": cnt / nsteps}
        if dom in ("basis",) and kind in ("tv", "hpn", "tvf", "tvsplit", "decoder"):
            # the basis is FP32-FMA bound: 23 chains x 22 FMA per sample
            fl = 2.0 * (M + 1) * M * lp_rows * T_k / t_step / 1e12
            fp32_peak = 148 * 128 * 2 * 1.965e-3  # TFLOP/s at the max SM clock (derived)
            roof["fp32_tflops"] = round(fl, 2)
            roof["fp32_frac_of_derived_peak"] = round(fl / fp32_peak, 4)
    step_gbs = algorithmic_bytes_per_sample(cfg) * B * T / (ms * 1e-3) / 1e9

    # e2e: pinned host buffers through the public API (HpN: the host batch of
    # both filters' rows, H(z) then C(z), through the pipelined host API)
    if kind == "decoder":
        # host: the frame parameters, noise and target in; the output signal,
        # the per-item losses and every parameter gradient out
        ph = {k: v.detach().cpu().pin_memory() for k, v in A.items()}
        nh, th = e.cpu().pin_memory(), g.cpu().pin_memory()
        yh = torch.empty((B, T + 1), dtype=torch.float32, pin_memory=True)
        lh = torch.empty(B, dtype=torch.float32, pin_memory=True)
        gh_ = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in ph.items()}
        h2d = sum(x.numel() * x.element_size() for x in list(ph.values()) + [nh, th])
        d2h = sum(x.numel() * x.element_size() for x in list(gh_.values()) + [yh, lh])

        # every step copies its inputs up and its results down, on a second
        # stream through device staging buffers so the copies overlap the
        # neighbouring steps' graph replays: step i+1's inputs land while step
        # i replays, step i's results drain while step i+1 replays (double-
        # buffered); e2e_flush() joins the copy stream before the clock stops
        cstream = torch.cuda.Stream(dev)    # host -> device
        dstream = torch.cuda.Stream(dev)    # device -> host (the other copy engine)
        s_in = {k: torch.empty_like(v, device=dev) for k, v in ph.items()}
        s_n, s_t = torch.empty_like(e), torch.empty_like(g)
        s_out = [({k: torch.empty_like(A[k]) for k in ph}, torch.empty_like(gstep.y),
                  torch.empty_like(gstep.loss)) for _ in range(2)]
        pipe = {"i": 0, "in_ready": None, "drained": [None, None]}

        def stage_inputs():
            with torch.cuda.stream(cstream):
                for k, v in ph.items():
                    s_in[k].copy_(v, non_blocking=True)
                s_n.copy_(nh, non_blocking=True)
                s_t.copy_(th, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cstream)
            return ev

        def e2e_step():
            main = torch.cuda.current_stream(dev)
            if pipe["in_ready"] is None:
                pipe["in_ready"] = stage_inputs()
            main.wait_event(pipe["in_ready"])
            with torch.no_grad():
                for k in ph:
                    A[k].copy_(s_in[k])
                e.copy_(s_n)
                g.copy_(s_t)
            consumed = torch.cuda.Event()
            consumed.record(main)
            cstream.wait_event(consumed)
            pipe["in_ready"] = stage_inputs()          # the next step's inputs
            y, L, _ = step()
            j = pipe["i"] % 2
            if pipe["drained"][j] is not None:
                main.wait_event(pipe["drained"][j])
            og, oy, ol = s_out[j]
            with torch.no_grad():
                oy.copy_(y.detach())
                ol.copy_(L.detach())
                for k in ph:
                    og[k].copy_(A[k].grad)
            ready = torch.cuda.Event()
            ready.record(main)
            dstream.wait_event(ready)
            with torch.cuda.stream(dstream):
                yh.copy_(oy, non_blocking=True)
                lh.copy_(ol, non_blocking=True)
                for k in ph:
                    gh_[k].copy_(og[k], non_blocking=True)
                drained = torch.cuda.Event()
                drained.record(dstream)
            pipe["drained"][j] = drained
            pipe["i"] += 1

        def e2e_flush():
            torch.cuda.current_stream(dev).wait_stream(cstream)
            torch.cuda.current_stream(dev).wait_stream(dstream)
    elif kind == "hpn":
        eh, Ah, gh = (torch.cat([y.cpu() for y in x]).pin_memory() for x in (e, A, g))
        oh = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in (eh, eh, Ah)]
    else:
        eh, Ah, gh = (x.cpu().pin_memory() for x in (e, A, g))
        outs = step()
        oh = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in outs]
    if kind != "decoder":
        h2d = sum(x.numel() * x.element_size() for x in (eh, Ah, gh))
        d2h = sum(x.numel() * x.element_size() for x in oh)

    if kind == "decoder":
        pass  # e2e_step defined above
    elif kind in ("tv", "hpn"):
        from paper_2406_05128_b200 import stream as pstream

        def e2e_step():
            # host batches through the pipelined public API: chunk copies in
            # both directions overlap the kernels of the neighbouring chunks
            pstream.lp_tv_fwd_bwd_host(eh, Ah, gh, out=oh, device=dev)
            if allreduce is not None:
                allreduce().wait()
    else:
        # every step copies its own inputs up and results down on a second
        # stream: the next step's inputs land in the other device buffer set
        # while this step runs, and this step's results drain while the next
        # one runs (results are fresh tensors, held by the allocator until then)
        cstream2 = torch.cuda.Stream(dev)   # host -> device
        dstream2 = torch.cuda.Stream(dev)   # device -> host (the other copy engine)
        bufs_in = [tuple(torch.empty(x.shape, dtype=x.dtype, device=dev) for x in (eh, Ah, gh))
                   for _ in range(2)]
        pipe2 = {"i": 0, "ready": [None, None], "free": [None, None]}

        def stage(j):
            with torch.cuda.stream(cstream2):
                if pipe2["free"][j] is not None:
                    cstream2.wait_event(pipe2["free"][j])
                for d, h in zip(bufs_in[j], (eh, Ah, gh)):
                    d.copy_(h, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cstream2)
            pipe2["ready"][j] = ev

        def e2e_step():
            main = torch.cuda.current_stream(dev)
            j = pipe2["i"] % 2
            if pipe2["ready"][j] is None:
                stage(j)
            stage(1 - j)                                  # the next step's inputs
            main.wait_event(pipe2["ready"][j])
            res = step(*bufs_in[j])
            done = torch.cuda.Event()
            done.record(main)
            pipe2["free"][j] = done
            pipe2["ready"][j] = None
            dstream2.wait_event(done)
            with torch.cuda.stream(dstream2):
                for o, r in zip(oh, res):
                    o.copy_(r, non_blocking=True)
                    r.record_stream(dstream2)             # not reused before the copy drains
            pipe2["i"] += 1

        def e2e_flush():
            torch.cuda.current_stream(dev).wait_stream(cstream2)
            torch.cuda.current_stream(dev).wait_stream(dstream2)

    if kind in ("tv", "hpn"):
        def e2e_flush():
            pass
    for _ in range(max(1, args.warmup)):
        e2e_step()
    e2e_flush()
    barrier()
    ev0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e2e_flush()
    ev1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = pdist.max_over_ranks(ev0.elapsed_time(ev1) / args.steps, dist, dev)

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong" if (kind == "tvsplit" or strong) else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic D1 (SURVEY.md §8(d)); inputs resident in HBM; working set "
                f"{round(algorithmic_bytes_per_sample(cfg) * B * T / 1e6)} MB > 126 MB L2 "
                "(no flush needed)",
        "config": {"workload": args.config, "baseline_config": cfg["baseline_cfg"],
                   "kind": kind, "B_per_gpu": B, "T": T, "M": M,
                   "global_B": B_glob, "parallelism": f"batch-shard x{world}",
                   "shard_of": args.shard_of if (strong and world == 1 and args.shard_of > 1) else None,
                   "cuda_graph": kind == "decoder",
                   "carry_precision": lpc.carry_precision(),
                   "subchunk": int(lib.tvlp_subchunk_len(2 * B if kind == "hpn" else B, T, M)) if kind in ("tv", "hpn", "tvf") else None,
                   "l2": "inputs larger than L2"},
        "gbs_algorithmic_step": round(step_gbs, 1),
        "step_roofline_frac": round(step_gbs / hbm, 4),
        **({"step_fp32_tflops": round(roof["step_flops_per_sample"] * B * T / (ms * 1e-3) / 1e12, 2),
            "step_fp32_frac": round(roof["step_flops_per_sample"] * B * T / (ms * 1e-3) / 1e12
                                    / fp32_peak_tflops(), 4)}
           if kind == "framewise" and roof else {}),
        "roofline": roof,
        "kernels": per_kernel,
        "e2e": {"value": round(samples / (e2e_ms * 1e-3), 1), "unit": UNIT,
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": round(e2e_ms, 3),
                "copies": ("every step's inputs up and results down on a second stream "
                           "(double-buffered device staging), overlapping the neighbouring "
                           "steps' graph replays" if kind == "decoder" else
                           "pipelined host API (chunks overlap kernels and both copy directions)"
                           if kind in ("tv", "hpn") else
                           "every step's inputs up and results down on a second stream, "
                           "overlapping the neighbouring steps")},
        "gpu_launches": int(launches),
        "nonfinite_outputs": bool(nonfinite_seen),
        "refined_sequences": int(refined),
        "clocks": clk.summary(),
    }
    return line, parity_sample


def run_reference(args, cfg):
    base = cpu_baseline(cfg, seconds=max(5.0, min(60.0, 2.0 * args.steps)))
    return {
        "metric": METRIC, "value": round(base["value"], 1), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic D1 (SURVEY.md §8(d))",
        "config": {"workload": args.config, "baseline_config": cfg["baseline_cfg"],
                   "kind": cfg["kind"], "B_per_gpu": cfg["B"], "T": cfg["T"], "M": cfg["M"]},
        "impl": "reference",
        "cpu_baseline": base,
        "e2e": {"value": round(base["value"], 1), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="default: the config's own (config 3: strong, global B=64)")
    ap.add_argument("--shard-of", type=int, default=0,
                    help="1-GPU probe: run rank 0's share of an S-way strong split")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.scaling is None:
        args.scaling = cfg.get("scaling", "weak")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, cfg)), flush=True)
        return 0

    from paper_2406_05128_b200 import dist as pdist

    dist = pdist.init("nccl") if world > 1 else None
    line, sample = run_b200(args, cfg, rank, world, dist)
    if rank == 0:
        if not (cfg["kind"] == "tvsplit" and world > 1):  # a rank holds a segment only
            line["parity_max_err"] = parity_check(cfg, sample)
            line["parity_items"] = len(sample)
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
