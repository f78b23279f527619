"""Kineto trace of the host pipeline (config 3): copy/kernel timelines per stream."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_05128_b200 import data, lpc, stream
lpc.set_validation("lazy")
B, T, M = 64, 48000, 22
e, A, g = data.d1_batch_torch(0, B, T, M, device="cuda")
eh, Ah, gh = (x.cpu().pin_memory() for x in (e, A, g))
oh = tuple(torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in (e, e, A))
for _ in range(3):
    stream.lp_tv_fwd_bwd_host(eh, Ah, gh, out=oh)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        stream.lp_tv_fwd_bwd_host(eh, Ah, gh, out=oh)
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
tr = json.load(open("gpurun_out/e2e_trace.json"))
ev = [x for x in tr["traceEvents"] if x.get("ph") == "X" and x.get("cat") in ("gpu_memcpy", "kernel", "gpu_memset")]
t0 = min(x["ts"] for x in ev)
rows = []
for x in sorted(ev, key=lambda x: x["ts"]):
    a = x.get("args", {})
    rows.append((round(x["ts"] - t0, 1), round(x["dur"], 1), a.get("stream"), x["cat"], x["name"][:40], a.get("bytes")))
with open("gpurun_out/e2e_timeline.txt", "w") as f:
    for r in rows:
        f.write(" ".join(str(v) for v in r) + "\n")
print(len(rows), "events")
