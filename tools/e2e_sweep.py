"""Time stream.lp_tv_fwd_bwd_host on config 3 for several chunk counts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_05128_b200 import data, lpc, stream
lpc.set_validation("lazy")
B, T, M = 64, 48000, 22
e, A, g = data.d1_batch_torch(0, B, T, M, device="cuda")
eh, Ah, gh = (x.cpu().pin_memory() for x in (e, A, g))
oh = tuple(torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in (e, e, A))
for ch in (2, 4, 8, 16, 32, 64):
    for _ in range(2):
        stream.lp_tv_fwd_bwd_host(eh, Ah, gh, out=oh, chunks=ch)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        stream.lp_tv_fwd_bwd_host(eh, Ah, gh, out=oh, chunks=ch)
    b.record(); torch.cuda.synchronize()
    print("chunks", ch, round(a.elapsed_time(b) / 5, 3), "ms")

# copy-only pipeline (same streams/events, no kernels)
bufs = stream._buffers(torch.device("cuda", 0), B, T, M, torch.float32, [B // 8], False)
h2d, comp, d2h = stream._streams(torch.device("cuda", 0), 3)
def copies(n):
    main = torch.cuda.current_stream()
    for st in (h2d, comp, d2h): st.wait_stream(main)
    for i in range(n):
        lo, hi = B * i // n, B * (i + 1) // n
        with torch.cuda.stream(h2d):
            for k, src in (("e", eh), ("A", Ah), ("g", gh)):
                bufs[k][lo:hi].copy_(src[lo:hi], non_blocking=True)
            ev = torch.cuda.Event(); ev.record(h2d)
        d2h.wait_event(ev)
        with torch.cuda.stream(d2h):
            for dst, k in ((oh[0], "s"), (oh[1], "ge"), (oh[2], "gA")):
                dst[lo:hi].copy_(bufs[k][lo:hi], non_blocking=True)
    for st in (h2d, comp, d2h): main.wait_stream(st)
for n in (4, 8, 16):
    copies(n); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): copies(n)
    b.record(); torch.cuda.synchronize()
    print("copies only, chunks", n, round(a.elapsed_time(b) / 5, 3), "ms")
