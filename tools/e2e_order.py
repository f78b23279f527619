"""Copy-ordering variants of the host pipeline (config 3), same kernels as
stream.lp_tv_fwd_bwd_host.  base: per-chunk e, A, g up / s, ge, gA down.
bulk: e and g of the whole batch as single copies ahead of the A chunks; s
and ge of the whole batch as single copies after the last chunk.
split: chunk 0 as in base, the remaining e/g (and s/ge of all but the last
chunk) as single copies."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_05128_b200 import _native as N, data, lpc, stream
lpc.set_validation("lazy")
B, T, M = 64, 48000, 22
dev = torch.device("cuda", 0)
e, A, g = data.d1_batch_torch(0, B, T, M, device="cuda")
eh, Ah, gh = (x.cpu().pin_memory() for x in (e, A, g))
oh = tuple(torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in (e, e, A))
lib = N.load()
n = 8
bounds = [(B * i // n, B * (i + 1) // n) for i in range(n)]
bufs = stream._buffers(dev, B, T, M, torch.float32, B // n, False)
h2d, comp, d2h = stream._streams(dev, 3)
flag = lpc._flag(dev)

def run(order):
    main = torch.cuda.current_stream(dev)
    for st in (h2d, comp, d2h):
        st.wait_stream(main)
    if order == "bulk":
        with torch.cuda.stream(h2d):
            bufs["e"].copy_(eh, non_blocking=True)
            bufs["g"].copy_(gh, non_blocking=True)
    for i, (lo, hi) in enumerate(bounds):
        nb = hi - lo
        with torch.cuda.stream(h2d):
            if order == "base" or (order == "split" and i == 0):
                bufs["e"][lo:hi].copy_(eh[lo:hi], non_blocking=True)
            if order == "split" and i == 0:
                bufs["g"][lo:hi].copy_(gh[lo:hi], non_blocking=True)
            bufs["A"][lo:hi].copy_(Ah[lo:hi], non_blocking=True)
            if order == "base":
                bufs["g"][lo:hi].copy_(gh[lo:hi], non_blocking=True)
            if order == "split" and i == 0:
                bufs["e"][hi:].copy_(eh[hi:], non_blocking=True)
                bufs["g"][hi:].copy_(gh[hi:], non_blocking=True)
            ready = torch.cuda.Event(); ready.record(h2d)
        comp.wait_event(ready)
        carry = bufs["carry"][:lib.tvlp_carry_elems(nb, T, M)]
        cs = ctypes.c_void_p(comp.cuda_stream)
        ed, Ad, gd = bufs["e"][lo:hi], bufs["A"][lo:hi], bufs["g"][lo:hi]
        sd, ged, gAd = bufs["s"][lo:hi], bufs["ge"][lo:hi], bufs["gA"][lo:hi]
        N.check(lib.tvlp_lp_forward_tv(0, N.ptr(ed), N.ptr(Ad), None, N.ptr(sd), nb, T, M,
                                       N.ptr(carry), lpc._carry_code(), N.ptr(bufs["ws"]),
                                       bufs["nws"], N.ptr(flag), cs))
        N.check(lib.tvlp_lp_backward_tv(0, N.ptr(gd), N.ptr(Ad), N.ptr(sd), None, N.ptr(ged),
                                        N.ptr(gAd), nb, T, M, N.ptr(carry), lpc._carry_code(),
                                        N.ptr(bufs["ws"]), bufs["nws"], cs))
        done = torch.cuda.Event(); done.record(comp)
        d2h.wait_event(done)
        with torch.cuda.stream(d2h):
            if order == "base" or (order == "split" and i == n - 1):
                oh[0][lo:hi].copy_(sd, non_blocking=True)
                oh[1][lo:hi].copy_(ged, non_blocking=True)
            oh[2][lo:hi].copy_(gAd, non_blocking=True)
            if order == "split" and i == n - 2:
                oh[0][:hi].copy_(bufs["s"][:hi], non_blocking=True)
                oh[1][:hi].copy_(bufs["ge"][:hi], non_blocking=True)
            if order == "bulk" and i == n - 1:
                oh[0].copy_(bufs["s"], non_blocking=True)
                oh[1].copy_(bufs["ge"], non_blocking=True)
    for st in (h2d, comp, d2h):
        main.wait_stream(st)

ref = stream.lp_tv_fwd_bwd_host(eh, Ah, gh)
torch.cuda.synchronize()  # (lazy validation: the host results land asynchronously)
ref = tuple(x.clone() for x in ref)
for rep in range(2):
    for order in ("base", "bulk", "split"):
        for _ in range(2):
            run(order)
        torch.cuda.synchronize()
        ok = all(torch.equal(a, b) for a, b in zip(ref, oh))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            run(order)
        b.record(); torch.cuda.synchronize()
        print(order, round(a.elapsed_time(b) / 5, 3), "ms", "identical" if ok else "MISMATCH", flush=True)
