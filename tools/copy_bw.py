"""Host<->device copy bandwidth on this box: H2D, D2H, and both concurrently."""
import torch
n = 295 * 2**20 // 4
h1 = torch.empty(n, pin_memory=True); h2 = torch.empty(n, pin_memory=True)
d1 = torch.empty(n, device="cuda"); d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    for s in (s1, s2): torch.cuda.current_stream().wait_stream(s)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    for st in (s1, s2): st.wait_stream(torch.cuda.current_stream())
    ms = t(fn)
    print(name, round(ms, 3), "ms", round(n * 4 * (2 if name == "both" else 1) / ms / 1e6, 1), "GB/s")
