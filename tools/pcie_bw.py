"""Pinned host <-> device copy bandwidth on this box (the bound of bench.py's
e2e number): H2D alone, D2H alone, and both directions at once, 800 MB each
(one C3 grid), CUDA events, best of 5."""
import json

import torch

nb = 800_080_000
n = nb // 8
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"bytes": nb, "h2d_gbs": nb / t1 / 1e6, "d2h_gbs": nb / t2 / 1e6, "h2d_ms": t1, "d2h_ms": t2,
                  "both_ms": t3, "both_gbs_each": nb / t3 / 1e6}))
