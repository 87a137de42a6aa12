"""PCIe floor of the streamed e2e copy pattern (lap2d-4096: 64 bands of
2 MB): b in doubling chunks up to IN bands on one stream, x out in OUT-band
chunks on another, both directions at once, no kernel. Compare with the
measured e2e of sptrsv_solve to see what the kernel dependency costs."""
import json
import sys
import time

import torch

band = 64 * 4096
nt = 64
n = band * nt
h_in = torch.ones(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.ones(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(in_max, out_n, lag_bands):
    """D2H chunk k waits for the H2D of band k + lag (a proxy for the kernel's dependency)."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    evs = [None] * nt
    t, w = 0, 1
    with torch.cuda.stream(s1):
        while t < nt:
            t1 = min(nt, t + w)
            d_a[t * band:t1 * band].copy_(h_in[t * band:t1 * band], non_blocking=True)
            e = torch.cuda.Event()
            e.record(s1)
            for k in range(t, t1):
                evs[k] = e
            t, w = t1, min(2 * w, in_max)
    with torch.cuda.stream(s2):
        for t in range(0, nt, out_n):
            t1 = min(nt, t + out_n)
            s2.wait_event(evs[min(nt - 1, t1 - 1 + lag_bands)])
            h_out[t * band:t1 * band].copy_(d_b[t * band:t1 * band], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


res = {}
for in_max, out_n in ((4, 2), (8, 4), (16, 8), (64, 64)):
    for lag in (0, 4):
        run(in_max, out_n, lag)
        res[f"in{in_max}_out{out_n}_lag{lag}"] = round(min(run(in_max, out_n, lag) for _ in range(5)), 3)
print(json.dumps(res))
