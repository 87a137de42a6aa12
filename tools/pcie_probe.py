"""Host<->device copy bandwidth on this box: H2D alone, D2H alone, both at once
(separate streams), whole-buffer and in 2 MB chunks. Explains the e2e floor."""
import json
import time

import torch

n = 16 * 1024 * 1024
h_in = torch.ones(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.ones(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
chunk = 64 * 4096


def run(h2d, d2h, chunked):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step = chunk if chunked else n
    for off in range(0, n, step):
        if h2d:
            with torch.cuda.stream(s1):
                d_a[off:off + step].copy_(h_in[off:off + step], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out[off:off + step].copy_(d_b[off:off + step], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


res = {}
for name, a, b in (("h2d", 1, 0), ("d2h", 0, 1), ("both", 1, 1)):
    for ch in (False, True):
        run(a, b, ch)
        t = min(run(a, b, ch) for _ in range(3))
        res[f"{name}{'_chunked' if ch else ''}"] = {"ms": round(t * 1e3, 3),
                                                      "GBps_per_dir": round(8 * n / t / 1e9, 1)}
print(json.dumps(res))
