"""HBM throughput of plain library streams on this box, beside the copy figure
in MEASURED_PEAKS.json: read-only (sum), copy, 2 reads + 1 write (add),
3 reads + 1 write (addcmul), write-only (fill).  Context for the roofline
fractions of K6 (read-dominated) and K7; python tools/membw_probe.py"""
import json

import torch

n = 1 << 29  # 4 GiB of fp64 per array
a = torch.rand(n, dtype=torch.float64, device="cuda")
b = torch.rand(n, dtype=torch.float64, device="cuda")
c = torch.rand(n, dtype=torch.float64, device="cuda")
d = torch.empty_like(a)


def timed(fn, nbytes, reps=10):
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return nbytes / best / 1e6


out = {
    "read_only_sum_GBps": timed(lambda: torch.sum(a), 8 * n),
    "copy_GBps": timed(lambda: d.copy_(a), 16 * n),
    "add_2r1w_GBps": timed(lambda: torch.add(a, b, out=d), 24 * n),
    "addcmul_3r1w_GBps": timed(lambda: torch.addcmul(a, b, c, out=d), 32 * n),
    "fill_write_only_GBps": timed(lambda: d.fill_(1.0), 8 * n),
}
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
