"""Measured write-only and copy HBM bandwidth on this GPU (torch fill_/copy_, CUDA events)."""
import json
import torch

n = 1 << 30   # 8 GiB of fp64
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(3):
    a.fill_(1.0)
    b.copy_(a)
torch.cuda.synchronize()
res = {}
for name, fn, nbytes in (("write_only_fill", lambda: a.fill_(2.0), 8 * n),
                         ("copy_read_write", lambda: b.copy_(a), 16 * n)):
    best = 0.0
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    res[name + "_GBps"] = best
print(json.dumps(res))
