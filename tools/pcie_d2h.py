"""Raw device->host bandwidth into pinned memory (the e2e ceiling): one
stream vs two copy streams, 1 GiB pieces."""
import time

import torch

n = 1 << 30
src = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(2)]
dst = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
for _ in range(2):
    dst[0].copy_(src[0])
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(8):
    dst[0].copy_(src[0], non_blocking=True)
torch.cuda.synchronize()
one = 8 * n / (time.perf_counter() - t) / 1e9
ss = [torch.cuda.Stream() for _ in range(2)]
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(4):
    for k in range(2):
        with torch.cuda.stream(ss[k]):
            dst[k].copy_(src[k], non_blocking=True)
torch.cuda.synchronize()
two = 8 * n / (time.perf_counter() - t) / 1e9
print({"d2h_GBps_one_stream": round(one, 2), "d2h_GBps_two_streams": round(two, 2)})
