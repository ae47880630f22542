"""C1 (1e5-event phsp_generate) split: device time of the generation kernel
back to back through the C ABI, against the host cost of one API call."""
import ctypes, os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1711_05683_b200 as hk
from paper_1711_05683_b200 import _lib
M, ms = 5.27966, (3.0969, 0.493677, 0.13957039)
spec, mother = hk.DecaySpec(M, ms), hk.FourVector.at_rest(M)
L = _lib.lib(); st = torch.cuda.current_stream()
for n in (100_000, 1_000_000):
    d, k = _lib.make_decay(spec), _lib.make_key(hk.RngKey(1, 1))
    blk = torch.empty(13, n + 2, dtype=torch.float64, device="cuda")
    cols = _lib.ptr_rows(blk)
    wpart = _lib.empty(2 * _lib.num_weight_slices(n))
    for _ in range(20): L.hk_phsp_generate(d, k, 0, n, cols, _lib.ptr(wpart), st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(500): L.hk_phsp_generate(d, k, 0, n, cols, _lib.ptr(wpart), st.cuda_stream)
    e1.record(); e1.synchronize()
    dev = e0.elapsed_time(e1) / 500 * 1e3
    for _ in range(50): hk.phsp_generate(spec, mother, n, hk.RngKey(1, 1))
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(500): hk.phsp_generate(spec, mother, n, hk.RngKey(1, 1))
    host = (time.perf_counter() - t) / 500 * 1e6
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(500): hk.phsp_generate(spec, mother, n, hk.RngKey(1, 1))
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t) / 500 * 1e6
    print({"n": n, "kernel_us_back_to_back": round(dev, 2), "api_host_us_per_call": round(host, 2),
           "api_us_per_call_synced_at_end": round(tot, 2)})
