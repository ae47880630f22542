"""CSV writer throughput on the GPU: device formatting of phase-space rows
(hk_format_csv) and the end-to-end ColumnStore.write_csv stream to a file."""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1711_05683_b200 as hk  # noqa: E402
from paper_1711_05683_b200 import _lib  # noqa: E402

M, ms = 5.27966, (3.0969, 0.493677, 0.13957039)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
blk = hk.phsp_generate(hk.DecaySpec(M, ms), hk.FourVector.at_rest(M), n, hk.RngKey(1, 1))
L = _lib.lib()
C = 13
rows = 1 << 21
scratch = torch.empty(int(L.hk_csv_scratch_bytes(rows, C)), dtype=torch.uint8, device="cuda")
out = torch.empty(rows * C * 25, dtype=torch.uint8, device="cuda")
cols = blk.device_columns()
ln = ctypes.c_int64()
ptrs = _lib.ptr_array([c[:rows] for c in cols])
st = torch.cuda.current_stream()
for _ in range(2):
    L.hk_format_csv(ptrs, C, rows, _lib.ptr(scratch), _lib.ptr(out), out.numel(), ctypes.byref(ln), st.cuda_stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(5):
    L.hk_format_csv(ptrs, C, rows, _lib.ptr(scratch), _lib.ptr(out), out.numel(), ctypes.byref(ln), st.cuda_stream)
e1.record(st)
e1.synchronize()
kt = e0.elapsed_time(e1) / 5 * 1e-3
res = {"rows": rows, "text_bytes": ln.value, "format_s": kt, "format_rows_per_s": rows / kt,
       "format_text_GBps": ln.value / kt / 1e9}
t0 = time.perf_counter()
with open(os.devnull, "wb") as fh:
    blk.write_csv(fh)
dt = time.perf_counter() - t0
res.update({"e2e_rows": n, "e2e_s": dt, "e2e_rows_per_s": n / dt})
host = blk.to_host()
small = 20000
sub = hk.ColumnStore.from_columns(host.schema, [host.column(nm)[:small] for nm in host.schema.names])
t0 = time.perf_counter()
sub.write_csv(open(os.devnull, "w"))
pt = time.perf_counter() - t0
res.update({"python_reference_rows_per_s": small / pt})
print(json.dumps(res))
