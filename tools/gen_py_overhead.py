"""Per-call host cost of phsp_generate pieces at C1 size (1e5 events), us."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1711_05683_b200 as hk  # noqa: E402
from paper_1711_05683_b200 import _lib, phasespace as P  # noqa: E402

M, ms = 5.27966, (3.0969, 0.493677, 0.13957039)
spec, mother = hk.DecaySpec(M, ms), hk.FourVector.at_rest(M)
key = hk.RngKey(1, 1)
n = 100_000
for _ in range(50):
    hk.phsp_generate(spec, mother, n, key)
torch.cuda.synchronize()
N = 2000


def t(fn, n=N):
    t0 = time.perf_counter()
    for i in range(n):
        fn()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t0) / n * 1e6, 2)


cols = P._columns(13, n)
out = {
    "phsp_generate": t(lambda: hk.phsp_generate(spec, mother, n, key)),
    "check_mother": t(lambda: P._check_mother(spec, mother)),
    "make_decay": t(lambda: _lib.make_decay(spec, mother, M)),
    "make_key": t(lambda: _lib.make_key(key, 0)),
    "columns13": t(lambda: P._columns(13, n)),
    "schema": t(lambda: P.phsp_schema(3)),
    "store": t(lambda: hk.ColumnStore._from_device(P.phsp_schema(3), cols)),
    "wpart_empty": t(lambda: _lib.empty(2 * _lib.num_weight_slices(n))),
    "ptr_array": t(lambda: _lib.ptr_array(cols)),
    "stream_ptr": t(lambda: _lib.stream_ptr()),
}
print(out)
