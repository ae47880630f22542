#!/bin/bash
# A/B: shared back-to-back dot product at the generator's last step (product) vs previous (variants/prev);
# outputs must be bit-identical
cd "$(dirname "$0")/.."
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_jit_gpu.py tests/test_parity_pins_gpu.py 2>&1 | tail -1
python - <<'PY'
import subprocess, json, os
def run(lib):
    env = dict(os.environ); 
    if lib: env["HK_LIB_PATH"] = lib
    code = """
import sys, numpy as np; sys.path.insert(0, '.')
import paper_1711_05683_b200 as hk
spec = hk.DecaySpec(5.27966, (3.0969, 0.493677, 0.13957039))
b = hk.phsp_generate(spec, hk.FourVector(6.0, 0.5, -1.0, 2.0), 300001, hk.RngKey(3, 1))
c = hk.phsp_generate(hk.DecaySpec(1.0, (0.0, 0.2, 0.3)), hk.FourVector.at_rest(1.0), 100000, hk.RngKey(3, 1))
import hashlib
h = hashlib.sha256()
for blk in (b, c):
    for n in blk.schema.names: h.update(np.asarray(blk.column(n)).tobytes())
print(h.hexdigest())
"""
    return subprocess.run(["python", "-c", code], env=env, capture_output=True, text=True).stdout.strip()
print("identical:", run(None) == run("variants/prev/libhepkit_cuda.so"))
PY
for rep in 1 2; do for lib in default prev; do
  if [ "$lib" = default ]; then timeout 120 python tools/bench_gen.py --n 1e8 --reps 20 | sed "s/^{/{\"v\": \"$lib\", /";
  else HK_LIB_PATH=variants/$lib/libhepkit_cuda.so timeout 120 python tools/bench_gen.py --n 1e8 --reps 20 | sed "s/^{/{\"v\": \"$lib\", /"; fi
done; done
