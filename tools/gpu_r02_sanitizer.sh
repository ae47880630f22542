#!/bin/bash
# compute-sanitizer probe: is it usable on this pool? (small smoke workload)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/sanitizer_memcheck.txt 2>&1; echo "memcheck rc=$?"
tail -5 gpurun_out/sanitizer_memcheck.txt
