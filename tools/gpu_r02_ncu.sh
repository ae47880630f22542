#!/bin/bash
# ncu --set full captures (one launch each) of the C3 fused chain, the Philox C2 generator and the FCN
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
P="python tools/prof_kernels.py --n 50000000"
timeout 300 $P > gpurun_out/prof_plain.log 2>&1 || { echo "plain failed"; tail gpurun_out/prof_plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_generate_chain -s 1 -c 1 \
    -o gpurun_out/chain_full -f $P > gpurun_out/ncu_chain.log 2>&1; echo "chain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_generate -s 1 -c 1 \
    -o gpurun_out/gen_philox_full -f python tools/prof_kernels.py --n 50000000 --rng philox > gpurun_out/ncu_philox.log 2>&1; echo "philox rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_nll' -s 2 -c 1 \
    -o gpurun_out/fcn_full -f $P > gpurun_out/ncu_fcn.log 2>&1; echo "fcn rc=$?"
ls -la gpurun_out
