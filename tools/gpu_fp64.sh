cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o /tmp/fp64_peak && for i in 1 2 3; do /tmp/fp64_peak; done > gpurun_out/fp64_peak.jsonl
cat gpurun_out/fp64_peak.jsonl
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second
timeout 300 python tools/prof_kernels.py > gpurun_out/prof_plain.log 2>&1 && echo plain ok && \
timeout 900 ncu --metrics $M --clock-control none -k regex:'k_generate|hk_jit_integrate|k_nll' --csv --log-file gpurun_out/dp_counts.csv python tools/prof_kernels.py > gpurun_out/dp_ncu.log 2>&1
echo "ncu rc=$?"
