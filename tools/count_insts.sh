#!/bin/bash
# dynamic instruction mix of the SN/SS stage kernels at 256^3 (ncu metrics only)
python tools/profile_stage.py --n 256 --variants ${1:-SN} --stages 1 > gpurun_out/pc.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__inst_executed_op_shared_ld.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv -k regex:k_stage_tiled python tools/profile_stage.py --n 256 --variants ${1:-SN} --stages 1 2>/dev/null | grep k_stage | awk -F'","' '{print $13, $15}'
