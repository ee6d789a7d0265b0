#!/bin/bash
# ncu --set full of four tcgen05 GEMM launches of layer 0 in one C3 plan_keep
# (the memory refresh before it launches 4 x 48 GEMMs, skipped).
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 192 -c 4 -o gpurun_out/gemm_full python tools/one_plan_keep.py > gpurun_out/ncu_gemm.log 2>&1
python tools/ncu_summary.py gpurun_out/gemm_summary.csv gpurun_out/gemm_full.ncu-rep
tail -2 gpurun_out/ncu_gemm.log; cut -c1-300 gpurun_out/gemm_summary.csv
