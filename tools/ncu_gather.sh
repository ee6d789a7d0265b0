#!/bin/bash
# ncu --set full of the gather/scatter kernels of one C3 plan_keep: merged-KV
# assembly from cached blocks (K4) and the active-row compaction (K2).
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"copy_cached_kernel|gather_rows_kernel" -c 4 -o gpurun_out/gather_full python tools/one_plan_keep.py > gpurun_out/ncu_gather.log 2>&1
python tools/ncu_summary.py gpurun_out/gather_summary.csv gpurun_out/gather_full.ncu-rep
tail -2 gpurun_out/ncu_gather.log; cut -c1-330 gpurun_out/gather_summary.csv
