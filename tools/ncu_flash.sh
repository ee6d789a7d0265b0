#!/bin/bash
# ncu --set full of layer 0's CTX pass (summary bins) and layer 1's single-pass
# FLASH attention in one C3 plan_keep (the memory refresh before it launches
# 48 block-diagonal FLASH kernels, skipped).
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc2_kernel -s 49 -c 2 -o gpurun_out/flash_full python tools/one_plan_keep.py > gpurun_out/ncu_flash.log 2>&1
python tools/ncu_summary.py gpurun_out/flash_summary.csv gpurun_out/flash_full.ncu-rep
tail -3 gpurun_out/ncu_flash.log; cut -c1-420 gpurun_out/flash_summary.csv
