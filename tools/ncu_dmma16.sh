#!/bin/bash
# ncu --set full of the first m16n8k16 flash launch of one C3 PARITY plan_keep (layer 1)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"dmma16" -s 0 -c 1 -o gpurun_out/dmma16 python tools/one_plan_keep.py parity > gpurun_out/ncu_dmma16.log 2>&1
python tools/ncu_summary.py gpurun_out/dmma16_summary.csv gpurun_out/dmma16.ncu-rep
tail -2 gpurun_out/ncu_dmma16.log
