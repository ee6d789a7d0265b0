#!/bin/bash
# ncu --set full of the PARITY DMMA attention kernels of one C3 plan_keep
# (layer 0: stats, ctx, bins; layer 1: flash), setup excluded.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"attn_dmma" \
    -c ${1:-5} -o gpurun_out/dmma_full python tools/one_plan_keep.py parity > gpurun_out/ncu_dmma.log 2>&1
python tools/ncu_summary.py gpurun_out/dmma_summary.csv gpurun_out/dmma_full.ncu-rep
