#!/bin/bash
# ncu --set full of ONE PARITY FLASH DMMA launch (C3 layer 1) + the layer-0
# context pass with fused bins; setup excluded.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"attn_dmma_ws_kernel" -s ${1:-2} -c 1 -o gpurun_out/flash_dmma${1:-2} python tools/one_plan_keep.py parity > gpurun_out/ncu_flash_dmma.log 2>&1
python tools/ncu_summary.py gpurun_out/flash_dmma${1:-2}_summary.csv gpurun_out/flash_dmma${1:-2}.ncu-rep
tail -3 gpurun_out/ncu_flash_dmma.log
