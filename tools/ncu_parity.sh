#!/bin/bash
# ncu --set full of the PARITY kernels of layers 0-1 in one C3 plan_keep:
# Ozaki int8 GEMMs (gemm_oz_kernel) and DMMA attention (attn_dmma*).  The
# canonical-KV refresh before it launches 48 x 5 of them (skipped).
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_oz_kernel|attn_dmma" -s 240 -c 9 \
    -o gpurun_out/parity_full python tools/one_plan_keep.py parity > gpurun_out/ncu_parity.log 2>&1
python tools/ncu_summary.py gpurun_out/parity_summary.csv gpurun_out/parity_full.ncu-rep
tail -2 gpurun_out/ncu_parity.log; cut -c1-400 gpurun_out/parity_summary.csv
