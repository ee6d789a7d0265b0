#!/bin/bash
# ncu --set full of one Ozaki GEMM launch of a C3 PARITY plan_keep (layer 0 QKV, CTA pairs)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"gemm_oz_kernel" -s ${1:-0} -c 1 -o gpurun_out/oz${1:-0} python tools/one_plan_keep.py parity > gpurun_out/ncu_oz.log 2>&1
python tools/ncu_summary.py gpurun_out/oz${1:-0}_summary.csv gpurun_out/oz${1:-0}.ncu-rep
tail -2 gpurun_out/ncu_oz.log
