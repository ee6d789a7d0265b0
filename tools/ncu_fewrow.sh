#!/bin/bash
# ncu --set full of the few-row kernels (decode attention, skinny GEMM) in the
# deep layers of one C3 plan_keep, plus the launch list of a bench step.
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_decode_kernel|gemm_skinny_kernel" -s 8 -c 6 -o gpurun_out/fewrow_full python tools/one_plan_keep.py > gpurun_out/ncu_fewrow.log 2>&1
python tools/ncu_summary.py gpurun_out/fewrow_summary.csv gpurun_out/fewrow_full.ncu-rep
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-quality > /dev/null 2>&1
tail -3 gpurun_out/ncu_fewrow.log; cat gpurun_out/fewrow_summary.csv | cut -c1-400
