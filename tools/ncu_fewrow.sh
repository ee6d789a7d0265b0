#!/bin/bash
# ncu --set full of the few-row kernels (decode attention, skinny GEMM) in the
# deep layers of one C3 plan_keep, plus the launch list of a bench step.
mkdir -p gpurun_out
cat > gpurun_out/one_pk.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import bench, paper_2602_23592_b200 as kb
cfg = bench.CONFIGS["c3"]
lay, q = bench.workload(cfg, 20250807)
ctx = kb.Context(cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, kb.FAST)
ctx.model_init(); ctx.memory_compute_layout(lay)
ctx.plan_keep(lay, q, kb.ratio_schedule(cfg["L"], cfg["r_avg"]), final_hidden=False)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_decode_kernel|gemm_skinny_kernel" -s 8 -c 6 -o gpurun_out/fewrow_full python gpurun_out/one_pk.py > gpurun_out/ncu_fewrow.log 2>&1
python tools/ncu_summary.py gpurun_out/fewrow_summary.csv gpurun_out/fewrow_full.ncu-rep
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-quality > /dev/null 2>&1
tail -3 gpurun_out/ncu_fewrow.log; cat gpurun_out/fewrow_summary.csv | cut -c1-400
