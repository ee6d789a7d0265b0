#!/bin/bash
# BASELINE configs[4] at its stated size: Qwen2.5-32B dims, 128K-token memory
# bank in pinned host DRAM (deepest layers in HBM under a budget), a batch of
# 16 planning queries (FAST numerics: the fp32 PARITY weights alone are 105 GB).
mkdir -p gpurun_out
free -g | head -2
for a in ${C5_VARIANTS:-"--sub-batch 2 --hbm-budget-gb 50"}; do
  tag=$(echo $a | tr -d ' -')
  timeout 1800 python bench.py --config c5 --numerics fast --batch 16 --memory host $a --steps 1 --warmup 1 \
      --no-sequential > gpurun_out/bench_c5_$tag.json 2> gpurun_out/bench_c5_$tag.err
  echo "== $a rc=$?"; grep "#" gpurun_out/bench_c5_$tag.err; grep -iE "error|Killed" gpurun_out/bench_c5_$tag.err | tail -2
  python -c "
import json; d=json.loads(open('gpurun_out/bench_c5_$tag.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['batch'], d['e2e']['ttft_ms'], d['phase_ms_per_step'])" 2>&1 | tail -1
  [ -n "$C5_FIRST_ONLY" ] && [ -s gpurun_out/bench_c5_$tag.json ] && break
done
