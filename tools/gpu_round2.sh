#!/bin/bash
# Evidence run: tests, smoke, default bench (+CPU baseline), reference arm, host-memory bench, launch list, ncu full of the top kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --memory host --no-cpu > gpurun_out/bench_host.json 2> gpurun_out/bench_host.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 420 ncu --set full --clock-control none --import-source on -k regex:attn_tc2_kernel -s 96 -c 2 -o gpurun_out/attn_full python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_attn.log 2>&1
timeout 420 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 192 -c 4 -o gpurun_out/gemm_full python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_gemm.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
true
