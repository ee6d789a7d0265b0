#!/bin/bash
# Round evidence: GPU tests, smoke, default bench (+CPU baseline), reference
# arm, host-memory / updates / batched benches, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 180 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --memory host --no-cpu --no-quality > gpurun_out/bench_host.json 2> gpurun_out/bench_host.err
timeout 600 python bench.py --updates 0.35 --no-cpu --no-quality > gpurun_out/bench_upd.json 2> gpurun_out/bench_upd.err
timeout 600 python bench.py --batch 16 --steps 2 --warmup 1 > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err
timeout 600 python bench.py --batch 16 --memory host --steps 2 --warmup 1 > gpurun_out/bench_batch_host.json 2> gpurun_out/bench_batch_host.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-quality > /dev/null 2>&1
tail -n 2 gpurun_out/pytest_gpu.log; tail -n 3 gpurun_out/smoke.log
for f in bench bench_ref bench_host bench_upd bench_batch bench_batch_host; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, d.get("value"), d.get("ttft_ms"), (d.get("batch") or {}).get("batch_ttft_ms"), (d.get("e2e") or {}).get("ttft_ms"))
except Exception as e:
    print(f, "ERR", e)
PY
done
true
