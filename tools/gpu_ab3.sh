#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
tail -n 3 gpurun_out/pytest_q.log
for v in "" "KEEP_CACHED_KERNEL=1"; do
env $v timeout 300 python bench.py --no-cpu --steps 3 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
echo "== $v"; python -c "
import json; j=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]); print(round(j['ttft_ms'],2), j['plan_segments_per_layer'][:3], j['phase_ms_per_step'], j['e2e']['ttft_ms'])" || tail -5 gpurun_out/bench_q.err
done
