#!/bin/bash
# quick check: FAST tests, then A/B bench (v1 vs v2 attention)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
tail -3 gpurun_out/pytest_quick.log
timeout 300 python bench.py --no-cpu --steps 3 > gpurun_out/bench_v2.json 2> gpurun_out/bench_v2.err
KEEP_ATTN_V1=1 timeout 300 python bench.py --no-cpu --steps 3 > gpurun_out/bench_v1.json 2> gpurun_out/bench_v1.err
python - <<'PY'
import json
for f in ['v1','v2']:
    try:
        j=json.loads(open(f'gpurun_out/bench_{f}.json').read().strip().splitlines()[-1])
        print(f, j['ttft_ms'], j['phase_ms_per_step'])
    except Exception as e: print(f, 'fail', e, open(f'gpurun_out/bench_{f}.err').read()[-2000:])
PY
