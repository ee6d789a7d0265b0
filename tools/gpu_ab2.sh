#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_ab.log 2>&1; echo "pytest(default) rc=$?" >> gpurun_out/pytest_ab.log
KEEP_BINS=scan timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_sharded.py -q -x > gpurun_out/pytest_ab_mma.log 2>&1; echo "pytest(scan-v1) rc=$?" >> gpurun_out/pytest_ab_mma.log
tail -n 3 gpurun_out/pytest_ab.log; tail -n 3 gpurun_out/pytest_ab_mma.log
for mode in scan mma; do
  KEEP_BINS=$mode timeout 300 python bench.py --no-cpu --steps 3 > gpurun_out/bench_$mode.json 2> gpurun_out/bench_$mode.err
done
python - <<'PY'
import json
for f in ['scan','mma']:
    try:
        j=json.loads(open(f'gpurun_out/bench_{f}.json').read().strip().splitlines()[-1])
        print(f, round(j['ttft_ms'],2), j['plan_segments_per_layer'][:3], j['phase_ms_per_step'])
    except Exception as e: print(f, 'fail', e, open(f'gpurun_out/bench_{f}.err').read()[-1500:])
PY
timeout 600 python tools/seed_scan.py 1 12 fast gpurun_out/scan_mma.json > gpurun_out/scan_mma.log 2>&1
python -c "
import json
b=json.load(open('gpurun_out/scan_mma.json'))
print({k:v[0] for k,v in b.items()})
"
