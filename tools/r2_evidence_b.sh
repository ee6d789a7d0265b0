#!/bin/bash
# Round-2 evidence: full GPU suite, smoke, default bench (PARITY headline),
# reference arm, PARITY with host-resident memory (K10 loader), launch list.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --memory host --no-cpu --no-compare --updates 0 > gpurun_out/bench_host.json 2> gpurun_out/bench_host.err
bash tools/launch_list.sh parity c3 700 > gpurun_out/ll_parity.txt 2>&1
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 4 gpurun_out/smoke.log
python - <<'PY'
import json
for f in ("bench", "bench_host"):
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, d.get("value"), d.get("ttft_ms"), (d.get("e2e") or {}).get("ttft_ms"), d.get("phase_ms_per_step"), (d.get("loader") or {}))
    except Exception as e:
        print(f, "ERR", e)
PY
head -12 gpurun_out/ll_parity.txt
