#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
tail -n 3 gpurun_out/pytest_q.log
timeout 300 python bench.py --no-cpu --steps 3 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python -c "
import json; j=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]); print(round(j['ttft_ms'],2), j['plan_segments_per_layer'][:3], j['phase_ms_per_step'])" || tail -5 gpurun_out/bench_q.err
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:attn_tc2 -s 96 -c 4 --csv --log-file gpurun_out/attn_t.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/attn_t.csv')) if len(r)>10 and r[0].isdigit()]
for r in rows: print(r[4][:35], r[-3][:30], r[-1])
"
timeout 600 python tools/seed_scan.py 1 12 fast gpurun_out/scan_t.json > gpurun_out/scan_t.log 2>&1
python -c "
import json; b=json.load(open('gpurun_out/scan_t.json')); print({k:v[0] for k,v in b.items()})"
