# PARITY attention change check: parity tests (one-pass / forced rerun / max pass), goldens, then the C3 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_refmax.py tests/test_gpu_parity.py tests/test_gpu_batch.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python - <<'P'
import json; d=json.loads(open('gpurun_out/bench_c3.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e']['value'], d.get('phase_ms_per_step'))
print({k: d['exact_mode'][k] for k in ('plans_equal', 'orders_equal', 'hops_equal', 'selections_identical')})
print({k: v for k, v in d['selection_parity'].items() if not isinstance(v, (list, dict))})
P
