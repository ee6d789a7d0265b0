#!/bin/bash
# Round-2 closing evidence on one B200: GPU tests, smoke, the C3 PARITY bench and
# the reference arm, the full launch list of one C3 PARITY plan_keep, and ncu
# --set full of the few-row kernels (weight stream, fp64 decode attention).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash tools/launch_list.sh parity c3 3000 > gpurun_out/launch_summary_parity_c3.txt
cap() {  # name regex skip
    timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
        -k regex:"$2" -s $3 -c 1 -o gpurun_out/$1 python tools/one_plan_keep.py parity > gpurun_out/ncu_$1.log 2>&1
}
cap stream_l20 "gemm_f64_stream_kernel" 0
cap decode_l20 "attn_f64_decode_kernel" 0
python tools/ncu_summary.py gpurun_out/r02_ncu_fewrow_parity_full.csv gpurun_out/stream_l20.ncu-rep gpurun_out/decode_l20.ncu-rep
tail -n 4 gpurun_out/pytest_gpu.log; tail -n 4 gpurun_out/smoke.log; head -12 gpurun_out/launch_summary_parity_c3.txt
python - <<'P'
import json
d = json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e']['ttft_ms'], d['clocks'], d['phase_ms_per_step'])
print(d['exact_mode']['selections_identical'], d['selection_parity'])
P
cut -c1-300 gpurun_out/r02_ncu_fewrow_parity_full.csv
