#!/bin/bash
# PARITY correctness after an attention / GEMM change: tensor-core-path
# parity tests, goldens, batch vs oracle, smoke; then per-layer phases at C3.
mkdir -p gpurun_out
free -g > gpurun_out/free.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity_tc.py tests/test_gpu_parity.py tests/test_gpu_batch.py \
    tests/test_gpu_c3_golden.py tests/test_gpu_episode.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pt_parity.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pt_parity.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python tools/layer_phase_probe.py c3 parity > gpurun_out/lpp_parity.txt 2>&1
tail -3 gpurun_out/pt_parity.log; tail -4 gpurun_out/smoke.log; head -3 gpurun_out/lpp_parity.txt | cut -c1-200; grep -E "^19 " gpurun_out/lpp_parity.txt | cut -c1-200; tail -1 gpurun_out/lpp_parity.txt; cat gpurun_out/free.txt
