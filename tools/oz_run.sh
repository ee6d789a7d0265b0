# Ozaki GEMM: parity tests, timing at the C3 layer-0 shapes, split kernels under ncu
mkdir -p gpurun_out
python -m pytest tests/test_gpu_gemm_oz.py tests/test_gpu_parity_tc.py -x -q -p no:cacheprovider 2>&1 | tail -2
python tools/bench_oz.py 4 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:oz_split -c 2 python tools/bench_oz.py 1 2>&1 | grep -E "  unnamed|gpu__time|dram__|fp64|issue"
