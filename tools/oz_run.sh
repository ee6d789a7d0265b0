# Ozaki GEMM: parity tests + timing at the C3 layer-0 shapes + one ncu metrics pass
mkdir -p gpurun_out
python -m pytest tests/test_gpu_gemm_oz.py tests/test_gpu_parity_tc.py -x -q 2>&1 | tail -2
for u in 10 12 14; do KEEP_OZ_MODULI=$u python tools/bench_oz.py 4; done 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_oz_kernel -c 1 python tools/bench_oz.py 1 2>&1 | grep -E "gpu__time|dram__bytes|hit_rate|tensor|issue"
