mkdir -p gpurun_out
for u in 8 10 12 14; do KEEP_OZ_MODULI=$u python tools/bench_oz.py 2; done > gpurun_out/oz_sweep.log 2>&1
KEEP_OZ_PAIR=0 python tools/bench_oz.py 2 >> gpurun_out/oz_sweep.log 2>&1
for u in 8 14; do KEEP_OZ_MODULI=$u timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_oz_kernel -c 2 python tools/bench_oz.py 1 ; done > gpurun_out/oz_sweep_ncu.log 2>&1
cat gpurun_out/oz_sweep.log; grep -E "U=|gpu__time|dram__bytes|hit_rate|tensor" gpurun_out/oz_sweep_ncu.log
