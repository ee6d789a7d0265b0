mkdir -p gpurun_out
KEEP_DEBUG_NO_BINS=1 timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:attn_tc2 -s 96 -c 4 --csv --log-file gpurun_out/nobins.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
cat gpurun_out/nobins.csv | grep -v "^==" | cut -d, -f5,13-15 | head -20
