mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v6.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 420 ncu --set full --clock-control none --import-source on -k regex:attn_tc2_kernel -s 96 -c 4 -o gpurun_out/attn6 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_attn2.log 2>&1
