mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 96 -c 4 -o gpurun_out/attn_prefill python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 200 -c 3 -o gpurun_out/gemm_prefill python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_gemm.log 2>&1
