set -x
timeout 300 python tools/layer_phase_probe.py c3 parity > gpurun_out/layer_parity.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"attn_dmma" -c 5 \
    -o gpurun_out/dmma_full python tools/one_plan_keep.py parity > gpurun_out/ncu_dmma.log 2>&1
python tools/ncu_summary.py gpurun_out/dmma_summary.csv gpurun_out/dmma_full.ncu-rep
