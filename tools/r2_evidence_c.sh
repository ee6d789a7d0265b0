#!/bin/bash
# Round-2 kernel evidence after the Ozaki-epilogue / one-pass changes (one B200):
# ncu --set full of the layer-0 and layer-1 QKV Ozaki GEMMs, the layer-0 one-pass
# context pass with fused bins, the layer-0 row split; the full launch list of one
# C3 PARITY plan_keep.  Setup is excluded (--profile-from-start off).
mkdir -p gpurun_out
cap() {  # name regex skip
    timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
        -k regex:"$2" -s $3 -c 1 -o gpurun_out/$1 python tools/one_plan_keep.py parity > gpurun_out/ncu_$1.log 2>&1
    tail -1 gpurun_out/ncu_$1.log
}
cap oz_l0 "gemm_oz_kernel" 0
cap oz_l1 "gemm_oz_kernel" 4
cap ctx_l0 "attn_dmma_ws_kernel" 0
cap split_l0 "oz_split_rows_kernel" 0
python tools/ncu_summary.py gpurun_out/r02_ncu_gemm_oz_full.csv gpurun_out/oz_l0.ncu-rep gpurun_out/oz_l1.ncu-rep
python tools/ncu_summary.py gpurun_out/r02_ncu_ctx_bins_onepass_full.csv gpurun_out/ctx_l0.ncu-rep
python tools/ncu_summary.py gpurun_out/r02_ncu_oz_split_full.csv gpurun_out/split_l0.ncu-rep
bash tools/launch_list.sh parity c3 3000 > gpurun_out/launch_summary_parity_c3.txt
head -24 gpurun_out/launch_summary_parity_c3.txt
cat gpurun_out/r02_ncu_gemm_oz_full.csv gpurun_out/r02_ncu_ctx_bins_onepass_full.csv | cut -c1-400
