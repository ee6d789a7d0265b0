mkdir -p gpurun_out
timeout 600 python tools/seed_scan.py 1 40 fast gpurun_out/scan_v2.json > gpurun_out/scan_v2.log 2>&1
KEEP_ATTN_V1=1 timeout 600 python tools/seed_scan.py 1 40 fast gpurun_out/scan_v1.json > gpurun_out/scan_v1.log 2>&1
timeout 900 python tools/seed_scan.py 1 6 parity gpurun_out/scan_par.json > gpurun_out/scan_par.log 2>&1
