mkdir -p gpurun_out
for v in "" "KEEP_DEBUG_ATTN=1" "KEEP_DEBUG_ATTN=2" "KEEP_DEBUG_NO_BINS=1"; do
env $v timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:attn_tc2 -s 96 -c 2 --csv --log-file gpurun_out/dbg.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
echo "== $v"
python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/dbg.csv')) if len(r)>10 and r[0].isdigit()]
for r in rows: print(r[4][:35], r[-3][:30], r[-1])
"
done
