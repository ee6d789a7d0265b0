mkdir -p gpurun_out
for v in "" "KEEP_ATTN_SMALL_N=32"; do
env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sn.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
echo "== $v"
python - <<'PY'
import csv,collections
rows=[r for r in csv.reader(open('gpurun_out/sn.csv')) if len(r)>10 and r[0].isdigit()]
names=[r[4] for r in rows]
idx=[i for i,n in enumerate(names) if n.startswith('embed_kernel')]
seq=rows[idx[-1]-1:]
agg=collections.defaultdict(float)
for r in seq[-200:]:
    n=r[4].split('(')[0].replace('void ','').replace('unnamed>::','')
    agg[n]+=float(r[-1])/1e3
for k,v in sorted(agg.items(),key=lambda x:-x[1])[:10]: print(f"  {k[:40]:40s} {v:9.1f} us (last 200 launches)")
PY
env $v timeout 300 python bench.py --no-cpu --steps 3 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python -c "
import json; j=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]); print(round(j['ttft_ms'],2), j['plan_segments_per_layer'][:3], j['plan_segments_per_layer'][19:22], j['phase_ms_per_step'])" || tail -5 gpurun_out/bench_q.err
done
