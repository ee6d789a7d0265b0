#!/bin/bash
# Per-launch device times of one plan_keep (setup excluded):
#   bash tools/launch_list.sh [fast|parity] [c3|c2|...] [max launches]
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c ${3:-400} --csv \
    --log-file gpurun_out/launches_${1:-parity}_${2:-c3}.csv python tools/one_plan_keep.py ${1:-parity} ${2:-c3} \
    > gpurun_out/launch_list.log 2>&1
python - "$1" "$2" <<'PY'
import csv, sys, collections
rows = list(csv.reader(open(f"gpurun_out/launches_{sys.argv[1] or 'parity'}_{sys.argv[2] or 'c3'}.csv")))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= vi: continue
    k = r[ki].split("(")[0][:70]; v = float(r[vi].replace(",", "")) / 1e6
    a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += v
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{ms:10.3f} ms {n:5d}  {k}")
PY
