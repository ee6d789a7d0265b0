"""Summarise ncu reports into a small CSV of the metrics the roofline uses.

    python tools/ncu_summary.py out.csv rep1.ncu-rep [rep2.ncu-rep ...]
"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum.per_second",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]

out = []
for rep in sys.argv[2:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if len(rows) < 3:
        continue
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        rec = {"report": rep.split("/")[-1], "kernel": r[idx["Kernel Name"]][:80]}
        for k in KEYS:
            if k in idx:
                rec[f"{k} [{units[idx[k]]}]"] = r[idx[k]]
        out.append(rec)
with open(sys.argv[1], "w", newline="") as f:
    fields = []
    for rec in out:
        fields += [k for k in rec if k not in fields]
    w = csv.DictWriter(f, fieldnames=fields)
    w.writeheader()
    w.writerows(out)
print(f"{len(out)} kernels -> {sys.argv[1]}")
