"""Measured int8 tensor-core peak on this B200 (the roofline denominator of the
PARITY Ozaki GEMM): cuBLASLt int8 GEMM through torch._int_mm, 8192^3,
best of 10 (burst) and back to back for 4 s (sustained); and the fp64 DMMA
peak from tools/micro/fp64_peak (compiled binary).  Writes profiles/<out>."""
import json, os, subprocess, sys, time
import torch
out = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_peaks_int8_fp64.json"
n = 8192
a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); torch._int_mm(a, b); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
burst = 2 * n ** 3 / (best / 1e3) / 1e12
t0 = time.time(); k = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    for _ in range(20):
        torch._int_mm(a, b)
    k += 20
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
sust = 2 * n ** 3 * k / (e0.elapsed_time(e1) / 1e3) / 1e12
fp64 = None
exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fp64_peak")
if os.path.exists(exe):
    txt = subprocess.run([exe], capture_output=True, text=True).stdout
    vals = [float(l.split(":")[1].split()[0]) for l in txt.splitlines() if l.startswith("DMMA")]
    fp64 = max(vals) if vals else None
res = {"int8_tops_burst": burst, "int8_tops_sustained": sust, "fp64_dmma_tflops": fp64,
       "how": "torch._int_mm (cuBLASLt int8, int32 out) 8192^3 best of 10 / 4 s back to back; "
              "fp64: tools/micro/fp64_peak.cu mma.sync.m8n8k4.f64 loop, 296 CTAs",
       "gpu": torch.cuda.get_device_name()}
os.makedirs(os.path.dirname(out), exist_ok=True)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
