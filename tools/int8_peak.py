"""Measure the dense int8 tensor-core peak on this B200 the same way the
driver measured bf16 (MEASURED_PEAKS.json 'how'): torch._int_mm 8192^3,
best of 10 (burst), then back to back for 4 s (sustained).  Writes
profiles/int8_peak.json."""
import json
import os
import time

import torch

M = N = K = 8192
a = torch.randint(-128, 127, (M, K), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (K, N), dtype=torch.int8, device="cuda")
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); torch._int_mm(a, b); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e) / 1e3)
burst = 2 * M * N * K / best / 1e12
n = 0
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.time()
s.record()
while time.time() - t0 < 4.0:
    for _ in range(20):
        torch._int_mm(a, b)
    n += 20
    torch.cuda.synchronize()
e.record(); torch.cuda.synchronize()
sust = 2 * M * N * K * n / (s.elapsed_time(e) / 1e3) / 1e12
out = {"int8_tops_burst": round(burst, 1), "int8_tops_sustained": round(sust, 1),
       "how": "torch._int_mm int8 8192^3 (2*N^3 ops): best of 10 (burst); back to back for 4 s (sustained)",
       "gpu": torch.cuda.get_device_name()}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/int8_peak.json", "w"), indent=1)
print(json.dumps(out))
