"""Pinned host -> device copy rate of this box (the ceiling of bench.py's e2e leg)."""
import json

import torch

out = {}
for mib in (16, 64, 800):
    n = mib << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    out[f"{mib}MiB"] = round(5 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
print(json.dumps({"pinned_h2d_gbs": out}))
