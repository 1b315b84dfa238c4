"""Pinned host -> device copy bandwidth for the e2e step's input size (60 MB), alone."""
import json

import torch

n = 16 * 2 * 441_000 + 2 * 441_000
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record()
    for _ in range(20):
        d.copy_(h, non_blocking=True)
    e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"bytes": 4 * n, "ms_per_copy": ms, "GB_per_s": 4 * n / ms / 1e6}))
