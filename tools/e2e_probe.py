"""Where does the e2e step lose time against the device step?  (config 2, 1 GPU)

(a) device loop: step_async x N on resident inputs (CUDA events)
(b) train_segments x N with pinned host segments (wall clock)
(c) the same with the segments already on the device (no H2D)
(d) H2D copy of one segment alone (CUDA events)
(e) CPU time of the train_segments loop body with the GPU work stubbed is not separable;
    instead report the host-side enqueue time of (b) (time until the loop returns minus sync)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2509_15948_b200.engine import TrainEngine  # noqa: E402
from paper_2509_15948_b200.optimizer import TrainConfig, _EngineCfg, make_optimizer, train_segments  # noqa: E402
from paper_2509_15948_b200.scheduler import execute_batched  # noqa: E402

N = 48
dev = torch.device("cuda", 0)
K, S, L = bench.K_TRACKS, bench.S_GROUPS, bench.L_SAMPLES


def render(graph, tparams, stems):
    y, _ = execute_batched(graph, tparams, stems, device=dev)
    return y.cpu().numpy()


graph, params, stems, target = bench.make_inputs(0, K, S, L, render)
cfg = TrainConfig(segment_seconds=L / 30000, steps=1)
opt = make_optimizer(params, cfg, device=dev)
eng = TrainEngine(graph, L, _EngineCfg(opt, cfg), device=dev)
eng.load_params(params)
eng.plan.set_stems(stems)
eng.target.copy_(torch.from_numpy(target))
for _ in range(5):
    eng.step_async()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(N):
    eng.step_async()
b.record()
torch.cuda.synchronize()
print(f"(a) device step      {a.elapsed_time(b) / N:.3f} ms")

st_pin = torch.from_numpy(stems).pin_memory()
tg_pin = torch.from_numpy(target).pin_memory()
opt2 = make_optimizer(params, cfg, device=dev)
p2 = params.copy()
train_segments(graph, p2, [(st_pin, tg_pin)] * 4, cfg, opt2)
torch.cuda.synchronize()
t0 = time.perf_counter()
train_segments(graph, p2, [(st_pin, tg_pin)] * N, cfg, opt2)
print(f"(b) train_segments   {(time.perf_counter() - t0) * 1e3 / N:.3f} ms/step (pinned host)")
st_d, tg_d = st_pin.to(dev), tg_pin.to(dev)
torch.cuda.synchronize()
t0 = time.perf_counter()
train_segments(graph, p2, [(st_d, tg_d)] * N, cfg, opt2)
print(f"(c) train_segments   {(time.perf_counter() - t0) * 1e3 / N:.3f} ms/step (device-resident segments)")
buf = torch.empty_like(st_d)
a.record()
for _ in range(10):
    buf.copy_(st_pin, non_blocking=True)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
print(f"(d) H2D stems        {ms:.3f} ms  ({st_pin.numel() * 4 / ms / 1e6:.1f} GB/s)")
s2 = torch.cuda.Stream()
with torch.cuda.stream(s2):
    a.record(s2)
    for _ in range(10):
        buf.copy_(st_pin, non_blocking=True)
    b.record(s2)
for _ in range(20):
    eng.step_async()
torch.cuda.synchronize()
print(f"(e) H2D stems under load {a.elapsed_time(b) / 10:.3f} ms")
t0 = time.perf_counter()
for _ in range(N):
    eng.step_async()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"(f) enqueue-only host time per step_async {(t1 - t0) * 1e3 / N:.3f} ms")
