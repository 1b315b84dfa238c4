"""Per-level critical-path durations inside the CAPTURED train step: a globaltimer stamp
(mgb_timestamp) on the main stream before and after every level's forward and backward
launches, captured into the CUDA graph with the side streams running as usual."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_15948_b200 import engine as En  # noqa: E402
from paper_2509_15948_b200._lib import lib  # noqa: E402
from paper_2509_15948_b200.engine import TrainEngine  # noqa: E402
from paper_2509_15948_b200.optimizer import TrainConfig, _EngineCfg, make_optimizer  # noqa: E402
from paper_2509_15948_b200.scheduler import execute_batched  # noqa: E402

dev = torch.device("cuda", 0)
L = int(sys.argv[1]) if len(sys.argv) > 1 else 441_000


def render(graph, tparams, stems):
    return execute_batched(graph, tparams, stems, device=dev)[0].cpu().numpy()


graph, params, stems, target = bench.make_inputs(0, 16, 4, L, render)
cfg = TrainConfig(segment_seconds=L / 30000, steps=1)
eng = TrainEngine(graph, L, _EngineCfg(make_optimizer(params, cfg), cfg), device=dev)
eng.load_params(params)
eng.plan.set_stems(stems)
eng.target.copy_(torch.from_numpy(target))
Ld = lib()
stamps = torch.zeros(256, dtype=torch.int64, device=dev)
labels = []


def stamp(label):
    if len(labels) < 256:
        Ld.mgb_timestamp(En.ptr(stamps, len(labels)), En.stream_ptr())
        labels.append(label)


# wrap the library's per-level entry points as the engine calls them on the main stream
orig = {n: getattr(Ld, n) for n in ("mgb_level_forward_phase", "mgb_level_backward_phase", "mgb_bus_sum")}


class Wrapped:
    def __getattr__(self, n):
        return getattr(Ld, n)

    def mgb_level_forward_phase(self, st, ph, s):
        lv = getattr(st, "_obj", None)
        rc = orig["mgb_level_forward_phase"](st, ph, s)
        if ph == 2:
            stamp(f"fwd {lv.tag.decode()} B={lv.B}" if lv is not None else "fwd")
        return rc

    def mgb_level_backward_phase(self, st, ph, s):
        lv = getattr(st, "_obj", None)
        rc = orig["mgb_level_backward_phase"](st, ph, s)
        if ph == 1:
            stamp(f"bwd {lv.tag.decode()} B={lv.B}" if lv is not None else "bwd")
        return rc


wrapped = Wrapped()
En.lib = lambda: wrapped  # the engine resolves lib() at call time
orig_body = eng._body


def body():
    labels.clear()
    stamp("start")
    orig_body()
    stamp("end")


eng._body = body
for _ in range(5):
    eng.step_async()
torch.cuda.synchronize()
res = {}
for _ in range(5):
    eng.step_async()
    torch.cuda.synchronize()
    t = stamps.cpu().tolist()
    for i in range(1, len(labels)):
        res.setdefault(f"{i:02d} {labels[i]}", []).append((t[i] - t[i - 1]) / 1e3)
print(json.dumps({k: round(sorted(v)[len(v) // 2], 1) for k, v in res.items()}, indent=0))
