"""Phase boundaries of the CAPTURED train step (timing events recorded on the main
stream inside the CUDA graph): where the critical path spends its time once the
side streams run concurrently."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_15948_b200 import engine as En  # noqa: E402
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
from paper_2509_15948_b200._lib import lib  # noqa: E402

names = ["start", "forward_done", "loss_fwd_done", "loss_bwd_done", "backward_done", "end"]
stamps = torch.zeros(len(names), dtype=torch.int64, device=dev)
plan, lp = eng.plan, eng.lossp
orig_fwd, orig_lf, orig_lb, orig_bwd = plan.forward, lp.forward, lp.backward, plan.backward


def mark(n):  # a globaltimer stamp on the main stream (captured into the graph)
    lib().mgb_timestamp(En.ptr(stamps, names.index(n)), En.stream_ptr())


def fwd(*a, **k):
    mark("start")
    r = orig_fwd(*a, **k)
    mark("forward_done")
    return r


def lf(*a, **k):
    r = orig_lf(*a, **k)
    mark("loss_fwd_done")
    return r


def lb(*a, **k):
    r = orig_lb(*a, **k)
    mark("loss_bwd_done")
    return r


def bwd(*a, **k):
    r = orig_bwd(*a, **k)
    mark("backward_done")
    return r


plan.forward, lp.forward, lp.backward, plan.backward = fwd, lf, lb, bwd
orig_body = eng._body


def body():
    orig_body()
    mark("end")


eng._body = body
for _ in range(5):
    eng.step_async()
torch.cuda.synchronize()
out = {n: [] for n in names[1:]}
for _ in range(10):
    eng.step_async()
    torch.cuda.synchronize()
    t = stamps.cpu().tolist()
    for i in range(1, len(names)):
        out[names[i]].append((t[i] - t[i - 1]) / 1e6)  # ms
print(json.dumps({"L": L, **{k: round(sorted(v)[len(v) // 2], 4) for k, v in out.items()}}))
