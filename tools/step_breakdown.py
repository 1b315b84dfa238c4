"""Critical-path breakdown of one train step (eager, one stream, CUDA events):
FIR syntheses, render forward, target spectra, MRSTFT forward, MRSTFT backward,
render backward, optimiser.  Also the captured step (all streams) for reference."""

import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2509_15948_b200._lib import check, lib  # noqa: E402
from paper_2509_15948_b200.engine import TrainEngine, ptr, stream_ptr  # noqa: E402
from paper_2509_15948_b200.optimizer import TrainConfig, _EngineCfg, make_optimizer  # noqa: E402
from paper_2509_15948_b200.scheduler import execute_batched  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tracks", type=int, default=16)
    ap.add_argument("--subgroups", type=int, default=4)
    ap.add_argument("--length", type=int, default=441_000)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)

    def render(graph, tparams, stems):
        return execute_batched(graph, tparams, stems, device=dev)[0].cpu().numpy()

    graph, params, stems, target = bench.make_inputs(0, a.tracks, a.subgroups, a.length, render)
    cfg = TrainConfig(segment_seconds=a.length / 30000, steps=1)
    eng = TrainEngine(graph, a.length, _EngineCfg(make_optimizer(params, cfg), cfg), device=dev, use_graph=True)
    eng.load_params(params)
    eng.plan.set_stems(stems)
    eng.target.copy_(torch.from_numpy(target))
    L, ws = eng.L, eng.ws
    plan, lp = eng.plan, eng.lossp
    Ld = lib()
    lay = eng.layout

    phases = {
        "fir_synthesis": lambda: plan.prepare(),
        "render_fwd": lambda: plan.forward(use_mask=False, prepared=True, norms="inline"),
        "target_spectra": lambda: lp.target(ptr(eng.target, ws), ptr(eng.target, L + ws)),
        "loss_fwd": lambda: lp.forward(ptr(plan.y, ws), ptr(plan.y, L + ws)),
        "loss_bwd": lambda: lp.backward(ptr(plan.y, ws), ptr(plan.y, L + ws), ptr(plan.dY, ws),
                                        ptr(plan.dY, L + ws)),
        "render_bwd": lambda: plan.backward(),
        "optimizer": lambda: check(Ld.mgb_adamw_step(ptr(eng.params), ptr(eng.grads), ptr(eng.m), ptr(eng.v), lay.n,
                                                     lay.off["d"], eng.d_rows, lay.w_off, lay.P, ptr(plan.gw), None,
                                                     ptr(eng.scalars), ptr(eng.vals), None, stream_ptr()), "adamw"),
    }
    eng._set_scalars(0.0)
    out = {}
    snap = [eng.params.clone(), eng.m.clone(), eng.v.clone()]
    for _ in range(2):
        for f in phases.values():
            f()
    torch.cuda.synchronize()
    for name, f in phases.items():
        best = 1e9
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name] = round(best, 4)
    eng.params.copy_(snap[0]); eng.m.copy_(snap[1]); eng.v.copy_(snap[2])  # noqa: E702
    out["sum_eager_ms"] = round(sum(out.values()), 4)
    for _ in range(5):
        eng.step_async()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        eng.step_async()
    e1.record()
    torch.cuda.synchronize()
    out["captured_step_ms"] = round(e0.elapsed_time(e1) / 20, 4)
    print(json.dumps({"config": [a.tracks, a.subgroups, a.length], **out}))


if __name__ == "__main__":
    main()
