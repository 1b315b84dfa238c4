"""Multi-step training trajectory on the device vs the float64 oracle (diagnostic).

python tools/trajectory.py [--steps 30] [--tracks 4 --subgroups 1 --length 132300] [--oracle]
Prints L_a per step for the CUDA-graph engine (and, with --oracle, the CPU oracle).
fp32 and fp64 trajectories separate slowly (noise-level gradients are sign-normalised
by Adam), so the check is that both descend alike, not bitwise agreement."""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_15948_b200.console import build_console, init_params  # noqa: E402
from paper_2509_15948_b200.engine import TrainEngine  # noqa: E402
from paper_2509_15948_b200.optimizer import TrainConfig, _EngineCfg, make_optimizer  # noqa: E402
from paper_2509_15948_b200.scheduler import execute_batched  # noqa: E402
from workloads import SynthSpec, make_stems_f32, manifest_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--tracks", type=int, default=4)
    ap.add_argument("--subgroups", type=int, default=1)
    ap.add_argument("--length", type=int, default=132_300)
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--eager", action="store_true")
    a = ap.parse_args()
    K, S, L = a.tracks, a.subgroups, a.length
    spec = SynthSpec(tracks=K, subgroups=S, duration_seconds=L / 30000)
    stems = make_stems_f32(spec, 0, L)
    graph, zeros = build_console(manifest_for(spec))
    params = init_params(zeros, 0)
    tp = init_params(zeros, 1)
    y, _ = execute_batched(graph, tp, stems)
    target = y.cpu().numpy()
    cfg = TrainConfig(segment_seconds=L / 30000, steps=1)
    eng = TrainEngine(graph, L, _EngineCfg(make_optimizer(params, cfg), cfg), use_graph=not a.eager)
    eng.load_params(params)
    eng.plan.set_stems(stems)
    eng.target.copy_(torch.from_numpy(target))
    gpu = []
    for _ in range(a.steps):
        eng.step_async()
        gpu.append(eng.read_values())
    ora = []
    if a.oracle:
        from oracle import mixgraph_oracle as O
        p = {t: v.copy() for t, v in params.params.items()}
        raw = params.raw_weights.copy()
        opt = O.AdamW({**p, "w": raw})
        for _ in range(a.steps):
            v, _ = O.train_step(graph, p, raw, stems.astype(np.float64), target.astype(np.float64), 30000,
                                O.LossConfig(), opt)
            ora.append(v)
    for i, v in enumerate(gpu):
        o = f"  oracle L_a={ora[i]['L_a']:.6g}" if ora else ""
        print(f"step {i:3d} gpu L_a={v['L_a']:.6g} L_g={v['L_g']:.4g}{o}", flush=True)


if __name__ == "__main__":
    main()
