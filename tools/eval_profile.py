"""Eager pruning-trial evaluations of the config-2 console (for ncu): masked forward + MRSTFT."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2509_15948_b200.engine import EvalEngine  # noqa: E402
from paper_2509_15948_b200.optimizer import TrainConfig  # noqa: E402
from paper_2509_15948_b200.scheduler import execute_batched  # noqa: E402

dev = torch.device("cuda", 0)
K, S, L = bench.K_TRACKS, bench.S_GROUPS, bench.L_SAMPLES


def render(graph, tparams, stems):
    y, _ = execute_batched(graph, tparams, stems, device=dev)
    return y.cpu().numpy()


graph, params, stems, target = bench.make_inputs(0, K, S, L, render)
cfg = TrainConfig(segment_seconds=L / 30000, steps=1)
ev = EvalEngine(graph, [(stems, target)], bench.WARMUP, cfg.loss, device=dev, params=params,
                use_graph=False)
mask = np.ones(ev.layout.P)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    ev.run_async(mask)
torch.cuda.synchronize()
from paper_2509_15948_b200 import _lib  # noqa: E402
print("clusters", _lib.lib().mgb_launch_count())
