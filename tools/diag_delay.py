"""d-bank gradient of a short console step, device vs the oracle, largest differences by tap (degenerate delay case)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import mixgraph_oracle as O  # noqa: E402
from paper_2509_15948_b200.console import build_console, init_params  # noqa: E402
from paper_2509_15948_b200.engine import TrainEngine  # noqa: E402
from paper_2509_15948_b200.optimizer import TrainConfig, _EngineCfg, make_optimizer  # noqa: E402
from workloads import SynthSpec, make_stems_f32, manifest_for  # noqa: E402

for L in [int(a) for a in sys.argv[1:]] or [1231, 2000, 2999, 3100, 4999]:
    ws = 1000
    spec = SynthSpec(tracks=3, subgroups=1, duration_seconds=L / 30000)
    stems = make_stems_f32(spec, 9, L)
    graph, zeros = build_console(manifest_for(spec))
    params = init_params(zeros, 0)
    target = (0.3 * np.random.default_rng(L).standard_normal((2, L))).astype(np.float32)
    cfg = TrainConfig(segment_seconds=L / 30000, warmup_seconds=ws / 30000, steps=1)
    eng = TrainEngine(graph, L, _EngineCfg(make_optimizer(params, cfg), cfg), device="cuda", use_graph=False)
    eng.load_params(params)
    eng.plan.set_stems(stems)
    eng.target.copy_(torch.as_tensor(target))
    vals, grads, gw, y = eng.grads_only()
    _, og, _ = O.render_loss_and_grads(graph, {t: v.copy() for t, v in params.params.items()},
                                       params.raw_weights.copy(), stems.astype(np.float64),
                                       target.astype(np.float64), ws, O.LossConfig(),
                                       loss_point=y.astype(np.float64))
    d, od = grads["d"], og["d"]
    err = np.abs(d - od)
    i = np.unravel_index(np.argmax(err), err.shape)
    row, col = i
    ch, off = divmod(col, 440)
    part = "re" if off < 20 else ("im" if off < 40 else f"colour tap {(off - 40) // 20} bin {(off - 40) % 20}")
    print(f"L={L}: max |err| {err.max():.3e} at row {row} ch {ch} {part} (tap {off % 20 if off < 40 else ''}): "
          f"dev {d[i]:.6e} oracle {od[i]:.6e}; |oracle| max {np.abs(od).max():.3e}", flush=True)
    big = np.argsort(-err.ravel())[:6]
    for b in big:
        r, c = divmod(int(b), 880)
        print("   ", r, c, f"{d.ravel()[b]:.4e} {od.ravel()[b]:.4e}")
