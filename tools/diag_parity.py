"""Where does a step's gradient error come from?  Device vs float64 oracle at a
given (K, S, L): the mix y, the loss gradient dL/dy, and every bank, with the
oracle's loss gradient evaluated both at its own y and at the device's y."""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

from conftest import normrel  # noqa: E402
from oracle import mixgraph_oracle as O  # noqa: E402
from paper_2509_15948_b200.console import build_console, init_params  # noqa: E402
from paper_2509_15948_b200.engine import TrainEngine  # noqa: E402
from paper_2509_15948_b200.optimizer import TrainConfig, _EngineCfg, make_optimizer  # noqa: E402
from paper_2509_15948_b200.scheduler import execute_batched  # noqa: E402
from workloads import SynthSpec, make_stems_f32, manifest_for  # noqa: E402


def run(K, S, L, seed):
    spec = SynthSpec(tracks=K, subgroups=S, duration_seconds=L / 30000)
    stems = make_stems_f32(spec, seed, L)
    graph, zeros = build_console(manifest_for(spec))
    params = init_params(zeros, 0)
    target = execute_batched(graph, init_params(zeros, 1), stems)[0].cpu().numpy()
    cfg = TrainConfig(segment_seconds=L / 30000, steps=1)
    eng = TrainEngine(graph, L, _EngineCfg(make_optimizer(params, cfg), cfg), device="cuda", use_graph=False)
    eng.load_params(params)
    eng.plan.set_stems(stems)
    eng.target.copy_(torch.as_tensor(target))
    vals, grads, gw, y = eng.grads_only()
    dY = eng.plan.dY.cpu().numpy().astype(np.float64)
    ov, og, oy = O.render_loss_and_grads(graph, {t: v.copy() for t, v in params.params.items()},
                                         params.raw_weights.copy(), stems.astype(np.float64),
                                         target.astype(np.float64), 30000, O.LossConfig())
    tg = target.astype(np.float64)
    res = {}
    for name, yy in (("oracle_y", oy), ("device_y", y.astype(np.float64))):
        yt = torch.tensor(yy, requires_grad=True)
        O.mrstft(yt[:, 30000:], tg[:, 30000:], O.LossConfig()).backward()
        res[name] = yt.grad.numpy()
    out = {"L_a_rel": abs(vals["L_a"] - ov["L_a"]) / ov["L_a"], "y": normrel(y, oy),
           "dY_vs_oracle": normrel(dY, res["oracle_y"]), "dY_vs_oracle_at_device_y": normrel(dY, res["device_y"]),
           "oracle_dY_shift_from_y_error": normrel(res["device_y"], res["oracle_y"])}
    for t in "gsecnrd":
        out[t] = normrel(grads[t], og[t], floor=1e-6)
    print(f"K={K} S={S} L={L} seed={seed}: " + " ".join(f"{k}={v:.2e}" for k, v in out.items()), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="*", default=["16,4,441000,0", "4,1,441000,0", "16,4,132300,0", "4,1,132300,3",
                                                  "16,4,441000,3"])
    for c in ap.parse_args().cases:
        run(*[int(x) for x in c.split(",")])
