"""MRSTFT timing at config-2 size (eager, CUDA events on the launching stream).

Times the target spectra, the forward and the backward of the device MRSTFT
(three resolutions forked onto their side streams, as inside the train step)
for a scored length of 411,000 samples; prints one JSON line.

usage: python tools/loss_bench.py [--Ls 411000] [--reps 50]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_15948_b200.engine import LossPlan, ptr  # noqa: E402
from paper_2509_15948_b200.losses import LossConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--Ls", type=int, default=411_000)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--sizes", default="512,1024,4096")
    ap.add_argument("--save", default=None, help="write the gradient (npy) here")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    nb = a.batch
    y = torch.from_numpy(rng.standard_normal((nb, 2, a.Ls)).astype(np.float32) * 0.1).to(dev)
    t = torch.from_numpy(rng.standard_normal((nb, 2, a.Ls)).astype(np.float32) * 0.1).to(dev)
    g = torch.zeros_like(y)
    lp = LossPlan(LossConfig(fft_sizes=tuple(int(v) for v in a.sizes.split(","))), a.Ls, dev, batch=nb, sig_stride=2 * a.Ls)
    out = {}

    def timed(name, fn):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[name + "_ms"] = float(np.median(ts))

    timed("target", lambda: lp.target(ptr(t), ptr(t, a.Ls)))
    timed("forward", lambda: lp.forward(ptr(y), ptr(y, a.Ls)))
    # the backward consumes the frame spectra its forward kept: time the pair
    def fwd_bwd():
        lp.forward(ptr(y), ptr(y, a.Ls))
        lp.backward(ptr(y), ptr(y, a.Ls), ptr(g), ptr(g, a.Ls))

    timed("fwd_plus_bwd", fwd_bwd)
    out["backward_ms"] = out["fwd_plus_bwd_ms"] - out["forward_ms"]
    out["loss"] = float(lp.loss.sum())
    out["grad_norm"] = float(g.double().norm())
    out["Ls"], out["batch"] = a.Ls, nb
    if a.save:
        np.save(a.save, g.cpu().numpy())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
