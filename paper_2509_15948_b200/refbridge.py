"""Device level ops behind the reference's own foreign-op hook.

The reference substitutes hand-written forward/backward pairs into its tape
through ``engine.custom_gradient(forward_fn, backward_fn)``
(mg/engine.py:673-704; its multitap delay uses it, mg/processors.py:303).
``foreign_kernels(E)`` builds, for a caller-supplied reference ``engine``
module ``E``, a table with the shape of ``processors.KERNELS``
(mg/processors.py:321-329): ``table[tag](u, p) -> (ybar, reg | None)`` where
the work runs in this library's CUDA level kernels and the reference's tape
records one op per call whose adjoint is the level's hand-written backward.

A reference user swaps it in with
``mixgraph.processors.KERNELS.update(foreign_kernels(mixgraph.engine))``; the
reference's ``execute_batched`` / ``train_step`` / ``eval_loss`` then render
every level on the GPU while everything else (graph, schedule, loss, tape,
optimizer) stays the reference's.  This module never imports the reference:
the engine module is passed in.

Layout of the recorded op: its output is the flattened wet signal followed by
the level's gain-staging term (``B*2*L + 1`` float64 values); ``ybar`` and
``reg`` are a reshape and an index of it on the reference's tape.
"""

from __future__ import annotations

import numpy as np
import torch

from .engine import F32, F64, ensure_device
from .processors import KERNELS

TAGS = "gsercnd"


def _kernel(E, tag, device):
    dev = ensure_device(device)

    def to_dev(u, p, grad):
        ut = torch.as_tensor(np.asarray(u), dtype=F32).to(dev).contiguous()
        pt = torch.as_tensor(np.asarray(p, dtype=np.float64), dtype=F64).to(dev).contiguous()
        return ut.requires_grad_(grad), pt.requires_grad_(grad)

    def forward_fn(u, p):
        ut, pt = to_dev(u, p, False)
        with torch.no_grad():
            ybar, reg = KERNELS[tag](ut, pt)
        out = np.empty(ut.numel() + 1, dtype=np.float64)
        out[:-1] = ybar.double().reshape(-1).cpu().numpy()
        out[-1] = float(reg) if reg is not None else 0.0
        return out

    def backward_fn(g, u, p):
        # the level's adjoint needs its forward workspace: re-run the forward on the
        # device, then the hand-written backward (mgb_level_backward)
        ut, pt = to_dev(u, p, True)
        ybar, reg = KERNELS[tag](ut, pt)
        g = np.asarray(g, dtype=np.float64)
        outs = [ybar]
        grads = [torch.from_numpy(np.ascontiguousarray(g[:-1].reshape(ybar.shape))).to(dev, F32)]
        if reg is not None:
            outs.append(reg)
            grads.append(torch.tensor(g[-1], dtype=F64, device=dev))
        torch.autograd.backward(outs, grads)
        return (ut.grad.double().cpu().numpy().reshape(np.shape(u)),
                pt.grad.cpu().numpy().reshape(np.shape(p)))

    op = E.custom_gradient(forward_fn, backward_fn)

    def run(u, p):
        shape = np.shape(E.value_of(u))
        out = op(u, p)
        ybar = E.reshape(E.getitem(out, slice(0, -1)), shape)
        reg = E.getitem(out, -1) if tag in "erd" else None
        return ybar, reg

    run.__name__ = KERNELS[tag].__name__
    return run


def foreign_kernels(E, device="cuda"):
    """{tag: kernel} for the reference's tape; E is the reference's engine module."""
    return {t: _kernel(E, t, device) for t in TAGS}


__all__ = ["foreign_kernels", "TAGS"]
