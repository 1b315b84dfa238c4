"""``execute_batched`` on the device (mg/scheduler.py:225-263).

Planning (schedules, index plans) is host Python in ``schedule.py``; the
render itself runs as one ``RenderPlan`` of level kernels.  Returns device
tensors: ``y`` (2, L) float32 and the gain-staging sum ``reg`` (float64).
"""

from __future__ import annotations

import numpy as np
import torch

from .engine import F32, F64, ParamLayout, RenderPlan, ensure_device
from .graph import topological_order, validate
from .schedule import (CONSOLE_SEQUENCE, GREEDY_TIE_ORDER, LengthMismatch, NotAConsole, Schedule,  # noqa: F401
                       SchedulerError, StepPlan, console_chains, plan_indices, schedule_console,
                       schedule_for, schedule_greedy)


def _check_sources(graph, sources):
    """mg/scheduler.py:207-215: the source count, then equal lengths (same errors)."""
    k = len(graph.nodes_of_type("i"))
    n = sources.shape[0] if (torch.is_tensor(sources) or isinstance(sources, np.ndarray)) else len(sources)
    if n != k:
        raise LengthMismatch(f"graph has {k} inputs, got {n} sources")
    if torch.is_tensor(sources):
        return sources
    if isinstance(sources, (list, tuple)):
        lengths = {np.asarray(s).shape[-1] if not torch.is_tensor(s) else s.shape[-1] for s in sources}
        if len(lengths) != 1:
            raise LengthMismatch(f"sources have mixed lengths {sorted(lengths)}")
        return torch.stack([torch.as_tensor(np.asarray(s)) if not torch.is_tensor(s) else s for s in sources])
    return torch.as_tensor(np.asarray(sources))


def execute_batched(graph, params, sources, schedule=None, mask=None, device="cuda"):
    """Render the graph through its schedule; returns (y (2, L), reg) on the device."""
    src = _check_sources(graph, sources)  # host checks first: the reference's errors on any device
    dev = ensure_device(device)
    L = src.shape[-1]
    if schedule is None:
        schedule = schedule_greedy(graph)
    if schedule.plans is None:
        schedule = plan_indices(graph, schedule)
    lay = ParamLayout(graph)
    flat = torch.from_numpy(lay.pack(params)).to(dev)
    plan = RenderPlan(graph, schedule, L, dev, flat, None, lay, backward=False)
    plan.set_stems(src)
    if mask is not None:
        plan.mask[: lay.P].copy_(torch.as_tensor(np.asarray(mask, dtype=np.float64)))
    plan.forward(use_mask=mask is not None)
    return plan.y.clone(), plan.reg_total()


def node_schedule(graph) -> Schedule:
    """One node per step in topological order (inputs first, the output last):
    the visiting order of the reference's one-node-at-a-time executor."""
    validate(graph)
    inputs = set(graph.nodes_of_type("i"))
    output = graph.nodes_of_type("o")[0]
    order = [v for v in topological_order(graph) if v not in inputs and v != output]
    subsets = [sorted(inputs)] + [[v] for v in order] + [[output]]
    seq = "i" + "".join(graph.node_types[v] for v in order) + "o"
    return plan_indices(graph, Schedule(seq, subsets))


def execute_reference(graph, params, sources, device="cuda"):
    """One-node-at-a-time executor (mg/scheduler.py:266-298), same contract as
    ``execute_batched``: every processor node is its own level launch of batch 1,
    visited in topological order.  The unbatched check of the batched path."""
    return execute_batched(graph, params, sources, node_schedule(graph), device=device)


def effective_weights(params, mask=None):
    w = params.effective_weights()
    return w * np.asarray(mask, dtype=np.float64) if mask is not None else w


__all__ = ["execute_batched", "execute_reference", "node_schedule", "effective_weights", "Schedule", "StepPlan",
           "schedule_greedy", "schedule_console", "plan_indices", "console_chains", "NotAConsole",
           "LengthMismatch", "SchedulerError", "F32", "F64"]
