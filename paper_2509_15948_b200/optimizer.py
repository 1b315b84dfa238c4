"""Gradient-descent training of console parameters on the device.

Same API and semantics as ``mg/optimizer.py``: each step samples a segment,
runs render + MRSTFT forward and the full backward, replaces the delay
z-gradients by the sign-normalised rule, applies AdamW with decoupled weight
decay and projects delay frequencies into the unit disk.  Here the whole step
is one CUDA-graph replay of ``engine.TrainEngine``; parameters and AdamW
moments stay on the device for a whole ``train()`` call (fresh moments per
call, mg/optimizer.py:205) and are written back to the host ``ParamStore``
at the end.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .common import rng_for, seconds_to_samples
from .engine import F32, TrainEngine, ensure_device, host_wait, own_stream
from .graph import MixGraph, ParamStore
from .losses import LossConfig
from .schedule import plan_indices, schedule_for


# train() captures its step only for runs at least this long
GRAPH_MIN_STEPS = int(os.environ.get("MG_GRAPH_MIN_STEPS", "200"))


class SongTooShort(Exception):
    pass


class NonFiniteLoss(Exception):
    pass


@dataclass
class Session:
    stems: np.ndarray   # (K, 2, L)
    target: np.ndarray  # (2, L)
    name: str = "session"

    @property
    def length(self):
        return self.stems.shape[-1]

    def on_device(self, dev):
        """(stems, target) as float32 device tensors, uploaded once per device and
        reused by every ``train`` call of a search (13 per desk-recipe song).
        Assign new arrays to change the session; in-place edits are not seen."""
        key = (str(dev), id(self.stems), id(self.target))
        hit = self.__dict__.get("_dev")
        if hit is None or hit[0] != key:
            st = torch.as_tensor(np.asarray(self.stems), dtype=F32).to(dev)
            tg = torch.as_tensor(np.asarray(self.target), dtype=F32).to(dev)
            hit = self.__dict__["_dev"] = (key, st, tg)
        return hit[1], hit[2]


@dataclass
class TrainConfig:
    lr: float = 0.01
    steps: int = 12_000
    segment_seconds: float = 3.8
    warmup_seconds: float = 1.0
    seed: int = 0
    weight_decay: float = 1e-2
    betas: tuple = (0.9, 0.999)
    eps: float = 1e-8
    loss: LossConfig = field(default_factory=LossConfig)

    def __post_init__(self):
        if self.segment_seconds <= self.warmup_seconds:
            raise ValueError("segment must be longer than the warm-up exclusion")

    @property
    def segment_len(self):
        return seconds_to_samples(self.segment_seconds)

    @property
    def warmup_len(self):
        return seconds_to_samples(self.warmup_seconds)


class AdamW:
    """Decoupled-weight-decay Adam whose moments live on the device.

    Holds one ``TrainEngine`` per (graph, segment length): a new optimiser is
    fresh state, exactly like constructing the reference's AdamW."""

    def __init__(self, arrays=None, lr=0.01, betas=(0.9, 0.999), eps=1e-8, weight_decay=1e-2,
                 device="cuda"):
        self.lr, self.betas, self.eps, self.weight_decay = lr, tuple(betas), eps, weight_decay
        self.t = 0
        self.device = device
        self._engines = {}

    def engine(self, graph: MixGraph, L: int, cfg: TrainConfig, schedule=None, use_graph=True) -> TrainEngine:
        key = (id(graph), graph.node_types, graph.edges, int(L), int(cfg.warmup_len), cfg.loss, bool(use_graph))
        eng = self._engines.get(key)
        if eng is None:
            ecfg = _EngineCfg(self, cfg)
            eng = TrainEngine(graph, L, ecfg, device=self.device, schedule=schedule, use_graph=use_graph)
            self._engines = {key: eng}  # one live engine per optimiser
        eng.cfg = _EngineCfg(self, cfg)
        return eng


class _EngineCfg:
    """Hyper-parameters the engine reads each step (optimiser's lr/betas + cfg's loss/warm-up)."""

    def __init__(self, opt: AdamW, cfg: TrainConfig):
        self.lr, self.betas, self.eps, self.weight_decay = opt.lr, opt.betas, opt.eps, opt.weight_decay
        self.loss = cfg.loss
        self.warmup_len = cfg.warmup_len


def make_optimizer(params: ParamStore, cfg: TrainConfig, device="cuda"):
    return AdamW(None, lr=cfg.lr, betas=cfg.betas, eps=cfg.eps, weight_decay=cfg.weight_decay,
                 device=device)


def sample_segment(session: Session, segment_len, rng):
    total = session.length
    if total < segment_len:
        raise SongTooShort(f"song has {total} samples, segment needs {segment_len}")
    offset = int(rng.integers(0, total - segment_len + 1))
    return (session.stems[..., offset:offset + segment_len],
            session.target[..., offset:offset + segment_len], offset)


def train_step(graph, params: ParamStore, segment, cfg: TrainConfig, opt: AdamW, schedule=None,
               alpha_p=0.0):
    """One forward/backward/update on an aligned (stems, target) segment (mg/optimizer.py:140-186).

    Host arrays in, host ``params`` updated in place, metrics dict out."""
    stems, target = segment
    L = np.asarray(stems).shape[-1] if not torch.is_tensor(stems) else stems.shape[-1]
    eng = opt.engine(graph, L, cfg, schedule)
    eng.load_params(params)
    eng.plan.set_stems(stems)
    eng.target.copy_(torch.as_tensor(np.asarray(target) if not torch.is_tensor(target) else target,
                                     dtype=F32), non_blocking=True)
    eng.t = opt.t
    eng.halt.zero_()
    eng.step_async(alpha_p)
    values = eng.read_values()
    if not np.isfinite(values["loss"]):
        eng.t -= 1  # the device left params and moments untouched
        raise NonFiniteLoss(f"non-finite loss: {values}")
    opt.t = eng.t
    eng.store_params(params)
    return values


def _graph_min_steps():
    from .engine import _host
    return getattr(_host, "graph_min_steps", None) or GRAPH_MIN_STEPS


def _pinned_f32(a):
    t = a if torch.is_tensor(a) else torch.from_numpy(np.ascontiguousarray(a))
    if t.dtype != F32:
        t = t.to(dtype=F32)
    if t.device.type == "cpu" and not t.is_pinned():
        t = t.pin_memory()
    return t


def train_segments(graph, params: ParamStore, segments, cfg: TrainConfig, opt: AdamW = None,
                   schedule=None, alpha_p_fn=None, history=None):
    """One optimiser step per host ``(stems, target)`` segment of an iterable, pipelined.

    The streaming form of ``train_step`` for segments that live on the host
    (a data loader): segment k+1's host→device copy runs on a copy stream
    into a staging slot while step k computes, each step's metrics are read
    back into a pinned ring without stalling the stream, and ``params`` is
    updated once at the end.  Same arithmetic and per-step semantics as
    calling ``train_step`` in a loop (mg/optimizer.py:140-186); a non-finite
    loss leaves that step's update undone on the device and raises
    ``NonFiniteLoss`` after the run, like ``train``: no update happens from
    the first non-finite step on, ``params`` and ``opt.t`` are those after the
    last finite step and ``history`` holds the finite steps only.  Pass pinned
    torch tensors to avoid a pinning copy per segment."""
    history = history if history is not None else []
    it = iter(segments)
    seg = next(it, None)
    if seg is None:
        return history
    opt = opt or make_optimizer(params, cfg)
    L = seg[0].shape[-1]
    eng = opt.engine(graph, L, cfg, schedule)
    eng.load_params(params)
    eng.halt.zero_()
    t_start = eng.t = opt.t
    dev = eng.device
    comp = torch.cuda.current_stream(dev)
    copy = own_stream(dev, "copy")
    stage = [(torch.empty_like(eng.plan.stems), torch.empty_like(eng.target)) for _ in range(2)]
    freed = [None, None]  # event: the compute stream is done reading the slot

    def upload(seg, slot):
        st, tg = _pinned_f32(seg[0]), _pinned_f32(seg[1])
        if st.shape != eng.plan.stems.shape or tg.shape != eng.target.shape:
            raise ValueError(f"segment shapes {tuple(st.shape)}, {tuple(tg.shape)} differ from the first")
        with torch.cuda.stream(copy):
            if freed[slot] is not None:
                copy.wait_event(freed[slot])
            stage[slot][0].copy_(st, non_blocking=True)
            stage[slot][1].copy_(tg, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
        return ev, (st, tg)  # keep the host tensors alive until the copy ran

    ring = torch.zeros((64, 4), dtype=torch.float64).pin_memory()
    ring_ev = [None] * 64
    out = []
    t0 = time.perf_counter()
    ready, keep = upload(seg, 0)
    k = 0
    while seg is not None:
        slot = k % 2
        comp.wait_event(ready)
        eng.plan.stems.copy_(stage[slot][0], non_blocking=True)
        eng.target.copy_(stage[slot][1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(comp)
        freed[slot] = ev
        seg = next(it, None)
        if seg is not None:
            nxt = upload(seg, 1 - slot)
        eng.step_async(alpha_p_fn(k) if alpha_p_fn else 0.0)
        r = k % 64
        if ring_ev[r] is not None:
            host_wait(ring_ev[r])
            out.append(ring[r].tolist())
        ring[r].copy_(eng.vals, non_blocking=True)
        ring_ev[r] = torch.cuda.Event()
        ring_ev[r].record(comp)
        if seg is not None:
            ready, keep = nxt
        k += 1
    for j in range(k - min(k, 64), k):
        r = j % 64
        host_wait(ring_ev[r])
        out.append(ring[r].tolist())
    del keep
    wall = (time.perf_counter() - t0) / k
    bad = _first_nonfinite([v[0] for v in out])
    opt.t = eng.t = t_start + (k if bad is None else bad)
    eng.store_params(params)
    base = len(history)
    for i, v in enumerate(out[:bad]):
        history.append({"loss": v[0], "L_a": v[1], "L_g": v[2], "L_p": v[3], "step": base + i,
                        "wall_s": wall})
    if bad is not None:
        raise NonFiniteLoss(f"non-finite loss at step {bad}: {out[bad]}")
    return history


def _first_nonfinite(losses):
    for i, v in enumerate(losses):
        if not np.isfinite(v):
            return i
    return None


def train(graph, params: ParamStore, session: Session, cfg: TrainConfig, schedule=None,
          alpha_p_fn=None, rng=None, history=None, device="cuda"):
    """Optimise params in place for cfg.steps (mg/optimizer.py:196-216)."""
    if schedule is None:
        schedule = schedule_for(graph)
    elif schedule.plans is None:
        schedule = plan_indices(graph, schedule)
    opt = make_optimizer(params, cfg, device)
    rng = rng or rng_for(cfg.seed, "segments")
    history = history if history is not None else []
    seg = cfg.segment_len
    if session.length < seg:
        raise SongTooShort(f"song has {session.length} samples, segment needs {seg}")
    if cfg.steps <= 0:
        return history
    dev = ensure_device(device)
    # a short run (a fine-tune round) is as fast eager as replayed: skip the capture
    eng = opt.engine(graph, seg, cfg, schedule, use_graph=cfg.steps >= _graph_min_steps())
    eng.load_params(params)
    full = session.length == seg
    st_dev, tg_dev = session.on_device(dev)
    if full:
        eng.plan.stems.copy_(st_dev)
        eng.target.copy_(tg_dev)
    vals = torch.zeros((cfg.steps, 4), dtype=torch.float64, device=dev)
    eng.halt.zero_()
    rng_state = rng.bit_generator.state
    t0 = time.perf_counter()
    for step in range(cfg.steps):
        offset = int(rng.integers(0, session.length - seg + 1))
        if not full:
            eng.plan.stems.copy_(st_dev[..., offset:offset + seg])
            eng.target.copy_(tg_dev[..., offset:offset + seg])
        eng.step_async(alpha_p_fn(step) if alpha_p_fn else 0.0)
        vals[step].copy_(eng.vals)
    host_wait(torch.cuda.current_stream())
    host = vals.cpu().numpy()
    wall = (time.perf_counter() - t0) / cfg.steps
    # NonFiniteLoss (mg/optimizer.py:170-171): the reference stops at the first
    # non-finite step.  The device's sticky flag skipped that step's update and
    # every later one, so the parameters are those after the last finite step;
    # the step count, history and segment RNG are put where the reference leaves them.
    bad = _first_nonfinite(host[:, 0])
    opt.t = eng.t = cfg.steps if bad is None else bad
    eng.store_params(params)
    for i, v in enumerate(host[:bad]):
        history.append({"loss": float(v[0]), "L_a": float(v[1]), "L_g": float(v[2]), "L_p": float(v[3]),
                        "step": len(history), "wall_s": wall})
    if bad is not None:
        rng.bit_generator.state = rng_state
        for _ in range(bad + 1):
            rng.integers(0, session.length - seg + 1)
        raise NonFiniteLoss(f"non-finite loss at step {bad}: {host[bad].tolist()}")
    return history
