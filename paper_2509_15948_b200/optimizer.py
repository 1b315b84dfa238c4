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

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .common import rng_for, seconds_to_samples
from .engine import F32, TrainEngine, ensure_device
from .graph import MixGraph, ParamStore
from .losses import LossConfig
from .schedule import plan_indices, schedule_for


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

    def engine(self, graph: MixGraph, L: int, cfg: TrainConfig, schedule=None) -> TrainEngine:
        key = (id(graph), graph.node_types, graph.edges, int(L), int(cfg.warmup_len), cfg.loss)
        eng = self._engines.get(key)
        if eng is None:
            ecfg = _EngineCfg(self, cfg)
            eng = TrainEngine(graph, L, ecfg, device=self.device, schedule=schedule)
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
    eng.step_async(alpha_p)
    values = eng.read_values()
    if not np.isfinite(values["loss"]):
        eng.t -= 1
        raise NonFiniteLoss(f"non-finite loss: {values}")
    opt.t = eng.t
    eng.store_params(params)
    return values


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
    eng = opt.engine(graph, seg, cfg, schedule)
    eng.load_params(params)
    full = session.length == seg
    st_dev = torch.as_tensor(np.asarray(session.stems), dtype=F32).to(dev)
    tg_dev = torch.as_tensor(np.asarray(session.target), dtype=F32).to(dev)
    if full:
        eng.plan.stems.copy_(st_dev)
        eng.target.copy_(tg_dev)
    vals = torch.zeros((cfg.steps, 4), dtype=torch.float64, device=dev)
    t0 = time.perf_counter()
    for step in range(cfg.steps):
        offset = int(rng.integers(0, session.length - seg + 1))
        if not full:
            eng.plan.stems.copy_(st_dev[..., offset:offset + seg])
            eng.target.copy_(tg_dev[..., offset:offset + seg])
        eng.step_async(alpha_p_fn(step) if alpha_p_fn else 0.0)
        vals[step].copy_(eng.vals)
    host = vals.cpu().numpy()
    wall = (time.perf_counter() - t0) / cfg.steps
    opt.t = eng.t
    eng.store_params(params)
    for i, v in enumerate(host):
        if not np.all(np.isfinite(v[:1])):
            raise NonFiniteLoss(f"non-finite loss at step {i}: {v.tolist()}")
        history.append({"loss": float(v[0]), "L_a": float(v[1]), "L_g": float(v[2]), "L_p": float(v[3]),
                        "step": len(history), "wall_s": wall})
    return history
