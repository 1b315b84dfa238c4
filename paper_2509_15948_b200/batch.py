"""Several songs' consoles trained as ONE device program.

A desk-recipe search trains on 57,000-sample segments, where one level launch
of one song fills only part of the 148 SMs.  Here the consoles of G songs are
joined into a disjoint union: node ids are offset per song, and level k of
the union schedule is the union of every song's level k of the console
sequence ``iecnsgdrmecnsgdro`` (mg/scheduler.py:135-154; a pruned song simply
contributes nothing to a stage it lost), so each level type is ONE launch
over all songs' nodes, the output level has one row per song.  Each song keeps
its own loss (one MRSTFT per song), its own segment stream (its RNG draws its
own offsets, mg/optimizer.py:97-105) and its own parameters; the optimiser is
one fused AdamW over the union's flat vector (AdamW is elementwise, and songs
in lock-step share the step count t and the sparsity weight).

Every level kernel computes a node's rows independently of which other nodes
share the launch (grids are (per-row blocks) x rows), so a song trained in a
union makes bit-for-bit the updates it makes alone (GPU test).

``prune_songs_lockstep`` runs G searches through ``pruning.prune_song_steps``
(the single copy of the reference's search control flow): trials run per song,
and whenever every search has reached its next train() (the console fit, each
round's fine-tune: the same step counts for all songs of a recipe) the requests
are served together by one ``BatchTrainEngine``.
"""

from __future__ import annotations

import time

import numpy as np
import torch

from ._lib import check, lib
from .engine import (F32, F64, LossPlan, ParamLayout, RenderPlan, capture_graph, current_stream, ensure_device,
                     host_wait, on_stream, own_stream, ptr, stream_ptr)
from .graph import PROCESSOR_TYPES, MixGraph, ParamStore
from .optimizer import NonFiniteLoss, SongTooShort, _EngineCfg, _graph_min_steps, make_optimizer
from .schedule import CONSOLE_SEQUENCE, Schedule, plan_indices, schedule_console


class SongUnion:
    """Disjoint union of console graphs with the stage-merged console schedule."""

    def __init__(self, graphs):
        self.graphs = list(graphs)
        types, edges = [], []
        self.node_off, self.in_off, self.proc_off = [], [], []
        n_in = n_proc = 0
        stages = [[] for _ in CONSOLE_SEQUENCE]
        schedules = {}  # a graph repeated in the union (eval segments) is scheduled once
        for g in self.graphs:
            off = len(types)
            self.node_off.append(off)
            self.in_off.append(n_in)
            self.proc_off.append(n_proc)
            n_in += len(g.nodes_of_type("i"))
            n_proc += len(g.processor_nodes())
            types.extend(g.node_types)
            edges.extend((a + off, b + off) for a, b in g.edges)
            sch = schedules.get(id(g))
            if sch is None:  # NotAConsole for anything but a console or its prunings
                sch = schedules[id(g)] = schedule_console(g)
            pos = 0
            for step, tag in enumerate(sch.type_sequence):
                while CONSOLE_SEQUENCE[pos] != tag:
                    pos += 1
                stages[pos].extend(v + off for v in sch.subsets[step])
                pos += 1
        self.n_in, self.n_proc = n_in, n_proc
        self.graph = MixGraph("".join(types), tuple(edges))
        seq = "".join(t for t, sub in zip(CONSOLE_SEQUENCE, stages) if sub)
        self.schedule = plan_indices(self.graph, Schedule(seq, [sub for sub in stages if sub]))
        self.layout = ParamLayout(self.graph)
        # per type: the union bank rows of each song (songs appear in node-id order)
        self.rows = {t: [len(g.nodes_of_type(t)) for g in self.graphs] for t in PROCESSOR_TYPES}

    def pack(self, params_list) -> np.ndarray:
        banks = {t: np.concatenate([np.asarray(p.params[t], dtype=np.float64).reshape(-1, self.layout_cols(t))
                                    for p in params_list], axis=0) for t in PROCESSOR_TYPES}
        raw = np.concatenate([np.asarray(p.raw_weights, dtype=np.float64) for p in params_list])
        return self.layout.pack(ParamStore(banks, raw))

    def unpack_into(self, flat: np.ndarray, params_list) -> None:
        parts = self.layout.split(flat)
        for t in PROCESSOR_TYPES:
            o = 0
            for p, n in zip(params_list, self.rows[t]):
                p.params[t] = parts[t][o:o + n].copy()
                o += n
        o = 0
        for p, g in zip(params_list, self.graphs):
            n = len(g.processor_nodes())
            p.raw_weights = parts["w"][o:o + n].copy()
            o += n

    @staticmethod
    def layout_cols(t):
        from .graph import PARAM_COUNTS
        return PARAM_COUNTS[t]


class BatchTrainEngine:
    """``train_step`` (mg/optimizer.py:140-186) for G songs at once on a ``SongUnion``."""

    def __init__(self, union: SongUnion, L: int, cfg, device="cuda"):
        self.device = dev = ensure_device(device)
        self.union, self.cfg, self.L = union, cfg, int(L)
        self.ws = int(cfg.warmup_len)
        G = self.G = len(union.graphs)
        lay = self.layout = union.layout
        self.params = torch.zeros(lay.n, dtype=F64, device=dev)
        self.grads = torch.zeros(lay.n, dtype=F64, device=dev)
        self.m = torch.zeros(lay.n, dtype=F64, device=dev)
        self.v = torch.zeros(lay.n, dtype=F64, device=dev)
        self.plan = RenderPlan(union.graph, union.schedule, self.L, dev, self.params, self.grads, lay, backward=True)
        assert self.plan.n_out == G
        # one MRSTFT call set for all songs (signals 2L apart in ys / targets / dYs)
        self.lossp = LossPlan(cfg.loss, self.L - self.ws, dev, batch=G, sig_stride=2 * self.L)
        self.targets = torch.zeros((G, 2, self.L), dtype=F32, device=dev)
        self.scalars = torch.zeros(8, dtype=F64, device=dev)
        self.vals = torch.zeros((G, 4), dtype=F64, device=dev)  # per song: loss, L_a, L_g, L_p
        self.guard = torch.zeros((), dtype=F64, device=dev)     # sum of the songs' losses
        self.halt = torch.zeros((), dtype=F64, device=dev)
        self.sparsity = torch.zeros(G, dtype=F64, device=dev)
        self.plan.greg.fill_(float(cfg.loss.gain_staging_weight))
        # song of every gain-staging slot (plan.reg: the e/r/d level rows in level order)
        owner = []
        sched = union.schedule
        bounds = np.asarray(union.node_off + [union.graph.num_nodes])
        for s in range(1, len(sched.subsets)):
            if sched.type_sequence[s] in "erd":
                owner.extend(int(np.searchsorted(bounds, v, side="right") - 1) for v in sched.subsets[s])
        # the gain-staging rows of each song, in level order: (offsets, row indices)
        order = sorted(range(len(owner)), key=lambda i: (owner[i], i))
        counts = np.bincount(np.asarray(owner, dtype=np.int64), minlength=G) if owner else np.zeros(G, np.int64)
        self.reg_off = torch.tensor(np.concatenate([[0], np.cumsum(counts)]).astype(np.int32), device=dev)
        self.reg_idx = torch.tensor(order if order else [0], dtype=torch.int32, device=dev)
        self.t = 0
        self.side = own_stream(dev, "side")
        self._graph = None
        self._ring = torch.zeros((64, 8 + G), dtype=F64).pin_memory()
        self._ring_ev = [None] * 64
        self.song_off = torch.zeros(G, dtype=torch.int64, device=dev)
        self.gather = None  # (src ptrs, dst ptrs, row song, rows): set_sessions

    def set_sessions(self, sessions):
        """Device sessions (stems (K_i, 2, T_i), target (2, T_i)) per song: every step
        gathers each song's segment at its offset (song_off) into the union's inputs."""
        L, u = self.L, self.union
        src, dst, song = [], [], []
        for i, (st, tg) in enumerate(sessions):
            T = st.shape[-1]
            for k in range(st.shape[0]):
                for c in range(2):
                    src.append(ptr(st, (k * 2 + c) * T))
                    dst.append(ptr(self.plan.stems, ((u.in_off[i] + k) * 2 + c) * L))
                    song.append(i)
            for c in range(2):
                src.append(ptr(tg, c * T))
                dst.append(ptr(self.targets, (i * 2 + c) * L))
                song.append(i)
        self._sessions = sessions  # keep the source buffers alive
        t = [torch.tensor(np.asarray(a, dtype=np.int64), device=self.device) for a in (src, dst)]
        self.gather = (t[0], t[1], torch.tensor(song, dtype=torch.int32, device=self.device), len(src))

    def load_params(self, params_list):
        self.params.copy_(torch.from_numpy(self.union.pack(params_list)))

    def store_params(self, params_list):
        self.union.unpack_into(self.params.cpu().numpy(), params_list)

    def _body(self):
        L, ws, G = self.L, self.ws, self.G
        plan = self.plan
        Ld = lib()
        main, side = current_stream(), self.side
        if self.gather is not None:
            src, dst, song, rows = self.gather
            check(Ld.mgb_gather_rows(ptr(src), ptr(dst), ptr(song), ptr(self.song_off), rows, L, stream_ptr()),
                  "mgb_gather_rows")
        prepared = plan.prepare(side)
        with on_stream(side):
            plan.dYs[:, :, :ws].zero_()
            self.lossp.target(ptr(self.targets, ws), ptr(self.targets, L + ws))
            tev = torch.cuda.Event()
            tev.record(side)
        plan.forward(use_mask=False, prepared=prepared, norms=side)
        main.wait_event(tev)
        self.lossp.forward(ptr(plan.ys, ws), ptr(plan.ys, L + ws))
        main.wait_stream(side)
        side.wait_stream(main)
        with on_stream(side):  # loss assembly per song (read by the optimiser only)
            lay, u = self.layout, self.union
            sp = stream_ptr()
            for i, g in enumerate(u.graphs):
                n = len(g.processor_nodes())
                if n:
                    check(Ld.mgb_sparsity(ptr(self.params, lay.w_off + u.proc_off[i]), n, ptr(self.sparsity, i), sp),
                          "mgb_sparsity")
            check(Ld.mgb_loss_assembly(ptr(self.lossp.loss), ptr(plan.reg), ptr(self.reg_off), ptr(self.reg_idx),
                                       ptr(self.sparsity), ptr(self.scalars),
                                       float(self.cfg.loss.gain_staging_weight), G, ptr(self.vals), ptr(self.guard),
                                       sp), "mgb_loss_assembly")
        self.lossp.backward(ptr(plan.ys, ws), ptr(plan.ys, L + ws), ptr(plan.dYs, ws), ptr(plan.dYs, L + ws))
        plan.backward(side)
        main.wait_stream(side)
        check(Ld.mgb_adamw_step(ptr(self.params), ptr(self.grads), ptr(self.m), ptr(self.v), lay.n,
                                lay.off["d"], lay.rows["d"], lay.w_off, lay.P, ptr(plan.gw), None,
                                ptr(self.scalars), ptr(self.guard), ptr(self.halt), stream_ptr()),
              "mgb_adamw_step")

    def _set_scalars(self, alpha_p, offsets=None):
        """Per-step [lr, b1, b2, eps, wd, c1, c2, alpha_p] and the songs' segment offsets
        -> device, through a ring of pinned slots."""
        c = self.cfg
        self.t += 1
        b1, b2 = c.betas
        i = self.t % 64
        if self._ring_ev[i] is not None:
            host_wait(self._ring_ev[i])
        row = self._ring[i].numpy()
        row[:8] = (c.lr, b1, b2, c.eps, c.weight_decay, 1.0 - b1 ** self.t, 1.0 - b2 ** self.t, float(alpha_p))
        if offsets is not None:
            row[8:] = offsets  # exact in float64 (< 2^53)
        self.scalars.copy_(self._ring[i, :8], non_blocking=True)
        if offsets is not None:
            self.song_off.copy_(self._ring[i, 8:], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._ring_ev[i] = ev

    def step_async(self, alpha_p=0.0, use_graph=True, offsets=None):
        self._set_scalars(alpha_p, offsets)
        if not use_graph:
            self._body()
            return
        if self._graph is None:
            s = own_stream(self.device, "warm")
            s.wait_stream(current_stream())
            with torch.cuda.stream(s):
                snap = [x.clone() for x in (self.params, self.m, self.v, self.halt)]
                self._body()
                for x, y in zip((self.params, self.m, self.v, self.halt), snap):
                    x.copy_(y)
            current_stream().wait_stream(s)
            current_stream().synchronize()
            self._graph = capture_graph(self._body, self.device)
        self._graph.replay()


# a batched train() call replays a captured step when it is at least this long (one capture
# serves all songs of the batch; the 50-step fine-tunes of the desk recipe qualify)
BATCH_GRAPH_MIN_STEPS = 10


def train_batch(reqs, device="cuda"):
    """Serve several ``pruning.TrainRequest``s (one per song, same step count and
    hyper-parameters) with one ``BatchTrainEngine``: each step draws every song's
    segment offset from its own RNG, copies the segments into the union's input
    rows, and replays the union step.  Same per-song semantics as ``optimizer.train``
    (histories, parameters written back, fresh AdamW state per call, NonFiniteLoss)."""
    cfg = reqs[0].cfg
    for r in reqs[1:]:
        if (r.cfg.steps, r.cfg.segment_len, r.cfg.warmup_len, r.cfg.lr, r.cfg.betas, r.cfg.eps,
                r.cfg.weight_decay, r.cfg.loss) != (cfg.steps, cfg.segment_len, cfg.warmup_len, cfg.lr, cfg.betas,
                                                     cfg.eps, cfg.weight_decay, cfg.loss):
            raise ValueError("batched train requests must share steps, segment length and hyper-parameters")
    if cfg.steps <= 0:
        return
    seg = cfg.segment_len
    for r in reqs:
        if r.session.length < seg:
            raise SongTooShort(f"song has {r.session.length} samples, segment needs {seg}")
    dev = ensure_device(device)
    union = SongUnion([r.graph for r in reqs])
    eng = BatchTrainEngine(union, seg, _EngineCfg(make_optimizer(None, cfg), cfg), device=dev)
    eng.load_params([r.params for r in reqs])
    eng.set_sessions([r.session.on_device(dev) for r in reqs])
    rng_states = [r.rng.bit_generator.state for r in reqs]
    vals = torch.zeros((cfg.steps, eng.G, 4), dtype=F64, device=dev)
    use_graph = cfg.steps >= BATCH_GRAPH_MIN_STEPS
    t0 = time.perf_counter()
    for step in range(cfg.steps):
        offs = [int(r.rng.integers(0, r.session.length - seg + 1)) for r in reqs]
        alphas = {r.alpha_p_fn(step) if r.alpha_p_fn else 0.0 for r in reqs}
        if len(alphas) != 1:
            raise ValueError("batched songs must share the sparsity weight of every step")
        eng.step_async(alphas.pop(), use_graph=use_graph, offsets=offs)
        vals[step].copy_(eng.vals)
    host_wait(torch.cuda.current_stream())
    host = vals.cpu().numpy()
    wall = (time.perf_counter() - t0) / cfg.steps
    bad = [next((k for k in range(cfg.steps) if not np.isfinite(host[k, i, 0])), None) for i in range(eng.G)]
    if any(b is not None for b in bad):
        # a non-finite loss stopped the whole union at its first occurrence; the reference
        # stops only the failing song: let the caller rerun these songs one at a time
        for r, st in zip(reqs, rng_states):
            r.rng.bit_generator.state = st
        raise BatchNonFinite([i for i, b in enumerate(bad) if b is not None])
    eng.store_params([r.params for r in reqs])
    for i, r in enumerate(reqs):
        for v in host[:, i]:
            r.history.append({"loss": float(v[0]), "L_a": float(v[1]), "L_g": float(v[2]), "L_p": float(v[3]),
                              "step": len(r.history), "wall_s": wall})


class BatchNonFinite(NonFiniteLoss):
    def __init__(self, songs):
        super().__init__(f"non-finite loss in batched songs {songs}")
        self.songs = songs


class BatchEvalEngine:
    """Pruning trials of several songs in one device program: ``eval_loss``
    (mg/pruning.py:115-123) of every song at once, each song with its own graph,
    mask, parameters and eval set (same segment count and length for all songs of
    a recipe).  The unit of the union is a (segment, song) pair: every eval segment
    of every song is its own copy of the song's console in ONE render plan (SURVEY
    §8f rank 1 (iii): all eval segments in one launch per level type), and ONE
    batched MRSTFT scores all of them against device-resident target spectra.
    Renders are incremental like ``engine.EvalEngine``'s: a trial starts at the
    first level where any unit's mask changed; per-row kernels make each song's
    loss bit-identical to its own ``EvalEngine``."""

    def __init__(self, graphs, eval_sets, device="cuda"):
        self.device = dev = ensure_device(device)
        es0 = eval_sets[0]
        self.G = G = len(graphs)
        self.nseg, self.ws = len(es0.segments), int(es0.warmup_len)
        L = self.L = np.asarray(es0.segments[0][0]).shape[-1]
        for es in eval_sets:
            if (len(es.segments), int(es.warmup_len), np.asarray(es.segments[0][0]).shape[-1], es.loss_cfg) != \
                    (self.nseg, self.ws, L, es0.loss_cfg):
                raise ValueError("batched eval sets must share segment count, length, warm-up and loss")
        # unit u = j * G + i: segment j of song i
        self.union = union = SongUnion([g for _ in range(self.nseg) for g in graphs])
        lay = self.layout = union.layout
        self.params = torch.zeros(lay.n, dtype=F64, device=dev)
        self._packed = None
        self._prep_dirty = True
        self._last = None
        self.plan = plan = RenderPlan(union.graph, union.schedule, L, dev, self.params, None, lay, backward=False)
        U, ws = G * self.nseg, self.ws
        t = torch.zeros((U, 2, L), dtype=F32, device=dev)  # targets laid out like the output rows
        for i, es in enumerate(eval_sets):
            for j, (st, tg) in enumerate(es.device_segments(dev)):  # uploaded once per search
                u = j * G + i
                plan.stems[union.in_off[u]:union.in_off[u] + st.shape[0]].copy_(st)
                t[u, :, ws:].copy_(tg)
        self.lossp = LossPlan(es0.loss_cfg, L - ws, dev, backward=False, batch=U, sig_stride=2 * L) if U > 1 else \
            LossPlan(es0.loss_cfg, L - ws, dev, backward=False)
        self.lossp.target(ptr(t, ws), ptr(t, L + ws))
        self._targets = t
        self.acc = torch.zeros(U, dtype=F64, device=dev)
        self.acc_host = torch.zeros(U, dtype=F64).pin_memory()
        self.mask_host = torch.ones(max(lay.P, 1), dtype=F64).pin_memory()

    def load_params(self, params_list):
        packed = self.union.pack([p for _ in range(self.nseg) for p in params_list])
        if self._packed is not None and np.array_equal(packed, self._packed):
            return
        self._packed = packed.copy()
        self.params.copy_(torch.from_numpy(packed))
        self._prep_dirty = True

    def losses_for(self, masks):
        """Per-song mean eval loss for per-song masks (a list, one mask per song)."""
        u = self.union
        m = np.ones(max(self.layout.P, 1))
        for j in range(self.nseg):
            for i, mk in enumerate(masks):
                o = u.proc_off[j * self.G + i]
                m[o:o + len(mk)] = mk
        self.mask_host.copy_(torch.from_numpy(m))
        L, ws, plan = self.L, self.ws, self.plan
        if self._prep_dirty:
            plan.prepare()
        plan.mask.copy_(self.mask_host, non_blocking=True)
        start = 0
        if not self._prep_dirty and self._last is not None:
            changed = np.nonzero(m != self._last)[0]
            start = int(plan.proc_level[changed].min()) if changed.size else len(plan.levels)
        plan.forward(use_mask=True, prepared=True, norms=None, start=start)
        self._last = m
        self.lossp.forward(ptr(plan.ys, ws), ptr(plan.ys, L + ws))
        self.acc.copy_(self.lossp.loss)
        self._prep_dirty = False
        self.acc_host.copy_(self.acc, non_blocking=True)
        host_wait(current_stream())
        a = self.acc_host.numpy()
        out = []
        for i in range(self.G):
            total = 0.0
            for j in range(self.nseg):  # per-segment float() then mean, as mg/pruning.py:120-123
                total += float(a[j * self.G + i])
            out.append(total / self.nseg)
        return out


def prune_songs_lockstep(jobs, device="cuda", batch_trials=True):
    """Run several ``prune_song`` searches in lock-step; ``jobs`` = list of
    (graph, params, session, PruneConfig).  Each search is ``pruning.prune_song_steps``
    (the reference's control flow, one copy); its train requests are served together by
    one ``train_batch`` once every search has reached one, and its trials together by a
    ``BatchEvalEngine`` over the songs' current graphs (a song whose pass has ended
    keeps its last graph and mask in the union until the next round, so the union is
    rebuilt once per round).  Returns each search's (graph, params, state, report,
    history), identical to running them one by one."""
    from .pruning import EvalRequest, eval_losses, prune_song, prune_song_steps, run_train_request
    gens = [prune_song_steps(g, p, s, c, None, device) for g, p, s, c in jobs]
    out = [None] * len(gens)
    reqs, last_eval = {}, {}

    def advance(i, value):
        try:
            reqs[i] = gens[i].send(value) if value is not _START else next(gens[i])
            if isinstance(reqs[i], EvalRequest):
                last_eval[i] = reqs[i]
        except StopIteration as done:
            out[i] = done.value
            reqs.pop(i, None)
            last_eval.pop(i, None)

    for i in range(len(gens)):
        advance(i, _START)
    engines, trained = {}, 0  # per eval-set shape: (engine key, engine, loaded-params key)
    while reqs:
        evals = sorted(i for i, r in reqs.items() if isinstance(r, EvalRequest))
        if evals:
            if not batch_trials:
                for i in evals:
                    r = reqs[i]
                    advance(i, eval_losses(r.graph, r.params, r.masks, r.eval_set))
                continue
            # songs whose eval sets share a shape form one union (every song of one recipe)
            groups = {}
            for i in sorted(last_eval):
                es = last_eval[i].eval_set
                shape = (len(es.segments), np.shape(es.segments[0][0])[-1], int(es.warmup_len), es.loss_cfg)
                groups.setdefault(shape, []).append(i)
            for shape, ids in groups.items():
                if not any(i in evals for i in ids):
                    continue
                key = tuple((i, id(last_eval[i].graph), id(last_eval[i].eval_set)) for i in ids)
                t0 = time.perf_counter()
                ekey, beval, loaded = engines.get(shape, (None, None, None))
                if key != ekey:
                    beval = BatchEvalEngine([last_eval[i].graph for i in ids],
                                            [last_eval[i].eval_set for i in ids], device)
                    ekey, loaded = key, None
                    PHASE_S["trial_engine_build"] += time.perf_counter() - t0
                pkey = (tuple(id(last_eval[i].params) for i in ids), trained)
                if pkey != loaded:  # parameters change only in training: no repack per trial
                    beval.load_params([last_eval[i].params for i in ids])
                    loaded = pkey
                engines[shape] = (ekey, beval, loaded)
                losses = beval.losses_for([last_eval[i].mask for i in ids])
                PHASE_S["trials"] += time.perf_counter() - t0
                PHASE_S["trial_slots"] += 1
                for k, i in enumerate(ids):
                    if i in evals:
                        advance(i, [losses[k]])
            continue
        # every pending search waits on a train(): requests with the same step count,
        # hyper-parameters and sparsity schedule run as one batch
        batches = {}
        for i in sorted(reqs):
            r = reqs[i]
            c = r.cfg
            alphas = tuple(r.alpha_p_fn(s) if r.alpha_p_fn else 0.0 for s in range(c.steps))
            batches.setdefault((c.steps, c.segment_len, c.warmup_len, c.lr, tuple(c.betas), c.eps,
                                c.weight_decay, c.loss, alphas), []).append(i)
        t0 = time.perf_counter()
        for ids in batches.values():
            try:
                if len(ids) == 1:
                    run_train_request(reqs[ids[0]], device)
                else:
                    train_batch([reqs[i] for i in ids], device)
            except NonFiniteLoss:
                # rare: rerun these searches one by one from the start (the reference's
                # per-song semantics: only a failing song stops)
                for i in ids:
                    g, p, s, c = jobs[i]
                    try:
                        out[i] = prune_song(g, p, s, c, device=device, speculate=1)
                    except NonFiniteLoss as e:
                        out[i] = e
                    reqs.pop(i, None)
                    last_eval.pop(i, None)
                continue
            trained += 1
            for i in ids:
                advance(i, None)
        PHASE_S["train"] += time.perf_counter() - t0
    return out


_START = object()

# wall seconds per phase of prune_songs_lockstep (tools/songs_bench.py reports them)
PHASE_S = {"train": 0.0, "trials": 0.0, "trial_engine_build": 0.0, "trial_slots": 0, "host_other": 0.0}


__all__ = ["SongUnion", "BatchTrainEngine", "BatchEvalEngine", "train_batch", "prune_songs_lockstep",
           "BatchNonFinite"]
