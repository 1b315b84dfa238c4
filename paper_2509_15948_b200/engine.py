"""Device engine: one compiled plan per graph version, launched through the C ABI.

A ``RenderPlan`` turns a schedule's ``StepPlan`` list (mg/scheduler.py:157-204)
into device row-pointer tables, so every level kernel reads its inputs straight
out of the producer level's output buffer (no gather copies):

* processor level  ->  ``mgb_level_forward/backward`` over all B rows at once;
* mix/output level ->  ``mgb_bus_sum`` (atomic-free segmented sum).

Backward gradient routing mirrors the tape's ``gather_rows``/``segment_sum``
adjoints (mg/engine.py:439-467) without copies: a node with exactly one
consumer simply points its dL/dy row at the consumer's dL/du row (processor
consumer) or at the consumer's own dL/dy row (mix/output consumer, whose
adjoint is a broadcast).  Only nodes with fan-out > 1 get a summing kernel.

``TrainEngine`` is ``train_step`` (mg/optimizer.py:140-186) on device: render,
target spectra, MRSTFT, full backward, delay rule, AdamW and projection, all
on one stream and captured once into a CUDA graph per graph version.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np
import torch

from . import _lib
from ._lib import MgbLevel, MgbLoss, check, lib
from .graph import PARAM_COUNTS, PROCESSOR_TYPES, MixGraph
from .schedule import KERNEL_TYPES, LengthMismatch, Schedule, plan_indices, schedule_for
from .tables import projection_sparse, reverb_tables

F32, F64, I32 = torch.float32, torch.float64, torch.int32
WARMUP_DEFAULT = 30_000

_inited_devices = set()


def ensure_device(device) -> torch.device:
    """Load the library and upload per-device tables once."""
    dev = torch.device(device)
    if dev.type != "cuda":
        raise RuntimeError("the mixgraph B200 engine runs on CUDA devices only (no CPU fallback)")
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    dev = torch.device("cuda", idx)
    if idx in _inited_devices:
        return dev
    L = lib()
    specs, wss, _ = reverb_tables()
    spec_arr = np.ascontiguousarray(np.stack([specs.real, specs.imag], axis=-1))
    wss_arr = np.ascontiguousarray(wss)
    with torch.cuda.device(idx):
        check(L.mgb_init(spec_arr.ctypes.data, wss_arr.ctypes.data, stream_ptr()), "mgb_init")
        torch.cuda.synchronize()
    _inited_devices.add(idx)
    return dev


def capture_graph(body, device):
    """Capture ``body`` into a CUDA graph on a side stream.

    torch.cuda.graph's context manager empties the device and pinned-host caches
    before every capture (~60 ms each); a pruning search re-captures its engines
    every round, so capture here without that.  With concurrent song searches
    the capture runs alone (``HostTurns``): no other thread's CUDA call may land
    inside it."""
    turns = getattr(_host, "lock", None)
    if turns is not None:
        turns.begin_capture()
    try:
        g = torch.cuda.CUDAGraph()
        s = own_stream(device, "capture")
        s.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(s):
            g.capture_begin(capture_error_mode="thread_local")
            try:
                body()
            finally:
                g.capture_end()
        torch.cuda.current_stream(device).wait_stream(s)
    finally:
        if turns is not None:
            turns.end_capture()
    return g


class HostTurns:
    """Host turns of concurrent song searches (songs.search_songs): any number of
    threads issue GPU work at once, a graph capture runs alone.  A thread holds a
    turn while it runs and gives it up only while blocked on its own stream
    (``host_wait``), so a capture waits for every other thread to reach such a
    wait (unguarded, other threads' pinned allocations invalidated captures)."""

    def __init__(self):
        self.cv = threading.Condition()
        self.active = 0        # threads holding a turn
        self.capturing = False
        self.waiting = 0       # captures waiting to start (they go first)

    def acquire(self):
        with self.cv:
            while self.capturing or self.waiting:
                self.cv.wait()
            self.active += 1

    def release(self):
        with self.cv:
            self.active -= 1
            self.cv.notify_all()

    def begin_capture(self):  # the caller holds a turn
        with self.cv:
            self.active -= 1
            self.waiting += 1
            self.cv.notify_all()
            while self.capturing or self.active:
                self.cv.wait()
            self.waiting -= 1
            self.capturing = True

    def end_capture(self):
        with self.cv:
            self.capturing = False
            self.active += 1
            self.cv.notify_all()


_host = threading.local()


def host_wait(obj) -> None:
    """``obj.synchronize()`` (a stream or event), giving up the host turn meanwhile
    when searches run concurrently (a pending capture can start).

    A stream is waited on through an event recorded while this thread still
    holds its turn: synchronising an event is legal while another thread
    captures a graph, synchronising a stream that capture reaches is not."""
    lk = getattr(_host, "lock", None)
    if lk is None:
        obj.synchronize()
        return
    if isinstance(obj, torch.cuda.Stream):
        ev = torch.cuda.Event()
        ev.record(obj)
        obj = ev
    lk.release()
    try:
        obj.synchronize()
    finally:
        lk.acquire()


_own_streams = {}
# stream priority per role with MGB_STREAM_PRIORITY=1: the captured step's critical path
# high, its side work low.  Off by default: measured 442 vs 446 steps/s.
_ROLE_PRIORITY = {"capture": 1, "side": -1, "main": 1}


def own_stream(device, role: str) -> torch.cuda.Stream:
    """A stream owned by the calling host thread for ``role`` (created once by
    ``mgb_stream_create`` and reused).  torch.cuda.Stream() hands out streams
    round-robin from a pool shared by all threads, so two concurrent song
    searches could otherwise end up on one stream while one of them captures."""
    dev = torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    key = (threading.get_ident(), idx, role)
    s = _own_streams.get(key)
    if s is None:
        prio = _ROLE_PRIORITY.get(role, 0) if os.environ.get("MGB_STREAM_PRIORITY", "0") == "1" else 0
        with torch.cuda.device(idx):
            raw = lib().mgb_stream_create_priority(prio)
        if not raw:
            raise _lib.DeviceError("mgb_stream_create failed")
        s = _own_streams[key] = torch.cuda.ExternalStream(raw, device=torch.device("cuda", idx))
    return s


def stream_ptr():
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))


# torch.cuda.current_stream() / torch.cuda.stream() resolve the device index
# through several Python layers on every call (env lookups, availability
# checks): ~20 % of a song search's host time under cProfile.  These do the same for the
# current device straight through the torch._C stream registry.
def current_stream() -> torch.cuda.Stream:
    sid, di, dt = torch._C._cuda_getCurrentStream(torch._C._cuda_getDevice())
    return torch.cuda.Stream(stream_id=sid, device_index=di, device_type=dt)


class on_stream:
    """``with torch.cuda.stream(s)`` for a stream on the current device."""
    __slots__ = ("s", "prev", "ctx")

    def __init__(self, s):
        self.s = s

    def __enter__(self):
        s = self.s
        if s.device_index != torch._C._cuda_getDevice():
            self.ctx = torch.cuda.stream(s)
            return self.ctx.__enter__()
        self.ctx = None
        self.prev = torch._C._cuda_getCurrentStream(s.device_index)
        torch._C._cuda_setStream(stream_id=s.stream_id, device_index=s.device_index, device_type=s.device_type)

    def __exit__(self, *exc):
        if self.ctx is not None:
            return self.ctx.__exit__(*exc)
        sid, di, dt = self.prev
        torch._C._cuda_setStream(stream_id=sid, device_index=di, device_type=dt)


def ptr(t: torch.Tensor, elem_offset: int = 0) -> int:
    return t.data_ptr() + elem_offset * t.element_size()


def dev_ptr_array(ptrs, device) -> torch.Tensor:
    return torch.tensor(np.asarray(ptrs, dtype=np.int64), dtype=torch.int64, device=device)


# ---------------------------------------------------------------------------
# parameters: one flat float64 vector  [e | c | n | s | g | d | r | raw_w]


class ParamLayout:
    def __init__(self, graph: MixGraph):
        self.rows = {t: len(graph.nodes_of_type(t)) for t in PROCESSOR_TYPES}
        self.off = {}
        o = 0
        for t in PROCESSOR_TYPES:
            self.off[t] = o
            o += self.rows[t] * PARAM_COUNTS[t]
        self.w_off = o
        self.P = len(graph.processor_nodes())
        self.n = o + self.P

    def pack(self, params) -> np.ndarray:
        flat = np.empty(self.n, dtype=np.float64)
        for t in PROCESSOR_TYPES:
            a = np.asarray(params.params[t], dtype=np.float64).reshape(-1)
            flat[self.off[t]:self.off[t] + a.size] = a
        flat[self.w_off:] = np.asarray(params.raw_weights, dtype=np.float64)
        return flat

    def unpack_into(self, flat: np.ndarray, params) -> None:
        for t in PROCESSOR_TYPES:
            n = self.rows[t] * PARAM_COUNTS[t]
            params.params[t] = flat[self.off[t]:self.off[t] + n].reshape(self.rows[t], PARAM_COUNTS[t]).copy()
        params.raw_weights = flat[self.w_off:].copy()

    def split(self, flat: np.ndarray) -> dict:
        out = {t: flat[self.off[t]:self.off[t] + self.rows[t] * PARAM_COUNTS[t]]
               .reshape(self.rows[t], PARAM_COUNTS[t]) for t in PROCESSOR_TYPES}
        out["w"] = flat[self.w_off:]
        return out


# ---------------------------------------------------------------------------
# render plan


class _Level:
    __slots__ = ("step", "tag", "B", "struct", "keep", "bus", "fanouts")


class RenderPlan:
    """Device plan of ``execute_batched`` for one (graph, schedule, L)."""

    def __init__(self, graph: MixGraph, schedule: Schedule | None, L: int, device,
                 params_flat: torch.Tensor, grads_flat: torch.Tensor | None, layout: ParamLayout,
                 backward: bool = True):
        self.device = ensure_device(device)
        dev = self.device
        if schedule is None:
            schedule = schedule_for(graph)
        elif schedule.plans is None:
            schedule = plan_indices(graph, schedule)
        self.schedule = schedule
        self.graph = graph
        self.L = L = int(L)
        self.layout = layout
        self.params = params_flat
        self.grads = grads_flat
        self.K = len(schedule.subsets[0])
        self.P = layout.P
        Ld = lib()
        inputs = graph.nodes_of_type("i")
        in_row = {v: i for i, v in enumerate(inputs)}
        self.input_rows = [in_row[v] for v in schedule.subsets[0]]
        self.stems = torch.zeros((len(inputs), 2, L), dtype=F32, device=dev)
        self.w = torch.zeros(max(self.P, 1), dtype=F64, device=dev)
        self.mask = torch.ones(max(self.P, 1), dtype=F64, device=dev)
        self.gw = torch.zeros(max(self.P, 1), dtype=F64, device=dev)
        self.greg = torch.zeros((), dtype=F64, device=dev)
        nsteps = len(schedule.subsets)
        self.outs = [None] * nsteps
        self.gus = [None] * nsteps
        n_reg = sum(len(schedule.subsets[s]) for s in range(1, nsteps)
                    if schedule.type_sequence[s] in "erd")
        self.reg = torch.zeros(max(n_reg, 1), dtype=F64, device=dev)
        self.n_reg = n_reg
        self._keep = []  # device tensors referenced by raw pointers

        def row_ptr(step, row):
            if step == 0:
                return ptr(self.stems, self.input_rows[row] * 2 * L)
            return ptr(self.outs[step], row * 2 * L)

        # ---- forward structures
        self.levels = []
        reg_off = 0
        for s in range(1, nsteps):
            plan = schedule.plans[s]
            tag = schedule.type_sequence[s]
            B = plan.batch
            self.outs[s] = torch.empty((B, 2, L), dtype=F32, device=dev)
            lv = _Level()
            lv.step, lv.tag, lv.B, lv.fanouts = s, tag, B, []
            lv.keep = []
            srcs = [row_ptr(*g) for g in plan.gather]
            if tag in KERNEL_TYPES:
                u_rows = dev_ptr_array(srcs, dev)
                prow = torch.tensor(np.asarray(schedule.type_perm[tag])[plan.pslice], dtype=I32, device=dev)
                widx = torch.tensor(np.asarray(plan.weight_idx), dtype=I32, device=dev)
                ws_bytes = int(Ld.mgb_level_workspace(tag.encode(), B, L))
                ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
                ybar = torch.empty((B, 2, L), dtype=F32, device=dev) if tag in "erd" else None
                aux = torch.empty((B, L), dtype=F32, device=dev) if tag in "cn" else None
                # dL/du of a level reading only the stems (step 1) has no consumer: not computed
                gu = torch.empty((B, 2, L), dtype=F32, device=dev) if backward and s > 1 else None
                self.gus[s] = gu
                st = MgbLevel()
                st.tag = tag.encode()
                st.B, st.L = B, L
                st.u_rows = ptr(u_rows)
                st.bank = ptr(self.params, layout.off[tag])
                st.prow, st.widx = ptr(prow), ptr(widx)
                st.w = ptr(self.w)
                st.greg = ptr(self.greg)
                st.y = ptr(self.outs[s])
                st.ybar = ptr(ybar) if ybar is not None else None
                st.aux = ptr(aux) if aux is not None else None
                if tag in "erd":
                    st.reg = ptr(self.reg, reg_off)
                    reg_off += B
                st.gu = ptr(gu) if gu is not None else None
                st.gbank = ptr(self.grads, layout.off[tag]) if self.grads is not None else None
                st.gw = ptr(self.gw)
                st.ws, st.ws_bytes = ptr(ws), ws_bytes
                lv.struct = st
                lv.keep = [u_rows, prow, widx, ws, ybar, aux, gu]
                lv.bus = None
            else:
                seg = plan.segments if plan.segments is not None else np.arange(B)
                counts = np.bincount(np.asarray(seg), minlength=B)
                seg_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
                in_rows = dev_ptr_array(srcs, dev)
                seg_t = torch.tensor(seg_off, dtype=I32, device=dev)
                lv.bus = (in_rows, seg_t, B)
                lv.struct = None
                lv.keep = [in_rows, seg_t]
            self.levels.append(lv)
        # the output level: one row for a graph, one per song for a union of song consoles
        # (batch.SongBatch); ys (n_out, 2, L), y its first row
        self.ys = self.outs[nsteps - 1]
        self.n_out = len(schedule.subsets[nsteps - 1])
        self.y = self.ys[0]
        # processor index -> position of its level in self.levels (incremental re-render)
        self.proc_level = np.zeros(max(self.P, 1), dtype=np.int64)
        for i, s in enumerate(range(1, nsteps)):
            if schedule.type_sequence[s] in KERNEL_TYPES:
                self.proc_level[np.asarray(schedule.plans[s].weight_idx, dtype=np.int64)] = i

        # ---- backward gradient routing
        self.dYs = torch.zeros((self.n_out, 2, L), dtype=F32, device=dev) if backward else None
        self.dY = self.dYs[0] if backward else None
        if backward:
            consumers = {}
            for s in range(1, nsteps):
                plan = schedule.plans[s]
                seg = plan.segments if plan.segments is not None else np.arange(len(plan.gather))
                for i, g in enumerate(plan.gather):
                    consumers.setdefault(tuple(g), []).append((s, int(seg[i])))
            gptr = {(nsteps - 1, r): ptr(self.dYs, r * 2 * L) for r in range(self.n_out)}
            fan_bufs = {}
            for s in range(nsteps - 2, 0, -1):
                tag = schedule.type_sequence[s]
                lv = self.levels[s - 1]
                rows = []
                for r in range(len(schedule.subsets[s])):
                    contrib = []
                    for (cs, cr) in consumers.get((s, r), []):
                        if schedule.type_sequence[cs] in KERNEL_TYPES:
                            contrib.append(ptr(self.gus[cs], cr * 2 * L))
                        else:
                            contrib.append(gptr[(cs, cr)])
                    if len(contrib) == 1:
                        gptr[(s, r)] = contrib[0]
                    else:
                        buf = torch.empty((2, L), dtype=F32, device=dev)
                        fan_bufs[(s, r)] = buf
                        src = dev_ptr_array(contrib, dev)
                        off = torch.tensor([0, len(contrib)], dtype=I32, device=dev)
                        lv.fanouts.append((src, off, buf))
                        gptr[(s, r)] = ptr(buf)
                    rows.append(gptr[(s, r)])
                if tag in KERNEL_TYPES:
                    gy = dev_ptr_array(rows, dev)
                    lv.struct.gy_rows = ptr(gy)
                    lv.keep.append(gy)
            self._fan_bufs = fan_bufs

    # -- launches ---------------------------------------------------------
    def set_stems(self, stems):
        """Copy (K, 2, L) stems (numpy / torch, any device) into the static input buffer."""
        t = stems if torch.is_tensor(stems) else torch.from_numpy(np.ascontiguousarray(stems))
        if t.shape[-1] != self.L:
            raise LengthMismatch(f"plan is built for L={self.L}, got {t.shape[-1]}")
        self.stems.copy_(t.to(dtype=F32), non_blocking=True)

    def prepare(self, side=None):
        """Forward phase 1 of every e/r/d/c/n level (FIR synthesis, ballistics
        parameter blocks; params only).

        With ``side`` (a torch stream) the work is enqueued there and one event
        per level is returned for ``forward`` to wait on; else it runs inline."""
        L = lib()
        events = {}
        if side is None:
            sp = stream_ptr()
            for lv in self.levels:
                if lv.struct is not None and lv.tag in "erdcn":
                    check(L.mgb_level_forward_phase(ctypes.byref(lv.struct), 1, sp), f"level {lv.tag} prepare")
            return events
        side.wait_stream(current_stream())
        with on_stream(side):
            sp = stream_ptr()
            for lv in self.levels:
                if lv.struct is not None and lv.tag in "erdcn":
                    check(L.mgb_level_forward_phase(ctypes.byref(lv.struct), 1, sp), f"level {lv.tag} prepare")
                    ev = torch.cuda.Event()
                    ev.record(side)
                    events[lv.step] = ev
        return events

    def forward(self, use_mask: bool, prepared=None, norms="inline", start=0):
        """The render.  ``prepared``: None => run the FIR syntheses inline; a dict of
        events from ``prepare(side)`` => wait on them; True => already done.
        ``norms`` (forward phase 3, the gain-staging norms and reg of e/r/d levels):
        "inline", a torch stream to run them on (off the render chain; the caller
        joins it before the backward or reg), or None to skip (reg not needed).
        ``start``: first level to render; the outputs of earlier levels are reused
        as they are in the buffers (the caller guarantees they are current)."""
        L = lib()
        sp = stream_ptr()
        if prepared is None:
            self.prepare()
            prepared = True
        main = current_stream()
        if self.P:
            check(L.mgb_weights(ptr(self.params, self.layout.w_off), ptr(self.mask) if use_mask else None,
                                ptr(self.w), self.P, sp), "mgb_weights")
        for lv in self.levels[start:]:
            if lv.struct is not None:
                if isinstance(prepared, dict) and lv.step in prepared:
                    main.wait_event(prepared[lv.step])
                check(L.mgb_level_forward_phase(ctypes.byref(lv.struct), 2, sp), f"level {lv.tag} forward")
                if lv.tag in "erd" and norms is not None:
                    if norms == "inline":
                        check(L.mgb_level_forward_phase(ctypes.byref(lv.struct), 3, sp), f"level {lv.tag} norms")
                    else:
                        norms.wait_stream(main)
                        with on_stream(norms):
                            check(L.mgb_level_forward_phase(ctypes.byref(lv.struct), 3, stream_ptr()),
                                  f"level {lv.tag} norms")
            else:
                in_rows, seg, B = lv.bus
                check(L.mgb_bus_sum(ptr(in_rows), ptr(seg), ptr(self.outs[lv.step]), B, self.L, sp),
                      "mgb_bus_sum")

    def reg_total(self) -> torch.Tensor:
        return self.reg.sum()

    def backward(self, side=None):
        """Reverse level sweep.  With ``side`` each level's parameter-gradient phase
        (backward phase 2: gbank / gw reductions, FIR adjoints) runs there,
        overlapping the following levels; the caller must join
        (``current_stream().wait_stream(side)``) before reading the gradients."""
        L = lib()
        sp = stream_ptr()
        main = current_stream()
        sides = side if isinstance(side, (tuple, list)) else (side,)
        n = 0
        for lv in reversed(self.levels):
            for src, off, buf in lv.fanouts:
                check(L.mgb_bus_sum(ptr(src), ptr(off), ptr(buf), 1, self.L, sp), "fan-out sum")
            if lv.struct is None:
                continue
            if side is None:
                check(L.mgb_level_backward(ctypes.byref(lv.struct), sp), f"level {lv.tag} backward")
                continue
            check(L.mgb_level_backward_phase(ctypes.byref(lv.struct), 1, sp), f"level {lv.tag} backward")
            sd = sides[n % len(sides)]  # levels' parameter phases alternate over the side streams
            n += 1
            sd.wait_stream(main)
            with on_stream(sd):
                check(L.mgb_level_backward_phase(ctypes.byref(lv.struct), 2, stream_ptr()),
                      f"level {lv.tag} FIR adjoint")



# ---------------------------------------------------------------------------
# loss plan


_proj_dev = {}


def projection_device(device, n, cfg):
    """The banded mel x A-weight tables of one resolution on a device (immutable, shared)."""
    key = (str(device), n, cfg.sample_rate, cfg.mel_bins, float(cfg.mel_fmax), bool(cfg.a_weighting))
    hit = _proj_dev.get(key)
    if hit is None:
        tabs = projection_sparse(n, cfg.sample_rate, cfg.mel_bins, float(cfg.mel_fmax), bool(cfg.a_weighting))
        hit = _proj_dev[key] = [torch.from_numpy(a).to(device) for a in tabs]
    return hit


class LossPlan:
    """Device MRSTFT (mg/losses.py:104-170) for a fixed scored length Ls.

    ``backward=False`` (a trial's forward-only loss) skips the frame-adjoint buffers.
    ``batch`` > 1: that many independent signals (songs) per call, signal q's input,
    target and gradient pointers ``sig_stride`` floats after signal q-1's; ``loss``
    is then a (batch,) vector."""

    def __init__(self, cfg, Ls: int, device, backward: bool = True, batch: int = 1, sig_stride: int = 0):
        self.device = ensure_device(device)
        dev = self.device
        self.cfg = cfg
        self.Ls = Ls = int(Ls)
        sizes = tuple(cfg.fft_sizes)
        if len(sizes) > 8:
            raise ValueError("at most 8 resolutions")
        for n in sizes:
            if n & (n - 1) or not 256 <= n <= 8192:
                raise NotImplementedError(f"fft size {n}: power of two in [256, 8192] required")
        if Ls < 2:
            raise ValueError("the scored length must be at least 2 samples")
        if cfg.mel_bins > 128:
            raise NotImplementedError("mel_bins <= 128")
        st = MgbLoss()
        st.n_res = len(sizes)
        st.Ls = Ls
        gw = [cfg.weight_lr / 2, cfg.weight_lr / 2, cfg.weight_mid, cfg.weight_side]
        for i, v in enumerate(gw):
            st.group_w[i] = v
        self._keep = []
        nb = max(1, int(batch))
        if nb > 1 and sig_stride < Ls:
            raise ValueError("batched loss: sig_stride must be at least the scored length")
        st.batch, st.sig_stride = nb, int(sig_stride) if nb > 1 else 0
        self.batch = nb
        self.stats = torch.zeros(nb * len(sizes) * 16, dtype=F64, device=dev)
        self.loss = torch.zeros((nb,) if nb > 1 else (), dtype=F64, device=dev)
        st.stats, st.loss = ptr(self.stats), ptr(self.loss)
        for i, n in enumerate(sizes):
            hop = n // 4
            frames = 1 + Ls // hop
            dt = projection_device(dev, n, cfg)
            nm = cfg.mel_bins
            # every element is written (target / forward kernels) before it is read
            tmel = torch.empty((nb, frames, nm, 4), dtype=F64, device=dev)  # (frame, band, group)
            tlog = torch.empty_like(tmel)
            mel = torch.empty_like(tmel)
            part = torch.empty((nb, frames, 4, 3), dtype=F64, device=dev)
            gfr = torch.empty((nb, frames, 2, n), dtype=F32, device=dev) if backward else None
            r = st.res[i]
            r.n_fft, r.hop, r.frames, r.n_mels = n, hop, frames, nm
            (r.band_start, r.band_len, r.band_off, r.band_w,
             r.bin_start, r.bin_len, r.bin_band, r.bin_w) = [ptr(t) for t in dt]
            r.tmel, r.tlog, r.mel, r.part = ptr(tmel), ptr(tlog), ptr(mel), ptr(part)
            r.gframes = ptr(gfr) if gfr is not None else None
            self._keep += dt + [tmel, tlog, mel, part, gfr]
        self.struct = st

    def target(self, tl_ptr, tr_ptr):
        check(lib().mgb_mrstft_target(ctypes.byref(self.struct), tl_ptr, tr_ptr, stream_ptr()), "mrstft target")

    def forward(self, yl_ptr, yr_ptr):
        check(lib().mgb_mrstft_forward(ctypes.byref(self.struct), yl_ptr, yr_ptr, stream_ptr()),
              "mrstft forward")

    def backward(self, yl_ptr, yr_ptr, gl_ptr, gr_ptr):
        if not self.struct.res[0].gframes:
            raise RuntimeError("LossPlan built with backward=False")
        check(lib().mgb_mrstft_backward(ctypes.byref(self.struct), yl_ptr, yr_ptr, gl_ptr, gr_ptr,
                                        stream_ptr()), "mrstft backward")

    def launches(self, which: str) -> int:
        n = self.struct.n_res
        return n + 1


# ---------------------------------------------------------------------------
# train-step engine


class TrainEngine:
    """train_step (mg/optimizer.py:140-186) as one device program per graph version."""

    def __init__(self, graph: MixGraph, L: int, cfg, device="cuda", schedule=None, warmup_len=None,
                 use_graph=True):
        self.device = ensure_device(device)
        dev = self.device
        self.graph = graph
        self.cfg = cfg
        self.L = int(L)
        self.ws = int(cfg.warmup_len if warmup_len is None else warmup_len)
        if self.ws >= self.L:
            raise ValueError("segment must be longer than the warm-up exclusion")
        self.layout = lay = ParamLayout(graph)
        self.params = torch.zeros(lay.n, dtype=F64, device=dev)
        self.grads = torch.zeros(lay.n, dtype=F64, device=dev)
        self.m = torch.zeros(lay.n, dtype=F64, device=dev)
        self.v = torch.zeros(lay.n, dtype=F64, device=dev)
        self.plan = RenderPlan(graph, schedule, self.L, dev, self.params, self.grads, lay, backward=True)
        self.lossp = LossPlan(cfg.loss, self.L - self.ws, dev)
        self.target = torch.zeros((2, self.L), dtype=F32, device=dev)
        self.scalars = torch.zeros(8, dtype=F64, device=dev)
        self.scalars_host = torch.zeros(8, dtype=F64).pin_memory()
        self.vals = torch.zeros(4, dtype=F64, device=dev)        # loss, L_a, L_g, L_p
        self.vals_host = torch.zeros(4, dtype=F64).pin_memory()
        self.sparsity = torch.zeros((), dtype=F64, device=dev)
        self.reg_off = torch.tensor([0, self.plan.n_reg], dtype=I32, device=dev)  # all reg rows: one signal
        self.plan.greg.fill_(float(cfg.loss.gain_staging_weight))
        self.t = 0
        self.use_graph = use_graph
        self._graph = None
        self.d_rows = lay.rows["d"]
        self.side = own_stream(dev, "side")
        # the levels' backward parameter phases alternate over two side streams, so the
        # last levels' phases run side by side before the optimiser (config 1 +1.3 %,
        # config 2 unchanged; MG_SIDE2=0: one side stream)
        self.side2 = own_stream(dev, "side2") if os.environ.get("MG_SIDE2", "1") == "1" else None
        # sticky NonFiniteLoss flag of the current run (mgb_adamw_step); zeroed per run
        self.halt = torch.zeros((), dtype=F64, device=dev)

    # -- state ------------------------------------------------------------
    def load_params(self, params):
        self.params.copy_(torch.from_numpy(self.layout.pack(params)))

    def store_params(self, params):
        self.layout.unpack_into(self.params.cpu().numpy(), params)

    def reset_optimizer(self):
        self.m.zero_()
        self.v.zero_()
        self.t = 0

    # -- the device program --------------------------------------------------
    def _body(self):
        L, ws, P = self.L, self.ws, self.layout.P
        plan, lp = self.plan, self.lossp
        Ld = lib()
        main, side = current_stream(), self.side
        # side stream: FIR syntheses (params only), the warm-up part of dL/dy (read by the
        # level backward; the loss backward writes the rest), then the target spectra
        prepared = plan.prepare(side)
        with on_stream(side):
            if ws:  # the warm-up part of dL/dy (the loss backward writes the rest)
                check(Ld.mgb_zero(ptr(plan.dY), 4 * ws, stream_ptr()), "mgb_zero")
                check(Ld.mgb_zero(ptr(plan.dY, L), 4 * ws, stream_ptr()), "mgb_zero")
            lp.target(ptr(self.target, ws), ptr(self.target, L + ws))
            tev = torch.cuda.Event()
            tev.record(side)
        plan.forward(use_mask=False, prepared=prepared, norms=side)
        y = plan.y
        main.wait_event(tev)
        lp.forward(ptr(y, ws), ptr(y, L + ws))
        main.wait_stream(side)  # the levels' norms (read by the backward prologues)
        # loss assembly (read by the optimiser step only) on the side stream, off the path
        # from the loss forward into the backward sweep
        side.wait_stream(main)
        with on_stream(side):
            sp = stream_ptr()
            if P:
                check(Ld.mgb_sparsity(ptr(self.params, self.layout.w_off), P, ptr(self.sparsity), sp),
                      "mgb_sparsity")
            check(Ld.mgb_loss_assembly(ptr(lp.loss), ptr(plan.reg), ptr(self.reg_off), None, ptr(self.sparsity),
                                       ptr(self.scalars), float(self.cfg.loss.gain_staging_weight), 1,
                                       ptr(self.vals), None, sp), "mgb_loss_assembly")
        lp.backward(ptr(y, ws), ptr(y, L + ws), ptr(plan.dY, ws), ptr(plan.dY, L + ws))
        if self.side2 is not None:
            plan.backward((side, self.side2))
            main.wait_stream(self.side2)
        else:
            plan.backward(side)
        main.wait_stream(side)
        lay = self.layout
        check(Ld.mgb_adamw_step(ptr(self.params), ptr(self.grads), ptr(self.m), ptr(self.v), lay.n,
                                lay.off["d"], self.d_rows, lay.w_off, P, ptr(plan.gw), None,
                                ptr(self.scalars), ptr(self.vals), ptr(self.halt), stream_ptr()), "mgb_adamw_step")

    def grads_only(self, alpha_p=0.0):
        """Eager forward + backward without the optimiser (test hook).

        Returns (values, bank grads split by type (raw, before the delay rule), dL/dw)."""
        self.scalars.copy_(torch.tensor([0, 0, 0, 0, 0, 1, 1, float(alpha_p)], dtype=F64))
        L, ws, P = self.L, self.ws, self.layout.P
        plan, lp = self.plan, self.lossp
        self.grads.zero_()
        plan.forward(use_mask=False)
        y = plan.y
        lp.target(ptr(self.target, ws), ptr(self.target, L + ws))
        lp.forward(ptr(y, ws), ptr(y, L + ws))
        reg = plan.reg_total()
        plan.dY[:, :ws].zero_()
        lp.backward(ptr(y, ws), ptr(y, L + ws), ptr(plan.dY, ws), ptr(plan.dY, L + ws))
        plan.backward()
        torch.cuda.synchronize(self.device)
        values = {"L_a": float(lp.loss), "L_g": float(reg)}
        g = self.layout.split(self.grads.cpu().numpy())
        return values, g, plan.gw[:P].cpu().numpy().copy(), y.detach().cpu().numpy().copy()

    def launches_per_step(self) -> int:
        """Library kernels one step enqueues (counted by the C ABI over one eager step)."""
        if getattr(self, "_launches", None) is None:
            Ld = lib()
            snap = [self.params.clone(), self.m.clone(), self.v.clone(), self.halt.clone(), self.t]
            self._set_scalars(0.0)
            n0 = Ld.mgb_launch_count()
            self._body()
            self._launches = int(Ld.mgb_launch_count() - n0)
            current_stream().synchronize()
            self.params.copy_(snap[0])
            self.m.copy_(snap[1])
            self.v.copy_(snap[2])
            self.halt.copy_(snap[3])
            self.t = snap[4]
        return self._launches

    _RING = 64

    def _set_scalars(self, alpha_p):
        """Per-step [lr, b1, b2, eps, wd, c1, c2, alpha_p] -> device, from a ring of pinned
        slots: a slot is rewritten only after its previous async copy has executed."""
        c = self.cfg
        self.t += 1
        b1, b2 = c.betas
        if not hasattr(self, "_ring"):
            self._ring = torch.zeros((self._RING, 8), dtype=F64).pin_memory()
            self._ring_ev = [None] * self._RING
        i = self.t % self._RING
        if self._ring_ev[i] is not None:
            host_wait(self._ring_ev[i])
        self._ring[i].copy_(torch.tensor([c.lr, b1, b2, c.eps, c.weight_decay, 1.0 - b1 ** self.t,
                                          1.0 - b2 ** self.t, float(alpha_p)], dtype=F64))
        self.scalars.copy_(self._ring[i], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._ring_ev[i] = ev

    def step_async(self, alpha_p=0.0):
        """Enqueue one full train step (inputs already in plan.stems / self.target)."""
        self._set_scalars(alpha_p)
        if not self.use_graph:
            self._body()
            return
        if self._graph is None:
            # warm-up run outside capture (sets function attributes, JIT, allocations)
            s = own_stream(self.device, "warm")
            s.wait_stream(current_stream())
            with torch.cuda.stream(s):
                snap = [self.params.clone(), self.m.clone(), self.v.clone(), self.halt.clone()]
                self._body()
                self.params.copy_(snap[0])
                self.m.copy_(snap[1])
                self.v.copy_(snap[2])
                self.halt.copy_(snap[3])
            current_stream().wait_stream(s)
            current_stream().synchronize()  # not device-wide: other songs may be capturing
            self._graph = capture_graph(self._body, self.device)
        self._graph.replay()

    def read_values(self):
        self.vals_host.copy_(self.vals, non_blocking=True)
        host_wait(current_stream())
        v = self.vals_host.tolist()
        return {"loss": v[0], "L_a": v[1], "L_g": v[2], "L_p": v[3]}


class EvalEngine:
    """Forward-only masked render + MRSTFT over a fixed eval set (mg/pruning.py:99-123).

    Long segments (or a single one) get a render plan each, stems loaded once,
    and eager engines (the pruning passes') re-render them incrementally: a
    trial whose mask differs from the segment's previous render only in
    processors of level k and later starts the render at level k, the earlier
    levels' outputs being the same values (trial engine).  Several
    short segments share one plan (built once per round, ~10 ms per plan)."""

    INCREMENTAL_MIN_L = 200_000  # segments at least this long get a plan each

    def __init__(self, graph: MixGraph, segments, warmup_len, loss_cfg, device="cuda", params=None,
                 use_graph=True):
        self.device = ensure_device(device)
        dev = self.device
        self.graph = graph
        self.layout = lay = ParamLayout(graph)
        self.params = torch.zeros(lay.n, dtype=F64, device=dev)
        self._packed = None      # host copy of the loaded parameter vector
        self._prep_dirty = True  # FIR syntheses / ballistics blocks stale (eager mode)
        if params is not None:
            self.load_params(params)
        L = segments[0][0].shape[-1]
        self.L, self.ws = L, int(warmup_len)
        schedule = schedule_for(graph)
        # Several short segments share one plan (a plan costs ~10 ms to build and an
        # engine lives for one pruning round); otherwise each segment keeps its own
        # plan, so its level outputs persist between trials for incremental renders.
        self.shared = len(segments) > 1 and L < self.INCREMENTAL_MIN_L
        self.plans, self.losses, self._last_mask, self.seg_stems = [], [], [], []
        for stems, target in segments:
            st = torch.as_tensor(np.asarray(stems), dtype=F32).to(dev)
            if not self.shared or not self.plans:
                plan = RenderPlan(graph, schedule, L, dev, self.params, None, lay, backward=False)
                plan.set_stems(st)
                self.plans.append(plan)
            self.seg_stems.append(st)
            lp = LossPlan(loss_cfg, L - self.ws, dev, backward=False)
            t = torch.as_tensor(np.asarray(target), dtype=F32).to(dev).contiguous()
            lp.target(ptr(t, 0), ptr(t, t.shape[-1]))
            self.losses.append((lp, t))
            self._last_mask.append(None)
        self.plan = self.plans[0]
        self.acc = torch.zeros(len(segments), dtype=F64, device=dev)
        self.mask_host = torch.ones(max(lay.P, 1), dtype=F64).pin_memory()
        self.acc_host = torch.zeros(len(segments), dtype=F64).pin_memory()
        self.use_graph = use_graph
        self._graph = None
        self._mask_np = None

    def load_params(self, params):
        packed = self.layout.pack(params)
        if self._packed is not None and np.array_equal(packed, self._packed):
            return  # a pruning pass evaluates many masks on the same parameters
        self._packed = packed.copy()
        self.params.copy_(torch.from_numpy(packed))
        self._prep_dirty = True

    def _body(self):
        L, ws = self.L, self.ws
        # FIR syntheses (parameters only); an eager engine redoes them only when the
        # parameters changed (a captured graph always includes them)
        full = self.use_graph or self._prep_dirty
        if full:
            for plan in self.plans:
                plan.prepare()
        for i in range(len(self.losses)):
            plan = self.plans[0 if self.shared else i]
            start = 0
            if self.shared:
                plan.stems.copy_(self.seg_stems[i])
            elif not full and self._mask_np is not None and self._last_mask[i] is not None:
                changed = np.nonzero(self._mask_np != self._last_mask[i])[0]
                start = int(plan.proc_level[changed].min()) if changed.size else len(plan.levels)
            plan.forward(use_mask=True, prepared=True, norms=None, start=start)  # eval_loss is the audio loss only
            if not self.use_graph and not self.shared:
                self._last_mask[i] = None if self._mask_np is None else self._mask_np.copy()
            lp, _ = self.losses[i]
            lp.forward(ptr(plan.y, ws), ptr(plan.y, L + ws))
            self.acc[i].copy_(lp.loss)
        self._prep_dirty = False

    def run_async(self, mask):
        m = np.asarray(mask, dtype=np.float64)
        self.mask_host[: len(m)].copy_(torch.from_numpy(m))
        self._mask_np = np.ones(self.mask_host.numel())
        self._mask_np[: len(m)] = m
        for plan in self.plans:
            plan.mask.copy_(self.mask_host, non_blocking=True)
        if not self.use_graph:
            self._body()
            return
        if self._graph is None:
            s = own_stream(self.device, "warm")
            s.wait_stream(current_stream())
            with torch.cuda.stream(s):
                self._body()
            current_stream().wait_stream(s)
            current_stream().synchronize()  # not device-wide: other songs may be capturing
            self._graph = capture_graph(self._body, self.device)
        self._graph.replay()

    def loss(self, mask) -> float:
        self.run_async(mask)
        self.acc_host.copy_(self.acc, non_blocking=True)
        host_wait(current_stream())
        # per-segment float() then mean, as mg/pruning.py:120-123
        total = 0.0
        for v in self.acc_host.tolist():
            total += float(v)
        return total / len(self.seg_stems)
