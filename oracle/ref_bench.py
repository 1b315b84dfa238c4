"""CPU baseline: the REFERENCE's own train_step and eval trial timed on the host.

TEST / MEASUREMENT INFRASTRUCTURE ONLY: used by ``bench.py --impl reference``
and by the ``cpu_baseline`` leg of ``bench.py``; never by the product.

The reference (``mixgraph``, pure numpy/scipy, float64, single-threaded:
``scipy.fft`` runs with workers=1) is imported from its source tree or from
the archive ``oracle/build_ref.py`` ships to the GPU box.  Its CLI runs one
song per worker process (``mixgraph prune --threads N``, mg/cli.py:185-189);
the throughput arm here does the same with train steps: N forked worker
processes, each running whole ``train_step`` calls of the same console
(mg/optimizer.py:140-186), N = min(host cores, what the RAM allows at the
measured ~13.2 GB peak RSS of a config-2 step).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import platform
import time

import numpy as np

from . import build_ref

RSS_PER_PROC = {441_000: 14e9}  # bytes, measured peak RSS of one config-2 train_step (+ margin)


def cpu_info() -> dict:
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "os_cpu_count": os.cpu_count()}


def mem_available() -> float:
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    return float(line.split()[1]) * 1024
    except OSError:
        pass
    return 16e9


def ref_console(K, S, L, stems=None, seed=0, target=None):
    """Reference-built console, params (init_params(seed)), stems and target.

    ``stems`` / ``target`` given (e.g. the bench's arrays) are used as they are;
    otherwise the stems come from the reference's make_stems and the target is
    the reference's render of the console at init_params(seed + 1)."""
    mg = build_ref.load()
    if mg is None:
        raise RuntimeError("reference package unavailable (run oracle/build_ref.py where /root/reference exists)")
    from mixgraph import engine as E
    from mixgraph.console import SessionManifest, TrackEntry, build_console, init_params
    from mixgraph.scheduler import execute_batched, plan_indices, schedule_console
    from mixgraph.synth import SynthSpec, make_stems
    groups = [f"bus{j}" for j in range(S)]
    man = SessionManifest([TrackEntry(f"stems/track{k:02d}.wav", f"track{k:02d}", groups[k % S])
                           for k in range(K)], "target.wav")
    graph, zeros = build_console(man)
    sched = plan_indices(graph, schedule_console(graph))
    if stems is None:
        stems, _ = make_stems(SynthSpec(tracks=K, subgroups=S, duration_seconds=L / 30000), seed)
        stems = stems.astype(np.float32).astype(np.float64)[..., :L]
    stems = np.asarray(stems, dtype=np.float64)
    if target is None:
        target = np.asarray(E.value_of(execute_batched(graph, init_params(zeros, seed + 1), stems, sched)[0]))
    return graph, init_params(zeros, seed), stems, np.asarray(target, dtype=np.float64), sched


def time_train_steps(graph, params, stems, target, sched, steps) -> list:
    """Wall time of each of ``steps`` consecutive reference train_step calls (one process)."""
    from mixgraph.optimizer import TrainConfig, make_optimizer, train_step
    L = stems.shape[-1]
    cfg = TrainConfig(segment_seconds=L / 30000, warmup_seconds=1.0, steps=steps)
    p = params.copy()
    opt = make_optimizer(p, cfg)
    out = []
    for _ in range(steps):
        t0 = time.perf_counter()
        train_step(graph, p, (stems, target), cfg, opt, sched)
        out.append(time.perf_counter() - t0)
    return out


def time_eval_trial(graph, params, stems, target, sched) -> float:
    """One pruning trial segment: masked forward render + MRSTFT on a PreparedTarget."""
    from mixgraph import engine as E
    from mixgraph.losses import LossConfig, mrstft, prepare_target
    from mixgraph.scheduler import execute_batched
    prep = prepare_target(target[:, 30000:], LossConfig())
    mask = np.ones(len(graph.processor_nodes()))
    mask[0] = 0.0
    t0 = time.perf_counter()
    y, _ = execute_batched(graph, params, stems, sched, mask=mask)
    float(E.value_of(mrstft(y[:, 30000:], prep)))
    return time.perf_counter() - t0


_SHARED = {}


def _worker(i, steps, q, go):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)  # one core per worker process (BLAS/OpenMP pools would oversubscribe)
    g, p, st, tg, sc = _SHARED["inputs"]
    go.wait()
    t0 = time.perf_counter()
    times = time_train_steps(g, p, st, tg, sc, steps) if steps else []
    q.put((i, t0, time.perf_counter(), times))


def parallel_throughput(inputs, total_steps, workers) -> dict:
    """``total_steps`` reference train steps spread over ``workers`` forked processes that
    start together; steps/s = total_steps / (last finish - first start)."""
    _SHARED["inputs"] = inputs
    ctx = mp.get_context("fork")
    q, go = ctx.Queue(), ctx.Event()
    per = [total_steps // workers + (1 if i < total_steps % workers else 0) for i in range(workers)]
    procs = [ctx.Process(target=_worker, args=(i, per[i], q, go)) for i in range(workers) if per[i]]
    for pr in procs:
        pr.start()
    go.set()
    res = [q.get() for _ in procs]
    for pr in procs:
        pr.join()
    start, stop = min(r[1] for r in res), max(r[2] for r in res)
    times = [t for r in res for t in r[3]]
    return {"steps": sum(per), "workers": len(procs), "wall_s": stop - start,
            "value": sum(per) / (stop - start), "step_s_mean": float(np.mean(times)),
            "step_s_min": float(np.min(times))}


def default_workers(L) -> int:
    rss = RSS_PER_PROC.get(L, 14e9 * L / 441_000 + 1e9)
    return max(1, min(os.cpu_count() or 1, int(0.6 * mem_available() // rss)))
