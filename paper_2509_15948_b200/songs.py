"""Song-sharded multi-GPU search.

Songs are independent pruning searches, so the data-parallel unit is a whole
song: one process per GPU, songs assigned longest-processing-time-first by a
cost model, no collective inside any step.  Per-song results (the final
``.mixgraph.json`` bytes and the report) are gathered to rank 0 once at the
end with ``torch.distributed.gather_object`` (NCCL over NVLink on the GPU box,
gloo in the CPU tests).  This replaces the reference's process pool over
manifests (mg/cli.py:185-189).
"""

from __future__ import annotations

import heapq
import os
import time
from dataclasses import asdict, dataclass

import numpy as np


@dataclass
class SongSpec:
    index: int
    tracks: int
    subgroups: int
    length: int


def song_costs(specs):
    """Predicted cost ∝ (K + S) · L (render work per step)."""
    return [float((s.tracks + s.subgroups) * s.length) for s in specs]


def assign_lpt(costs, world):
    """Longest-processing-time-first: each song (cost-descending) goes to the least loaded rank.

    Deterministic: ties break on the lower rank, then the lower song index."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    out = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(x) for x in out]


def desk_specs(n_songs, seed=0, length=441_000, kmin=8, kmax=24):
    """Config 5 song list: K ~ U{kmin..kmax} from rng_for(seed, 'songs'), S = max(1, round(K/4))."""
    from .common import rng_for
    rng = rng_for(seed, "songs")
    ks = rng.integers(kmin, kmax + 1, size=n_songs)
    return [SongSpec(i, int(k), max(1, int(round(k / 4))), length) for i, k in enumerate(ks)]


def run_rank(specs, mine, run_song):
    """Run this rank's songs; ``run_song(spec) -> dict`` (JSON-serialisable)."""
    results = []
    for i in mine:
        t0 = time.perf_counter()
        res = run_song(specs[i])
        res["song"] = specs[i].index
        res["wall_s"] = time.perf_counter() - t0
        results.append(res)
    return results


def gather_results(results, rank, world, dist=None):
    """Collect every rank's result list on rank 0 (one gather at the very end; NCCL's
    gather_object when the process group is NCCL, also for a single rank)."""
    if dist is None or not dist.is_initialized():
        return results
    box = [None] * world if rank == 0 else None
    dist.gather_object(results, box, dst=0)
    if rank != 0:
        return None
    merged = [r for part in box for r in part]
    return sorted(merged, key=lambda r: r["song"])


DESK_SEGMENT = 57_000  # samples (1.9 "s" at the reference's 30 kHz constants)


def desk_prune_config(seed, iterations=12):
    """The reference README's desk search (pkg/README.md:54-58): console 600 steps, 12 hybrid
    rounds, 50 fine-tune steps, 1.9 s segments, 4 eval segments of 1.9 s, tolerance 0.02 relative."""
    from .optimizer import TrainConfig
    from .pruning import PruneConfig
    seg = DESK_SEGMENT / 30_000
    return PruneConfig(tolerance_relative=0.02, mode="hybrid", iterations=iterations, seed=seed,
                       console_steps=600, finetune_steps=50, eval_segments=4, eval_segment_seconds=seg,
                       train=TrainConfig(segment_seconds=seg, warmup_seconds=1.0, seed=seed))


def report_dict(rep) -> dict:
    """A PruneReport (mg/pruning.py:72-91) as plain JSON-able values, plus its derived ratio."""
    out = asdict(rep)
    out["pruning_ratio"] = rep.pruning_ratio
    return out


def song_result(spec, graph, params, state, rep, search_s, metrics=None) -> dict:
    """What one song's search hands to rank 0: the final ``.mixgraph.json`` bytes (the
    reference writer's exact format, mg/graph.py:276-293), the PruneReport, the
    surviving-processor mask, the trial ledger and the match metrics row (mg/cli.py:128-182
    writes the same artefacts per song)."""
    from .graph import serialize
    return {"song": spec.index, "tracks": spec.tracks, "subgroups": spec.subgroups, "search_s": search_s,
            "metrics": metrics,
            "trials": rep.trial_count, "pruning_ratio": rep.pruning_ratio, "console_loss": rep.console_loss,
            "final_loss": rep.final_loss, "report": report_dict(rep),
            "alive": [bool(a) for a in state.alive],
            "ledger": [(r.iteration, r.mode, [int(c) for c in r.candidates], float(r.loss), bool(r.accepted))
                       for r in state.ledger],
            "graph_json": serialize(graph, params).decode("utf-8")}


def search_song(spec, graph, params, stems, target, iterations=12, device="cuda"):
    """One song's full pruning search (``prune_song``) with the desk recipe; its JSON-able result."""
    from .optimizer import Session
    from .pruning import prune_song
    t0 = time.perf_counter()
    g, p, state, rep, _ = prune_song(graph, params, Session(stems, target), desk_prune_config(spec.index, iterations),
                                     device=device)
    return song_result(spec, g, p, state, rep, time.perf_counter() - t0, match_metrics(spec, g, p, stems, target, device))


def match_metrics(spec, graph, params, stems, target, device="cuda"):
    """The final graph rendered over the whole session and scored against the target on the
    device (mg/cli.py:164-170: match.wav + metrics.csv per song)."""
    from .metrics import render_match, song_metrics
    match = render_match(graph, params, stems, device=device)
    return song_metrics(f"song{spec.index:03d}", target, match, 30_000, device=device)


def search_songs_lockstep(specs, mine, inputs, group=4, iterations=12, device="cuda", threads=1):
    """This rank's songs in groups of ``group`` searched in lock-step (batch.prune_songs_lockstep):
    trials per song, every console fit and fine-tune of a group as ONE batched device program
    over the disjoint union of the group's consoles.  Songs are grouped costliest-first so a
    group's consoles are of similar size.  ``threads`` > 1 runs that many groups at once on
    host threads (one stream set each; engine builds and round bookkeeping of one group
    overlap the other groups' device work; measured slower on one B200: 5,369 vs 5,900
    songs/hour with 2 groups of 8 in flight, the lock-step programs already fill the GPU).
    Same results as searching the songs one by one."""
    from .batch import prune_songs_lockstep
    from .optimizer import Session
    order = sorted(mine, key=lambda i: (-song_costs([specs[i]])[0], i))
    groups = [order[g0:g0 + group] for g0 in range(0, len(order), group)]
    out = {}

    def run_group(ids):
        t0 = time.perf_counter()
        jobs = []
        for i in ids:
            graph, params, stems, target = inputs[i]
            jobs.append((graph, params, Session(stems, target), desk_prune_config(specs[i].index, iterations)))
        res = prune_songs_lockstep(jobs, device=device)
        dt = (time.perf_counter() - t0) / len(ids)
        for i, r in zip(ids, res):
            if isinstance(r, BaseException):
                raise r
            g, p, state, rep, _ = r
            _, _, stems, target = inputs[i]
            out[i] = song_result(specs[i], g, p, state, rep, dt,
                                 match_metrics(specs[i], g, p, stems, target, device))

    _run_on_threads(groups, run_group, threads, device)
    return [out[i] for i in mine]


def _run_on_threads(tasks, fn, threads, device, graph_min_steps=None):
    """fn(task) for every task, ``threads`` at a time on host threads that each own their
    CUDA streams; graph captures run alone (engine.HostTurns).  ``graph_min_steps``: the
    threads' train() calls replay a captured step from this many steps on."""
    if threads <= 1 or len(tasks) <= 1:
        for t in tasks:
            fn(t)
        return
    import threading

    import torch

    from . import engine
    dev = engine.ensure_device(device)
    queue, lock, errors = list(tasks), threading.Lock(), []
    turn = engine.HostTurns()

    def worker():
        torch.cuda.set_device(dev)
        stream = engine.own_stream(dev, "main")
        engine._host.lock = turn
        engine._host.graph_min_steps = graph_min_steps
        turn.acquire()
        try:
            with torch.cuda.stream(stream):
                while True:
                    with lock:
                        if not queue or errors:
                            break
                        task = queue.pop(0)
                    try:
                        fn(task)
                    except BaseException as e:  # surfaced on the calling thread
                        errors.append(e)
                        break
            engine.host_wait(stream)
        finally:
            engine._host.lock = engine._host.graph_min_steps = None
            turn.release()

    ths = [threading.Thread(target=worker, daemon=True) for _ in range(min(threads, len(tasks)))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errors:
        raise errors[0]


def search_songs(specs, mine, inputs, concurrent=1, iterations=12, device="cuda"):
    """Run this rank's songs, ``concurrent`` at a time on one GPU.

    A desk-recipe song trains on 57,000-sample segments, where one level
    launch fills only part of the 148 SMs; several songs in flight (one host
    thread and one CUDA stream each, songs taken costliest-first from a shared
    queue) let their kernels overlap.  Searches stay independent: each has its
    own engines, streams and graphs, and the results are the same as running
    the songs one after another.  The threads issue concurrently except around
    graph captures, which run alone (``engine.HostTurns``).  Returns the per-song summaries in ``mine``
    order."""
    order = sorted(mine, key=lambda i: (-song_costs([specs[i]])[0], i))
    out = {}

    def run(i):
        out[i] = search_song(specs[i], *inputs[i], iterations=iterations, device=device)

    # with songs in flight, fine-tunes replay a captured step too: fewer host launches per
    # step competing for the interpreter with the other songs' threads
    _run_on_threads(order if concurrent > 1 else list(mine), run, concurrent, device,
                    graph_min_steps=int(os.environ.get("MG_CONCURRENT_GRAPH_MIN_STEPS", "1")))
    return [out[i] for i in mine]


def songs_per_hour(results, wall_s):
    return len(results) / max(wall_s, 1e-9) * 3600.0


def spec_dict(spec):
    return asdict(spec)


__all__ = ["SongSpec", "song_costs", "assign_lpt", "desk_specs", "run_rank", "gather_results", "song_result",
           "search_songs_lockstep",
           "report_dict",
           "songs_per_hour", "spec_dict", "desk_prune_config", "search_song", "search_songs", "DESK_SEGMENT", "np"]
