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
    """Collect every rank's result list on rank 0 (one gather at the very end)."""
    if world == 1 or dist is None:
        return results
    box = [None] * world if rank == 0 else None
    dist.gather_object(results, box, dst=0)
    if rank != 0:
        return None
    merged = [r for part in box for r in part]
    return sorted(merged, key=lambda r: r["song"])


def songs_per_hour(results, wall_s):
    return len(results) / max(wall_s, 1e-9) * 3600.0


def spec_dict(spec):
    return asdict(spec)


__all__ = ["SongSpec", "song_costs", "assign_lpt", "desk_specs", "run_rank", "gather_results",
           "songs_per_hour", "spec_dict", "np"]
