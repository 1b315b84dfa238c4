"""World-size-2 gloo test of the song-sharded driver's host logic:
each rank runs its LPT share of songs, results are gathered once on rank 0."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_15948_b200.songs import assign_lpt, desk_specs, gather_results, run_rank, song_costs, song_result
    specs = desk_specs(10, seed=1, length=1000)
    mine = assign_lpt(song_costs(specs), world)[rank]

    def run_song(spec):  # the device search replaced by a deterministic pruning of the song's console
        graph, params, state, rep = _fake_search(spec)
        res = song_result(spec, graph, params, state, rep, 0.0)
        res["rank"] = rank
        return res

    res = run_rank(specs, mine, run_song)
    merged = gather_results(res, rank, world, dist)
    if rank == 0:
        out.put(merged)
    dist.barrier()
    dist.destroy_process_group()


def _fake_search(spec):
    """A song's console pruned by a seeded rule, with its PruneState / PruneReport."""
    import numpy as np

    from paper_2509_15948_b200.console import SessionManifest, TrackEntry, build_console, init_params
    from paper_2509_15948_b200.graph import PROCESSOR_TYPES, bypass_remove
    from paper_2509_15948_b200.pruning import PruneReport, PruneState, TrialRecord
    man = SessionManifest([TrackEntry(f"t{k}.wav", f"t{k}", f"bus{k % spec.subgroups}")
                           for k in range(spec.tracks)], "m.wav")
    graph, zeros = build_console(man)
    params = init_params(zeros, spec.index)
    procs = graph.processor_nodes()
    rng = np.random.default_rng(spec.index)
    drop = sorted(int(i) for i in rng.choice(len(procs), size=len(procs) // 3, replace=False))
    counts = {t: len(graph.nodes_of_type(t)) for t in PROCESSOR_TYPES}
    state = PruneState(alive=np.ones(len(procs), dtype=bool), la_min=1.0, tolerance=0.02)
    state.alive[drop] = False
    state.ledger.append(TrialRecord(1, "bruteforce", tuple(drop[:2]), 0.99, 1.0, True))
    g2, p2 = bypass_remove(graph, params, {procs[i] for i in drop})
    pruned = {t: counts[t] - len(g2.nodes_of_type(t)) for t in PROCESSOR_TYPES}
    rep = PruneReport(1.0, 0.99, 0.99, 0.02, "hybrid", counts, pruned, 1, 0.0)
    return g2, p2, state, rep


@pytest.mark.timeout(120)
def test_two_rank_song_sharding_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=100)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2509_15948_b200.graph import deserialize, serialize
    from paper_2509_15948_b200.songs import desk_specs
    assert [r["song"] for r in got] == list(range(10))
    assert {r["rank"] for r in got} == {0, 1}
    for r, spec in zip(got, desk_specs(10, seed=1, length=1000)):
        # the gathered .mixgraph.json bytes round-trip and equal this process's own search
        g, p = deserialize(r["graph_json"].encode("utf-8"))
        g0, p0, state0, rep0 = _fake_search(spec)
        assert serialize(g, p) == serialize(g0, p0) == r["graph_json"].encode("utf-8")
        assert r["alive"] == [bool(a) for a in state0.alive]
        assert r["report"]["pruned_counts"] == rep0.pruned_counts and r["report"]["trial_count"] == 1
        assert r["report"]["pruning_ratio"] == rep0.pruning_ratio
