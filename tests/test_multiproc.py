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
    from paper_2509_15948_b200.songs import assign_lpt, desk_specs, gather_results, run_rank, song_costs
    specs = desk_specs(10, seed=1, length=1000)
    mine = assign_lpt(song_costs(specs), world)[rank]

    def run_song(spec):  # stand-in for prune_song on the device: a deterministic per-song result
        return {"graph_bytes": len(f"{spec.tracks}-{spec.subgroups}"), "rank": rank}

    res = run_rank(specs, mine, run_song)
    merged = gather_results(res, rank, world, dist)
    if rank == 0:
        out.put([(r["song"], r["rank"]) for r in merged])
    dist.barrier()
    dist.destroy_process_group()


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
    songs = [s for s, _ in got]
    ranks = {r for _, r in got}
    assert songs == list(range(10))
    assert ranks == {0, 1}
