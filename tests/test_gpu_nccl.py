"""The song-sharded driver's end-of-run gather over NCCL on the device.

One rank per GPU; this box has one GPU, so the NCCL group has world size 1 — the
gather_object path (pickled results staged through device tensors by NCCL) runs
for real, the sharding itself is covered by the gloo world-size-2 test."""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_results_gathered_over_nccl():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.distributed as dist
    from paper_2509_15948_b200.graph import deserialize, serialize
    from paper_2509_15948_b200.songs import assign_lpt, desk_specs, gather_results, run_rank, song_result
    from test_multiproc import _fake_search
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        assert dist.get_backend() == "nccl"
        specs = desk_specs(4, seed=2, length=1000)
        mine = assign_lpt([1.0] * 4, 1)[0]

        def run_song(spec):
            g, p, state, rep = _fake_search(spec)
            return song_result(spec, g, p, state, rep, 0.0)

        merged = gather_results(run_rank(specs, mine, run_song), 0, 1, dist)
        assert [r["song"] for r in merged] == list(range(4))
        for r, spec in zip(merged, specs):
            g, p = deserialize(r["graph_json"].encode())
            g0, p0, _, _ = _fake_search(spec)
            assert serialize(g, p) == serialize(g0, p0)
    finally:
        dist.destroy_process_group()
