"""Config 5: songs searched per hour.

Each song is a full iterative-pruning search with the reference README's desk
recipe (pkg/README.md:54-58): console fit 600 steps, 12 hybrid rounds with 50
fine-tune steps each, 57,000-sample training segments, 4 eval segments of
57,000 samples, tolerance 0.02 relative.  Songs are synthetic consoles with
K ~ U{8..24} tracks and S = max(1, round(K/4)) subgroups at L = 441,000
(`songs.desk_specs`), the target rendered from a second parameter draw.

One process per GPU: under torchrun each rank takes its longest-processing-
time-first share of the songs (`songs.assign_lpt`) and the per-song reports
are gathered once on rank 0 (`songs.gather_results`); no collective runs
inside a search.  Input synthesis is outside the timed region; the timed
region is each rank's `prune_song` calls, max over ranks.

usage: python tools/songs_bench.py --songs 4   (or torchrun --nproc-per-node N ...)
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_15948_b200.scheduler import execute_batched  # noqa: E402
from paper_2509_15948_b200.songs import (assign_lpt, desk_specs, gather_results, search_songs,  # noqa: E402
                                         search_songs_lockstep, song_costs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--songs", type=int, default=4)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--iterations", type=int, default=12)
    ap.add_argument("--concurrent", type=int, default=1, help="songs in flight per GPU (threads + streams)")
    ap.add_argument("--lockstep", type=int, default=0,
                    help="search songs in lock-step groups of this size (batched training), 0 = off")
    ap.add_argument("--group-threads", type=int, default=1, help="lock-step groups in flight (host threads)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    def render(graph, tparams, stems):
        y, _ = execute_batched(graph, tparams, stems, device=dev)
        return y.cpu().numpy()

    specs = desk_specs(args.songs, seed=args.seed)
    mine = assign_lpt(song_costs(specs), world)[rank]
    inputs = {i: bench.make_inputs(1000 + specs[i].index, specs[i].tracks, specs[i].subgroups, specs[i].length,
                                   render) for i in mine}
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if args.lockstep:
        results = search_songs_lockstep(specs, mine, inputs, group=args.lockstep, iterations=args.iterations,
                                        device=dev, threads=args.group_threads)
    else:
        results = search_songs(specs, mine, inputs, concurrent=args.concurrent, iterations=args.iterations,
                               device=dev)
    torch.cuda.synchronize()
    wall = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(wall, op=dist.ReduceOp.MAX)
    merged = gather_results(results, rank, world, dist)
    if rank == 0:
        w = float(wall.item())
        print(json.dumps({"metric": "songs searched/hour (config 5 desk recipe)",
                          "value": len(merged) / w * 3600.0, "unit": "songs/hour", "n_gpus": world,
                          "songs": len(merged), "wall_s": w, "iterations": args.iterations, "concurrent": args.concurrent,
                          "lockstep": args.lockstep,
                          "lockstep_phase_s": __import__("paper_2509_15948_b200.batch", fromlist=["PHASE_S"]).PHASE_S,
                          "max_mem_gb": torch.cuda.max_memory_allocated(dev) / 1e9,
                          "reserved_gb": torch.cuda.memory_reserved(dev) / 1e9,
                          "per_song": [{k: v for k, v in r.items() if k not in ("graph_json", "ledger", "alive")}
                                       for r in merged]}))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
