"""Full pruning searches on the device vs the REFERENCE's own search (SURVEY §8c
protocol item 4: fp32 full runs reported as consistency against the oracle graph).

Whole searches cannot match decision for decision between an fp32 device and
the float64 reference (the optimiser turns noise-level gradients into lr-sized
steps), so each song is searched twice from the same
console, parameters, session and seeds — by ``prune_song`` on the GPU and by the
reference's ``mixgraph.pruning.prune_song`` on the host (one worker process per
song) — and the final graphs are compared with the reference's own
``metrics.consistency_score`` (per-slot, per-type presence: accuracy / F1),
together with both searches' final losses and trial counts.

usage: python tools/full_run_consistency.py [--songs 8] [--out gpurun_out/consistency.json]
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

RECIPE = dict(tolerance_relative=0.02, mode="hybrid", iterations=4, console_steps=150, finetune_steps=20,
              eval_segments=2, eval_segment_seconds=57_000 / 30_000)
SEG = 57_000 / 30_000


def song_inputs(i):
    from workloads import SynthSpec, make_stems_f32
    k = (4, 6, 5, 4, 6, 5, 4, 6)[i % 8]
    s = 1 if k < 6 else 2
    L = 90_000
    stems = make_stems_f32(SynthSpec(tracks=k, subgroups=s, duration_seconds=L / 30000), 500 + i, L)
    return k, s, L, stems


def run_reference(i, q):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    from oracle import build_ref
    build_ref.load()
    from mixgraph import engine as E
    from mixgraph.console import SessionManifest, TrackEntry, build_console, init_params
    from mixgraph.graph import serialize
    from mixgraph.optimizer import Session, TrainConfig
    from mixgraph.pruning import PruneConfig, prune_song
    from mixgraph.scheduler import execute_reference
    k, s, L, stems = song_inputs(i)
    man = SessionManifest([TrackEntry(f"t{j}.wav", f"t{j}", f"bus{j % s}") for j in range(k)], "m.wav")
    graph, zeros = build_console(man)
    st64 = stems.astype(np.float64)
    target = np.asarray(E.value_of(execute_reference(graph, init_params(zeros, 77 + i), st64)[0]))
    target = target.astype(np.float32).astype(np.float64)
    cfg = PruneConfig(**RECIPE, seed=i, train=TrainConfig(segment_seconds=SEG, warmup_seconds=1.0, seed=i))
    t0 = time.perf_counter()
    g, p, state, rep, _ = prune_song(graph, init_params(zeros, i), Session(st64, target), cfg)
    q.put((i, serialize(g, p).decode(), target.astype(np.float32), float(rep.final_loss), rep.trial_count,
           time.perf_counter() - t0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--songs", type=int, default=8)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "consistency.json"))
    a = ap.parse_args()
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    procs = [ctx.Process(target=run_reference, args=(i, q)) for i in range(a.songs)]
    for pr in procs:
        pr.start()
    ref = {}
    for _ in procs:
        i, gj, target, fl, trials, wall = q.get()
        ref[i] = (gj, target, fl, trials, wall)
    for pr in procs:
        pr.join()
    # the device searches (after the host workers are done: no CUDA in forked children)
    import torch  # noqa: F401
    from oracle import build_ref
    build_ref.load()
    from mixgraph.graph import deserialize as rdeserialize
    from mixgraph.metrics import consistency_score
    from paper_2509_15948_b200.console import build_console, init_params
    from paper_2509_15948_b200.graph import serialize
    from paper_2509_15948_b200.optimizer import Session, TrainConfig
    from paper_2509_15948_b200.pruning import PruneConfig, prune_song
    from workloads import SynthSpec, manifest_for
    rows = []
    for i in range(a.songs):
        k, s, L, stems = song_inputs(i)
        graph, zeros = build_console(manifest_for(SynthSpec(tracks=k, subgroups=s)))
        gj, target, fl, trials, wall = ref[i]
        cfg = PruneConfig(**RECIPE, seed=i, train=TrainConfig(segment_seconds=SEG, warmup_seconds=1.0, seed=i))
        t0 = time.perf_counter()
        g, p, state, rep, _ = prune_song(graph, init_params(zeros, i), Session(stems, target), cfg)
        dev_s = time.perf_counter() - t0
        g_ref, _ = rdeserialize(gj.encode())
        g_dev, _ = rdeserialize(serialize(g, p))
        sc = consistency_score(g_ref, g_dev)
        rows.append({"song": i, "tracks": k, "subgroups": s, "micro": sc["micro"],
                     "processors_ref": len(g_ref.processor_nodes()), "processors_dev": len(g_dev.processor_nodes()),
                     "final_loss_ref": fl, "final_loss_dev": rep.final_loss, "trials_ref": trials,
                     "trials_dev": rep.trial_count, "search_s_ref": wall, "search_s_dev": dev_s})
        print(json.dumps(rows[-1]), flush=True)
    summary = {"recipe": RECIPE, "length": 90_000, "songs": rows,
               "mean_micro_f1": float(np.mean([r["micro"]["f1"] for r in rows])),
               "mean_micro_accuracy": float(np.mean([r["micro"]["accuracy"] for r in rows])),
               "what": "device fp32 prune_song vs the reference's float64 prune_song from identical inputs; "
                       "final graphs compared with the reference's metrics.consistency_score"}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(summary, open(a.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "songs"}))


if __name__ == "__main__":
    main()
