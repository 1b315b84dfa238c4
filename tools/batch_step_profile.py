"""The lock-step trainer's batched step (G desk-recipe songs, 57,000-sample segments):
captured-step time, and with --eager N an eager run for an ncu launch list."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_15948_b200.batch import BatchTrainEngine, SongUnion  # noqa: E402
from paper_2509_15948_b200.optimizer import Session, TrainConfig, _EngineCfg, make_optimizer  # noqa: E402
from paper_2509_15948_b200.scheduler import execute_batched  # noqa: E402
from paper_2509_15948_b200.songs import DESK_SEGMENT, desk_specs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--songs", type=int, default=8)
ap.add_argument("--eager", type=int, default=0)
a = ap.parse_args()
dev = torch.device("cuda", 0)


def render(graph, tparams, stems):
    return execute_batched(graph, tparams, stems, device=dev)[0].cpu().numpy()


specs = desk_specs(a.songs, seed=0)
ins = [bench.make_inputs(1000 + s.index, s.tracks, s.subgroups, s.length, render) for s in specs]
cfg = TrainConfig(segment_seconds=DESK_SEGMENT / 30000, steps=1)
union = SongUnion([g for g, _, _, _ in ins])
eng = BatchTrainEngine(union, DESK_SEGMENT, _EngineCfg(make_optimizer(None, cfg), cfg), device=dev)
eng.load_params([p for _, p, _, _ in ins])
eng.set_sessions([Session(st, tg).on_device(dev) for _, _, st, tg in ins])
offs = [0] * a.songs
if a.eager:
    for _ in range(a.eager):
        eng.step_async(0.0, use_graph=False, offsets=offs)
    torch.cuda.synchronize()
    sys.exit(0)
for _ in range(5):
    eng.step_async(0.0, offsets=offs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    eng.step_async(0.0, offsets=offs)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"songs": a.songs, "tracks": sum(s.tracks for s in specs), "batched_step_ms": e0.elapsed_time(e1) / 50}))
