"""Benchmark: console fwd+bwd train steps/s on B200 (BASELINE.json metric).

Workload: full console, 16 tracks + 4 subgroups
(140 processors, 161 nodes), L = 441,000 samples per channel ("10 s @ 44.1 kHz"
read as a sample count, processed with the reference's 30 kHz constants),
warm-up 30,000 samples excluded from the loss.  One step = render fwd + MRSTFT
fwd + full backward + delay rule + AdamW + projection (mg/optimizer.py:140-186).
Synthetic stems (mg/synth.py recipe, seed = rank), params init_params(seed),
target = the same console rendered at init_params(seed + 1).

value: device-resident inputs, CUDA-graph replays, CUDA events, max over ranks.
e2e:   the public ``train_segments`` with pinned host stems/target in per step, loss out
       (``train_step``, synchronous, reported beside it).
--impl reference: the float64 CPU oracle port (the reference is pure
numpy/scipy and cannot travel to the GPU box) timed on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "console fwd+bwd steps/s (16 trk, 10 s stereo); songs searched/hour at 1-8 B200"
K_TRACKS, S_GROUPS, L_SAMPLES, WARMUP = 16, 4, 441_000, 30_000


def b_step(L, K, S, P):
    """Design-neutral compulsory HBM bytes per step."""
    return 40 * L * P + 16 * L * (K + S) + 16 * L * (S + 1) + 32 * (L - WARMUP)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--song-concurrency", type=int, default=4,
                    help="songs searched concurrently per GPU (host threads + CUDA streams), with --song-lockstep 0")
    ap.add_argument("--song-lockstep", type=int, default=8,
                    help="songs per GPU searched in lock-step groups of this size: each group's training steps and "
                         "trials run as one batched device program (0: threads instead)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the BASELINE config 3 and 4 sub-lines (tools/configs_bench.py)")
    ap.add_argument("--songs", type=int, default=32,
                    help="config-5 desk-recipe pruning searches per GPU for songs/hour (0: skip)")
    ap.add_argument("--tracks", type=int, default=K_TRACKS)
    ap.add_argument("--subgroups", type=int, default=S_GROUPS)
    ap.add_argument("--length", type=int, default=L_SAMPLES)
    ap.add_argument("--eager-profile", type=int, default=0,
                    help="run N eager (non-graph) steps and exit: for ncu launch lists")
    ap.add_argument("--profile-level", default="",
                    help="e.g. d@step6: after one eager step, run only that level's forward+backward "
                         "(--eager-profile times) and exit: per-level ncu traffic")
    return ap.parse_args()


def make_inputs(seed, K, S, L, render_target):
    from paper_2509_15948_b200.console import build_console, init_params
    from workloads import SynthSpec, make_stems_f32, manifest_for
    spec = SynthSpec(tracks=K, subgroups=S, duration_seconds=L / 30000)
    stems = make_stems_f32(spec, seed, L)
    graph, zeros = build_console(manifest_for(spec))
    params = init_params(zeros, seed)
    tparams = init_params(zeros, seed + 1)
    target = render_target(graph, tparams, stems)
    return graph, params, stems, np.ascontiguousarray(target, dtype=np.float32)


class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.samples = []
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7 and f[0].isdigit():
                self.samples.append(f)

    def summary(self):
        if not getattr(self, "samples", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [int(f[0]) for f in self.samples]
        reasons = set()
        for f in self.samples:
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"),
                               f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(self.samples[0][1]),
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_baseline(K, S, L, stems, target, songs=None):
    """The reference's own train_step (numpy/scipy float64, one core) on the same
    console and inputs, and a derived CPU songs/hour for the config-5 desk recipe."""
    from oracle import ref_bench
    g, p, st, tg, sc = ref_console_timed = ref_bench.ref_console(K, S, L, stems=stems, target=target)
    dt = ref_bench.time_train_steps(g, p, st, tg, sc, 1)[0]
    out = {"value": 1.0 / dt, "unit": "steps/s", "cores": 1, "kind": "reference",
           "sample": f"1 reference train_step (mixgraph.optimizer.train_step, {K} trk + {S} sub, L={L}) "
                     "on one host core", "cpu": ref_bench.cpu_info()}
    del ref_console_timed
    if songs:
        out["songs_per_hour_derived"] = cpu_songs_per_hour(songs)
    return out


def cpu_songs_per_hour(songs):
    """Derived CPU songs/hour for the desk recipe: one measured reference
    train_step and one eval-trial segment of a 16 + 4 console at the desk segment length,
    scaled per song by (K+S)/20, times each song's measured trial count (from the GPU
    searches of the same songs), on N concurrent worker processes (mixgraph prune
    --threads N, mg/cli.py:185-189)."""
    from oracle import ref_bench
    from paper_2509_15948_b200.songs import DESK_SEGMENT
    g, p, st, tg, sc = ref_bench.ref_console(16, 4, DESK_SEGMENT)
    t_step = ref_bench.time_train_steps(g, p, st, tg, sc, 1)[0]
    t_trial = ref_bench.time_eval_trial(g, p, st, tg, sc)
    per_song = []
    for k, trials in zip(songs["tracks"], songs["trials"]):
        scale = (k + max(1, round(k / 4))) / 20.0
        per_song.append(scale * ((600 + 12 * 50) * t_step + (trials + 2) * 4 * t_trial))
    workers = min(os.cpu_count() or 1, max(1, int(0.6 * ref_bench.mem_available() // 2.5e9)))
    return {"value": workers * 3600.0 / float(np.mean(per_song)), "unit": "songs/hour", "kind": "derived",
            "workers": workers, "step_s": t_step, "trial_segment_s": t_trial,
            "how": "per song: (600 console + 12 x 50 fine-tune steps) x reference step + (trials + 2) x 4 "
                   "eval segments x reference trial, both measured here at 16 trk + 4 sub, 57,000 samples, "
                   "scaled by (K+S)/20; trials = the GPU searches' counts for the same songs; "
                   "N worker processes as mixgraph prune --threads N"}


def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if (torch.cuda.is_available() and args.impl == "ours") else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend, device_id=torch.device("cuda", local) if backend == "nccl" else None)
    return world, rank, local


def run_reference(args, world, rank):
    """The reference arm: the REFERENCE's own train_step (oracle/_ref archive of the
    unmodified mixgraph package) on this host's cores: args.steps steps of the same
    console spread over N forked worker processes, as its CLI spreads songs
    (mg/cli.py:185-189)."""
    if rank != 0:
        return
    from oracle import ref_bench
    try:
        inputs = ref_bench.ref_console(args.tracks, args.subgroups, args.length)
    except RuntimeError as exc:
        print(json.dumps({"impl": "reference", "unavailable": str(exc)}), flush=True)
        return
    workers = ref_bench.default_workers(args.length)
    res = ref_bench.parallel_throughput(inputs, args.steps, workers)
    v = res["value"]
    line = {"metric": METRIC, "value": v, "unit": "steps/s", "n_gpus": args.gpus, "steps": res["steps"],
            "warmup": 0, "ms_per_step": 1000.0 / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "config2: full console 16 trk + 4 sub, L=441000 (10 s @44.1k as samples)",
                       "tracks": args.tracks, "subgroups": args.subgroups, "length": args.length},
            "cpu_baseline": {"value": v, "unit": "steps/s", "cores": res["workers"], "kind": "reference",
                             "sample": f"{res['steps']} reference train_step calls (unmodified mixgraph "
                                       f"package, numpy/scipy float64) over {res['workers']} concurrent worker "
                                       f"processes, one core each; wall {res['wall_s']:.1f} s; mean step "
                                       f"{res['step_s_mean']:.2f} s (no warm-up: no JIT on this path)",
                             "cpu": ref_bench.cpu_info()},
            "e2e": {"value": v, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import torch
    import torch.distributed as dist

    from paper_2509_15948_b200.engine import TrainEngine
    from paper_2509_15948_b200.optimizer import (TrainConfig, _EngineCfg, make_optimizer, train_segments,
                                                 train_step)
    from paper_2509_15948_b200.scheduler import execute_batched

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    K, S, L = args.tracks, args.subgroups, args.length

    def render(graph, tparams, stems):
        y, _ = execute_batched(graph, tparams, stems, device=dev)
        return y.cpu().numpy()

    graph, params, stems, target = make_inputs(rank, K, S, L, render)
    cfg = TrainConfig(segment_seconds=L / 30000, steps=1)
    opt = make_optimizer(params, cfg, device=dev)
    eng = TrainEngine(graph, L, _EngineCfg(opt, cfg), device=dev, use_graph=not args.eager_profile)
    eng.load_params(params)
    if args.eager_profile and args.profile_level:
        import ctypes

        from paper_2509_15948_b200._lib import check, lib
        from paper_2509_15948_b200.engine import stream_ptr
        eng.plan.set_stems(stems)
        eng.target.copy_(torch.from_numpy(target))
        eng.grads_only()
        lv = next(lv for lv in eng.plan.levels if lv.struct is not None and f"{lv.tag}@step{lv.step}" == args.profile_level)
        Ld = lib()
        n0 = Ld.mgb_launch_count()
        for _ in range(args.eager_profile):
            check(Ld.mgb_level_forward(ctypes.byref(lv.struct), stream_ptr()), "fwd")
            check(Ld.mgb_level_backward(ctypes.byref(lv.struct), stream_ptr()), "bwd")
        torch.cuda.synchronize()
        per = (Ld.mgb_launch_count() - n0) // args.eager_profile
        print(json.dumps({"profile_level": args.profile_level, "reps": args.eager_profile, "launches_per_rep": per}))
        return
    if args.eager_profile:
        eng.plan.set_stems(stems)
        eng.target.copy_(torch.from_numpy(target))
        for _ in range(args.eager_profile):
            eng.step_async()
        torch.cuda.synchronize()
        print(json.dumps({"eager_profile_steps": args.eager_profile, "launches_per_step": eng.launches_per_step()}))
        return
    eng.plan.set_stems(stems)
    eng.target.copy_(torch.from_numpy(target))
    for _ in range(max(3, args.warmup)):
        eng.step_async()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record()
        for _ in range(args.steps):
            eng.step_async()
        stop.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(stop)
    t_local = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_max = float(t_local.item())
    ms_step = ms_max / args.steps
    value = world * args.steps / (ms_max / 1000.0)
    vals = eng.read_values()

    # per-level kernel-group timing (eager, CUDA events on the launching stream)
    level_ms = time_levels(eng, reps=3)
    # e2e through the public API with pinned host buffers
    st_pin = torch.from_numpy(stems).pin_memory()
    tg_pin = torch.from_numpy(target).pin_memory()
    opt2 = make_optimizer(params, cfg, device=dev)
    p2 = params.copy()
    train_step(graph, p2, (st_pin, tg_pin), cfg, opt2)  # builds + captures
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # (1) the streaming API: every step uploads its own segment (copy overlapped with the
    # previous step's compute) and reads its metrics back
    runs = []
    for _ in range(3):  # three timed runs of e2e_steps steps each; the median is reported
        t0 = time.perf_counter()
        train_segments(graph, p2, [(st_pin, tg_pin)] * args.e2e_steps, cfg, opt2)
        runs.append(time.perf_counter() - t0)
    e2e_s = statistics.median(runs)
    # (2) the synchronous single-step API, for reference
    t0 = time.perf_counter()
    for _ in range(max(3, args.e2e_steps // 4)):
        train_step(graph, p2, (st_pin, tg_pin), cfg, opt2)
    sync_s = (time.perf_counter() - t0) / max(3, args.e2e_steps // 4)
    e2e_t = torch.tensor([e2e_s, sync_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    sync_val = world / float(e2e_t[1].item())
    e2e_t = e2e_t[:1]
    e2e_val = world * args.e2e_steps / float(e2e_t.item())
    # one pruning trial (masked forward-only render + MRSTFT, mg/pruning.py:115-123) on the
    # same clip
    from paper_2509_15948_b200.engine import EvalEngine
    ev = EvalEngine(graph, [(stems, target)], WARMUP, cfg.loss, device=dev, params=params)
    mask = np.ones(eng.layout.P)
    for _ in range(3):
        ev.run_async(mask)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ev.run_async(mask)
    e1.record()
    torch.cuda.synchronize()
    trial_ms = e0.elapsed_time(e1) / 20
    # config 5: full pruning searches (desk recipe), this rank's LPT share of songs*world songs
    songs = None
    if args.songs > 0:
        from paper_2509_15948_b200.songs import (assign_lpt, desk_specs, gather_results, search_songs,
                                                 search_songs_lockstep, song_costs)
        specs = desk_specs(args.songs * world, seed=0)
        mine = assign_lpt(song_costs(specs), world)[rank]
        inputs = {i: make_inputs(1000 + specs[i].index, specs[i].tracks, specs[i].subgroups, specs[i].length,
                                 render) for i in mine}
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if args.song_lockstep > 0:
            res = search_songs_lockstep(specs, mine, inputs, group=args.song_lockstep, device=dev)
        else:
            res = search_songs(specs, mine, inputs, concurrent=args.song_concurrency, device=dev)
        torch.cuda.synchronize()
        sw = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(sw, op=dist.ReduceOp.MAX)
        res = gather_results(res, rank, world, dist if world > 1 else None)
        if rank == 0:
            songs = {"value": len(res) / float(sw.item()) * 3600.0, "unit": "songs/hour", "songs": len(res),
                     "wall_s": float(sw.item()), "recipe": "desk (pkg/README.md:54-58): console 600, 12 hybrid "
                     "rounds x 50 fine-tune, 57,000-sample segments, 4 eval segments, tau_rel 0.02",
                     "mode": (f"lock-step groups of {args.song_lockstep} (one batched device program per group "
                              "for training and for trials)") if args.song_lockstep > 0 else
                             f"{args.song_concurrency} songs in flight (threads + streams)",
                     "tracks": [r["tracks"] for r in res],
                     "trials": [r["trials"] for r in res],
                     "gathered": {"songs": len(res), "graph_json_bytes": sum(len(r["graph_json"]) for r in res),
                                  "what": "final .mixgraph.json + PruneReport + survivors + ledger per song, "
                                          "one gather_object to rank 0 (NCCL when N > 1)"}}
    # BASELINE config 1 (4 tracks + 1 subgroup, L = 132,300): launch-bound, CUDA-graph replays
    cfg1 = time_config(dev, 4, 1, 132_300, rank, render, steps=200, warmup=max(3, args.warmup))
    # BASELINE configs 3 (c/n-heavy, 32 trk, 1,323,000 samples) and 4 (e/r-heavy, 6-resolution loss)
    secondary = None
    if not args.no_secondary:
        import importlib.util
        spec_ = importlib.util.spec_from_file_location("configs_bench", os.path.join(ROOT, "tools", "configs_bench.py"))
        cb = importlib.util.module_from_spec(spec_)
        spec_.loader.exec_module(cb)
        secondary = {}
        for cid in (3, 4):
            r = cb.run(cid, 10, dev)
            secondary[f"config{cid}"] = {k: r[k] for k in ("chains", "tracks", "subgroups", "length", "processors",
                                                           "steps_per_s", "ms_per_step", "step_roofline")}
            for k in ("scan_ns_per_sample_row", "fft"):
                if k in r and (k != "fft" or cid == 4):
                    secondary[f"config{cid}"][k] = r[k]
            torch.cuda.empty_cache()
    lay = eng.layout
    # per step: its segment and the 8 step scalars in, the 4 metrics out (params move once per run)
    h2d = stems.nbytes + target.nbytes + 8 * 8
    d2h = 4 * 8

    P = lay.P
    bytes_step = b_step(L, K, S, P)
    hbm, peak_src = _peak_hbm()
    dom = max(level_ms.items(), key=lambda kv: kv[1]["ms"]) if level_ms else None
    roof = None
    if dom:
        name, rec = dom
        ach = rec["bytes"] / (rec["ms"] / 1e3) / 1e9
        traffic, traffic_src = None, None
        try:  # DRAM bytes of every conv level's kernels, one ncu capture each (tools/ncu_traffic.sh)
            with open(os.path.join(ROOT, "profiles", "level_traffic_config2.json")) as fh:
                lt = json.load(fh)
            rec_t = lt["levels"].get(name.split("(")[0])
            if rec_t is not None:
                traffic, traffic_src = rec_t["dram_bytes_per_rep"], lt.get("source")
        except (OSError, ValueError, KeyError):
            pass
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": traffic, "traffic_source": traffic_src, "kernel": name, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": rec["bytes"], "launch_ms": rec["ms"],
                "unit_of_launch": "one level forward+backward (SURVEY 8d: 40 L bytes per node)"}
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_reference_baseline(K, S, L, stems, target, songs)
            except Exception as exc:  # pragma: no cover
                cpu = {"value": None, "unit": "steps/s", "cores": 0, "kind": "reference",
                       "sample": f"failed: {exc}"}
        line = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (f64 scans/loss/optimizer)",
            "data": "synthetic",
            "config": {"workload": "config2: full console 16 trk + 4 sub, L=441000 (10 s @44.1k as samples)",
                       "tracks": K, "subgroups": S, "length": L, "processors": P, "seed": "rank",
                       "l2": "working set per step >> 126 MB L2 (no flush needed)",
                       "parallelism": f"song-sharded x{world} (no collective in the step)"},
            "e2e": {"value": e2e_val, "unit": "steps/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "paper_2509_15948_b200.train_segments (pinned host stems/target per step, "
                           "H2D overlapped with the previous step)",
                    "steps": args.e2e_steps, "runs": 3, "statistic": "median of 3 timed runs",
                    "includes": "engine param load, first (unoverlapped) upload, final param read-back",
                    "train_step_sync": sync_val},
            "config1": cfg1,
            "configs34": secondary,
            "eval_trial_ms": trial_ms,
            "songs_per_hour": songs,
            "gpu_launches": eng.launches_per_step() * args.steps,
            "clocks": clk.summary(),
            "roofline": roof,
            "step_roofline": {"bound": "hbm", "algorithmic_bytes": bytes_step,
                              "achieved": bytes_step / (ms_step / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                              "frac": bytes_step / (ms_step / 1e3) / 1e9 / hbm},
            "levels_ms": {k: round(v["ms"], 4) for k, v in level_ms.items()},
            "loss": vals,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def time_config(dev, K, S, L, seed, render, steps, warmup):
    """steps/s of another BASELINE config on this GPU (graph replays, CUDA events) + its step roofline."""
    import torch

    from paper_2509_15948_b200.engine import TrainEngine
    from paper_2509_15948_b200.optimizer import TrainConfig, _EngineCfg, make_optimizer
    graph, params, stems, target = make_inputs(seed, K, S, L, render)
    cfg = TrainConfig(segment_seconds=L / 30000, steps=1)
    eng = TrainEngine(graph, L, _EngineCfg(make_optimizer(params, cfg), cfg), device=dev)
    eng.load_params(params)
    eng.plan.set_stems(stems)
    eng.target.copy_(torch.from_numpy(target))
    for _ in range(warmup):
        eng.step_async()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        eng.step_async()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    hbm = _peak_hbm()[0]
    by = b_step(L, K, S, eng.layout.P)
    return {"workload": f"config1: full console {K} trk + {S} sub, L={L} (3 s @44.1k as samples)",
            "value": 1000.0 / ms, "unit": "steps/s", "ms_per_step": ms, "steps": steps,
            "launches_per_step": eng.launches_per_step(),
            "step_roofline": {"algorithmic_bytes": by, "achieved": by / (ms / 1e3) / 1e9, "peak": hbm,
                              "frac": by / (ms / 1e3) / 1e9 / hbm}}


def _peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
        return float(peaks["hbm_gbs"]), "measured"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback"


def time_levels(eng, reps=3):
    """CUDA-event time of each level's forward+backward (eager) and its algorithmic bytes."""
    import ctypes

    import torch

    from paper_2509_15948_b200._lib import check, lib
    from paper_2509_15948_b200.engine import stream_ptr
    Ld = lib()
    L = eng.L
    out = {}
    plan = eng.plan
    # run one eager forward/backward so all buffers hold a consistent state
    eng.grads_only()
    for lv in plan.levels:
        if lv.struct is None:
            continue
        key = f"{lv.tag}@step{lv.step}(B={lv.B})"
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        fwd, bwd = [], []
        for _ in range(reps):
            ev[0].record()
            check(Ld.mgb_level_forward(ctypes.byref(lv.struct), stream_ptr()), "fwd")
            ev[1].record()
            check(Ld.mgb_level_backward(ctypes.byref(lv.struct), stream_ptr()), "bwd")
            ev[2].record()
            torch.cuda.synchronize()
            fwd.append(ev[0].elapsed_time(ev[1]))
            bwd.append(ev[1].elapsed_time(ev[2]))
        # compulsory bytes of one processor: 40 * L per node (fwd 16 L + bwd 24 L)
        out[key] = {"ms": min(fwd) + min(bwd), "fwd_ms": min(fwd), "bwd_ms": min(bwd),
                    "bytes": 40 * L * lv.B}
    return out


if __name__ == "__main__":
    main()
