"""Configs 3 and 4 of BASELINE.md §2.2 (secondary lines; bench.py's headline is config 2).

config 3  c/n-heavy: 32 tracks + 4 subgroups, console bypass-removed to chains "cn"
          (72 processors), L = 1,323,000; also the envelope-scan latency in ns per
          sample per row for the c and n levels (forward and backward).
config 4  e/r-heavy: 16 tracks + 4 subgroups, chains "er" (40 processors),
          L = 1,323,000, MRSTFT at 6 resolutions (256..8192); also the FFT-FLOP
          fraction: BASELINE's reference-formulation FFT GFLOP per step (58.2) over
          step time, against the FP32 CUDA-core peak at the measured SM clock.

One JSON line per config: steps/s (CUDA events over the captured train step on
resident inputs), the step HBM roofline fraction (B_step), per-level
fwd/bwd times.  usage: python tools/configs_bench.py [--configs 3 4] [--steps 10]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_15948_b200.engine import TrainEngine  # noqa: E402
from paper_2509_15948_b200.graph import bypass_remove  # noqa: E402
from paper_2509_15948_b200.losses import LossConfig  # noqa: E402
from paper_2509_15948_b200.optimizer import TrainConfig, _EngineCfg, make_optimizer  # noqa: E402
from paper_2509_15948_b200.scheduler import execute_batched  # noqa: E402

CONFIGS = {
    3: dict(K=32, S=4, L=1_323_000, keep="cn", fft_sizes=(512, 1024, 4096), fft_gflop=4.8),
    4: dict(K=16, S=4, L=1_323_000, keep="er", fft_sizes=(256, 512, 1024, 2048, 4096, 8192), fft_gflop=58.2),
}
FP32_LANES = 148 * 128  # FP32 lanes per B200


def run(cfg_id, steps, dev):
    c = CONFIGS[cfg_id]
    K, S, L = c["K"], c["S"], c["L"]

    def render(graph, tparams, stems):
        y, _ = execute_batched(graph, tparams, stems, device=dev)
        return y.cpu().numpy()

    graph, params, stems, target = bench.make_inputs(300 + cfg_id, K, S, L, render)
    drop = [v for v in graph.processor_nodes() if graph.node_types[v] not in c["keep"]]
    graph, params = bypass_remove(graph, params, drop)
    P = len(graph.processor_nodes())
    tcfg = TrainConfig(segment_seconds=L / 30000, steps=1, loss=LossConfig(fft_sizes=c["fft_sizes"]))
    eng = TrainEngine(graph, L, _EngineCfg(make_optimizer(params, tcfg, device=dev), tcfg), device=dev)
    eng.load_params(params)
    eng.plan.set_stems(stems)
    eng.target.copy_(torch.from_numpy(target))
    for _ in range(3):
        eng.step_async()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with bench.ClockSampler(dev.index or 0) as clk:
        a.record()
        for _ in range(steps):
            eng.step_async()
        b.record()
        torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    clocks = clk.summary()
    levels = bench.time_levels(eng, reps=3)
    hbm = json.load(open(os.path.join(bench.ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6549.8) \
        if os.path.exists(os.path.join(bench.ROOT, "MEASURED_PEAKS.json")) else 6549.8
    bstep = bench.b_step(L, K, S, P)
    out = {"config": cfg_id, "chains": c["keep"], "tracks": K, "subgroups": S, "length": L, "processors": P,
           "steps_per_s": 1000.0 / ms, "ms_per_step": ms,
           "step_roofline": {"bound": "hbm", "algorithmic_bytes": bstep,
                             "frac": bstep / (ms / 1e3) / (hbm * 1e9), "peak_gbs": hbm},
           "clocks": clocks,
           "levels_ms": {k: {"fwd": round(v["fwd_ms"], 4), "bwd": round(v["bwd_ms"], 4)} for k, v in levels.items()}}
    if cfg_id == 3:  # envelope scan latency per sample per row
        out["scan_ns_per_sample_row"] = {
            k: {"fwd": v["fwd_ms"] * 1e6 / (int(k.split("B=")[1][:-1]) * L),
                "bwd": v["bwd_ms"] * 1e6 / (int(k.split("B=")[1][:-1]) * L)}
            for k, v in levels.items() if k[0] in "cn"}
    sm_mhz = clocks.get("sm_mhz") or 1965.0
    peak_tf = FP32_LANES * 2 * sm_mhz * 1e6 / 1e12
    out["fft"] = {"gflop_per_step_reference_formulation": c["fft_gflop"],
                  "achieved_tflops": c["fft_gflop"] / ms, "fp32_peak_tflops_at_clock": peak_tf,
                  "frac": c["fft_gflop"] / ms / peak_tf}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[3, 4])
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    for cid in args.configs:
        print(json.dumps(run(cid, args.steps, dev)), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
