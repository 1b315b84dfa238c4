"""Generate tests/golden/*.npz by running the REFERENCE itself (float64 CPU).

Run in the build container, where ``/root/reference`` exists:

    python oracle/make_golden.py

The fixtures pin both the oracle restatement (``oracle/mixgraph_oracle.py``)
and the device path.  Inputs are regenerated in the tests from the same numpy
seeds, so only outputs (and small parameter arrays) are stored.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from mixgraph import engine as E  # noqa: E402
from mixgraph import losses as Lo  # noqa: E402
from mixgraph import processors as P  # noqa: E402
from mixgraph.console import SessionManifest, TrackEntry, build_console, init_params  # noqa: E402
from mixgraph.graph import PARAM_COUNTS, ParamStore  # noqa: E402
from mixgraph.optimizer import TrainConfig, make_optimizer, train_step  # noqa: E402
from mixgraph.scheduler import execute_reference, plan_indices, schedule_console  # noqa: E402
from mixgraph.synth import SynthSpec, make_stems  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")

def main():
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
    from golden_inputs import SCAN_ALPHAS, config1_spec, kernel_inputs, mrstft_inputs, scan_inputs, step_spec

    os.makedirs(OUT, exist_ok=True)

    # 1. per-kernel forward + adjoints (loss = sum(ybar * w) + reg)
    kern = {}
    for tag in "gsecndr":
        u, p, w = kernel_inputs(tag)
        t = E.Tape()
        ub, pb = t.leaf(u), t.leaf(p)
        ybar, reg = P.KERNELS[tag](ub, pb)
        loss = E.array_sum(E.mul(ybar, w))
        if reg is not None:
            loss = E.add(loss, reg)
        t.backward(loss)
        kern[f"{tag}_ybar"] = E.value_of(ybar)
        kern[f"{tag}_reg"] = np.asarray(0.0 if reg is None else E.value_of(reg))
        kern[f"{tag}_gu"] = ub.grad
        kern[f"{tag}_gp"] = pb.grad
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **kern)

    # 2. FIR synthesis (zero-phase EQ / colour FIRs, reverb FIR head + norms)
    rng = np.random.default_rng(77)
    pe = 0.1 * rng.standard_normal((1, 1024))
    pc = 0.1 * rng.standard_normal((1, 20))
    pr = 0.1 * rng.standard_normal((1, 768))
    for lo in (192, 576):
        pr[:, lo:lo + 192] = -np.abs(pr[:, lo:lo + 192]) - 0.01
    fir_r = E.value_of(P.reverb_fir(pr))
    specs, wss, nfr = P._reverb_tables()
    np.savez_compressed(
        os.path.join(OUT, "fir.npz"), pe=pe, pc=pc, pr=pr,
        eq=E.value_of(P.zero_phase_fir(pe, P.EQ_FIR_LEN)),
        color=E.value_of(P.zero_phase_fir(pc, P.COLOR_LEN)),
        reverb_head=fir_r[..., :4096], reverb_tail=fir_r[..., -1024:],
        reverb_norm=np.sqrt((fir_r ** 2).sum(-1)),
        wss=wss, spec_mid_head=specs["mid"][:4], spec_side_head=specs["side"][:4],
        mel512=Lo._projection(512, Lo.LossConfig()),
        mel4096_rowsum=Lo._projection(4096, Lo.LossConfig()).sum(0))

    # 3. MRSTFT value + gradient (default and 6-resolution configs)
    mr = {}
    for name, sizes in (("std", (512, 1024, 4096)), ("six", (256, 512, 1024, 2048, 4096, 8192))):
        cfg = Lo.LossConfig(fft_sizes=sizes)
        y_hat, tgt = mrstft_inputs()
        t = E.Tape()
        yb = t.leaf(y_hat)
        val = Lo.mrstft(yb, tgt, cfg)
        t.backward(val)
        mr[f"{name}_loss"] = np.asarray(E.value_of(val))
        mr[f"{name}_grad"] = yb.grad
    # short scored signals: the 4096- and 8192-point frames' reflect pads span several
    # reflections (mg/engine.py:640-645)
    y_hat, tgt = mrstft_inputs()
    for name, ls in (("short1000", 1000), ("short3000", 3000)):
        cfg = Lo.LossConfig(fft_sizes=(256, 512, 1024, 2048, 4096, 8192))
        t = E.Tape()
        yb = t.leaf(y_hat[:, :ls].copy())
        val = Lo.mrstft(yb, tgt[:, :ls].copy(), cfg)
        t.backward(val)
        mr[f"{name}_loss"] = np.asarray(E.value_of(val))
        mr[f"{name}_grad"] = yb.grad
    np.savez_compressed(os.path.join(OUT, "mrstft.npz"), **mr)

    # 4. one full train_step on a small console (K=2, S=1)
    K, S, L, seed_stems, seed_p, seed_t = step_spec()
    groups = [f"bus{j}" for j in range(S)]
    man = SessionManifest([TrackEntry(f"t{k}.wav", f"t{k}", groups[k % S]) for k in range(K)], "m.wav")
    graph, zeros = build_console(man)
    stems, _ = make_stems(SynthSpec(tracks=K, subgroups=S, duration_seconds=L / 30000), seed_stems)
    stems = stems.astype(np.float32).astype(np.float64)[..., :L]
    tgt_params = init_params(zeros, seed_t)
    target = np.asarray(E.value_of(execute_reference(graph, tgt_params, stems)[0]))
    params = init_params(zeros, seed_p)
    cfg = TrainConfig(segment_seconds=L / 30000, warmup_seconds=1.0, steps=1)
    sched = plan_indices(graph, schedule_console(graph))
    before = params.copy()

    # capture raw grads by wrapping the delay rule
    import mixgraph.optimizer as O
    captured = {}
    orig_rule = O._delay_gradient_rule

    def spy(p_rows, g_rows):
        out = orig_rule(p_rows, g_rows)
        captured.setdefault("d_raw", g_rows.copy())
        captured.setdefault("d_rule", out.copy())
        return out

    orig_step = O.AdamW.step

    def spy_step(self, arrays, grads):
        for k, v in grads.items():
            captured.setdefault(f"grad_{k}", np.array(v, copy=True))
        return orig_step(self, arrays, grads)

    O._delay_gradient_rule = spy
    O.AdamW.step = spy_step
    try:
        opt = make_optimizer(params, cfg)
        values = train_step(graph, params, (stems, target), cfg, opt, sched)
        values2 = train_step(graph, params, (stems, target), cfg, opt, sched)
    finally:
        O._delay_gradient_rule = orig_rule
        O.AdamW.step = orig_step
    y0 = np.asarray(E.value_of(
        __import__("mixgraph.scheduler", fromlist=["execute_batched"]).execute_batched(
            graph, before, stems, sched)[0]))
    out = {"target": target, "y": y0, "stems_head": stems[..., :64],
           "stems_sum": stems.sum(axis=-1)}
    for k in ("loss", "L_a", "L_g", "L_p"):
        out[f"v_{k}"] = np.asarray(values[k])
        out[f"v2_{k}"] = np.asarray(values2[k])
    for k, v in captured.items():
        out[k] = v
    for t_, v in params.params.items():
        out[f"after2_{t_}"] = v
    out["after2_w"] = params.raw_weights
    np.savez_compressed(os.path.join(OUT, "step.npz"), **out)

    # 5. compressor / gate in the envelope scan's hard regime (alpha_raw 8..12, L = 40,000:
    #    five 8192-sample chunks; the truncation term alpha^8192 is 0.05..0.95)
    scan = {}
    for tag in "cn":
        for a in SCAN_ALPHAS:
            u, p, w = scan_inputs(tag, a)
            t = E.Tape()
            ub, pb = t.leaf(u), t.leaf(p)
            ybar, _ = P.KERNELS[tag](ub, pb)
            t.backward(E.array_sum(E.mul(ybar, w)))
            key = f"{tag}{int(a)}"
            # signals stored as float32 (the device gates are 1e-4; float32 storage is 3e-8)
            scan[f"{key}_ybar"] = E.value_of(ybar).astype(np.float32)
            scan[f"{key}_gu"] = ub.grad.astype(np.float32)
            scan[f"{key}_gp"] = pb.grad
    np.savez_compressed(os.path.join(OUT, "scan.npz"), **scan)

    # 6. BASELINE config 1: one full train_step, K=4 tracks + 1 subgroup, L = 132,300.
    #    The target is rounded to float32 first so the device (float32 signals) and the
    #    reference see the same target values.
    K, S, L, seed_stems, seed_p, seed_t = config1_spec()
    man = SessionManifest([TrackEntry(f"t{k}.wav", f"t{k}", f"bus{k % S}") for k in range(K)], "m.wav")
    graph, zeros = build_console(man)
    stems, _ = make_stems(SynthSpec(tracks=K, subgroups=S, duration_seconds=L / 30000), seed_stems)
    stems = stems.astype(np.float32).astype(np.float64)[..., :L]
    target = np.asarray(E.value_of(execute_reference(graph, init_params(zeros, seed_t), stems)[0]))
    target = target.astype(np.float32).astype(np.float64)
    params = init_params(zeros, seed_p)
    cfg = TrainConfig(segment_seconds=L / 30000, warmup_seconds=1.0, steps=1)
    sched = plan_indices(graph, schedule_console(graph))
    y0 = np.asarray(E.value_of(
        __import__("mixgraph.scheduler", fromlist=["execute_batched"]).execute_batched(
            graph, params, stems, sched)[0]))
    captured = {}
    O._delay_gradient_rule, O.AdamW.step = spy, spy_step
    try:
        opt = make_optimizer(params, cfg)
        values = train_step(graph, params, (stems, target), cfg, opt, sched)
    finally:
        O._delay_gradient_rule = orig_rule
        O.AdamW.step = orig_step
    out = {"target": target.astype(np.float32), "y": y0.astype(np.float32),
           "stems_head": stems[..., :64], "stems_sum": stems.sum(axis=-1)}
    for k in ("loss", "L_a", "L_g", "L_p"):
        out[f"v_{k}"] = np.asarray(values[k])
    for k, v in captured.items():
        out[k] = v
    for t_, v in params.params.items():
        out[f"after_{t_}"] = v
    out["after_w"] = params.raw_weights
    np.savez_compressed(os.path.join(OUT, "config1_step.npz"), **out)
    print("golden fixtures written to", os.path.abspath(OUT))


if __name__ == "__main__":
    main()
