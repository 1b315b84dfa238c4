"""The drop-in boundary on the device, driven by the REFERENCE's own objects.

north_star: the reference package's classes, console construction and prune
entry points stay the API surface.  Here graphs, parameter stores and
schedules are built with the reference (imported from its source tree, or
from the archive ``oracle/build_ref.py`` ships to the GPU box) and passed
through this repo's device path; and the reference's own tape runs with this
repo's level kernels swapped in through its foreign-op hook
(``engine.custom_gradient``, mg/engine.py:673-704).  Tolerances are
north_star's: mix and gradients 1e-4 norm-relative, loss 1e-5 relative."""

import numpy as np
import pytest
import torch

from conftest import normrel
from oracle import build_ref

MG = build_ref.load()
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(MG is None, reason="reference package unavailable")]


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2509_15948_b200.engine import ensure_device
    return ensure_device("cuda")


def _ref_console(K, S, L, seed_stems=3, seed_p=0, seed_t=1):
    from mixgraph import engine as E
    from mixgraph.console import SessionManifest, TrackEntry, build_console, init_params
    from mixgraph.scheduler import execute_reference
    from mixgraph.synth import SynthSpec, make_stems
    groups = [f"bus{j}" for j in range(S)]
    man = SessionManifest([TrackEntry(f"t{k}.wav", f"t{k}", groups[k % S]) for k in range(K)], "m.wav")
    graph, zeros = build_console(man)
    stems, _ = make_stems(SynthSpec(tracks=K, subgroups=S, duration_seconds=L / 30000), seed_stems)
    stems = stems.astype(np.float32).astype(np.float64)[..., :L]
    target = np.asarray(E.value_of(execute_reference(graph, init_params(zeros, seed_t), stems)[0]))
    return graph, init_params(zeros, seed_p), stems, target


def test_reference_objects_render_on_device(dev):
    """Reference MixGraph + ParamStore + planned Schedule -> this repo's execute_batched
    (and the node-at-a-time execute_reference) == the reference's execute_batched."""
    from mixgraph import engine as E
    from mixgraph import scheduler as RS
    from paper_2509_15948_b200.scheduler import execute_batched, execute_reference
    graph, params, stems, _ = _ref_console(3, 2, 20_000)
    sched = RS.plan_indices(graph, RS.schedule_console(graph))
    want, want_reg = RS.execute_batched(graph, params, stems, sched)
    want = np.asarray(E.value_of(want))
    y, reg = execute_batched(graph, params, stems.astype(np.float32), sched)
    assert normrel(y.cpu().numpy(), want) < 1e-5
    np.testing.assert_allclose(float(reg), float(E.value_of(want_reg)), rtol=1e-5)
    mask = np.ones(len(graph.processor_nodes()))
    mask[[0, 4, 9, 17]] = 0.0
    want_m = np.asarray(E.value_of(RS.execute_batched(graph, params, stems, sched, mask=mask)[0]))
    ym, _ = execute_batched(graph, params, stems.astype(np.float32), sched, mask=mask)
    assert normrel(ym.cpu().numpy(), want_m) < 1e-5
    yr, _ = execute_reference(graph, params, stems.astype(np.float32))
    assert normrel(yr.cpu().numpy(), want) < 1e-5


def test_reference_objects_train_step_on_device(dev, monkeypatch):
    """The reference's ParamStore trained in place by this repo's train_step: the loss
    matches the reference's train_step, and the update lands on the same parameters
    wherever the reference's gradient sign is determined (test_gpu_parity_configs)."""
    from mixgraph import optimizer as RO
    from paper_2509_15948_b200.optimizer import TrainConfig, make_optimizer, train_step
    from test_gpu_parity_configs import _significant
    graph, params, stems, target = _ref_console(2, 1, 33_000)
    ref_p = params.copy()
    rcfg = RO.TrainConfig(segment_seconds=33_000 / 30000, steps=1)
    got = _spy_grads(monkeypatch)
    raw_d = {}
    orig_rule = RO._delay_gradient_rule

    def rule(p_rows, g_rows):
        raw_d["d"] = g_rows.copy()
        return orig_rule(p_rows, g_rows)

    monkeypatch.setattr(RO, "_delay_gradient_rule", rule)
    rv = RO.train_step(graph, ref_p, (stems, target), rcfg, RO.make_optimizer(ref_p, rcfg))
    cfg = TrainConfig(segment_seconds=33_000 / 30000, steps=1)
    ours = params.copy()
    v = train_step(graph, ours, (stems.astype(np.float32), target.astype(np.float32)), cfg,
                   make_optimizer(ours, cfg))
    assert type(ours) is type(params)  # the reference's own ParamStore, updated in place
    np.testing.assert_allclose(v["L_a"], rv["L_a"], rtol=1e-5)
    np.testing.assert_allclose(v["L_g"], rv["L_g"], rtol=1e-5)
    for t in "gsecnrdw":
        sig = _significant(raw_d["d"] if t == "d" else got[t], t)
        a = ours.raw_weights if t == "w" else ours.params[t]
        b = ref_p.raw_weights if t == "w" else ref_p.params[t]
        np.testing.assert_allclose(a[sig], b[sig], rtol=0, atol=1e-8, err_msg=t)


def _spy_grads(monkeypatch):
    import mixgraph.optimizer as RO
    got = {}
    orig = RO.AdamW.step

    def spy(self, arrays, grads):
        for k, v in grads.items():
            got[k] = np.array(v, copy=True)
        return orig(self, arrays, grads)

    monkeypatch.setattr(RO.AdamW, "step", spy)
    return got


def test_reference_tape_runs_device_kernels_through_custom_gradient(dev, monkeypatch):
    """The reference's own train_step (its tape, loss, optimizer) with every level op
    replaced by this repo's CUDA kernels through engine.custom_gradient: the same loss
    and gradients as the pure reference."""
    from mixgraph import engine as E
    from mixgraph import optimizer as RO
    from mixgraph import processors as RP
    from paper_2509_15948_b200.refbridge import foreign_kernels
    graph, params, stems, target = _ref_console(2, 1, 33_000)
    rcfg = RO.TrainConfig(segment_seconds=33_000 / 30000, steps=1)
    got = _spy_grads(monkeypatch)
    p_ref = params.copy()
    v_ref = RO.train_step(graph, p_ref, (stems, target), rcfg, RO.make_optimizer(p_ref, rcfg))
    g_ref = dict(got)
    for tag, fn in foreign_kernels(E, dev).items():
        monkeypatch.setitem(RP.KERNELS, tag, fn)
    p_dev = params.copy()
    v_dev = RO.train_step(graph, p_dev, (stems, target), rcfg, RO.make_optimizer(p_dev, rcfg))
    np.testing.assert_allclose(v_dev["L_a"], v_ref["L_a"], rtol=1e-5)
    np.testing.assert_allclose(v_dev["L_g"], v_ref["L_g"], rtol=1e-5)
    for t in "gsecnr":
        assert normrel(got[t], g_ref[t], floor=1e-6) < 1e-4, t
    assert normrel(got["w"], g_ref["w"], floor=1e-6) < 1e-4


def test_reference_eval_loss_with_device_kernels(dev, monkeypatch):
    """The reference's eval_loss (a pruning trial) with the device level ops swapped in."""
    from mixgraph import engine as E
    from mixgraph import processors as RP
    from mixgraph import pruning as RPr
    from mixgraph.losses import LossConfig, prepare_target
    from paper_2509_15948_b200.refbridge import foreign_kernels
    graph, params, stems, target = _ref_console(3, 1, 40_000)
    es = RPr.EvalSet([(stems, prepare_target(target[:, 30000:], LossConfig()))], 30000)
    mask = np.ones(len(graph.processor_nodes()))
    mask[[2, 11]] = 0.0
    want = RPr.eval_loss(graph, params, mask, es)
    for tag, fn in foreign_kernels(E, dev).items():
        monkeypatch.setitem(RP.KERNELS, tag, fn)
    got = RPr.eval_loss(graph, params, mask, es)
    np.testing.assert_allclose(got, want, rtol=1e-5)


def test_song_metrics_match_the_reference(dev):
    """Post-hoc metrics on the device (mg/metrics.py:45-112, mg/cli.py:55-63) against the
    reference's own functions on the same float32 signals: SI-SDR, the MIR feature
    distances over two 8-second segments, and the L_a of the match."""
    from mixgraph import metrics as RM
    from mixgraph.losses import mrstft as rmrstft
    from paper_2509_15948_b200 import metrics as M
    rng = np.random.default_rng(3)
    L = 2 * 240_000 + 1_000
    t = np.arange(L) / 30000.0
    base = np.stack([np.sin(2 * np.pi * 220 * t), 0.7 * np.sin(2 * np.pi * 331 * t + 0.3)])
    target = (0.3 * base + 0.05 * rng.standard_normal((2, L))).astype(np.float32)
    match = (0.27 * base + 0.02 * np.roll(base, 40, axis=1) + 0.05 * rng.standard_normal((2, L))).astype(np.float32)
    tg, mt = target.astype(np.float64), match.astype(np.float64)
    assert abs(M.si_sdr(target, match) - RM.si_sdr(tg, mt)) < 1e-9
    got = M.mir_distances(target, match)
    errs = {}
    for f in M.FEATURES:
        want = RM.mir_distance(tg, mt, f)
        errs[f] = abs(got[f] - want)
    print("metrics |device - reference| (log10 units):", {k: f"{v:.2e}" for k, v in errs.items()})
    assert max(errs[f] for f in ("rms", "cf", "sw", "si")) < 1e-9
    assert errs["bs"] < 1e-6  # float32 Bluestein FFT of a 240,000-point segment (measured 6e-8)
    row = M.song_metrics("s", target, match, 30000)
    from mixgraph import engine as E
    la = float(E.value_of(rmrstft(mt[:, 30000:], tg[:, 30000:])))
    np.testing.assert_allclose(row["L_a"], la, rtol=1e-5)
    for f in M.FEATURES:
        assert abs(row[f"d_{f}"] - got[f]) == 0.0
    with pytest.raises(M.TooShort):
        M.mir_distances(target[:, :1000], match[:, :1000])
