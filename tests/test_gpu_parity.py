"""Device parity: the CUDA path through the C ABI vs the reference's golden
fixtures and the float64 oracle.  Tolerances (north_star): rendered mix and
gradients 1e-4 norm-relative (fp32), loss 1e-5 relative."""

import numpy as np
import pytest
import torch

from conftest import golden, normrel
from golden_inputs import kernel_inputs, mrstft_inputs, step_spec

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2509_15948_b200.engine import ensure_device
    return ensure_device("cuda")


@pytest.mark.parametrize("log2n", [5, 8, 10, 11, 13, 14, 16, 18, 19, 21])
def test_fft_matches_numpy(dev, log2n):
    from paper_2509_15948_b200 import _lib
    from paper_2509_15948_b200.engine import ptr, stream_ptr
    n, B = 1 << log2n, 3
    rng = np.random.default_rng(log2n)
    x = (rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))).astype(np.complex64)
    xt = torch.from_numpy(x).to(dev)
    out = torch.empty_like(xt)
    tmp = torch.empty_like(xt)
    L = _lib.lib()
    _lib.check(L.mgb_fft(ptr(xt), ptr(out), ptr(tmp), B, log2n, 0, 1.0, stream_ptr()), "fft")
    ref = np.fft.fft(x.astype(np.complex128), axis=-1)
    assert normrel(out.cpu().numpy(), ref) < 3e-6
    _lib.check(L.mgb_fft(ptr(out), ptr(out), ptr(tmp), B, log2n, 1, 1.0 / n, stream_ptr()), "ifft")
    assert normrel(out.cpu().numpy(), x) < 3e-6


@pytest.mark.parametrize("tag", list("gsecndr"))
def test_kernel_matches_reference_golden(dev, tag):
    from paper_2509_15948_b200.processors import KERNELS
    gk = golden("kernels.npz")
    u, p, w = kernel_inputs(tag)
    ut = torch.tensor(u, dtype=torch.float32, device=dev, requires_grad=True)
    pt = torch.tensor(p, dtype=torch.float64, device=dev, requires_grad=True)
    ybar, reg = KERNELS[tag](ut, pt)
    loss = torch.sum(ybar.double() * torch.tensor(w, device=dev))
    if reg is not None:
        loss = loss + reg
    loss.backward()
    assert normrel(ybar.detach().cpu().numpy(), gk[f"{tag}_ybar"]) < 2e-6
    if tag in "erd":
        # reg = sum_b |log||ybar_mid|| - log||u_mid|||: near-identity rows make it a difference of
        # nearly equal logs, so the fp32 bound is absolute on the log scale (~1e-6 per row)
        np.testing.assert_allclose(float(reg.detach()), float(gk[f"{tag}_reg"]), rtol=1e-5, atol=2e-6)
    assert normrel(ut.grad.cpu().numpy(), gk[f"{tag}_gu"]) < 1e-4
    # gradient banks: norm-relative, excluding FFT-noise-level reference entries
    assert normrel(pt.grad.cpu().numpy(), gk[f"{tag}_gp"], floor=1e-6) < 1e-4


@pytest.mark.parametrize("name,sizes", [("std", (512, 1024, 4096)),
                                        ("six", (256, 512, 1024, 2048, 4096, 8192))])
def test_mrstft_matches_reference_golden(dev, name, sizes):
    from paper_2509_15948_b200.losses import LossConfig, mrstft
    gm = golden("mrstft.npz")
    y_hat, tgt = mrstft_inputs()
    yt = torch.tensor(y_hat, dtype=torch.float32, device=dev, requires_grad=True)
    val = mrstft(yt, tgt.astype(np.float32), LossConfig(fft_sizes=sizes))
    val.backward()
    # inputs are rounded to fp32 on the device: compare against the oracle on the same fp32 inputs
    from oracle import mixgraph_oracle as O
    yo = torch.tensor(y_hat.astype(np.float32).astype(np.float64), requires_grad=True)
    ov = O.mrstft(yo, tgt.astype(np.float32).astype(np.float64), O.LossConfig(fft_sizes=sizes))
    ov.backward()
    np.testing.assert_allclose(float(val), float(ov), rtol=1e-5)
    np.testing.assert_allclose(float(val), float(gm[f"{name}_loss"]), rtol=1e-3)
    assert normrel(yt.grad.cpu().numpy(), yo.grad.numpy()) < 1e-4


@pytest.mark.parametrize("name,ls", [("short1000", 1000), ("short3000", 3000)])
def test_mrstft_short_signals_match_reference_golden(dev, name, ls):
    """Scored signals shorter than the 4096/8192-point frames' reflect pad: the pad spans
    several reflections (mg/engine.py:640-645), in the forward and in the adjoint."""
    from paper_2509_15948_b200.losses import LossConfig, mrstft
    gm = golden("mrstft.npz")
    y_hat, tgt = mrstft_inputs()
    yt = torch.tensor(y_hat[:, :ls].astype(np.float32), device=dev, requires_grad=True)
    val = mrstft(yt, tgt[:, :ls].astype(np.float32), LossConfig(fft_sizes=(256, 512, 1024, 2048, 4096, 8192)))
    val.backward()
    from oracle import mixgraph_oracle as O
    yo = torch.tensor(y_hat[:, :ls].astype(np.float32).astype(np.float64), requires_grad=True)
    ov = O.mrstft(yo, tgt[:, :ls].astype(np.float32).astype(np.float64),
                  O.LossConfig(fft_sizes=(256, 512, 1024, 2048, 4096, 8192)))
    ov.backward()
    np.testing.assert_allclose(float(val.detach()), float(ov.detach()), rtol=1e-5)
    np.testing.assert_allclose(float(val.detach()), float(gm[f"{name}_loss"]), rtol=1e-3)
    assert normrel(yt.grad.cpu().numpy(), yo.grad.numpy()) < 1e-4


def _step_setup():
    from paper_2509_15948_b200.console import build_console, init_params
    from workloads import SynthSpec, make_stems_f32, manifest_for
    K, S, L, s_stems, s_p, s_t = step_spec()
    spec = SynthSpec(tracks=K, subgroups=S, duration_seconds=L / 30000)
    stems = make_stems_f32(spec, s_stems, L)
    graph, zeros = build_console(manifest_for(spec))
    return graph, init_params(zeros, s_p), stems, L


def test_train_step_gradients_match_reference(dev):
    from paper_2509_15948_b200.engine import TrainEngine
    from paper_2509_15948_b200.optimizer import TrainConfig, _EngineCfg, make_optimizer
    gs = golden("step.npz")
    graph, params, stems, L = _step_setup()
    cfg = TrainConfig(segment_seconds=L / 30000, steps=1)
    eng = TrainEngine(graph, L, _EngineCfg(make_optimizer(params, cfg), cfg), device=dev, use_graph=False)
    eng.load_params(params)
    eng.plan.set_stems(stems)
    eng.target.copy_(torch.as_tensor(gs["target"], dtype=torch.float32))
    vals, grads, gw, y = eng.grads_only()
    assert normrel(y, gs["y"]) < 1e-5
    np.testing.assert_allclose(vals["L_a"], float(gs["v_L_a"]), rtol=1e-5)
    np.testing.assert_allclose(vals["L_g"], float(gs["v_L_g"]), rtol=1e-5)
    for t in "gsecnr":
        assert normrel(grads[t], gs[f"grad_{t}"], floor=1e-6) < 1e-4, t
    s = 1.0 / (1.0 + np.exp(-params.raw_weights))
    assert normrel(gw * s * (1 - s), gs["grad_w"], floor=1e-6) < 1e-4
    assert normrel(grads["d"], gs["d_raw"], floor=1e-6) < 1e-4


def test_public_train_step_two_steps(dev):
    from paper_2509_15948_b200.optimizer import TrainConfig, make_optimizer, train_step
    gs = golden("step.npz")
    graph, params, stems, L = _step_setup()
    cfg = TrainConfig(segment_seconds=L / 30000, steps=1)
    opt = make_optimizer(params, cfg)
    v1 = train_step(graph, params, (stems, gs["target"]), cfg, opt)
    v2 = train_step(graph, params, (stems, gs["target"]), cfg, opt)
    np.testing.assert_allclose(v1["L_a"], float(gs["v_L_a"]), rtol=1e-5)
    np.testing.assert_allclose(v2["L_a"], float(gs["v2_L_a"]), rtol=1e-3)
    for t in "gsecnr":
        np.testing.assert_allclose(params.params[t], gs[f"after2_{t}"], atol=5e-3)


def test_train_segments_equals_train_step_loop(dev):
    """The pipelined segment trainer makes exactly the updates of a train_step loop."""
    from paper_2509_15948_b200.optimizer import TrainConfig, make_optimizer, train_segments, train_step
    gs = golden("step.npz")
    graph, params, stems, L = _step_setup()
    rng = np.random.default_rng(3)
    segs = [(stems * (1.0 + 0.1 * i), gs["target"] + 0.01 * rng.standard_normal(gs["target"].shape))
            for i in range(5)]
    segs = [(torch.from_numpy(s.astype(np.float32)).pin_memory(), torch.from_numpy(t.astype(np.float32)))
            for s, t in segs]
    cfg = TrainConfig(segment_seconds=L / 30000, steps=1)
    p_loop, p_pipe = params.copy(), params.copy()
    opt = make_optimizer(p_loop, cfg)
    loop = [train_step(graph, p_loop, s, cfg, opt) for s in segs]
    opt_pipe = make_optimizer(p_pipe, cfg)
    pipe = train_segments(graph, p_pipe, segs, cfg, opt_pipe)
    # the pipelined run reads the stems from its staging slots; the next train_step on the
    # same engine must read its own input again
    loop.append(train_step(graph, p_loop, segs[2], cfg, opt))
    pipe.append(train_step(graph, p_pipe, segs[2], cfg, opt_pipe))
    assert len(pipe) == len(loop)
    for a, b in zip(loop, pipe):
        for key in ("loss", "L_a", "L_g", "L_p"):
            assert a[key] == b[key], key
    for t in "gsecnrd":
        np.testing.assert_array_equal(p_loop.params[t], p_pipe.params[t])
    np.testing.assert_array_equal(p_loop.raw_weights, p_pipe.raw_weights)


def _random_console(rng, kmax=4, prune=0.0):
    from paper_2509_15948_b200.console import SessionManifest, TrackEntry, build_console
    from paper_2509_15948_b200.graph import PARAM_COUNTS, ParamStore, bypass_remove
    k = int(rng.integers(1, kmax + 1))
    s = int(rng.integers(1, min(3, k) + 1))
    tracks = [TrackEntry(f"t{i}", f"t{i}", f"bus{i % s}") for i in range(k)]
    g, _ = build_console(SessionManifest(tracks, "m"))
    P = {t: 0.1 * rng.standard_normal((len(g.nodes_of_type(t)), PARAM_COUNTS[t])) for t in PARAM_COUNTS}
    for lo in (192, 576):
        P["r"][:, lo:lo + 192] = -np.abs(P["r"][:, lo:lo + 192]) - 0.01
    params = ParamStore(P, 0.1 * rng.standard_normal(len(g.processor_nodes())))
    if prune > 0:
        procs = g.processor_nodes()
        drop = rng.choice(procs, size=int(round(prune * len(procs))), replace=False)
        g, params = bypass_remove(g, params, set(int(v) for v in drop))
    return g, params


def _oracle_render(graph, params, src, mask=None):
    from oracle import mixgraph_oracle as O
    with torch.no_grad():
        y, reg = O.execute(graph, {t: torch.tensor(v) for t, v in params.params.items()},
                           torch.tensor(params.raw_weights), src.astype(np.float64), mask)
    return y.numpy(), float(reg)


@pytest.mark.parametrize("seed,L", [(0, 5000), (1, 5000), (2, 5000), (3, 5000), (4, 4999), (5, 8193), (6, 1231)])
def test_execute_batched_matches_oracle_on_random_consoles(dev, seed, L):
    """Random consoles and prunings; odd lengths take the scalar (non-float4) row paths."""
    from paper_2509_15948_b200.schedule import schedule_console
    from paper_2509_15948_b200.scheduler import execute_batched
    rng = np.random.default_rng(seed + 100)
    graph, params = _random_console(rng, kmax=5, prune=rng.uniform(0, 0.8))
    src = (0.3 * rng.standard_normal((len(graph.nodes_of_type("i")), 2, L))).astype(np.float32)
    y, reg = execute_batched(graph, params, src, schedule_console(graph))
    yo, rego = _oracle_render(graph, params, src)
    assert normrel(y.cpu().numpy(), yo) < 1e-5
    np.testing.assert_allclose(float(reg), rego, rtol=1e-5, atol=1e-9)


def test_execute_batched_matches_oracle_on_random_dags(dev):
    from paper_2509_15948_b200.graph import PARAM_COUNTS, PROCESSOR_TYPES, MixGraph, ParamStore
    from paper_2509_15948_b200.scheduler import execute_batched
    for seed in range(4):
        rng = np.random.default_rng(seed + 500)
        k = int(rng.integers(1, 5))
        types, edges = list("i" * k), []
        for _ in range(int(rng.integers(0, 13))):
            nid = len(types)
            if rng.random() < 0.7:
                types.append(PROCESSOR_TYPES[int(rng.integers(0, 7))])
                edges.append((int(rng.integers(0, nid)), nid))
            else:
                preds = rng.choice(nid, size=int(rng.integers(1, min(3, nid) + 1)), replace=False)
                types.append("m")
                edges.extend((int(p), nid) for p in preds)
        sinks = [v for v in range(len(types)) if all(a != v for a, _ in edges)]
        out = len(types)
        types.append("o")
        edges.extend((v, out) for v in sinks)
        graph = MixGraph("".join(types), tuple(edges))
        P = {t: 0.1 * rng.standard_normal((len(graph.nodes_of_type(t)), PARAM_COUNTS[t]))
             for t in PARAM_COUNTS}
        for lo in (192, 576):
            P["r"][:, lo:lo + 192] = -np.abs(P["r"][:, lo:lo + 192]) - 0.01
        params = ParamStore(P, 0.1 * rng.standard_normal(len(graph.processor_nodes())))
        src = (0.3 * rng.standard_normal((k, 2, 3000))).astype(np.float32)
        y, _ = execute_batched(graph, params, src)
        yo, _ = _oracle_render(graph, params, src)
        assert normrel(y.cpu().numpy(), yo) < 1e-5, seed


def test_mask_matches_structural_bypass_and_all_masked_is_stem_sum(dev):
    from paper_2509_15948_b200.graph import bypass_remove
    from paper_2509_15948_b200.schedule import schedule_console
    from paper_2509_15948_b200.scheduler import execute_batched
    rng = np.random.default_rng(7)
    graph, params = _random_console(rng, kmax=4)
    src = (0.3 * rng.standard_normal((len(graph.nodes_of_type("i")), 2, 4000))).astype(np.float32)
    procs = graph.processor_nodes()
    drop = set(int(v) for v in rng.choice(procs, size=len(procs) // 2, replace=False))
    mask = np.array([0.0 if v in drop else 1.0 for v in procs])
    ym, _ = execute_batched(graph, params, src, schedule_console(graph), mask=mask)
    g2, p2 = bypass_remove(graph, params, drop)
    yc, _ = execute_batched(g2, p2, src, schedule_console(g2))
    assert normrel(ym.cpu().numpy(), yc.cpu().numpy()) < 1e-6
    y0, _ = execute_batched(graph, params, src, schedule_console(graph), mask=np.zeros(len(procs)))
    np.testing.assert_allclose(y0.cpu().numpy(), src.astype(np.float64).sum(axis=0), atol=1e-6)


def test_eval_loss_matches_oracle(dev):
    from oracle import mixgraph_oracle as O
    from paper_2509_15948_b200.losses import LossConfig
    from paper_2509_15948_b200.pruning import EvalSet, eval_loss
    gs = golden("step.npz")
    graph, params, stems, L = _step_setup()
    segs = [(stems, gs["target"][:, 30000:])]
    es = EvalSet(segs, 30000, LossConfig(), device=dev)
    mask = np.ones(len(graph.processor_nodes()))
    mask[[1, 5, 9]] = 0.0
    got = eval_loss(graph, params, mask, es)
    prep = O.prepare_target(gs["target"][:, 30000:].astype(np.float32).astype(np.float64), O.LossConfig())
    want = O.eval_loss(graph, params.params, params.raw_weights, mask,
                       [(stems.astype(np.float64), prep)], 30000, O.LossConfig())
    np.testing.assert_allclose(got, want, rtol=1e-5)


@pytest.mark.parametrize("min_l", [0, 10 ** 9])  # per-segment plans (incremental) / one shared plan
def test_incremental_trial_render_equals_full_render(dev, monkeypatch, min_l):
    """The eager eval engine re-renders a trial from the first level whose mask changed;
    every loss must equal (bit for bit) a full render of the same mask."""
    from paper_2509_15948_b200.engine import EvalEngine
    monkeypatch.setattr(EvalEngine, "INCREMENTAL_MIN_L", min_l)
    from paper_2509_15948_b200.losses import LossConfig
    gs = golden("step.npz")
    graph, params, stems, L = _step_setup()
    segs = [(stems, gs["target"][:, 30000:]), (stems[..., ::-1].copy(), gs["target"][:, 30000:][..., ::-1].copy())]
    inc = EvalEngine(graph, segs, 30000, LossConfig(), device=dev, params=params, use_graph=False)
    full = EvalEngine(graph, segs, 30000, LossConfig(), device=dev, params=params, use_graph=True)
    P = len(graph.processor_nodes())
    rng = np.random.default_rng(5)
    base = np.ones(P)
    for trial in range(12):
        mask = base.copy()
        mask[rng.choice(P, size=int(rng.integers(1, 4)), replace=False)] = 0.0
        if trial == 6:
            base = mask.copy()  # an accepted trial: the next ones differ from a new base
        assert inc.loss(mask) == full.loss(mask), trial
    assert inc.loss(base) == full.loss(base)


# FFT-size coverage of the convolution levels (N = next_pow2(L + M - 1)): the
# register four-step at N1 = 128..1024 (2^17..2^20), the Stockham four-step at
# 2^21, and the overlap-save EQ at the production length, against the oracle.
@pytest.mark.parametrize("tag,L", [("d", 441_000), ("r", 441_000), ("e", 441_000), ("r", 132_300),
                                   ("d", 600_000), ("r", 1_100_000), ("d", 33_000)])
def test_conv_level_matches_oracle_at_length(dev, tag, L):
    from oracle import mixgraph_oracle as O
    from paper_2509_15948_b200.processors import KERNELS
    _, p, _ = kernel_inputs(tag)
    rng = np.random.default_rng(L + ord(tag))
    u = (0.3 * rng.standard_normal((2, 2, L))).astype(np.float32)
    w = rng.standard_normal((2, 2, L))
    ut = torch.tensor(u, device=dev, requires_grad=True)
    pt = torch.tensor(p, dtype=torch.float64, device=dev, requires_grad=True)
    ybar, reg = KERNELS[tag](ut, pt)
    (torch.sum(ybar.double() * torch.tensor(w, device=dev)) + reg).backward()
    uo = torch.tensor(u.astype(np.float64), requires_grad=True)
    po = torch.tensor(p, requires_grad=True)
    yo, rego = O.KERNELS[tag](uo, po)
    (torch.sum(yo * torch.tensor(w)) + rego).backward()
    assert normrel(ybar.detach().cpu().numpy(), yo.detach().numpy()) < 1e-5
    np.testing.assert_allclose(float(reg.detach()), float(rego.detach()), rtol=1e-5, atol=2e-6)
    assert normrel(ut.grad.cpu().numpy(), uo.grad.numpy()) < 1e-4
    assert normrel(pt.grad.cpu().numpy(), po.grad.numpy(), floor=1e-6) < 1e-4


@pytest.mark.parametrize("tag", list("erdcgs"))
def test_phase_split_equals_whole_level_calls(dev, tag):
    """mgb_level_{forward,backward}_phase 1 then 2 == mgb_level_{forward,backward} bit-exactly,
    and the library's launch counter advances."""
    import ctypes
    from golden_inputs import kernel_inputs
    from paper_2509_15948_b200._lib import check, lib
    from paper_2509_15948_b200.engine import dev_ptr_array, ptr, stream_ptr
    from paper_2509_15948_b200.processors import _Level
    Ld = lib()
    u, p, w = kernel_inputs(tag)
    ut = torch.tensor(u, dtype=torch.float32, device=dev)
    pt = torch.tensor(p, dtype=torch.float64, device=dev)
    B, _, L = ut.shape
    outs = []
    for split in (False, True):
        lv = _Level(tag, ut, pt)
        st = lv.struct()
        gy = torch.tensor(w, dtype=torch.float32, device=dev)
        gyr = dev_ptr_array([ptr(gy, b * 2 * L) for b in range(B)], dev)
        greg = torch.ones((), dtype=torch.float64, device=dev)
        gu = torch.empty((B, 2, L), dtype=torch.float32, device=dev)
        gp = torch.zeros_like(pt)
        gw = torch.zeros(B, dtype=torch.float64, device=dev)
        st.gy_rows, st.greg, st.gu, st.gbank, st.gw = ptr(gyr), ptr(greg), ptr(gu), ptr(gp), ptr(gw)
        n0 = Ld.mgb_launch_count()
        if split:
            for ph in (1, 2, 3):
                check(Ld.mgb_level_forward_phase(ctypes.byref(st), ph, stream_ptr()), "fwd phase")
            for ph in (1, 2):
                check(Ld.mgb_level_backward_phase(ctypes.byref(st), ph, stream_ptr()), "bwd phase")
        else:
            check(Ld.mgb_level_forward(ctypes.byref(st), stream_ptr()), "fwd")
            check(Ld.mgb_level_backward(ctypes.byref(st), stream_ptr()), "bwd")
        torch.cuda.synchronize()
        assert Ld.mgb_launch_count() > n0
        outs.append([t.cpu().numpy().copy() for t in (lv.y, gu, gp)])
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)
    assert Ld.mgb_level_forward_phase(None, 1, stream_ptr()) != 0  # bad argument -> status 1


def test_pruning_passes_make_the_oracles_decisions(dev, monkeypatch):
    """Teacher-forced pruning parity: from the same state, τ and RNG
    stream, a dry/wet pass and a brute-force pass with device trials produce the same
    ledger (candidates, accept bits) and survivors as with the float64 oracle's eval_loss;
    the smallest decision margin |L_a - (L_min + τ)| / τ is reported."""
    from oracle import mixgraph_oracle as O
    from paper_2509_15948_b200 import pruning as P
    from paper_2509_15948_b200.common import rng_for
    from paper_2509_15948_b200.losses import LossConfig
    gs = golden("step.npz")
    graph, params, stems, L = _step_setup()
    ws = 30000
    tgt = gs["target"].astype(np.float32)
    eval_set = P.EvalSet([(stems, tgt[:, ws:])], ws, LossConfig(), device=dev)
    prep = O.prepare_target(tgt[:, ws:].astype(np.float64), O.LossConfig())
    oseg = [(stems.astype(np.float64), prep)]

    def oracle_eval(graph, params, mask, eval_set, schedule=None):
        return O.eval_loss(graph, params.params, params.raw_weights, mask, oseg, ws, O.LossConfig())

    n = len(graph.processor_nodes())
    la0 = oracle_eval(graph, params, np.ones(n), None)
    tau = 0.02 * la0

    def run(pass_fn, fn):
        monkeypatch.setattr(P, "eval_loss", fn)
        state = P.PruneState(alive=np.ones(n, dtype=bool), la_min=la0, tolerance=tau, iteration=1)
        mask = pass_fn(state, graph, params, eval_set, np.ones(n), list(range(n)), rng_for(0, "prune-order"))
        return mask, state.ledger

    margins = []
    for pass_fn in (P.prune_drywet_pass, P.prune_bruteforce_pass):
        m_dev, led_dev = run(pass_fn, _device_eval)
        m_ora, led_ora = run(pass_fn, oracle_eval)
        assert [(r.candidates, r.accepted) for r in led_dev] == [(r.candidates, r.accepted) for r in led_ora]
        np.testing.assert_array_equal(m_dev, m_ora)
        margins += [abs(r.loss - (r.la_min_before + tau)) / tau for r in led_ora]
        for a, b in zip(led_dev, led_ora):
            np.testing.assert_allclose(a.loss, b.loss, rtol=1e-5)
    print(f"pruning parity: {len(margins)} trials, min decision margin {min(margins):.3e} tau")


def _device_eval(graph, params, mask, eval_set, schedule=None):
    return eval_set.engine(graph, params).loss(mask)


def test_desk_song_search_runs(dev):
    """Config-5 unit of work end to end on the device: one desk-recipe pruning search
    (console fit, a hybrid round with trials and a fine-tune) on a small synthetic song."""
    import bench
    from paper_2509_15948_b200.scheduler import execute_batched
    from paper_2509_15948_b200.songs import SongSpec, search_song

    def render(graph, tparams, stems):
        y, _ = execute_batched(graph, tparams, stems, device=dev)
        return y.cpu().numpy()

    spec = SongSpec(index=0, tracks=4, subgroups=1, length=132_300)
    graph, params, stems, target = bench.make_inputs(7, spec.tracks, spec.subgroups, spec.length, render)
    res = search_song(spec, graph, params, stems, target, iterations=1, device=dev)
    assert res["trials"] > 0 and 0.0 <= res["pruning_ratio"] <= 1.0
    assert np.isfinite(res["console_loss"]) and np.isfinite(res["final_loss"])


def test_concurrent_song_searches_equal_sequential(dev):
    """Songs searched concurrently on one GPU (one host thread + stream each) make the same
    decisions and losses as the same songs searched one after another."""
    import bench
    from paper_2509_15948_b200.scheduler import execute_batched
    from paper_2509_15948_b200.songs import SongSpec, search_songs

    def render(graph, tparams, stems):
        y, _ = execute_batched(graph, tparams, stems, device=dev)
        return y.cpu().numpy()

    specs = [SongSpec(index=i, tracks=k, subgroups=1, length=132_300) for i, k in enumerate((4, 5, 3))]
    inputs = {i: bench.make_inputs(20 + i, s.tracks, s.subgroups, s.length, render) for i, s in enumerate(specs)}
    mine = [0, 1, 2]
    seq = search_songs(specs, mine, inputs, concurrent=1, iterations=2, device=dev)
    par = search_songs(specs, mine, inputs, concurrent=3, iterations=2, device=dev)
    keys = ("song", "tracks", "trials", "pruning_ratio", "console_loss", "final_loss")
    assert [{k: r[k] for k in keys} for r in par] == [{k: r[k] for k in keys} for r in seq]


def test_nonfinite_loss_stops_the_run_where_the_reference_does(dev):
    """train() hits a non-finite loss at step i (mg/optimizer.py:170-171, 208-215): it raises
    NonFiniteLoss with the parameters, step count, history and segment RNG exactly where a
    run of i steps leaves them (the device skips every update from step i on)."""
    from paper_2509_15948_b200.common import rng_for
    from paper_2509_15948_b200.optimizer import NonFiniteLoss, Session, TrainConfig, train
    gs = golden("step.npz")
    graph, params, stems, L0 = _step_setup()
    stems = np.concatenate([stems, stems[..., :37_000]], axis=-1)  # a 70,000-sample session
    tgt = np.concatenate([gs["target"], gs["target"][:, :37_000]], axis=-1).astype(np.float64)
    L = stems.shape[-1]
    seg = L - 1000
    tgt[:, seg + 500] = np.nan  # inside every segment whose offset exceeds 500
    session = Session(stems, tgt)
    cfg = TrainConfig(segment_seconds=seg / 30000, steps=12, seed=7)
    probe = rng_for(7, "segments")
    offs = [int(probe.integers(0, L - seg + 1)) for _ in range(cfg.steps)]
    bad = next(i for i, o in enumerate(offs) if o > 500)
    assert 0 < bad < cfg.steps - 1
    p_fail, hist, rng = params.copy(), [], rng_for(7, "segments")
    with pytest.raises(NonFiniteLoss):
        train(graph, p_fail, session, cfg, rng=rng, history=hist)
    assert len(hist) == bad
    after = rng.integers(0, 1 << 30)
    p_ok, rng2 = params.copy(), rng_for(7, "segments")
    ok_cfg = TrainConfig(segment_seconds=seg / 30000, steps=bad, seed=7)
    hist2 = train(graph, p_ok, session, ok_cfg, rng=rng2)
    rng2.integers(0, L - seg + 1)  # the reference drew the failing step's offset too
    assert after == rng2.integers(0, 1 << 30)
    for t in "gsecnrd":
        np.testing.assert_array_equal(p_fail.params[t], p_ok.params[t])
    np.testing.assert_array_equal(p_fail.raw_weights, p_ok.raw_weights)
    assert [h["loss"] for h in hist] == [h["loss"] for h in hist2]


def test_batched_training_of_several_songs_equals_training_each_alone(dev):
    """Multi-song batching: three songs' consoles (one pruned) trained as
    one disjoint-union device program make bit-for-bit the updates each makes alone."""
    import bench
    from paper_2509_15948_b200.batch import train_batch
    from paper_2509_15948_b200.common import rng_for
    from paper_2509_15948_b200.graph import bypass_remove
    from paper_2509_15948_b200.optimizer import Session, TrainConfig, train
    from paper_2509_15948_b200.pruning import TrainRequest
    from paper_2509_15948_b200.scheduler import execute_batched

    def render(graph, tparams, stems):
        return execute_batched(graph, tparams, stems, device=dev)[0].cpu().numpy()

    songs = []
    for i, (k, s) in enumerate(((4, 1), (6, 2), (3, 1))):
        graph, params, stems, target = bench.make_inputs(40 + i, k, s, 70_000, render)
        if i == 1:
            procs = graph.processor_nodes()
            graph, params = bypass_remove(graph, params, set(procs[::4]))
        songs.append((graph, params, Session(stems, target)))
    cfg = TrainConfig(segment_seconds=57_000 / 30000, steps=6, seed=0)
    alone = []
    for i, (g, p, sess) in enumerate(songs):
        q, hist = p.copy(), []
        train(g, q, sess, cfg, rng=rng_for(i, "train-segments"), history=hist, alpha_p_fn=lambda s: 1e-4 * s)
        alone.append((q, hist))
    reqs = [TrainRequest(g, p.copy(), sess, cfg, rng_for(i, "train-segments"), [], lambda s: 1e-4 * s)
            for i, (g, p, sess) in enumerate(songs)]
    train_batch(reqs, device=dev)
    for (q, hist), r in zip(alone, reqs):
        for t in "gsecnrd":
            np.testing.assert_array_equal(r.params.params[t], q.params[t])
        np.testing.assert_array_equal(r.params.raw_weights, q.raw_weights)
        assert [h["loss"] for h in r.history] == [h["loss"] for h in hist]


def test_lockstep_song_searches_equal_sequential(dev):
    """Whole desk-recipe searches run in lock-step (every console fit and fine-tune of the
    group as one batched program) give the sequential searches' results: trials, ledgers,
    surviving sets, final .mixgraph.json bytes and losses."""
    import bench
    from paper_2509_15948_b200.scheduler import execute_batched
    from paper_2509_15948_b200.songs import SongSpec, search_songs, search_songs_lockstep

    def render(graph, tparams, stems):
        return execute_batched(graph, tparams, stems, device=dev)[0].cpu().numpy()

    specs = [SongSpec(index=i, tracks=k, subgroups=1, length=132_300) for i, k in enumerate((4, 5, 3))]
    inputs = {i: bench.make_inputs(20 + i, s.tracks, s.subgroups, s.length, render) for i, s in enumerate(specs)}
    seq = search_songs(specs, [0, 1, 2], inputs, concurrent=1, iterations=3, device=dev)
    lock = search_songs_lockstep(specs, [0, 1, 2], inputs, group=3, iterations=3, device=dev)
    keys = ("song", "tracks", "trials", "pruning_ratio", "console_loss", "final_loss", "alive", "ledger", "graph_json",
            "metrics")
    assert [{k: r[k] for k in keys} for r in lock] == [{k: r[k] for k in keys} for r in seq]


@pytest.mark.parametrize("sizes", [(512, 1024, 4096), (256, 512, 1024, 2048, 4096, 8192)])
def test_batched_mrstft_equals_per_signal_calls(dev, sizes):
    """MgbLoss.batch > 1 (several songs' losses in one call set): every signal's loss and
    gradient equal the single-signal calls bit for bit (six resolutions: the 8192-point
    one in its own launch beside the merged launch of the others)."""
    from paper_2509_15948_b200.engine import LossPlan, ptr
    from paper_2509_15948_b200.losses import LossConfig
    rng = np.random.default_rng(11)
    G, L, ws = 3, 70_000, 30_000
    y = torch.tensor(0.3 * rng.standard_normal((G, 2, L)), dtype=torch.float32, device=dev)
    t = torch.tensor(0.3 * rng.standard_normal((G, 2, L)), dtype=torch.float32, device=dev)
    cfg = LossConfig(fft_sizes=sizes)
    bl = LossPlan(cfg, L - ws, dev, batch=G, sig_stride=2 * L)
    gb = torch.zeros((G, 2, L), dtype=torch.float32, device=dev)
    bl.target(ptr(t, ws), ptr(t, L + ws))
    bl.forward(ptr(y, ws), ptr(y, L + ws))
    bl.backward(ptr(y, ws), ptr(y, L + ws), ptr(gb, ws), ptr(gb, L + ws))
    for i in range(G):
        lp = LossPlan(cfg, L - ws, dev)
        g1 = torch.zeros((2, L), dtype=torch.float32, device=dev)
        lp.target(ptr(t[i], ws), ptr(t[i], L + ws))
        lp.forward(ptr(y[i], ws), ptr(y[i], L + ws))
        lp.backward(ptr(y[i], ws), ptr(y[i], L + ws), ptr(g1, ws), ptr(g1, L + ws))
        assert float(bl.loss[i]) == float(lp.loss)
        assert torch.equal(gb[i], g1)


def test_speculative_bruteforce_trials_make_the_same_decisions(dev):
    """brute-force trials requested four per device render under
    the reject assumption give the sequential search's ledger, survivors and graph."""
    import bench
    from paper_2509_15948_b200.graph import serialize
    from paper_2509_15948_b200.optimizer import Session
    from paper_2509_15948_b200.pruning import prune_song
    from paper_2509_15948_b200.scheduler import execute_batched
    from paper_2509_15948_b200.songs import desk_prune_config

    def render(graph, tparams, stems):
        return execute_batched(graph, tparams, stems, device=dev)[0].cpu().numpy()

    graph, params, stems, target = bench.make_inputs(31, 5, 2, 132_300, render)
    cfg = desk_prune_config(3, iterations=4)  # hybrid: round 4 is brute force
    outs = [prune_song(graph, params, Session(stems, target), cfg, device=dev, speculate=s) for s in (1, 4)]
    (g1, p1, s1, r1, _), (g4, p4, s4, r4, _) = outs
    led = lambda st: [(r.iteration, r.mode, r.candidates, r.loss, r.accepted) for r in st.ledger]  # noqa: E731
    assert led(s1) == led(s4)
    assert any(r.mode == "bruteforce" for r in s1.ledger)
    np.testing.assert_array_equal(s1.alive, s4.alive)
    assert serialize(g1, p1) == serialize(g4, p4)
    assert r1.final_loss == r4.final_loss


def test_lockstep_with_mixed_recipes_equals_one_by_one(dev):
    """prune_songs_lockstep groups what it can batch: songs whose train() calls differ in
    step count, or whose eval sets differ in shape, run in separate batches, and every
    search still equals its own prune_song."""
    import bench
    from paper_2509_15948_b200.batch import prune_songs_lockstep
    from paper_2509_15948_b200.graph import serialize
    from paper_2509_15948_b200.optimizer import Session
    from paper_2509_15948_b200.pruning import prune_song
    from paper_2509_15948_b200.scheduler import execute_batched
    from paper_2509_15948_b200.songs import desk_prune_config

    def render(graph, tparams, stems):
        return execute_batched(graph, tparams, stems, device=dev)[0].cpu().numpy()

    jobs = []
    for i, (k, ft, segs) in enumerate(((4, 5, 2), (3, 8, 2), (4, 5, 3))):
        graph, params, stems, target = bench.make_inputs(60 + i, k, 1, 132_300, render)
        cfg = desk_prune_config(i, iterations=2)
        cfg.console_steps, cfg.finetune_steps, cfg.eval_segments = 20, ft, segs
        jobs.append((graph, params, Session(stems, target), cfg))
    lock = prune_songs_lockstep(jobs, device=dev)
    for (g, p, s, c), r in zip(jobs, lock):
        g1, p1, st1, rep1, _ = prune_song(g, p, s, c, device=dev, speculate=1)
        g2, p2, st2, rep2, _ = r
        assert serialize(g1, p1) == serialize(g2, p2)
        assert [(x.candidates, x.loss, x.accepted) for x in st1.ledger] == \
            [(x.candidates, x.loss, x.accepted) for x in st2.ledger]
        assert rep1.final_loss == rep2.final_loss


@pytest.mark.parametrize("L", [4999, 6151])
def test_train_step_gradients_at_odd_lengths_match_oracle(dev, L):
    """A full forward + backward at lengths that are not multiples of 4 (scalar row paths in
    every streaming kernel) and shorter than one 8192-sample scan chunk.  (Below ~3,000
    samples a delay node whose taps all fall past the signal has a wet output of pure FFT
    rounding noise, and the gain-staging term's 1/||ybar|| turns that noise into O(100)
    gradients that differ between any two implementations, the reference and its own
    float64 restatement included.)"""
    from oracle import mixgraph_oracle as O
    from paper_2509_15948_b200.console import build_console, init_params
    from paper_2509_15948_b200.engine import TrainEngine
    from paper_2509_15948_b200.optimizer import TrainConfig, _EngineCfg, make_optimizer
    from workloads import SynthSpec, make_stems_f32, manifest_for
    ws = 1000
    spec = SynthSpec(tracks=3, subgroups=1, duration_seconds=L / 30000)
    stems = make_stems_f32(spec, 9, L)
    graph, zeros = build_console(manifest_for(spec))
    params = init_params(zeros, 0)
    rng = np.random.default_rng(L)
    target = (0.3 * rng.standard_normal((2, L))).astype(np.float32)
    cfg = TrainConfig(segment_seconds=L / 30000, warmup_seconds=ws / 30000, steps=1)
    eng = TrainEngine(graph, L, _EngineCfg(make_optimizer(params, cfg), cfg), device=dev, use_graph=False)
    eng.load_params(params)
    eng.plan.set_stems(stems)
    eng.target.copy_(torch.as_tensor(target))
    vals, grads, gw, y = eng.grads_only()
    args = (graph, {t: v.copy() for t, v in params.params.items()}, params.raw_weights.copy(),
            stems.astype(np.float64), target.astype(np.float64), ws, O.LossConfig())
    ov, og, oy = O.render_loss_and_grads(*args)
    _, ogd, _ = O.render_loss_and_grads(*args, loss_point=y.astype(np.float64))
    assert normrel(y, oy) < 1e-5
    np.testing.assert_allclose(vals["L_a"], ov["L_a"], rtol=1e-5)
    for t in "gsecnrd":
        assert normrel(grads[t], ogd[t], floor=1e-6) < 1e-4, t
