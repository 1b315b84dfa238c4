"""Device parity at the BASELINE configurations and in the hard numeric regimes.

* config 1 (4 tracks + 1 subgroup, L = 132,300): one full train_step against
  the REFERENCE's own golden (tests/golden/config1_step.npz);
* config 2 (16 tracks + 4 subgroups, L = 441,000): one step against the
  float64 oracle on the same inputs;
* the compressor / gate envelope scan at alpha_raw 8..12 (reference golden)
  and at config 3's length (L = 1,323,000) against the oracle;
* the optimiser kernel (delay rule + AdamW + projection + raw-weight
  gradient) fed identical state as the reference's functions;
* teacher-forced pruning decisions at config-2 scale with the desk recipe's
  four 57,000-sample eval segments.

Tolerances (north_star): mix and every gradient bank 1e-4 norm-relative
(entries below 1e-6 of a bank's largest are float noise in the reference's
own FFTs), loss 1e-5 relative.
"""

import ctypes

import numpy as np
import pytest
import torch

from conftest import golden, normrel

pytestmark = pytest.mark.gpu

GATE, LOSS_GATE, FLOOR = 1e-4, 1e-5, 1e-6


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2509_15948_b200.engine import ensure_device
    return ensure_device("cuda")


def _console(K, S, L, s_stems, s_p):
    from paper_2509_15948_b200.console import build_console, init_params
    from workloads import SynthSpec, make_stems_f32, manifest_for
    spec = SynthSpec(tracks=K, subgroups=S, duration_seconds=L / 30000)
    stems = make_stems_f32(spec, s_stems, L)
    graph, zeros = build_console(manifest_for(spec))
    return graph, zeros, init_params(zeros, s_p), stems


def _engine(graph, params, stems, target, L, dev):
    from paper_2509_15948_b200.engine import TrainEngine
    from paper_2509_15948_b200.optimizer import TrainConfig, _EngineCfg, make_optimizer
    cfg = TrainConfig(segment_seconds=L / 30000, steps=1)
    eng = TrainEngine(graph, L, _EngineCfg(make_optimizer(params, cfg), cfg), device=dev, use_graph=False)
    eng.load_params(params)
    eng.plan.set_stems(stems)
    eng.target.copy_(torch.as_tensor(np.asarray(target), dtype=torch.float32))
    return eng


def _report(name, errs):
    print(f"{name}: " + " ".join(f"{k}={v:.2e}" for k, v in errs.items()))


# ---------------------------------------------------------------------------
# config 1 against the reference's golden step


def test_config1_train_step_matches_reference(dev):
    from golden_inputs import config1_spec
    gs = golden("config1_step.npz")
    K, S, L, s_stems, s_p, _ = config1_spec()
    graph, _, params, stems = _console(K, S, L, s_stems, s_p)
    eng = _engine(graph, params, stems, gs["target"], L, dev)
    vals, grads, gw, y = eng.grads_only()
    errs = {"y": normrel(y, gs["y"])}
    np.testing.assert_allclose(vals["L_a"], float(gs["v_L_a"]), rtol=LOSS_GATE)
    np.testing.assert_allclose(vals["L_g"], float(gs["v_L_g"]), rtol=LOSS_GATE)
    for t in "gsecnr":
        errs[t] = normrel(grads[t], gs[f"grad_{t}"], floor=FLOOR)
    errs["d"] = normrel(grads["d"], gs["d_raw"], floor=FLOOR)
    s = 1.0 / (1.0 + np.exp(-params.raw_weights))
    errs["w"] = normrel(gw * s * (1 - s), gs["grad_w"], floor=FLOOR)
    _report("config1 step", errs)
    assert max(errs.values()) < GATE, errs


def test_config1_full_step_update_matches_reference(dev):
    """Rule + AdamW + projection after the config-1 step against the reference's updated
    parameters.  Adam's first step is lr * g / (|g| + 1e-8) (+ weight decay): wherever the
    reference gradient is well above eps and the noise floor the update is fixed by its sign
    and the parameters agree to 1e-8; below that the step moves at most lr either way."""
    from golden_inputs import config1_spec
    from paper_2509_15948_b200.optimizer import TrainConfig, make_optimizer, train_step
    gs = golden("config1_step.npz")
    K, S, L, s_stems, s_p, _ = config1_spec()
    graph, _, params, stems = _console(K, S, L, s_stems, s_p)
    before = params.copy()
    cfg = TrainConfig(segment_seconds=L / 30000, steps=1)
    train_step(graph, params, (stems, gs["target"]), cfg, make_optimizer(params, cfg))
    for t in "gsecnrdw":
        got = params.raw_weights if t == "w" else params.params[t]
        want = gs["after_w"] if t == "w" else gs[f"after_{t}"]
        g = gs["d_raw"] if t == "d" else gs[f"grad_{t}"]
        sig = _significant(g, t)
        np.testing.assert_allclose(got[sig], want[sig], rtol=0, atol=1e-8, err_msg=t)
        p0 = before.raw_weights if t == "w" else before.params[t]
        assert np.all(np.abs(got - want) <= 2.05 * cfg.lr * (1 + abs(p0).max() * 0.01)), t
        assert sig.mean() > 0.5, (t, sig.mean())


def _significant(g, t):
    """Entries whose gradient sign is determined: |g| > 1e-4 of the bank's largest and > 1e-6
    (so Adam's eps = 1e-8 does not weigh in); the delay rule normalises each (re, im) tap pair
    and acts on the pair."""
    sig = (np.abs(g) > 1e-4 * np.abs(g).max()) & (np.abs(g) > 1e-6)
    if t == "d":
        sig = sig.copy()
        for c in range(2):
            b = 440 * c
            tap = sig[:, b:b + 20] & sig[:, b + 20:b + 40]
            sig[:, b:b + 20] = sig[:, b + 20:b + 40] = tap
    return sig


# ---------------------------------------------------------------------------
# config 2 against the oracle


def test_config2_train_step_matches_oracle(dev):
    """Config 2 (16 tracks + 4 subgroups, L = 441,000), one step against the oracle.

    The log-mel L1 gradient is dominated by weak spectral bins whose phase moves
    with any 1e-6-level change of the mix: the oracle's OWN dL/dy moves by several
    1e-4 between its float64 mix and the device's fp32 mix (measured,
    tools/diag_parity.py).  So the gates are: (1) the mix and loss
    end to end; (2) every bank's gradient with the oracle's loss linearised at the
    device's mix (same loss input on both sides), 1e-4; (3) end to end, every bank
    within 1e-4 plus twice the oracle's own gradient shift between the two mixes."""
    from oracle import mixgraph_oracle as O
    from paper_2509_15948_b200.console import init_params
    from paper_2509_15948_b200.scheduler import execute_batched
    K, S, L = 16, 4, 441_000
    graph, zeros, params, stems = _console(K, S, L, 0, 0)
    target = execute_batched(graph, init_params(zeros, 1), stems)[0].cpu().numpy()
    eng = _engine(graph, params, stems, target, L, dev)
    vals, grads, gw, y = eng.grads_only()
    args = (graph, {t: v.copy() for t, v in params.params.items()}, params.raw_weights.copy(),
            stems.astype(np.float64), target.astype(np.float64), 30000, O.LossConfig())
    ov, og, oy = O.render_loss_and_grads(*args)
    _, ogd, _ = O.render_loss_and_grads(*args, loss_point=y.astype(np.float64))
    np.testing.assert_allclose(vals["L_a"], ov["L_a"], rtol=LOSS_GATE)
    np.testing.assert_allclose(vals["L_g"], ov["L_g"], rtol=LOSS_GATE)
    s = 1.0 / (1.0 + np.exp(-params.raw_weights))
    grads = dict(grads, w=gw * s * (1 - s))
    forced = {t: normrel(grads[t], ogd[t], floor=FLOOR) for t in "gsecnrdw"}
    e2e = {t: normrel(grads[t], og[t], floor=FLOOR) for t in "gsecnrdw"}
    shift = {t: normrel(ogd[t], og[t], floor=FLOOR) for t in "gsecnrdw"}
    _report("config2 y", {"y": normrel(y, oy)})
    _report("config2 banks, loss at device mix", forced)
    _report("config2 banks end to end", e2e)
    _report("config2 oracle's own shift fp64 mix -> fp32 mix", shift)
    assert normrel(y, oy) < GATE
    assert max(forced.values()) < GATE, forced
    for t in e2e:
        assert e2e[t] < GATE + 2 * shift[t], (t, e2e[t], shift[t])


# ---------------------------------------------------------------------------
# the envelope scan's truncation regime


@pytest.mark.parametrize("tag", ["c", "n"])
@pytest.mark.parametrize("a_raw", [8.0, 10.0, 12.0])
def test_envelope_scan_regime_matches_reference_golden(dev, tag, a_raw):
    from golden_inputs import scan_inputs
    from paper_2509_15948_b200.processors import KERNELS
    gsn = golden("scan.npz")
    key = f"{tag}{int(a_raw)}"
    u, p, w = scan_inputs(tag, a_raw)
    ut = torch.tensor(u, dtype=torch.float32, device=dev, requires_grad=True)
    pt = torch.tensor(p, dtype=torch.float64, device=dev, requires_grad=True)
    ybar, _ = KERNELS[tag](ut, pt)
    torch.sum(ybar.double() * torch.tensor(w, device=dev)).backward()
    errs = {"ybar": normrel(ybar.detach().cpu().numpy(), gsn[f"{key}_ybar"]),
            "gu": normrel(ut.grad.cpu().numpy(), gsn[f"{key}_gu"]),
            "gp": normrel(pt.grad.cpu().numpy(), gsn[f"{key}_gp"])}
    _report(f"scan {key}", errs)
    assert max(errs.values()) < GATE, errs


@pytest.mark.parametrize("tag", ["c", "n"])
def test_envelope_scan_at_config3_length_matches_oracle(dev, tag):
    """L = 1,323,000 (config 3, 162 chunks), four rows from alpha_raw 5 to 11."""
    from golden_inputs import scan_inputs
    from oracle import mixgraph_oracle as O
    from paper_2509_15948_b200.processors import KERNELS
    L = 1_323_000
    u, p, w = scan_inputs(tag, 5.0, length=L, B=2, seed=11)
    u2, p2, w2 = scan_inputs(tag, 8.0, length=L, B=2, seed=12)
    u, w = np.concatenate([u, u2]), np.concatenate([w, w2])
    p = np.concatenate([p, p2])
    p[:, 0] = [5.0, 6.5, 8.0, 11.0]
    ut = torch.tensor(u, dtype=torch.float32, device=dev, requires_grad=True)
    pt = torch.tensor(p, dtype=torch.float64, device=dev, requires_grad=True)
    ybar, _ = KERNELS[tag](ut, pt)
    torch.sum(ybar.double() * torch.tensor(w, device=dev)).backward()
    uo = torch.tensor(u.astype(np.float32).astype(np.float64), requires_grad=True)
    po = torch.tensor(p, requires_grad=True)
    yo, _ = O.KERNELS[tag](uo, po)
    torch.sum(yo * torch.tensor(w)).backward()
    errs = {"ybar": normrel(ybar.detach().cpu().numpy(), yo.detach().numpy()),
            "gu": normrel(ut.grad.cpu().numpy(), uo.grad.numpy()),
            "gp": normrel(pt.grad.cpu().numpy(), po.grad.numpy())}
    _report(f"scan {tag} L=1323000", errs)
    assert max(errs.values()) < GATE, errs


# ---------------------------------------------------------------------------
# optimiser kernel


def _ref_optim():
    from oracle import build_ref
    mg = build_ref.load()
    if mg is None:
        return None
    import mixgraph.optimizer as RO
    return RO


def test_adamw_kernel_matches_reference_rule_adamw_projection(dev):
    """mgb_adamw_step on identical (p, g, dL/dw, m, v, t) vs the reference's
    _delay_gradient_rule + AdamW.step + project_delay_radius (mg/optimizer.py:82-137)
    and the raw-weight gradient of effective_weights + sparsity (alpha_p > 0), with
    |z| > 1, z = 0, zero raw gradients and a masked weight in the inputs."""
    from oracle import mixgraph_oracle as O
    from paper_2509_15948_b200._lib import check, lib
    from paper_2509_15948_b200.engine import ptr, stream_ptr
    rng = np.random.default_rng(42)
    rows = {"e": 3, "c": 3, "n": 3, "s": 3, "g": 3, "d": 3, "r": 3}
    counts = {"e": 1024, "c": 4, "n": 4, "s": 1, "g": 2, "d": 880, "r": 768}
    order = "ecnsgdr"
    banks = {t: rng.standard_normal((rows[t], counts[t])) for t in order}
    grads = {t: rng.standard_normal((rows[t], counts[t])) * 10.0 ** rng.uniform(-6, 0, (rows[t], counts[t]))
             for t in order}
    d, gd = banks["d"], grads["d"]
    d[0, 0], d[0, 20] = 0.0, 0.0            # z = 0
    d[1, 3], d[1, 23] = 2.0, -1.5           # |z| > 1 (projected)
    gd[2, 5], gd[2, 25] = 0.0, 0.0          # zero raw gradient: sgn(0) = 0
    gd[0, 440 + 7] = 0.0                    # real part only
    P = 21
    raw = rng.standard_normal(P) * 2
    gw = rng.standard_normal(P)
    mask = np.ones(P)
    mask[4] = 0.0
    alpha_p = 1e-4
    m0 = {k: rng.standard_normal(v.shape) * 1e-2 for k, v in banks.items()}
    v0 = {k: rng.random(v.shape) * 1e-3 for k, v in banks.items()}
    m0["w"], v0["w"] = rng.standard_normal(P) * 1e-2, rng.random(P) * 1e-3
    t_step, lr, b1, b2, eps, wd = 3, 0.01, 0.9, 0.999, 1e-8, 1e-2

    flat = lambda dct, w: np.concatenate([dct[t].ravel() for t in order] + [w])  # noqa: E731
    off = np.cumsum([0] + [rows[t] * counts[t] for t in order])
    d_off, w_off = int(off[order.index("d")]), int(off[-1])
    tp = lambda a: torch.tensor(a, dtype=torch.float64, device=dev)  # noqa: E731
    p_t, g_t = tp(flat(banks, raw)), tp(flat(grads, np.zeros(P)))
    m_t, v_t = tp(flat(m0, m0["w"])), tp(flat(v0, v0["w"]))
    sc = tp([lr, b1, b2, eps, wd, 1 - b1 ** t_step, 1 - b2 ** t_step, alpha_p])
    gw_t, mask_t, guard, halt = tp(gw), tp(mask), tp(1.5), tp(0.0)
    L = lib()
    check(L.mgb_adamw_step(ptr(p_t), ptr(g_t), ptr(m_t), ptr(v_t), p_t.numel(), d_off, rows["d"], w_off, P,
                           ptr(gw_t), ptr(mask_t), ptr(sc), ptr(guard), ptr(halt), stream_ptr()), "adamw")
    torch.cuda.synchronize()
    got_p, got_g = p_t.cpu().numpy(), g_t.cpu().numpy()

    # expected: the raw-weight gradient dL/draw = dL/dw * mask * s(1-s) + alpha_p * s(1-s)
    s = 1.0 / (1.0 + np.exp(-raw))
    g_raw = gw * mask * s * (1 - s) + alpha_p * s * (1 - s)
    np.testing.assert_allclose(got_g[w_off:], g_raw, rtol=1e-14, atol=0)
    for impl in filter(None, (_ref_optim(), O)):
        arrays = {t: banks[t].copy() for t in order}
        arrays["w"] = raw.copy()
        gr = {t: grads[t].copy() for t in order}
        gr["w"] = g_raw.copy()
        if impl is O:
            gr["d"] = O.delay_gradient_rule(arrays["d"], gr["d"])
            opt = O.AdamW(arrays, lr=lr, betas=(b1, b2), eps=eps, weight_decay=wd)
        else:
            gr["d"] = impl._delay_gradient_rule(arrays["d"], gr["d"])
            opt = impl.AdamW(arrays, lr=lr, betas=(b1, b2), eps=eps, weight_decay=wd)
        np.testing.assert_allclose(got_g[d_off:d_off + d.size], gr["d"].ravel(), rtol=1e-13, atol=1e-15)
        for k in arrays:
            opt.m[k][...] = m0[k]
            opt.v[k][...] = v0[k]
        opt.t = t_step - 1
        opt.step(arrays, gr)
        if impl is O:
            O.project_delay_radius(arrays["d"])
        else:
            class _PS:  # the reference projects a ParamStore's d bank
                pass
            ps = _PS()
            ps.params = {"d": arrays["d"]}
            impl.project_delay_radius(ps)
        want = flat(arrays, arrays["w"])
        np.testing.assert_allclose(got_p, want, rtol=1e-13, atol=1e-15)

    # non-finite guard: nothing moves, and the sticky flag keeps a later finite step frozen too
    snap = [x.clone() for x in (p_t, m_t, v_t)]
    guard.fill_(float("nan"))
    for g_val in (float("nan"), 2.0):
        guard.fill_(g_val)
        check(L.mgb_adamw_step(ptr(p_t), ptr(g_t), ptr(m_t), ptr(v_t), p_t.numel(), d_off, rows["d"], w_off, P,
                               ptr(gw_t), ptr(mask_t), ptr(sc), ptr(guard), ptr(halt), stream_ptr()), "adamw")
    torch.cuda.synchronize()
    assert float(halt) == 1.0
    for a, b in zip((p_t, m_t, v_t), snap):
        assert torch.equal(a, b)


def test_alpha_p_step_raw_weight_gradient_matches_oracle(dev):
    """A fine-tune step's sparsity term (alpha_p > 0, mg/optimizer.py:161-162): the raw-weight
    gradient assembled on the device and the rule-applied delay gradient vs the oracle."""
    from golden_inputs import step_spec
    from oracle import mixgraph_oracle as O
    gs = golden("step.npz")
    K, S, L, s_stems, s_p, _ = step_spec()
    graph, _, params, stems = _console(K, S, L, s_stems, s_p)
    eng = _engine(graph, params, stems, gs["target"], L, dev)
    ap = 1e-4
    eng.t = 0
    eng.step_async(ap)
    vals = eng.read_values()
    g = eng.grads.cpu().numpy()
    ov, og, _ = O.render_loss_and_grads(graph, {t: v.copy() for t, v in params.params.items()},
                                        params.raw_weights.copy(), stems.astype(np.float64), gs["target"], 30000,
                                        O.LossConfig(), alpha_p=ap)
    np.testing.assert_allclose(vals["loss"], ov["loss"], rtol=LOSS_GATE)
    np.testing.assert_allclose(vals["L_p"], ov["L_p"], rtol=1e-12)
    lay = eng.layout
    assert normrel(g[lay.w_off:], og["w"], floor=FLOOR) < GATE
    rule = O.delay_gradient_rule(params.params["d"], og["d"])
    got = g[lay.off["d"]:lay.off["d"] + rule.size].reshape(rule.shape)
    sig = np.abs(og["d"]) > FLOOR * np.abs(og["d"]).max()
    for c in range(2):
        b = 440 * c
        tap = sig[:, b:b + 20] | sig[:, b + 20:b + 40]
        sig[:, b:b + 20] = sig[:, b + 20:b + 40] = tap
    assert normrel(got[sig], rule[sig]) < GATE


# ---------------------------------------------------------------------------
# teacher-forced pruning rounds at config-2 scale (desk recipe eval set)


def test_pruning_rounds_config2_desk_recipe_make_the_oracles_decisions(dev, monkeypatch):
    """16 tracks + 4 subgroups (140 processors), a 441,000-sample session and the desk
    recipe's four 57,000-sample eval segments: a dry/wet pass and a brute-force pass,
    teacher-forced from the same state, tau and RNG stream, with device trials and with
    the float64 oracle's eval_loss give the same ledger and survivors."""
    from oracle import mixgraph_oracle as O
    from paper_2509_15948_b200 import pruning as P
    from paper_2509_15948_b200.common import rng_for
    from paper_2509_15948_b200.console import init_params
    from paper_2509_15948_b200.optimizer import Session, TrainConfig
    from paper_2509_15948_b200.scheduler import execute_batched
    from paper_2509_15948_b200.songs import DESK_SEGMENT
    K, S, L = 16, 4, 441_000
    graph, zeros, params, stems = _console(K, S, L, 5, 0)
    target = execute_batched(graph, init_params(zeros, 1), stems)[0].cpu().numpy()
    seg = DESK_SEGMENT / 30000
    cfg = P.PruneConfig(tolerance_relative=0.02, eval_segments=4, eval_segment_seconds=seg,
                        train=TrainConfig(segment_seconds=seg, warmup_seconds=1.0))
    session = Session(stems, target)
    eval_set = P.build_eval_set(session, cfg, device=dev)
    ws = cfg.train.warmup_len
    oseg = [(np.asarray(st, dtype=np.float64),
             O.prepare_target(np.asarray(tg, dtype=np.float32).astype(np.float64), O.LossConfig()))
            for st, tg in eval_set.segments]

    def oracle_eval(graph, params, mask, eval_set, schedule=None):
        return O.eval_loss(graph, params.params, params.raw_weights, mask, oseg, ws, O.LossConfig())

    def device_eval(graph, params, mask, es, schedule=None):
        return eval_set.engine(graph, params).loss(mask)

    n = len(graph.processor_nodes())
    la0 = oracle_eval(graph, params, np.ones(n), None)
    np.testing.assert_allclose(device_eval(graph, params, np.ones(n), None), la0, rtol=LOSS_GATE)
    tau = 0.02 * la0

    def run(pass_fn, fn):
        monkeypatch.setattr(P, "eval_loss", fn)
        state = P.PruneState(alive=np.ones(n, dtype=bool), la_min=la0, tolerance=tau, iteration=1)
        mask = pass_fn(state, graph, params, eval_set, np.ones(n), list(range(n)), rng_for(0, "prune-order"))
        return mask, state.ledger

    margins, worst = [], 0.0
    for pass_fn in (P.prune_drywet_pass, P.prune_bruteforce_pass):
        m_dev, led_dev = run(pass_fn, device_eval)
        m_ora, led_ora = run(pass_fn, oracle_eval)
        assert [(r.candidates, r.accepted) for r in led_dev] == [(r.candidates, r.accepted) for r in led_ora]
        np.testing.assert_array_equal(m_dev, m_ora)
        margins += [abs(r.loss - (r.la_min_before + tau)) / tau for r in led_ora]
        for a, b in zip(led_dev, led_ora):
            worst = max(worst, abs(a.loss - b.loss) / abs(b.loss))
        assert worst < LOSS_GATE
    print(f"config-2 desk pruning parity: {len(margins)} trials, min decision margin {min(margins):.3e} tau, "
          f"max trial-loss rel err {worst:.2e}")
