"""Pin the float64 oracle restatement against fixtures produced by the reference."""

import numpy as np
import pytest
import torch

from conftest import golden, normrel
from golden_inputs import kernel_inputs, mrstft_inputs, step_spec
from oracle import mixgraph_oracle as O


@pytest.mark.parametrize("tag", list("gsecndr"))
def test_oracle_kernel_matches_reference(tag):
    gk = golden("kernels.npz")
    u, p, w = kernel_inputs(tag)
    ut = torch.tensor(u, requires_grad=True)
    pt = torch.tensor(p, requires_grad=True)
    ybar, reg = O.KERNELS[tag](ut, pt)
    loss = torch.sum(ybar * torch.tensor(w))
    if reg is not None:
        loss = loss + reg
    loss.backward()
    assert normrel(ybar.detach().numpy(), gk[f"{tag}_ybar"]) < 1e-11
    assert abs(float(0.0 if reg is None else reg) - float(gk[f"{tag}_reg"])) <= 1e-10 * max(1, abs(float(gk[f"{tag}_reg"])))
    assert normrel(ut.grad.numpy(), gk[f"{tag}_gu"]) < 1e-10
    assert normrel(pt.grad.numpy(), gk[f"{tag}_gp"], floor=1e-9) < 1e-8


def test_oracle_tables_match_reference():
    gf = golden("fir.npz")
    specs, wss, nfr = O.reverb_tables()
    assert nfr == 313
    np.testing.assert_allclose(wss, gf["wss"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(specs["mid"][:4], gf["spec_mid_head"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(specs["side"][:4], gf["spec_side_head"], rtol=1e-12, atol=1e-12)
    cfg = O.LossConfig()
    np.testing.assert_allclose(O.projection(512, cfg), gf["mel512"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(O.projection(4096, cfg).sum(0), gf["mel4096_rowsum"], rtol=1e-12)
    fir = O.reverb_fir(torch.tensor(gf["pr"])).numpy()
    assert normrel(fir[..., :4096], gf["reverb_head"]) < 1e-12
    np.testing.assert_allclose(np.sqrt((fir ** 2).sum(-1)), gf["reverb_norm"], rtol=1e-12)
    eq = O.zero_phase_fir(torch.tensor(gf["pe"]), O.EQ_FIR_LEN).numpy()
    assert normrel(eq, gf["eq"]) < 1e-13


@pytest.mark.parametrize("name,sizes", [("std", (512, 1024, 4096)),
                                        ("six", (256, 512, 1024, 2048, 4096, 8192))])
def test_oracle_mrstft_matches_reference(name, sizes):
    gm = golden("mrstft.npz")
    y_hat, tgt = mrstft_inputs()
    yt = torch.tensor(y_hat, requires_grad=True)
    val = O.mrstft(yt, tgt, O.LossConfig(fft_sizes=sizes))
    val.backward()
    np.testing.assert_allclose(float(val), float(gm[f"{name}_loss"]), rtol=1e-12)
    assert normrel(yt.grad.numpy(), gm[f"{name}_grad"]) < 1e-10


def test_oracle_train_step_matches_reference():
    from paper_2509_15948_b200.console import build_console, init_params
    from workloads import SynthSpec, make_stems_f32, manifest_for

    gs = golden("step.npz")
    K, S, L, s_stems, s_p, s_t = step_spec()
    spec = SynthSpec(tracks=K, subgroups=S, duration_seconds=L / 30000)
    stems = make_stems_f32(spec, s_stems, L).astype(np.float64)
    np.testing.assert_array_equal(stems[..., :64], gs["stems_head"])
    graph, zeros = build_console(manifest_for(spec))
    params = init_params(zeros, s_p)
    p = {t: v.copy() for t, v in params.params.items()}
    raw = params.raw_weights.copy()
    cfg = O.LossConfig()
    values, grads, y = O.render_loss_and_grads(graph, p, raw, stems, gs["target"], 30000, cfg)
    assert normrel(y, gs["y"]) < 1e-11
    np.testing.assert_allclose(values["L_a"], float(gs["v_L_a"]), rtol=1e-10)
    np.testing.assert_allclose(values["L_g"], float(gs["v_L_g"]), rtol=1e-10)
    for t in "gsecnr":
        assert normrel(grads[t], gs[f"grad_{t}"], floor=1e-9) < 1e-7, t
    assert normrel(grads["w"], gs["grad_w"], floor=1e-9) < 1e-7
    assert normrel(grads["d"], gs["d_raw"], floor=1e-6) < 1e-6
    # two full steps (rule + AdamW + projection) on the reference's inputs
    opt = O.AdamW({**p, "w": raw})
    arrays_p = {t: v.copy() for t, v in params.params.items()}
    raw2 = params.raw_weights.copy()
    opt = O.AdamW({**arrays_p, "w": raw2})
    v1, _ = O.train_step(graph, arrays_p, raw2, stems, gs["target"], 30000, cfg, opt)
    v2, _ = O.train_step(graph, arrays_p, raw2, stems, gs["target"], 30000, cfg, opt)
    np.testing.assert_allclose(v2["L_a"], float(gs["v2_L_a"]), rtol=1e-9)
    for t in "gsecnr":
        np.testing.assert_allclose(arrays_p[t], gs[f"after2_{t}"], rtol=0, atol=1e-9)


@pytest.mark.parametrize("tag", ["c", "n"])
@pytest.mark.parametrize("a_raw", [8.0, 10.0, 12.0])
def test_oracle_envelope_scan_regime_matches_reference(tag, a_raw):
    """Compressor / gate at alpha_raw 8..12 over five 8192-sample chunks (the
    truncated-ballistics regime the device scan's correction term exists for)."""
    from golden_inputs import scan_inputs
    gsn = golden("scan.npz")
    key = f"{tag}{int(a_raw)}"
    u, p, w = scan_inputs(tag, a_raw)
    ut = torch.tensor(u, requires_grad=True)
    pt = torch.tensor(p, requires_grad=True)
    ybar, _ = O.KERNELS[tag](ut, pt)
    torch.sum(ybar * torch.tensor(w)).backward()
    # the golden signals are stored as float32 (relative rounding ~3e-8)
    assert normrel(ybar.detach().numpy(), gsn[f"{key}_ybar"]) < 1e-7
    assert normrel(ut.grad.numpy(), gsn[f"{key}_gu"]) < 1e-7
    assert normrel(pt.grad.numpy(), gsn[f"{key}_gp"]) < 1e-9


def test_oracle_config1_step_matches_reference():
    """BASELINE config 1 (4 tracks + 1 subgroup, L = 132,300): one train_step."""
    from golden_inputs import config1_spec
    from paper_2509_15948_b200.console import build_console, init_params
    from workloads import SynthSpec, make_stems_f32, manifest_for

    gs = golden("config1_step.npz")
    K, S, L, s_stems, s_p, s_t = config1_spec()
    spec = SynthSpec(tracks=K, subgroups=S, duration_seconds=L / 30000)
    stems = make_stems_f32(spec, s_stems, L).astype(np.float64)
    np.testing.assert_array_equal(stems[..., :64], gs["stems_head"])
    graph, zeros = build_console(manifest_for(spec))
    params = init_params(zeros, s_p)
    p = {t: v.copy() for t, v in params.params.items()}
    raw = params.raw_weights.copy()
    target = gs["target"].astype(np.float64)
    values, grads, y = O.render_loss_and_grads(graph, p, raw, stems, target, 30000, O.LossConfig())
    assert normrel(y, gs["y"]) < 1e-7  # golden y stored as float32
    np.testing.assert_allclose(values["L_a"], float(gs["v_L_a"]), rtol=1e-10)
    np.testing.assert_allclose(values["L_g"], float(gs["v_L_g"]), rtol=1e-10)
    for t in "gsecnr":
        assert normrel(grads[t], gs[f"grad_{t}"], floor=1e-9) < 1e-7, t
    assert normrel(grads["w"], gs["grad_w"], floor=1e-9) < 1e-7
    assert normrel(grads["d"], gs["d_raw"], floor=1e-6) < 1e-6
    opt = O.AdamW({**p, "w": raw})
    O.train_step(graph, p, raw, stems, target, 30000, O.LossConfig(), opt)
    for t in "gsecnr":
        np.testing.assert_allclose(p[t], gs[f"after_{t}"], rtol=0, atol=1e-9)


@pytest.mark.parametrize("name,ls", [("short1000", 1000), ("short3000", 3000)])
def test_oracle_mrstft_short_signals_match_reference(name, ls):
    """Scored signals shorter than the frames' reflect pad (mg/engine.py:640-645)."""
    gm = golden("mrstft.npz")
    y_hat, tgt = mrstft_inputs()
    yt = torch.tensor(y_hat[:, :ls].copy(), requires_grad=True)
    val = O.mrstft(yt, tgt[:, :ls].copy(), O.LossConfig(fft_sizes=(256, 512, 1024, 2048, 4096, 8192)))
    val.backward()
    np.testing.assert_allclose(float(val.detach()), float(gm[f"{name}_loss"]), rtol=1e-12)
    assert normrel(yt.grad.numpy(), gm[f"{name}_grad"]) < 1e-10
