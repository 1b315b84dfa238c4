"""CPU tests pinning the host-side API mirror to the REFERENCE itself.

The reference package's classes, console construction and prune entry points
stay the API (north_star).  This repo's host modules (graph, console,
schedule, pruning control flow, workloads) restate them so that the product
path does not import the reference; these tests build the same objects with
the reference (imported from /root/reference, or from the archive
``oracle/build_ref.py`` makes) and with this repo and require identical
objects, plans, bytes and decisions.  Skipped where the reference is absent.
"""

import math

import numpy as np
import pytest

from oracle import build_ref

MG = build_ref.load()
pytestmark = pytest.mark.skipif(MG is None, reason="reference package unavailable")


def _ref():
    import mixgraph.common as C
    import mixgraph.console as Co
    import mixgraph.graph as G
    import mixgraph.pruning as Pr
    import mixgraph.scheduler as S
    import mixgraph.synth as Sy
    return C, Co, G, S, Pr, Sy


def _manifests():
    out = []
    for k, s in ((1, 1), (4, 1), (5, 2), (16, 4), (24, 6)):
        out.append((k, s))
    return out


def _both_manifests(k, s):
    from paper_2509_15948_b200 import console as ours
    _, Co, *_ = _ref()
    tr = [(f"t{i}.wav", f"t{i}", f"bus{i % s}") for i in range(k)]
    return (ours.SessionManifest([ours.TrackEntry(*t) for t in tr], "m.wav"),
            Co.SessionManifest([Co.TrackEntry(*t) for t in tr], "m.wav"))


def _same_graph(a, b):
    assert a.node_types == b.node_types
    assert tuple(a.edges) == tuple(b.edges)


def _same_params(a, b):
    assert sorted(a.params) == sorted(b.params)
    for t in a.params:
        np.testing.assert_array_equal(a.params[t], b.params[t])
    np.testing.assert_array_equal(a.raw_weights, b.raw_weights)


def _same_schedule(a, b):
    assert a.type_sequence == b.type_sequence
    assert [list(x) for x in a.subsets] == [list(x) for x in b.subsets]
    assert sorted(a.type_perm) == sorted(b.type_perm)
    for t in a.type_perm:
        np.testing.assert_array_equal(a.type_perm[t], b.type_perm[t])
    assert len(a.plans) == len(b.plans)
    for pa, pb in zip(a.plans, b.plans):
        assert [tuple(x) for x in pa.gather] == [tuple(x) for x in pb.gather]
        assert pa.batch == pb.batch and pa.pslice == pb.pslice
        for x, y in ((pa.segments, pb.segments), (pa.weight_idx, pb.weight_idx)):
            assert (x is None) == (y is None)
            if x is not None:
                np.testing.assert_array_equal(x, y)


def test_common_helpers_match_reference():
    from paper_2509_15948_b200 import common as ours
    C, *_ = _ref()
    for seed, label in ((0, "segments"), (7, "prune-order"), (123, "stem-3"), (0x5EED0001, "reverb-mid")):
        np.testing.assert_array_equal(ours.rng_for(seed, label).standard_normal(16),
                                      C.rng_for(seed, label).standard_normal(16))
    for x in (-2.5, -1.5, -0.5, 0.5, 1.5, 2.5, 3.49, 7.0):
        assert ours.round_half_away(x) == C.round_half_away(x)
    for s in (0.0, 1.0, 1.9, 3.8, 441000 / 30000, 1323000 / 30000):
        assert ours.seconds_to_samples(s) == C.seconds_to_samples(s)
    assert ours.SAMPLE_RATE == C.SAMPLE_RATE


@pytest.mark.parametrize("k,s", _manifests())
def test_console_and_init_params_match_reference(k, s):
    from paper_2509_15948_b200 import console as ours
    _, Co, *_ = _ref()
    mo, mr = _both_manifests(k, s)
    go, zo = ours.build_console(mo)
    gr, zr = Co.build_console(mr)
    _same_graph(go, gr)
    _same_params(zo, zr)
    for seed in (0, 1, 5):
        _same_params(ours.init_params(zo, seed), Co.init_params(zr, seed))


@pytest.mark.parametrize("k,s", _manifests())
def test_console_schedules_and_plans_match_reference(k, s):
    from paper_2509_15948_b200 import console as ours
    from paper_2509_15948_b200 import schedule as osch
    from paper_2509_15948_b200.scheduler import node_schedule
    _, Co, G, S, *_ = _ref()
    mo, mr = _both_manifests(k, s)
    go, _ = ours.build_console(mo)
    gr, _ = Co.build_console(mr)
    _same_schedule(osch.plan_indices(go, osch.schedule_console(go)), S.plan_indices(gr, S.schedule_console(gr)))
    _same_schedule(osch.plan_indices(go, osch.schedule_greedy(go)), S.plan_indices(gr, S.schedule_greedy(gr)))
    # the node-at-a-time schedule visits the reference executor's topological order
    assert [v for sub in node_schedule(go).subsets[1:-1] for v in sub] == \
        [v for v in G.topological_order(gr) if gr.node_types[v] not in "io"]


def _random_dag(rng, MixGraph, PROCESSOR_TYPES):
    # tests/helpers.py:10-32 recipe (random valid typed DAG)
    k = int(rng.integers(1, 5))
    types, edges = list("i" * k), []
    for _ in range(int(rng.integers(0, 13))):
        nid = len(types)
        if rng.random() < 0.7:
            types.append(PROCESSOR_TYPES[int(rng.integers(0, len(PROCESSOR_TYPES)))])
            edges.append((int(rng.integers(0, nid)), nid))
        else:
            preds = rng.choice(nid, size=int(rng.integers(1, min(3, nid) + 1)), replace=False)
            types.append("m")
            edges.extend((int(p), nid) for p in preds)
    sinks = [v for v in range(len(types)) if all(a != v for a, _ in edges)]
    out = len(types)
    types.append("o")
    edges.extend((v, out) for v in sinks)
    return MixGraph("".join(types), tuple(edges))


def test_greedy_schedules_on_random_dags_match_reference():
    from paper_2509_15948_b200 import graph as og
    from paper_2509_15948_b200 import schedule as osch
    _, _, G, S, *_ = _ref()
    for seed in range(60):
        go = _random_dag(np.random.default_rng(seed), og.MixGraph, og.PROCESSOR_TYPES)
        gr = _random_dag(np.random.default_rng(seed), G.MixGraph, G.PROCESSOR_TYPES)
        _same_graph(go, gr)
        _same_schedule(osch.plan_indices(go, osch.schedule_greedy(go)), S.plan_indices(gr, S.schedule_greedy(gr)))
        assert list(og.topological_order(go)) == list(G.topological_order(gr))


def test_validation_errors_match_reference():
    from paper_2509_15948_b200 import graph as og
    _, _, G, *_ = _ref()
    bad = [("ipo", ((0, 1), (1, 2), (1, 2))), ("igo", ((0, 1), (1, 0), (1, 2))), ("iggo", ((0, 2), (1, 2), (2, 3))),
           ("igoo", ((0, 1), (1, 2), (1, 3))), ("igo", ((0, 1),)), ("io", ())]
    for types, edges in bad:
        errs = []
        for mod in (og, G):
            try:
                mod.validate(mod.MixGraph(types, edges))
                errs.append(None)
            except Exception as e:  # noqa: BLE001 — the class name and message are compared
                errs.append((type(e).__name__, str(e)))
        assert errs[0] == errs[1], (types, edges, errs)


def test_bypass_remove_and_serialize_match_reference():
    from paper_2509_15948_b200 import console as ours
    from paper_2509_15948_b200 import graph as og
    _, Co, G, *_ = _ref()
    mo, mr = _both_manifests(6, 2)
    go, zo = ours.build_console(mo)
    gr, zr = Co.build_console(mr)
    po, pr = ours.init_params(zo, 2), Co.init_params(zr, 2)
    rng = np.random.default_rng(0)
    for _ in range(8):
        procs = go.processor_nodes()
        drop = set(int(v) for v in rng.choice(procs, size=int(rng.integers(1, len(procs) // 3)), replace=False))
        g2o, p2o = og.bypass_remove(go, po, drop)
        g2r, p2r = G.bypass_remove(gr, pr, drop)
        _same_graph(g2o, g2r)
        _same_params(p2o, p2r)
        bo, br = og.serialize(g2o, p2o), G.serialize(g2r, p2r)
        assert bo == br  # byte-identical .mixgraph.json
        g3, p3 = og.deserialize(br)
        _same_graph(g3, g2r)
        _same_params(p3, p2r)
        go, po, gr, pr = g2o, p2o, g2r, p2r
        if len(go.processor_nodes()) < 6:
            break


def test_stems_match_reference_bitwise():
    from workloads import SynthSpec, make_stems
    *_, Sy = _ref()
    for k, s, seed in ((2, 1, 3), (5, 2, 11)):
        a, ka = make_stems(SynthSpec(tracks=k, subgroups=s, duration_seconds=0.5), seed)
        b, kb = Sy.make_stems(Sy.SynthSpec(tracks=k, subgroups=s, duration_seconds=0.5), seed)
        assert ka == kb
        np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------------------
# the whole prune_song control flow, with deterministic stand-ins for the device
# work (train / eval_loss): identical ledgers, survivors and final graphs


def _fake_eval(graph, params, mask, eval_set, schedule=None):
    # a deterministic function of the alive processors' parameters: removing a
    # processor adds a parameter-dependent amount (some negative), so passes both
    # accept and reject trials
    raw = np.asarray(params.raw_weights, dtype=np.float64)
    m = np.asarray(mask, dtype=np.float64)
    gone = (1.0 - m) * (0.004 * (0.35 + np.sin(17.0 * raw + 1.0)))
    return float(1.0 + gone.sum() + 1e-3 * len(graph.node_types))


def _fake_train(graph, params, session, cfg, *args, rng=None, history=None, alpha_p_fn=None, **kw):
    # deterministic "fine-tune": consumes the segment RNG like train() and nudges the weights
    history = history if history is not None else []
    for step in range(cfg.steps):
        rng.integers(0, session.length - cfg.segment_len + 1)
        a = alpha_p_fn(step) if alpha_p_fn else 0.0
        params.raw_weights = params.raw_weights * 0.999 + 0.01 * math.sin(len(history)) + a
        history.append({"step": len(history)})
    return history


@pytest.mark.parametrize("mode,speculate", [("hybrid", 1), ("bruteforce", 1), ("drywet", 1), ("hybrid", 4),
                                            ("bruteforce", 3)])
def test_prune_song_control_flow_matches_reference(monkeypatch, mode, speculate):
    """Also with speculative brute-force batches (``speculate`` trials requested per
    render under the reject assumption): the same ledger as the reference's sequential loop."""
    from paper_2509_15948_b200 import console as ours
    from paper_2509_15948_b200 import graph as og
    from paper_2509_15948_b200 import pruning as op
    from paper_2509_15948_b200.optimizer import Session, TrainConfig
    _, Co, G, _, Pr, _ = _ref()
    import mixgraph.optimizer as RO
    for mod in (op, Pr):
        monkeypatch.setattr(mod, "eval_loss", _fake_eval)
        monkeypatch.setattr(mod, "train", _fake_train)
    requests = []

    def fake_losses(g, p, masks, es, schedule=None):
        requests.append(len(masks))
        return [_fake_eval(g, p, m, es) for m in masks]

    monkeypatch.setattr(op, "eval_losses", fake_losses)
    mo, mr = _both_manifests(6, 2)
    go, zo = ours.build_console(mo)
    gr, zr = Co.build_console(mr)
    L = 45_000
    rng = np.random.default_rng(1)
    stems, target = 0.1 * rng.standard_normal((6, 2, L)), 0.1 * rng.standard_normal((2, L))
    kw = dict(tolerance_relative=0.02, mode=mode, iterations=8, seed=3, console_steps=5, finetune_steps=3,
              eval_segments=2, eval_segment_seconds=1.2, sparsity_ramp_steps=7)
    tc = dict(segment_seconds=1.2, warmup_seconds=1.0, seed=3)
    out_o = op.prune_song(go, ours.init_params(zo, 4), Session(stems, target),
                          op.PruneConfig(**kw, train=TrainConfig(**tc)), device="cpu", speculate=speculate)
    if speculate > 1 and mode != "drywet":
        assert max(requests) == speculate  # brute-force trials were requested in batches
    out_r = Pr.prune_song(gr, Co.init_params(zr, 4), RO.Session(stems, target),
                          Pr.PruneConfig(**kw, train=RO.TrainConfig(**tc)))
    (g_o, p_o, s_o, rep_o, _), (g_r, p_r, s_r, rep_r, _) = out_o, out_r
    assert [(r.iteration, r.mode, tuple(r.candidates), r.loss, r.la_min_before, r.accepted) for r in s_o.ledger] == \
        [(r.iteration, r.mode, tuple(r.candidates), r.loss, r.la_min_before, r.accepted) for r in s_r.ledger]
    assert any(r.accepted for r in s_r.ledger) and not all(r.accepted for r in s_r.ledger)
    np.testing.assert_array_equal(s_o.alive, s_r.alive)
    _same_graph(g_o, g_r)
    _same_params(p_o, p_r)
    assert og.serialize(g_o, p_o) == G.serialize(g_r, p_r)
    for f in ("console_loss", "final_loss", "la_min", "tolerance", "mode", "console_counts", "pruned_counts",
              "trial_count"):
        assert getattr(rep_o, f) == getattr(rep_r, f), f


def test_source_errors_match_reference():
    """execute_batched's input errors (mg/scheduler.py:207-215) are raised before any device
    work, with the reference's exception class and message."""
    from paper_2509_15948_b200 import console as ours
    from paper_2509_15948_b200.scheduler import execute_batched
    _, Co, _, S, *_ = _ref()
    mo, mr = _both_manifests(3, 1)
    go, zo = ours.build_console(mo)
    gr, zr = Co.build_console(mr)
    cases = [np.zeros((2, 2, 100)), [np.zeros((2, 100)), np.zeros((2, 100)), np.zeros((2, 90))]]
    for src in cases:
        errs = []
        for fn, g, z in ((execute_batched, go, zo), (S.execute_batched, gr, zr)):
            with pytest.raises(Exception) as e:
                fn(g, z, src)
            errs.append((type(e.value).__name__, str(e.value)))
        assert errs[0] == errs[1], errs
