"""GPU parity of the reference-parity path (residual-MLP block, fp64 / fp32)
against the reference's golden vectors (oracle/make_golden.py) and the
numpy oracle.  Tolerances:
  * counter-RNG init, recover_checkfree fp64, schedules: bit-exact
  * fp64 GPU pipeline vs the fp64 CPU reference: rel 1e-9 (FMA / summation order only)
  * fp32 mode: recovered weights rel <= 1e-5 (north_star), loss curves within 1%
"""
import math

import numpy as np
import pytest

import ckfree_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2506_15461_b200")


def test_counter_uniform_bit_exact(goldens):
    for key, lo, hi, want in goldens["rng"]["counter_uniform"]:
        assert P.counter_uniform(key, lo, hi, len(want)).tolist() == want
    big = P.counter_uniform(0xDEADBEEF, -0.37, 0.37, 1 << 20)
    assert np.array_equal(big, O.counter_uniform(0xDEADBEEF, -0.37, 0.37, 1 << 20))


def test_recover_checkfree_seam_bit_exact(goldens):
    for c in goldens["recovery"]["checkfree"]:
        out, deg = P.recover_checkfree(np.array(c["wp"]), np.array(c["wn"]), c["op"], c["on"])
        assert out.tolist() == c["out"]
        assert deg == c["degenerate"]
    # large vector, several omega pairs incl. degenerate and one-sided
    n = 3_000_017
    wp = O.counter_uniform(O.derive_key(5, 1), -1, 1, n)
    wn = O.counter_uniform(O.derive_key(5, 2), -1, 1, n)
    for op, on in ((4.0, 1.0), (0.0, 0.0), (1.0, 0.0), (0.0, 2.5), (1e-30, 3e-30), (123.456, 0.001)):
        out, deg = P.recover_checkfree(wp, wn, op, on)
        want, wdeg = O.recover_checkfree(wp, wn, op, on)
        assert np.array_equal(out, want), (op, on)
        assert deg == wdeg
    with pytest.raises(P.ConfigError):
        P.recover_checkfree(wp[:4], wn[:4], -1.0, 1.0)


def test_adam_and_omega_seam(goldens):
    a = goldens["recovery"]["adam"]
    g = O.counter_uniform(a["g_key"], -1, 1, 16)
    w = O.counter_uniform(a["w_key"], -1, 1, 16)
    m = np.zeros(16)
    v = np.zeros(16)
    for t in a["trace"]:
        w, m, v = P.adam_update(w, m, v, g * t["step"], a["lr"], t["step"])
        np.testing.assert_allclose(w, t["w"], rtol=1e-15, atol=0)
        np.testing.assert_allclose(m, t["m"], rtol=1e-15)
        np.testing.assert_allclose(v, t["v"], rtol=1e-15)
    for c in goldens["recovery"]["sum_squares"]:
        x = O.counter_uniform(c["key"], -1, 1, c["n"])
        assert P.sum_squares(x) == pytest.approx(c["sum_squares"], rel=1e-14)


@pytest.mark.parametrize("kind", ["nn", "nn_acc", "nt_acc", "tn_acc"])
def test_gemm_seam_vs_numpy(kind):
    rng = np.random.default_rng(3)
    for m, k, n in ((1, 1, 1), (5, 3, 7), (33, 65, 17), (128, 96, 200)):
        c0 = rng.standard_normal((m, n))
        if kind == "nn":
            a, b = rng.standard_normal((m, k)), rng.standard_normal((k, n))
            want = a @ b
        elif kind == "nn_acc":
            a, b = rng.standard_normal((m, k)), rng.standard_normal((k, n))
            want = c0 + a @ b
        elif kind == "nt_acc":
            a, b = rng.standard_normal((m, k)), rng.standard_normal((n, k))
            want = c0 + a @ b.T
        else:
            a, b = rng.standard_normal((k, m)), rng.standard_normal((k, n))
            want = c0 + a.T @ b
        got = P.gemm(kind, a, b, c0, m, k, n)
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


def _tiny_engine(goldens, precision="fp64"):
    cfg = goldens["model"]["tiny_cfg"]
    spec = P.ModelSpec(cfg["input-dim"], cfg["hidden-dim"], cfg["model-dim"], cfg["output-dim"], cfg["layers"],
                       cfg["stages"], precision=precision, max_rows=64)
    return P.Engine(spec)


def _flat(eng):
    return np.concatenate([eng.export_edge(0)[0], eng.export_edge(1)[0]] +
                          [eng.export_stage(s)[0] for s in range(1, eng.spec.num_stages + 1)])


def test_engine_init_bit_exact(goldens):
    eng = _tiny_engine(goldens)
    eng.init(42, 1e-3)
    assert _flat(eng).tolist() == goldens["model"]["tiny_init_seed42"]
    e32 = _tiny_engine(goldens, "fp32")
    e32.init(42, 1e-3)
    assert np.array_equal(_flat(e32), np.array(goldens["model"]["tiny_init_seed42"]).astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("precision,rtol", [("fp64", 1e-11), ("fp32", 2e-5)])
def test_run_iteration_vs_reference(goldens, precision, rtol):
    g = goldens["model"]
    x, y = np.array(g["tiny_batch_iter1"]["x"]), np.array(g["tiny_batch_iter1"]["y"])
    eng = _tiny_engine(goldens, precision)
    for mode, sw in (("standard", False), ("swapped_half", True)):
        eng.init(42, 1e-3)
        loss, om = eng.run_iteration(P.api.build_schedule(2, sw, 4), x, y, 1)
        want = g["tiny_run_iteration"][mode]
        assert loss == pytest.approx(want["loss"], rel=rtol)
        np.testing.assert_allclose(om, want["omegas"], rtol=rtol * 10)
        np.testing.assert_allclose(_flat(eng), want["flat"], rtol=rtol * 10, atol=1e-7 if precision == "fp32" else 1e-13)


def test_indivisible_batch_is_config_error(goldens):
    eng = _tiny_engine(goldens)
    eng.init(1, 1e-3)
    with pytest.raises(P.ConfigError):
        eng.run_iteration(P.api.build_schedule(4, False, 4), np.zeros((6, 3)), np.zeros((6, 3)), 1)
    with pytest.raises(P.ConfigError):
        eng.run_iteration([[1, 2, 2, 4]], np.zeros((2, 3)), np.zeros((2, 3)), 1)


def test_non_finite_raises_divergence_with_iteration(goldens):
    eng = _tiny_engine(goldens)
    eng.init(12, 1e-3)
    w, _, _ = eng.export_edge(0)
    w[0] = math.inf
    eng.import_edge(0, w)
    with pytest.raises(P.NumericDivergenceError) as ei:
        eng.run_iteration([[1, 2, 3, 4]], np.ones((2, 3)), np.zeros((2, 3)), 41)
    assert ei.value.iteration == 41


def _compare_run(run, precision, rel_loss, rel_red):
    cfg = dict(run["cfg"])
    cfg["precision"] = precision
    evals, events, unrec = P.run_experiment(cfg, run["trace"], run["seed"])
    w_evals, w_events, w_unrec = O.parse_full_record(run["full"])
    assert (unrec is not None) == w_unrec
    assert [e[0] for e in evals] == [e[0] for e in w_evals]
    for (it, tr, va), (_, wtr, wva) in zip(evals, w_evals):
        assert tr == pytest.approx(wtr, rel=rel_loss), ("train", it)
        assert va == pytest.approx(wva, rel=rel_loss), ("val", it)
    assert [(e[0], e[1], e[2]) for e in events] == [(e[0], e[1], e[2]) for e in w_events]
    for e, w in zip(events, w_events):
        assert e[3] == pytest.approx(w[3], rel=rel_red)
    return evals, events


TRAINER_CASES = ["checkfree_s2_at50", "checkfree_plus_s1_at50", "checkfree_plus_s4_s2_at30_70",
                 "checkfree_averaged_moments", "checkfree_plus_averaged_edge", "reinit_uniform_avg", "reinit_copy",
                 "reinit_random", "no_failures", "unrecoverable_adjacent", "checkfree_edge_unsupported",
                 "classification_checkfree", "relu_checkfree_plus", "failure_at_iter1", "checkfree_plus_swap_from_40",
                 "s8_checkfree_plus_trace", "checkpointing_s2_at50", "checkpointing_edge_and_adjacent",
                 "checkpointing_at_snapshot", "redundant_s2_at50", "redundant_edges_and_middle",
                 "redundant_adjacent_unrecoverable"]


@pytest.mark.parametrize("name", TRAINER_CASES)
def test_trainer_fp64_matches_reference(trainer_goldens, name):
    run = next(r for r in trainer_goldens["runs"] if r["name"] == name)
    _compare_run(run, "fp64", rel_loss=1e-8, rel_red=1e-8)


@pytest.mark.parametrize("name", ["checkfree_s2_at50", "checkfree_plus_s1_at50", "checkfree_averaged_moments",
                                  "classification_checkfree", "s8_checkfree_plus_trace", "checkpointing_s2_at50"])
def test_trainer_fp32_loss_curve_within_1pct(trainer_goldens, name):
    run = next(r for r in trainer_goldens["runs"] if r["name"] == name)
    _compare_run(run, "fp32", rel_loss=1e-2, rel_red=1e-2)


def test_fp32_recovered_weights_within_1e5(goldens):
    """north_star: fp32 mode <= 1e-5 relative on recovered weights."""
    cfg = goldens["model"]["tiny_cfg"]
    for precision in ("fp32", "fp64"):
        eng = _tiny_engine(goldens, precision)
        eng.init(42, 1e-3)
        x, y = np.array(goldens["model"]["tiny_batch_iter1"]["x"]), np.array(goldens["model"]["tiny_batch_iter1"]["y"])
        eng.run_iteration(P.api.build_schedule(2, False, 4), x, y, 1)
        wp, _, _ = eng.export_stage(1)
        wn, _, _ = eng.export_stage(3)
        op, _, _ = eng.scalars(1)
        on, _, _ = eng.scalars(3)
        lr_before = eng.scalars(2)[1]
        eng.kill_stage(2)
        r = eng.recover_stage(2, P._native.CKF_REC_CHECKFREE)
        got, m, v = eng.export_stage(2)
        want, _ = O.recover_checkfree(wp, wn, op, on)
        if precision == "fp64":
            assert np.array_equal(got, want)
        else:
            np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-7)
        assert not r.degenerate and r.latency_ms > 0
        assert np.all(m == 0) and np.all(v == 0)
        om, lr, step = eng.scalars(2)
        assert om == 0.0 and step == 0 and lr == pytest.approx(1.1 * lr_before, rel=1e-15)


def test_run_records_in_reference_schema(tmp_path, trainer_goldens):
    """run_experiment_to_dir (experiment.cpp:202-213): the four artefacts in the reference's schema;
    metrics.csv / events.csv equal the reference's own files except the time columns (modeled there,
    measured here)."""
    import json
    run = next(r for r in trainer_goldens["runs"] if r["name"] == "checkfree_s2_at50")
    P.api.run_experiment_to_dir(run["cfg"], run["trace"], run["seed"], str(tmp_path))

    def strip(text, col):  # drop one column (wall_hours / recovery_s)
        return [",".join(f for i, f in enumerate(l.split(",")) if i != col) if not l.startswith("#") else l
                for l in text.strip().splitlines()]

    ours = strip((tmp_path / "metrics.csv").read_text(), 3)
    ref = strip(run["metrics_csv"], 3)
    assert ours[:2] == ref[:2] and len(ours) == len(ref)
    for a, b in zip(ours[2:], ref[2:]):
        fa, fb = a.split(","), b.split(",")
        assert fa[0] == fb[0]
        for x, y in zip(fa[1:], fb[1:]):
            assert float(x) == pytest.approx(float(y), rel=1e-9)
    oe = strip((tmp_path / "events.csv").read_text(), 4)
    re_ = strip(run["events_csv"], 4)
    assert oe[:2] == re_[:2] and len(oe) == len(re_)
    for a, b in zip(oe[2:], re_[2:]):
        fa, fb = a.split(","), b.split(",")
        assert fa[:3] == fb[:3] and float(fa[3]) == pytest.approx(float(fb[3]), rel=1e-6)
    s = json.loads((tmp_path / "summary.json").read_text())
    assert s["format_version"] == 1 and s["strategy"] == "checkfree" and s["failure_events"] == 1
    assert "strategy = checkfree" in (tmp_path / "config.resolved").read_text()
