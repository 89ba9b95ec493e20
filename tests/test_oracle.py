"""Pins the numpy oracle restatement (oracle/ckfree_oracle.py) to the golden
vectors produced by the UNMODIFIED reference library (oracle/make_golden.py).
CPU only."""
import numpy as np
import pytest

import ckfree_oracle as O


def test_rng_goldens(goldens):
    g = goldens["rng"]
    for x, want in g["mix64"]:
        assert O.mix64(x) == want
    for args, want in g["derive_key"]:
        assert O.derive_key(*args) == want
    for args, want in g["unit_at"]:
        assert O.unit_at(*args) == want
    for key, lo, hi, want in g["counter_uniform"]:
        assert O.counter_uniform(key, lo, hi, len(want)).tolist() == want  # bit-exact
    # SURVEY §8 a1 literal values
    assert O.mix64(0) == 0xE220A8397B1DCDAF
    assert O.derive_key(1) == 0x5BFAC50FA2FDEED6
    assert O.unit_at(42, 1, 2) == 0.16375111789623975


def test_failure_trace_goldens(goldens):
    g = goldens["failures"]
    for p, s, want in g["p_iter"]:
        assert O.hourly_to_per_iteration(p, s) == want
    for c in g["traces"]:
        ev = O.generate_trace(c["seed"], c["p_hour"], c["iter_s"], c["iters"], c["stages"])
        text = O.serialize_trace(c["seed"], c["p_hour"], c["iter_s"], c["stages"], ev)
        assert text == c["trace"]  # byte-identical checkfree-trace v1
        seed, p, it_s, st, ev2 = O.parse_trace(c["trace"])
        assert (seed, st, ev2) == (c["seed"], c["stages"], ev)
    first = g["traces"][0]
    assert O.parse_trace(first["trace"])[4] == [(7, 5), (178, 2), (326, 4), (403, 2), (451, 3), (459, 5)]


def test_partition_and_schedule_goldens(goldens):
    g = goldens["partition_schedule"]
    for c in g["partitions"]:
        assert [list(r) for r in O.even_partition(c["layers"], c["stages"])] == [list(r) for r in c["ranges"]]
    for c in g["schedules"]:
        assert O.build_schedule(c["m"], c["swapped_half"], c["s"]) == c["orders"]
    for c in g["schedule_errors"]:
        with pytest.raises(ValueError):
            O.build_schedule(c["m"], c["swapped_half"], c["s"])


def test_recovery_goldens(goldens):
    g = goldens["recovery"]
    for c in g["checkfree"]:
        out, deg = O.recover_checkfree(np.array(c["wp"]), np.array(c["wn"]), c["op"], c["on"])
        assert out.tolist() == c["out"]  # bit-exact (no FMA on either side)
        assert deg == c["degenerate"]
    assert g["checkfree"][0]["out"] == [0.8, 0.2]
    c = g["checkfree"][3]
    wf = O.counter_uniform(g["reduction_error"]["wf_key"], -1, 1, 64)
    assert O.reduction_error(np.array(c["wp"]), wf, np.array(c["wn"]), c["op"], c["on"]) == pytest.approx(
        g["reduction_error"]["value"], rel=1e-14)
    for lr, f, want in g["bump_lr"]:
        assert O.bump_lr(lr, f) == want
    for c in g["sum_squares"]:
        x = O.counter_uniform(c["key"], -1, 1, c["n"])
        assert O.sum_squares(x) == c["sum_squares"]  # same reduction order -> bit-exact
    a = g["adam"]
    gg = O.counter_uniform(a["g_key"], -1, 1, 16)
    w = O.counter_uniform(a["w_key"], -1, 1, 16)
    m = np.zeros(16)
    v = np.zeros(16)
    for t in a["trace"]:
        w, m, v = O.adam_update(w, m, v, gg * t["step"], a["lr"], t["step"])
        assert w.tolist() == t["w"] and m.tolist() == t["m"] and v.tolist() == t["v"]


def test_model_goldens(goldens):
    g = goldens["model"]
    spec = O.Spec.from_cfg(g["tiny_cfg"])
    m = O.init_model(spec, 42, 1e-3)
    assert m.all_weights_flat().tolist() == g["tiny_init_seed42"]  # bit-exact init
    dspec = O.Spec.from_cfg(g["desk_cfg"])
    dm = O.init_model(dspec, g["desk_init_seed"], 3e-4)
    flat = dm.all_weights_flat()
    assert flat.size == g["desk_init_n"]
    assert flat[:32].tolist() == g["desk_init_head"]
    task = O.Task(dspec, 1)
    x, y = task.training_batch(1, 16)
    assert x.tolist() == g["desk_batch_iter1_rows16"]["x"]
    np.testing.assert_allclose(y, g["desk_batch_iter1_rows16"]["y"], rtol=1e-12, atol=1e-13)
    vx, vy = task.validation_set(4)
    assert vx.tolist() == g["desk_val_rows4"]["x"]
    # one pipeline iteration, standard and swapped-half
    tb = g["tiny_batch_iter1"]
    x, y = np.array(tb["x"]), np.array(tb["y"])
    for mode, sw in (("standard", False), ("swapped_half", True)):
        mm = O.init_model(spec, 42, 1e-3)
        loss, om = O.run_iteration(mm, O.build_schedule(2, sw, 4), x, y)
        want = g["tiny_run_iteration"][mode]
        assert loss == pytest.approx(want["loss"], rel=1e-12)
        np.testing.assert_allclose(om, want["omegas"], rtol=1e-11)
        np.testing.assert_allclose(mm.all_weights_flat(), want["flat"], rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("name", ["checkfree_s2_at50", "checkfree_plus_s1_at50", "checkfree_averaged_moments",
                                  "checkfree_plus_averaged_edge", "reinit_copy", "reinit_random",
                                  "unrecoverable_adjacent", "checkfree_edge_unsupported", "classification_checkfree",
                                  "relu_checkfree_plus", "checkfree_plus_swap_from_40", "checkpointing_s2_at50",
                                  "checkpointing_edge_and_adjacent", "checkpointing_at_snapshot"])
def test_trainer_loss_curves_match_reference(trainer_goldens, name):
    run = next(r for r in trainer_goldens["runs"] if r["name"] == name)
    cfg = dict(run["cfg"])
    evals, evs, unrec = O.run_experiment(cfg, run["trace"], run["seed"])
    w_evals, w_evs, w_unrec = O.parse_full_record(run["full"])
    assert unrec == w_unrec
    assert [e[0] for e in evals] == [e[0] for e in w_evals]
    for (i, tr, va), (_, wtr, wva) in zip(evals, w_evals):
        assert tr == pytest.approx(wtr, rel=1e-9) and va == pytest.approx(wva, rel=1e-9), i
    assert [(e[0], e[1], e[2]) for e in evs] == [(e[0], e[1], e[2]) for e in w_evs]
    for e, w in zip(evs, w_evs):
        assert e[3] == pytest.approx(w[3], rel=1e-9)
        assert e[4] == pytest.approx(w[4], rel=1e-7, abs=1e-12)
