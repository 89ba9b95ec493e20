"""CPU checks of the LLaMA-block oracle (oracle/llama_oracle.py) with the
reference's own test METHODS, since the reference has no LLaMA block:
central finite differences (tests/test_model.cpp:109-155), microbatch
accumulation == full batch (tests/test_pipeline.cpp:100-138), identity-stage
swap invariance (tests/test_pipeline.cpp:140-156), and the token stream's
determinism.  Fast: tiny shapes only."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import llama_oracle as LO  # noqa: E402
from ckfree_oracle import build_schedule, standard_order, swapped_order  # noqa: E402

SPEC = LO.LSpec(vocab=32, d=16, layers=4, heads=2, ffn=24, seq_len=8, stages=4)


def _toks(rows=2, seed=5):
    return LO.token_batch(seed, 1, 1, rows, SPEC.seq_len, SPEC.vocab)


def test_token_stream_deterministic_and_in_range():
    a = LO.token_batch(7, 1, 3, 16, 64, 4096)
    b = LO.token_batch(7, 1, 3, 16, 64, 4096)
    c = LO.token_batch(7, 1, 4, 16, 64, 4096)
    assert a.shape == (16, 65) and a.dtype == np.int32
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert a.min() >= 0 and a.max() < 4096
    # learnable: the bigram successor structure makes the stream far from uniform
    assert len(np.unique(a)) < 16 * 65


def test_finite_differences():
    model = LO.LModel(SPEC, 3, 1e-3)
    toks = _toks()
    order = standard_order(SPEC.stages)
    loss, gs, ge, gd = LO.microbatch(model, order, toks)
    rng = np.random.default_rng(0)
    h = 1e-5
    checked = 0
    for which in ["stage", "embed", "deembed"]:
        for _ in range(12):
            if which == "stage":
                sid = int(rng.integers(1, SPEC.stages + 1))
                arr, g = model.stages[sid - 1].flat, gs[sid - 1]
            elif which == "embed":
                arr, g = model.embed, ge
            else:
                arr, g = model.deembed, gd
            i = int(rng.integers(0, arr.size))
            if which == "embed" and abs(g[i]) == 0.0:
                continue
            old = arr[i]
            arr[i] = old + h
            lp = LO.eval_loss(model, order, toks)
            arr[i] = old - h
            lm = LO.eval_loss(model, order, toks)
            arr[i] = old
            fd = (lp - lm) / (2 * h)
            assert abs(fd - g[i]) <= 1e-4 * max(1.0, abs(fd), abs(g[i])) + 1e-7, (which, i, fd, g[i])
            checked += 1
    assert checked >= 24


def test_microbatch_accumulation_equals_full_batch():
    model = LO.LModel(SPEC, 4, 1e-3)
    toks = _toks(rows=4)
    order = standard_order(SPEC.stages)
    _, g_full, e_full, d_full = LO.microbatch(model, order, toks)
    l, g_acc, e_acc, d_acc = LO.accumulate_grads(model, [order] * 4, toks)
    for a, b in zip(g_full, g_acc):
        np.testing.assert_allclose(a, b / 4, rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(e_full, e_acc / 4, rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(d_full, d_acc / 4, rtol=1e-10, atol=1e-14)


def test_identity_stages_make_swap_invariant():
    model = LO.LModel(SPEC, 5, 1e-3)
    o = SPEC.layer_offsets()
    for st in model.stages:  # Wo = Wd = 0 -> every layer is the identity on h
        for li in range(st.flat.size // o["total"]):
            b = li * o["total"]
            st.flat[b + o["wo"]:b + o["g2"]] = 0.0
            st.flat[b + o["wd"]:b + o["total"]] = 0.0
    toks = _toks()
    a = LO.eval_loss(model, standard_order(SPEC.stages), toks)
    b = LO.eval_loss(model, swapped_order(SPEC.stages), toks)
    assert a == b


def test_run_iteration_adam_and_omega():
    model = LO.LModel(SPEC, 6, 1e-3)
    toks = _toks(rows=4)
    before = [s.flat.copy() for s in model.stages]
    loss, om = LO.run_iteration(model, build_schedule(2, True, SPEC.stages), toks)
    assert np.isfinite(loss) and all(o > 0 for o in om)
    for b, s in zip(before, model.stages):
        step = np.abs(s.flat - b)
        assert step.max() <= 1e-3 * 1.0001  # first Adam step moves each weight by <= lr
        assert s.opt.step == 1
