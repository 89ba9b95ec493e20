"""BASELINE.json configs[0] on the B200 trainer (ckf_run_experiment): tiny LLaMA
(8 layers, d=256, seq 128) as a 4-stage pipeline on synthetic tokens, stage 2
killed at step 50 with CheckFree recovery (and stage 1 with CheckFree+'s edge
copy), against the CPU fp64 LLaMA oracle's curves committed in
tests/golden/llama_tiny_checkfree.json (oracle/make_llama_golden.py).

Bars: failure handling is bit-exact (same slots, stages, actions); every
train / validation loss point within 1 % of the oracle (north_star); the
reduction error of the recovered stage within 5 % (it integrates 50 bf16 steps
of weight drift)."""
import json
import os

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _golden():
    with open(os.path.join(ROOT, "tests", "golden", "llama_tiny_checkfree.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["checkfree_stage2_at50", "checkfree_plus_stage1_at50"])
def test_llama_trainer_matches_oracle(name):
    import paper_2506_15461_b200 as P
    g = _golden()[name]
    evals, events, unrec = P.run_experiment(g["config"], g["trace"], g["seed"])
    assert not unrec and not g["unrecoverable"]
    assert [e[0] for e in evals] == [e[0] for e in g["evals"]]
    for (it, tr, va), (it2, tr2, va2) in zip(evals, g["evals"]):
        assert abs(tr - tr2) <= 1e-2 * abs(tr2), (it, tr, tr2)
        assert abs(va - va2) <= 1e-2 * abs(va2), (it, va, va2)
    assert [(e[0], e[1], e[2]) for e in events] == [(e[0], e[1], e[2]) for e in g["events"]]
    for e, e2 in zip(events, g["events"]):
        assert abs(e[3] - e2[3]) <= 5e-2 * abs(e2[3]), (e[3], e2[3])
        assert e[5] > 0.0  # measured recovery latency (ms)


@pytest.mark.parametrize("name", ["checkfree_stage2_at50", "checkfree_plus_stage1_at50"])
def test_llama_trainer_fp32_parity_mode(name):
    # the same configs[0] runs in the LLaMA fp32 parity mode (llama_f32.cu): every loss point
    # within 1e-3 of the fp64 oracle over 100 iterations with the failure and recovery, the
    # reduction error within 1e-3 (vs 1 % / 5 % for the bf16 tensor-core path)
    import paper_2506_15461_b200 as P
    g = _golden()[name]
    cfg = dict(g["config"])
    cfg["precision"] = "fp32"
    evals, events, unrec = P.run_experiment(cfg, g["trace"], g["seed"])
    assert not unrec
    assert [e[0] for e in evals] == [e[0] for e in g["evals"]]
    for (it, tr, va), (it2, tr2, va2) in zip(evals, g["evals"]):
        assert abs(tr - tr2) <= 1e-3 * abs(tr2), (it, tr, tr2)
        assert abs(va - va2) <= 1e-3 * abs(va2), (it, va, va2)
    assert [(e[0], e[1], e[2]) for e in events] == [(e[0], e[1], e[2]) for e in g["events"]]
    for e, e2 in zip(events, g["events"]):
        assert abs(e[3] - e2[3]) <= 1e-3 * abs(e2[3]), (e[3], e2[3])


# ------------------------------------------------------------------ learning regime
# tests/golden/llama_tiny_learning.json (oracle/make_llama_golden.py learning): lr 3e-3 over 200
# iterations -- the oracle's validation loss falls 8.38 -> 4.45 (CheckFree) -- with the failure at
# iteration 100 in the steepest part of the curve, where a wrong recovery shows.
def _learning():
    with open(os.path.join(ROOT, "tests", "golden", "llama_tiny_learning.json")) as f:
        return json.load(f)


def _log(rec):
    path = os.environ.get("CKF_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("name", ["learning_checkfree_stage2_at100", "learning_checkfree_plus_stage1_at100"])
def test_llama_trainer_learning_regime(name, precision):
    import paper_2506_15461_b200 as P
    g = _learning()[name]
    cfg = dict(g["config"], precision=precision)
    evals, events, unrec = P.run_experiment(cfg, g["trace"], g["seed"])
    assert not unrec
    assert [e[0] for e in evals] == [e[0] for e in g["evals"]]
    dev = [abs(va - va2) / abs(va2) for (_, _, va), (_, _, va2) in zip(evals, g["evals"])]
    devt = [abs(tr - tr2) / abs(tr2) for (_, tr, _), (_, tr2, _) in zip(evals, g["evals"])]
    assert [(e[0], e[1], e[2]) for e in events] == [(e[0], e[1], e[2]) for e in g["events"]]
    red = abs(events[0][3] - g["events"][0][3]) / abs(g["events"][0][3])
    spike, spike_o = events[0][4], g["events"][0][4]
    _log({"test": "trainer_learning", "name": name, "precision": precision, "max_val_dev": max(dev),
          "max_train_dev": max(devt), "val_dev": dev, "reduction_error_dev": red, "spike": spike,
          "spike_oracle": spike_o, "final_val": evals[-1][2], "final_val_oracle": g["evals"][-1][2]})
    bar = LEARNING_BARS[precision]
    assert max(dev) <= bar["curve"] and max(devt) <= bar["curve"], (max(dev), max(devt))
    assert red <= bar["reduction_error"], red
    assert abs(spike - spike_o) <= bar["spike_abs"], (spike, spike_o)


# Measured on the B200 (profiles/r02_parity_learning.jsonl).  In the learning phase the curve
# amplifies per-step differences: the fp32 parity mode, which matches a single step to 1e-5,
# drifts up to 0.93 % from the fp64 oracle over the 100 iterations after the onset of learning;
# bf16 up to 1.69 %.  Bars ~1.5x measured: curve 2.5 % (bf16) / 1.5 % (fp32) per point;
# reduction error (measured 0.67 % / 0.31 %) 1.5 % / 1 %; the loss spike of the recovery
# (oracle +0.045 for CheckFree, -0.006 for CheckFree+) within 0.02 absolute for fp32 and 0.04 for
# bf16 -- a recovery from the wrong neighbours or weights spikes by O(1).  The bf16 spike moves with
# the GEMM summation order: 0.0083 before the wave-balanced weight-gradient split-K, 0.0207 after
# (CheckFree+, stage 1; the spike is the difference of two validation losses near 5.5, each within
# 0.4 % of the oracle's).
LEARNING_BARS = {"bf16": {"curve": 2.5e-2, "reduction_error": 1.5e-2, "spike_abs": 0.04},
                 "fp32": {"curve": 1.5e-2, "reduction_error": 1e-2, "spike_abs": 0.02}}
