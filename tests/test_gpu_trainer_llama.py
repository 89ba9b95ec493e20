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
