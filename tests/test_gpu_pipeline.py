"""Engine-side checks of the multi-GPU pipeline path on ONE GPU.

* GPipe schedule (all forwards, then all backwards -- what the ranks of a
  multi-GPU pipeline run so that they overlap) is bit-identical to the
  sequential per-microbatch schedule: the per-stage accumulation order is the
  reference's (pipeline.cpp:66-81).
* With a VIRTUAL stage -> rank placement the engine logs every stage-boundary
  transfer it would issue; the log equals ckf_pipeline_plan's transfers, the
  plan that tests/test_pipeline_multirank.py executes across two gloo ranks.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import llama_oracle as LO  # noqa: E402


def _mlp_engine(seed=5):
    import paper_2506_15461_b200 as P
    spec = P.api.ModelSpec(16, 64, 32, 16, 8, 4, precision="fp64", max_rows=64)
    e = P.Engine(spec)
    e.init(seed, 1e-3)
    return e


def _llama_engine(seed=3):
    import paper_2506_15461_b200 as P
    spec = P.api.ModelSpec.llama(512, 128, 4, 2, 256, 128, 4, max_tokens=2 * 128)
    e = P.Engine(spec)
    e.init(seed, 1e-3)
    return e


def _batches(kind, it):
    rng = np.random.default_rng(100 + it)
    if kind == "mlp":
        return rng.uniform(-1, 1, (32, 16)), rng.uniform(-1, 1, (32, 16))
    return LO.token_batch(9, 1, it, 8, 128, 512), None


@pytest.mark.parametrize("kind", ["mlp", "llama"])
def test_gpipe_schedule_bit_identical_to_sequential(kind):
    from paper_2506_15461_b200 import api
    runs = []
    for schedule in (0, 1):
        e = _mlp_engine() if kind == "mlp" else _llama_engine()
        e.set_schedule(schedule)
        e.set_group_cap(1)  # per-microbatch passes (fusion re-associates the fp32 sums)
        out = []
        for it in (1, 2):
            x, y = _batches(kind, it)
            out.append(e.run_iteration(api.build_schedule(4, it == 2, 4), x, y, it))
        w = np.concatenate([e.export_stage(s)[0] for s in range(1, 5)] + [e.export_edge(0)[0], e.export_edge(1)[0]])
        runs.append((out, w))
        e.close()
    (o0, w0), (o1, w1) = runs
    for (l0, om0), (l1, om1) in zip(o0, o1):
        assert l0 == l1 and np.array_equal(om0, om1)
    assert np.array_equal(w0, w1)


@pytest.mark.parametrize("kind", ["mlp", "llama"])
@pytest.mark.parametrize("schedule", [0, 1])
@pytest.mark.parametrize("placement", [[0, 0, 1, 1], [0, 1, 2, 3]])
def test_engine_transfers_follow_the_plan(kind, schedule, placement):
    from paper_2506_15461_b200 import api
    e = _mlp_engine() if kind == "mlp" else _llama_engine()
    e.set_schedule(schedule)
    e.hop_log(placement)
    x, y = _batches(kind, 1)
    orders = api.build_schedule(4, True, 4)
    e.run_iteration(orders, x, y, 1)
    log = e.hop_log()
    plan = [op for op in api.pipeline_plan(orders, placement, schedule) if op["kind"] == "xfer"]
    assert [(a, b) for a, b, _ in log] == [(op["rank"], op["arg"]) for op in plan]
    per_mb = (8 * 32 * 8) if kind == "mlp" else (2 * 128 * 128 * 4)  # rows x width x bytes (fp64 MLP / fp32 LLaMA)
    assert all(nb == per_mb for _, _, nb in log)
    e.close()
