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


@pytest.mark.parametrize("placement", [[0, 0, 1, 1], [0, 1, 2, 3], [0, 1, 0, 1]])
@pytest.mark.parametrize("swapped", [False, True])
def test_1f1b_executor_bit_identical_to_sequential(placement, swapped):
    # schedule 2: the plan-driven 1F1B executor (Engine::run_plan + LlamaBlock::plan_op) walking
    # the global op order of a VIRTUAL placement on one GPU (every rank's ops run here, transfers
    # are logged pointer hand-offs; activation caches rotate over the in-flight slots) computes
    # exactly what the per-microbatch sequential loop computes
    from paper_2506_15461_b200 import api
    runs = []
    for schedule in (0, 2):
        e = _llama_engine()
        e.set_group_cap(1)
        e.set_schedule(schedule)
        if schedule == 2:
            e.hop_log(placement)
        out = []
        for it in (1, 2, 3):
            x, y = _batches("llama", it)
            out.append(e.run_iteration(api.build_schedule(8, swapped and it != 2, 4), x, y, it))
        w = np.concatenate([e.export_stage(s)[0] for s in range(1, 5)] + [e.export_edge(0)[0], e.export_edge(1)[0]])
        runs.append((out, w))
        e.close()
    (o0, w0), (o2, w2) = runs
    for (l0, om0), (l2, om2) in zip(o0, o2):
        assert l0 == l2 and np.array_equal(om0, om2)
    assert np.array_equal(w0, w2)


@pytest.mark.parametrize("kind", ["mlp", "llama"])
@pytest.mark.parametrize("schedule", [0, 1, 2])
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
    # the MLP parity block has no plan ops: schedule 2 runs it with the GPipe executor
    want = 1 if (schedule == 2 and kind == "mlp") else schedule
    sc, hc = e.plan_cost()  # the 1F1B simulation is weighted by the engine's stage / head costs
    plan = [op for op in api.pipeline_plan(orders, placement, want, sc, hc) if op["kind"] == "xfer"]
    assert [(a, b) for a, b, _ in log] == [(op["rank"], op["arg"]) for op in plan]
    per_mb = (8 * 32 * 8) if kind == "mlp" else (2 * 128 * 128 * 4)  # rows x width x bytes (fp64 MLP / fp32 LLaMA)
    assert all(nb == per_mb for _, _, nb in log)
    e.close()
