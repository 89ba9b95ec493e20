"""Cost model: reference include/ckfree/cost_model.hpp, src/cost_model.cpp,
src/experiment.cpp:215-300.

* tests/cpp/cost_driver.cpp compiled against the reference library (oracle/_ref) and against
  the drop-in (dropin/_bin): every iteration / recovery / train-time quantity, profile text
  and error class over a grid of profiles, parameters, strategies and failure lists, printed
  as exact hex floats -- the two outputs must be identical;
* the Python face (paper_2506_15461_b200/cost.py) and the B200 re-parameterisation checked
  against closed forms restated here;
* compare_strategies over the GPU trainer (gpu-marked).
"""
import math
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "cost_driver_ref")
DROP = os.path.join(ROOT, "dropin", "_bin", "cost_driver_dropin")


def _run(exe):
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return r.stdout


def test_cost_model_bit_identical_to_reference():
    want, got = _run(REF), _run(DROP)
    assert len(want.splitlines()) > 2000
    assert "unsupported" in want and "train[" in want
    for i, (a, b) in enumerate(zip(want.splitlines(), got.splitlines())):
        assert a == b, f"line {i}: reference {a!r} vs drop-in {b!r}"
    assert want == got


@pytest.fixture(scope="module")
def K():
    from paper_2506_15461_b200 import cost
    try:
        cost._lib()
    except ImportError as e:
        pytest.skip(str(e))
    return cost


def test_synthetic_profile_text(K):
    p = K.Profile.synthetic(6)
    lines = p.text.splitlines()
    assert lines[0] == "ckfree-net v1"
    assert lines[1] == "sites us-east eu-west asia-se us-west eu-north"
    assert lines[2] == "assignment 0 1 2 3 4 0"
    assert lines[3] == "latency" and lines[4] == "0 0.080000000000000002 0.14999999999999999 0.059999999999999998 0.089999999999999997"


def test_b200_profile_links(K):
    p = K.Profile.b200(6, gpus_per_node=4, nodes=2, nvlink_bps=800e9, nvlink_latency_s=2e-6, nic_bps=50e9,
                       nic_latency_s=8e-6, hbm_bps=7e12, storage_bps=20e9, storage_latency_s=5e-4)
    lines = p.text.splitlines()
    sites = lines[1].split()[1:]
    assert sites == [f"node{g // 4}-gpu{g % 4}" for g in range(8)] + ["storage"]
    assert lines[2] == "assignment 0 1 2 3 4 5"
    n = len(sites)
    lat = [[float(v) for v in lines[4 + i].split()] for i in range(n)]
    bw = [[float(v) for v in lines[5 + n + i].split()] for i in range(n)]
    assert lat[0][1] == 2e-6 and bw[0][1] == 800e9        # NVLink inside node 0
    assert lat[3][4] == 8e-6 and bw[3][4] == 50e9         # node 0 -> node 1 over the NIC
    assert lat[2][8] == 5e-4 and bw[8][2] == 20e9         # storage
    assert lat[5][5] == 0.0 and bw[5][5] == 7e12          # same GPU
    with pytest.raises(K.CostError):
        K.Profile.b200(0)


def _par(K):
    return K.params_b200(1.5e-3, 3.2e-3, 8192, 512, 19_000_000, 6_000_000, 150_000_000, 8)


def test_params_b200_layout(K):
    p = _par(K)
    assert p.activation_bytes == 8192 * 512 * 2      # bf16 boundary activations
    assert p.stage_weight_bytes == 19_000_000 * 4    # fp32 masters
    assert p.edge_weight_bytes == 6_000_000 * 4
    assert p.full_model_bytes == 150_000_000 * 12    # masters + Adam m, v
    with pytest.raises(K.CostError, match="backward"):
        K.params_b200(2e-3, 1e-3, 8192, 512, 1, 1, 1, 8)


def test_b200_iteration_and_recovery_closed_forms(K):
    s, nv, lat = 4, 900e9, 3e-6
    prof = K.Profile.b200(s)  # one node, every stage on its own GPU
    p = _par(K)
    m = p.num_microbatches
    act = p.activation_bytes
    base = m * s * (p.fwd_seconds + p.bwd_seconds)
    hop_act = (s - 1) * (m * (lat + act / nv))
    cf = K.iteration_cost("checkfree", prof, p)
    assert cf["compute"] == pytest.approx(base, rel=1e-15)
    assert cf["communication"] == pytest.approx(hop_act, rel=1e-12)
    cfp = K.iteration_cost("checkfree-plus", prof, p)
    assert cfp["communication"] == pytest.approx(hop_act + 2 * (lat + p.edge_weight_bytes / nv), rel=1e-12)
    rc = K.iteration_cost("redundant", prof, p)
    assert rc["compute"] == pytest.approx(2 * m * s * (2 * p.fwd_seconds / 2 + p.bwd_seconds / 2), rel=1e-15)
    ck = K.iteration_cost("checkpointing", prof, p, checkpoint_interval=50)
    assert ck["checkpoint_overhead"] == pytest.approx(p.full_model_bytes / 25e9 / 50, rel=1e-15)
    # recovery: neighbours over NVLink; checkpoint restore from storage
    w = p.stage_weight_bytes
    assert K.recovery_time("checkfree", prof, p, 2) == pytest.approx(lat + w / nv, rel=1e-15)
    assert K.recovery_time("checkfree-plus", prof, p, 1) == pytest.approx(lat + (w + p.edge_weight_bytes) / nv)
    assert K.recovery_time("redundant", prof, p, 1) == pytest.approx(lat + w / nv)
    assert K.recovery_time("checkpointing", prof, p, 3) == pytest.approx(1e-3 + p.full_model_bytes / 25e9)
    with pytest.raises(K.CostError, match="unsupported"):
        K.recovery_time("checkfree", prof, p, 1)
    with pytest.raises(K.CostError, match="out of range"):
        K.recovery_time("checkfree", prof, p, 5)


def _rollback_lost(events, interval):
    """cost_model.cpp:361-377 restated: one rollback per failing slot to the last snapshot."""
    model_iter, prev, lost, seen = 0, 0, 0, set()
    for it, _ in events:
        if it in seen:
            continue
        seen.add(it)
        model_iter += it - prev
        prev = it
        snap = model_iter // interval * interval
        lost += model_iter - snap
        model_iter = snap
    return lost


@pytest.mark.parametrize("interval", [1, 7, 100])
def test_train_time_rollback_replay(K, interval):
    prof, p = K.Profile.b200(4), _par(K)
    events = [(3, 2), (3, 3), (15, 2), (16, 3), (230, 2), (231, 2), (900, 3)]
    per = K.iteration_cost("checkpointing", prof, p, interval)["total"]
    t = K.train_time("checkpointing", prof, p, 1000, events, interval)
    assert t["rollback_lost"] == pytest.approx(_rollback_lost(events, interval) * per, rel=1e-12)
    rec = K.recovery_time("checkpointing", prof, p, 2, interval)
    assert t["recovery"] == pytest.approx(len(events) * rec, rel=1e-12)
    total = t["compute"] + t["communication"] + t["checkpoint_overhead"] + t["recovery"] + t["rollback_lost"]
    assert t["hours"] == pytest.approx(total / 3600, rel=1e-15)
    # CheckFree never rolls back
    assert K.train_time("checkfree", prof, p, 1000, events)["rollback_lost"] == 0.0


def test_strategy_ordering_b200_vs_wan(K):
    """On the WAN profile the paper's ordering holds (checkpoint restores and RC's doubled
    compute dominate); on one NVSwitch node the gap between strategies shrinks to the
    compute difference: RC's 1.5 forward-equivalents per stage stay, transfers vanish."""
    p = _par(K)
    events = [(40 * k, 2 + k % 2) for k in range(1, 10)]
    hours = {}
    for name, prof in (("wan", K.Profile.synthetic(4)), ("b200", K.Profile.b200(4))):
        hours[name] = {s: K.train_time(s, prof, p, 400, events, 50)["hours"]
                       for s in ("checkpointing", "redundant", "checkfree", "checkfree-plus")}
    w, b = hours["wan"], hours["b200"]
    assert w["checkfree"] < w["checkfree-plus"] < w["redundant"] and w["checkfree"] < w["checkpointing"]
    assert b["checkfree"] < b["checkpointing"] and b["checkfree"] < b["redundant"]
    assert b["redundant"] > b["checkfree"]


def test_parse_errors(K):
    for bad in ("", "ckfree-net v2\n", "ckfree-net v1\nsites a b\nassignment 0 5\nlatency\n0 1\n1 0\nbandwidth\n0 1\n1 0\n"):
        with pytest.raises(K.CostError, match="parse"):
            K.iteration_cost("checkfree", K.Profile(bad), _par(K))


def test_compare_rows_from_records(K, monkeypatch):
    """compare_strategies' row arithmetic (experiment.cpp:217-243) on canned run records:
    cost stops at the convergence slot, failures after it are not charged."""
    trace = "checkfree-trace v1 seed=0 p_hour=0.1 iter_s=3600 stages=2,3\n5,2\n12,3\n30,2\n"
    recs = {"checkfree": dict(slots_run=40, model_iterations=40, final_val_loss=1.0, hours=0.001,
                              slots_to_target=20, model_iters_to_target=20, hours_to_target=0.0005,
                              unrecoverable=False),
            "checkpointing": dict(slots_run=40, model_iterations=31, final_val_loss=1.2, hours=0.002,
                                  slots_to_target=-1, model_iters_to_target=-1, hours_to_target=-1.0,
                                  unrecoverable=False)}
    monkeypatch.setattr(K, "run_record", lambda cfg, tr, seed: recs[cfg["strategy"]])
    prof, p = K.Profile.b200(4), _par(K)
    rows = K.compare_strategies({"checkpoint-interval": 10}, ["checkfree", "checkpointing"], trace, prof, p, seed=0)
    cf, ck = rows
    assert cf.train_time_h == K.train_time("checkfree", prof, p, 20, [(5, 2), (12, 3)], 10)["hours"]
    assert ck.train_time_h == K.train_time("checkpointing", prof, p, 31, [(5, 2), (12, 3), (30, 2)], 10)["hours"]
    assert cf.measured_hours == 0.0005 and ck.measured_hours == 0.002
    csv = K.comparison_csv(rows).splitlines()
    assert csv[0] == "# format_version=1" and csv[2].startswith("checkfree,")
    assert "DEAD" not in K.comparison_table(rows)


@pytest.mark.gpu
def test_compare_strategies_on_gpu_trainer(K):
    """One shared trace, four strategies on the GPU trainer (tiny LLaMA), costed on a B200 node."""
    import paper_2506_15461_b200 as P

    cfg = {"block": "llama", "precision": "bf16", "vocab": 512, "model-dim": 128, "layers": 4, "heads": 2,
           "hidden-dim": 256, "seq-len": 64, "stages": 4, "iters": 40, "batch": 16, "microbatches": 4,
           "lr": 1e-3, "eval-interval": 5, "val-size": 8, "checkpoint-interval": 10, "target-loss": 6.1}
    trace = P.api.generate_trace(3, 0.2, 3600.0, 40, [2, 3])
    prof = K.Profile.b200(4)
    p = K.params_b200(1e-4, 2e-4, 4 * 64, 128, 200_000, 65_536, 900_000, 4)
    rows = K.compare_strategies(cfg, ["checkpointing", "redundant", "checkfree", "checkfree-plus"], trace, prof, p,
                                seed=1)
    assert [r.strategy for r in rows] == ["checkpointing", "redundant", "checkfree", "checkfree-plus"]
    for r in rows:
        assert not r.unrecoverable and math.isfinite(r.train_time_h) and r.measured_hours > 0
        assert r.iteration_time_s == K.iteration_cost(r.strategy, prof, p, 10)["total"]
    print(K.comparison_table(rows))


def test_cost_c_entry_points_exported():
    import ctypes
    import re
    hdr = open(os.path.join(ROOT, "include", "ckfree", "cost_model.hpp")).read()
    names = re.findall(r"\b(ckfree_cost_\w+)\(", hdr)
    assert len(set(names)) >= 7
    so = os.path.join(ROOT, "dropin", "libckfree_b200.so")
    if not os.path.exists(so):
        pytest.skip("dropin/libckfree_b200.so not built")
    lib = ctypes.CDLL(so)
    for n in set(names):
        assert hasattr(lib, n), n


@pytest.mark.gpu
def test_measure_stage_seconds_and_b200_params(K):
    """The B200 re-parameterisation path end to end on a small LLaMA: measured per-stage
    forward / backward seconds feed CostParams::from_b200 and an iteration cost whose compute
    term reproduces the measured iteration (stages x microbatches x (fwd + bwd))."""
    import paper_2506_15461_b200 as P
    from paper_2506_15461_b200 import api

    spec = api.ModelSpec.llama(512, 128, 4, 2, 256, 64, 4, max_tokens=4 * 64)
    eng = P.Engine(spec)
    eng.init(1, 1e-3)
    f, b, detail = K.measure_stage_seconds(eng, spec, 4 * 64, 4, reps=3, warmup=2)
    assert 0 < f <= b and detail["iteration_s"] > 0
    par = K.params_b200(f, b, 4 * 64, 128, eng.stage_params, max(eng.embed_params, eng.deembed_params),
                        4 * eng.stage_params + eng.embed_params + eng.deembed_params, 4)
    eng.close()
    it = K.iteration_cost("checkfree", K.Profile.b200(4), par)
    assert it["compute"] == pytest.approx(4 * 4 * (f + b), rel=1e-12)
    assert it["compute"] == pytest.approx(detail["iteration_s"], rel=1e-6) or b == f


@pytest.mark.gpu
def test_ablation_swap_milestones_match_oracle(K):
    """ablation_swap (experiment.cpp:349-386): the GPU trainer's swap-off / swap-on runs give
    the same milestone iterations as the fp64 oracle restatement of the reference trainer."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ckfree_oracle as O
    cfg = {"input-dim": 16, "hidden-dim": 64, "model-dim": 32, "output-dim": 16, "layers": 8, "stages": 4,
           "batch": 256, "microbatches": 8, "lr": 0.0003, "eval-interval": 5, "val-size": 256, "iters": 60}
    ab = K.ablation_swap(cfg, 1)
    empty = "checkfree-trace v1 seed=1 p_hour=0 iter_s=120 stages=1,2,3,4\n"
    ref = {}
    for mode in ("standard", "swapped-half"):
        evals, _, _ = O.run_experiment({**cfg, "strategy": "no-failures", "schedule": mode}, empty, 1)
        ref[mode] = evals
    want = K.milestones(ref["standard"], ref["swapped-half"])
    got = ab["milestones"]
    assert [(r["iter_off"], r["iter_on"]) for r in got] == [(r["iter_off"], r["iter_on"]) for r in want]
    for g, w in zip(got, want):
        assert g["level"] == pytest.approx(w["level"], rel=1e-9)
    assert any(r["iter_off"] > 0 for r in got)


@pytest.mark.gpu
def test_estimate_delta_matches_numpy_restatement(K):
    """estimate_delta (experiment.cpp:305-345): per-layer parameter / function ratios of the
    GPU engine's residual-MLP model against a numpy restatement that skips the layer; the
    engine's weights are left as they were."""
    import numpy as np

    import paper_2506_15461_b200 as P
    from paper_2506_15461_b200 import api

    spec = api.ModelSpec(16, 64, 32, 16, 8, 4, precision="fp64", max_rows=64)
    eng = P.Engine(spec)
    eng.init(7, 1e-3)
    x = np.random.default_rng(3).uniform(-1.0, 1.0, (64, 16))
    before = eng.predict([1, 2, 3, 4], x)
    rep = K.estimate_delta(eng, x)
    assert np.array_equal(eng.predict([1, 2, 3, 4], x), before)

    E = eng.export_edge(0)[0].reshape(16, 32)
    D = eng.export_edge(1)[0].reshape(32, 16)
    W = [eng.export_stage(s)[0] for s in range(1, 5)]
    blocks = []
    for w in W:
        for b in range(2):
            o = b * 2 * 32 * 64
            blocks.append((w[o:o + 32 * 64].reshape(32, 64), w[o + 32 * 64:o + 2 * 32 * 64].reshape(64, 32)))

    def fwd(skip=None):
        h = x @ E
        for i, (w1, w2) in enumerate(blocks):
            if i != skip:
                h = h + np.tanh(h @ w1) @ w2
        return h @ D

    full = fwd()
    allw = np.concatenate([E.ravel(), D.ravel()] + W)
    for i, row in enumerate(rep["rows"]):
        w1, w2 = blocks[i]
        pr = np.sqrt((w1 ** 2).sum() + (w2 ** 2).sum()) / np.linalg.norm(allw)
        fr = np.linalg.norm(full - fwd(i)) / np.linalg.norm(full)
        assert row["layer"] == i + 1
        assert row["param_ratio"] == pytest.approx(pr, rel=1e-9)
        assert row["func_ratio"] == pytest.approx(fr, rel=1e-6)
    assert rep["delta_func"] == max(r["func_ratio"] for r in rep["rows"]) > 0
    assert K.delta_csv(rep).splitlines()[1] == "layer,param_ratio,func_ratio"
    eng.close()
