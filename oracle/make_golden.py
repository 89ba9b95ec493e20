"""Generates tests/golden/*.json from the UNMODIFIED reference library
(oracle/_ref/libckfree_oracle.so, built by `make -C oracle` from
/root/reference/proj/src).  Test infrastructure only; re-run after changing
the fixture set:  python oracle/make_golden.py

Each fixture names the reference function (file:line) that produced it.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import refshim as R  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden")

TINY = {"input-dim": 3, "hidden-dim": 3, "model-dim": 4, "output-dim": 3, "layers": 4, "stages": 4,
        "microbatches": 2, "lr": 1e-3}
DESK = {"input-dim": 16, "hidden-dim": 64, "model-dim": 32, "output-dim": 16, "layers": 8, "stages": 4,
        "batch": 256, "microbatches": 8, "lr": 3e-4, "eval-interval": 10, "val-size": 1024, "iters": 100}


def trace_text(seed, stages, events, iter_s=120.0):
    head = f"checkfree-trace v1 seed={seed} p_hour=0 iter_s={iter_s:.17g} stages={','.join(map(str, stages))}\n"
    return head + "".join(f"{i},{s}\n" for i, s in events)


def rng_goldens():
    return {
        "source": "include/ckfree/rng.hpp:10-48",
        "mix64": [[x, R.mix64(x)] for x in (0, 1, 42, 0xFFFFFFFFFFFFFFFF)],
        "derive_key": [[list(a), R.derive_key(*a)] for a in ((1, 0, 0, 0), (42, 1, 2, 0), (7, 0, 0, 0), (5, 3, 9, 11))],
        "unit_at": [[list(a), R.unit_at(*a)] for a in ((42, 1, 2, 0), (1, 40, 6, 0), (3, 7, 0, 0))],
        "counter_uniform": [[R.derive_key(7, 0), -1.0, 1.0, R.counter_uniform(R.derive_key(7, 0), -1.0, 1.0, 8).tolist()],
                            [R.derive_key(9, 2), 0.0, 1.0, R.counter_uniform(R.derive_key(9, 2), 0.0, 1.0, 8).tolist()]],
    }


def failure_goldens():
    cases = []
    for seed, p, iters, iter_s, stages in ((42, 0.16, 500, 92.12, [2, 3, 4, 5]),
                                           (1, 0.10, 1000, 120.0, list(range(1, 9))),
                                           (7, 0.10, 3000, 120.0, [2, 3]),
                                           (3, 0.5, 200, 3600.0, [1, 2, 3, 4, 5, 6])):
        text = R.generate_trace(seed, p, iter_s, iters, stages)
        cases.append({"seed": seed, "p_hour": p, "iters": iters, "iter_s": iter_s, "stages": stages, "trace": text})
    return {
        "source": "src/failures.cpp:57-95,171-184",
        "p_iter": [[p, s, R.hourly_to_per_iteration(p, s)] for p, s in ((0.16, 92.12), (0.10, 120.0), (0.05, 3600.0), (0.0, 10.0))],
        "traces": cases,
    }


def partition_schedule_goldens():
    parts = []
    for L, s in ((10, 4), (8, 4), (12, 4), (24, 8), (24, 4), (7, 3), (5, 5), (8, 1)):
        parts.append({"layers": L, "stages": s, "ranges": R.even_partition(L, s)})
    scheds = []
    for m, sw, s in ((4, False, 6), (4, True, 6), (2, True, 4), (8, True, 8), (12, True, 9), (1, False, 4)):
        scheds.append({"m": m, "swapped_half": sw, "s": s, "orders": R.build_schedule(m, sw, s)})
    errors = []
    for m, sw, s in ((3, True, 6), (4, True, 3), (0, False, 4)):
        try:
            R.build_schedule(m, sw, s)
            errors.append({"m": m, "swapped_half": sw, "s": s, "error": None})
        except RuntimeError as e:
            errors.append({"m": m, "swapped_half": sw, "s": s, "error": str(e)})
    return {"source": "src/model.cpp:63-73, src/pipeline.cpp:11-56", "partitions": parts, "schedules": scheds,
            "schedule_errors": errors}


def recovery_goldens():
    cases = []
    cases.append({"wp": [1.0, 0.0], "wn": [0.0, 1.0], "op": 4.0, "on": 1.0})
    cases.append({"wp": [1.0, 2.0, 3.0], "wn": [3.0, 2.0, 1.0], "op": 0.0, "on": 0.0})
    cases.append({"wp": [1.0, -1.0], "wn": [5.0, 7.0], "op": 1.0, "on": 0.0})
    k1, k2 = R.derive_key(11, 1), R.derive_key(11, 2)
    cases.append({"wp": R.counter_uniform(k1, -1, 1, 64).tolist(), "wn": R.counter_uniform(k2, -1, 1, 64).tolist(),
                  "op": 0.3171, "on": 2.718})
    for c in cases:
        out, deg = R.recover_checkfree(np.array(c["wp"]), np.array(c["wn"]), c["op"], c["on"])
        c["out"] = out.tolist()
        c["degenerate"] = deg
    wf = R.counter_uniform(R.derive_key(11, 3), -1, 1, 64)
    red = R.reduction_error(np.array(cases[3]["wp"]), wf, np.array(cases[3]["wn"]), cases[3]["op"], cases[3]["on"])
    # sum_squares at the 1024-block boundaries (kernels_serial.cpp:104-115)
    ss = []
    for n in (1, 1023, 1024, 1025, 3089):
        x = R.counter_uniform(R.derive_key(12, n), -1, 1, n)
        ss.append({"n": n, "key": R.derive_key(12, n), "sum_squares": R.sum_squares(x)})
    # adam (kernels_serial.cpp:133-144), 3 steps on 16 values
    g = R.counter_uniform(R.derive_key(13, 1), -1, 1, 16)
    w = R.counter_uniform(R.derive_key(13, 2), -1, 1, 16)
    m = np.zeros(16)
    v = np.zeros(16)
    trace = []
    for step in (1, 2, 3):
        w, m, v = R.adam_update(w, m, v, g * step, 2e-3, step)
        trace.append({"step": step, "w": w.tolist(), "m": m.tolist(), "v": v.tolist()})
    return {"source": "src/recovery.cpp:57-126, src/kernels_serial.cpp:104-144", "checkfree": cases,
            "reduction_error": {"wf_key": R.derive_key(11, 3), "case": 3, "value": red},
            "bump_lr": [[3e-4, 1.1, R.lib().ref_bump_lr(3e-4, 1.1)], [3.3e-4, 1.1, R.lib().ref_bump_lr(3.3e-4, 1.1)]],
            "sum_squares": ss,
            "adam": {"g_key": R.derive_key(13, 1), "w_key": R.derive_key(13, 2), "lr": 2e-3, "trace": trace}}


def model_goldens():
    tiny = dict(TINY)
    flat = R.init_model_flat(tiny, 42)
    desk_flat = R.init_model_flat(DESK, R.derive_key(1, 11))
    x, y = R.batch(tiny, 1, 1, 8)
    loss, om, after = R.run_iteration(tiny, 42, False, x, y, 1, flat.size)
    loss_sw, om_sw, after_sw = R.run_iteration(tiny, 42, True, x, y, 1, flat.size)
    dx, dy = R.batch(DESK, 1, 1, 16)
    vx, vy = R.batch(DESK, 1, -1, 4)
    return {
        "source": "src/model.cpp:159-197,211-413, src/pipeline.cpp:58-95, src/dataset.cpp:15-57",
        "tiny_cfg": tiny,
        "tiny_init_seed42": flat.tolist(),
        "desk_cfg": DESK,
        "desk_init_seed": R.derive_key(1, 11),
        "desk_init_head": desk_flat[:32].tolist(),
        "desk_init_sum": float(desk_flat.sum()),
        "desk_init_n": int(desk_flat.size),
        "tiny_batch_iter1": {"x": x.tolist(), "y": y.tolist()},
        "desk_batch_iter1_rows16": {"x": dx.tolist(), "y": dy.tolist()},
        "desk_val_rows4": {"x": vx.tolist(), "y": vy.tolist()},
        "tiny_run_iteration": {"standard": {"loss": loss, "omegas": om.tolist(), "flat": after.tolist()},
                               "swapped_half": {"loss": loss_sw, "omegas": om_sw.tolist(), "flat": after_sw.tolist()}},
    }


def trainer_goldens():
    runs = []
    base = dict(DESK)
    specs = [
        ("checkfree_s2_at50", {"strategy": "checkfree"}, trace_text(1, [2, 3], [(50, 2)])),
        ("checkfree_plus_s1_at50", {"strategy": "checkfree-plus"}, trace_text(1, [1, 2, 3, 4], [(50, 1)])),
        ("checkfree_plus_s4_s2_at30_70", {"strategy": "checkfree-plus"}, trace_text(1, [1, 2, 3, 4], [(30, 4), (70, 2)])),
        ("checkfree_averaged_moments", {"strategy": "checkfree", "recovered-moments": "averaged"},
         trace_text(1, [2, 3], [(20, 3), (60, 2)])),
        ("checkfree_plus_averaged_edge", {"strategy": "checkfree-plus", "recovered-moments": "averaged"},
         trace_text(1, [1, 2, 3, 4], [(40, 4)])),
        ("reinit_uniform_avg", {"strategy": "reinit-uniform-avg"}, trace_text(1, [2, 3], [(50, 2)])),
        ("reinit_copy", {"strategy": "reinit-copy"}, trace_text(1, [2, 3], [(50, 3)])),
        ("reinit_random", {"strategy": "reinit-random"}, trace_text(1, [2, 3], [(50, 2)])),
        ("no_failures", {"strategy": "no-failures"}, trace_text(1, [2, 3], [])),
        ("unrecoverable_adjacent", {"strategy": "checkfree"}, trace_text(1, [2, 3], [(25, 2), (25, 3)])),
        ("checkfree_edge_unsupported", {"strategy": "checkfree", "eligible": "all"}, trace_text(1, [1, 2, 3, 4], [(15, 1)])),
        ("classification_checkfree", {"strategy": "checkfree", "task": "classification"}, trace_text(1, [2, 3], [(50, 2)])),
        ("relu_checkfree_plus", {"strategy": "checkfree-plus", "activation": "relu"}, trace_text(1, [1, 2, 3, 4], [(50, 3)])),
        ("failure_at_iter1", {"strategy": "checkfree"}, trace_text(1, [2, 3], [(1, 2)])),
        ("checkfree_plus_swap_from_40", {"strategy": "checkfree-plus", "swap-from": 40}, trace_text(1, [1, 2, 3, 4], [(60, 1)])),
        ("s8_checkfree_plus_trace", {"strategy": "checkfree-plus", "layers": 8, "stages": 8, "iters": 60,
                                     "eval-interval": 5}, None),
        # redundant-computation baseline (trainer.cpp:162-171): the hot copy survives, state untouched
        ("redundant_s2_at50", {"strategy": "redundant"}, trace_text(1, [2, 3], [(50, 2)])),
        ("redundant_edges_and_middle", {"strategy": "redundant", "eligible": "all"},
         trace_text(1, [1, 2, 3, 4], [(20, 1), (45, 4), (45, 2), (70, 3)])),
        ("redundant_adjacent_unrecoverable", {"strategy": "redundant"}, trace_text(1, [2, 3], [(30, 2), (30, 3)])),
        # checkpointing baseline (trainer.cpp:173-193, checkpoint.cpp:70-83): rollback + data replay
        ("checkpointing_s2_at50", {"strategy": "checkpointing", "checkpoint-interval": 20},
         trace_text(1, [1, 2, 3, 4], [(50, 2)])),
        ("checkpointing_edge_and_adjacent", {"strategy": "checkpointing", "checkpoint-interval": 15},
         trace_text(1, [1, 2, 3, 4], [(20, 1), (47, 2), (47, 3), (80, 4)])),
        ("checkpointing_at_snapshot", {"strategy": "checkpointing", "checkpoint-interval": 25},
         trace_text(1, [1, 2, 3, 4], [(50, 3), (51, 3)])),
    ]
    for name, over, ttext in specs:
        cfg = dict(base)
        cfg.update(over)
        if ttext is None:
            stages = list(range(1, int(cfg["stages"]) + 1))
            for tseed in range(1, 200):  # first generated trace that is recoverable with >= 2 events
                ttext = R.generate_trace(tseed, 0.02, 3600.0, int(cfg["iters"]), stages)
                m, e = R.run_experiment(cfg, ttext, 1)
                if "unrecoverable" not in e and len(ttext.splitlines()) >= 3:
                    break
        m, e = R.run_experiment(cfg, ttext, 1)
        full = R.run_experiment_full(cfg, ttext, 1)
        runs.append({"name": name, "cfg": cfg, "seed": 1, "trace": ttext, "metrics_csv": m, "events_csv": e,
                     "full": full})
    return {"source": "src/trainer.cpp:63-289 via harness::run_experiment; src/experiment.cpp:156-174", "runs": runs}


def main():
    os.makedirs(OUT, exist_ok=True)
    if "--append-trainer" in sys.argv:  # add runs missing from trainer_runs.json, keep the others byte-identical
        path = os.path.join(OUT, "trainer_runs.json")
        with open(path) as f:
            cur = json.load(f)
        have = {r["name"] for r in cur["runs"]}
        new = [r for r in trainer_goldens()["runs"] if r["name"] not in have]
        cur["runs"].extend(new)
        with open(path, "w") as f:
            json.dump(cur, f, indent=1)
        print("appended", [r["name"] for r in new])
        return
    payload = {
        "rng": rng_goldens(),
        "failures": failure_goldens(),
        "partition_schedule": partition_schedule_goldens(),
        "recovery": recovery_goldens(),
        "model": model_goldens(),
    }
    with open(os.path.join(OUT, "reference_goldens.json"), "w") as f:
        json.dump(payload, f, indent=1)
    with open(os.path.join(OUT, "trainer_runs.json"), "w") as f:
        json.dump(trainer_goldens(), f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
