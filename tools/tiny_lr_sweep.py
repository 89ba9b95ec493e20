#!/usr/bin/env python
"""Picks a LEARNING regime for the configs[0] golden (tiny LLaMA, 4 stages, stage 2 killed
mid-run, CheckFree): runs the GPU trainer (fp32 parity mode) at several learning rates, horizons
and failure iterations and prints the validation curve and the loss spike.  Tool, not a test."""
import json
import sys

sys.path.insert(0, ".")
import paper_2506_15461_b200 as P  # noqa: E402

BASE = {"block": "llama", "precision": "fp32", "vocab": 4096, "model-dim": 256, "layers": 8, "heads": 4,
        "hidden-dim": 768, "seq-len": 128, "stages": 4, "batch": 32, "microbatches": 8,
        "val-size": 8, "strategy": "checkfree"}
for lr, iters, kill, ev in [(3e-3, 200, 100, 10), (3e-3, 200, 150, 10), (4e-3, 200, 120, 10), (5e-3, 200, 120, 10),
                            (3e-3, 300, 200, 25), (2e-3, 300, 200, 25), (3e-3, 150, 100, 10)]:
    trace = f"checkfree-trace v1 seed=0 p_hour=0 iter_s=3600 stages=1,2,3,4\n{kill},2\n"
    cfg = dict(BASE, lr=lr, iters=iters, **{"eval-interval": ev})
    evl, evs, un = P.run_experiment(cfg, trace, 1)
    print(json.dumps({"lr": lr, "iters": iters, "kill": kill, "val": [(e[0], round(e[2], 4)) for e in evl],
                      "events": [(e[0], e[1], e[2], round(e[3], 2), round(e[4], 4)) for e in evs]}), flush=True)
