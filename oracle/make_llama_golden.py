#!/usr/bin/env python
"""Generates tests/golden/llama_tiny_checkfree.json: the CPU fp64 LLaMA oracle
(oracle/llama_oracle.py) running BASELINE.json configs[0] -- tiny LLaMA
(8 layers, d=256, seq 128) as a 4-stage pipeline, synthetic tokens, stage 2
killed at step 50, CheckFree recovery -- plus the same with CheckFree+ and
stage 1 killed (edge copy).  Test infrastructure: the GPU trainer
(ckf_run_experiment) is compared against these curves in tests/test_gpu_trainer_llama.py.
Takes ~10-20 minutes on 8 CPU cores.  `make_llama_golden.py learning` writes the
learning-regime cases (tests/golden/llama_tiny_learning.json, ~20 minutes)."""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import torch  # noqa: E402

import llama_oracle as LO  # noqa: E402

torch.set_num_threads(os.cpu_count() or 8)

BASE = {"block": "llama", "precision": "bf16", "vocab": 4096, "model-dim": 256, "layers": 8, "heads": 4,
        "hidden-dim": 768, "seq-len": 128, "stages": 4, "iters": 100, "batch": 32, "microbatches": 8, "lr": 1e-3,
        "eval-interval": 10, "val-size": 8}


def trace(events):
    head = "checkfree-trace v1 seed=0 p_hour=0 iter_s=3600 stages=1,2,3,4\n"
    return head + "".join(f"{i},{s}\n" for i, s in events)


# learning regime (tests/golden/llama_tiny_learning.json): lr 3e-3 over 200 iterations, where the
# validation loss falls from 8.38 to ~4.4 (-47 %) and the failure at iteration 100 lands in the
# steepest part of the curve (lr / horizon / failure slot chosen with tools/tiny_lr_sweep.py on the GPU)
LEARNING = {"lr": 3e-3, "iters": 200}


def main():
    learning = len(sys.argv) > 1 and sys.argv[1] == "learning"
    out = {}
    cases = [("checkfree_stage2_at50", "checkfree", [(50, 2)]),
             ("checkfree_plus_stage1_at50", "checkfree-plus", [(50, 1)])]
    if learning:
        cases = [("learning_checkfree_stage2_at100", "checkfree", [(100, 2)]),
                 ("learning_checkfree_plus_stage1_at100", "checkfree-plus", [(100, 1)])]
    for name, strat, evs in cases:
        cfg = dict(BASE, strategy=strat, **(LEARNING if learning else {}))
        t0 = time.time()
        evals, events, unrec = LO.run_experiment(cfg, trace(evs), 1)
        out[name] = {"config": cfg, "trace": trace(evs), "seed": 1, "evals": evals, "events": events,
                     "unrecoverable": unrec, "seconds": time.time() - t0}
        print(name, "done in", round(time.time() - t0, 1), "s", evals[-1], flush=True)
    path = os.path.join(os.path.dirname(HERE), "tests", "golden",
                        "llama_tiny_learning.json" if learning else "llama_tiny_checkfree.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
