#!/usr/bin/env python
"""End-to-end failure-injected training of the LLaMA-124M configuration (BASELINE.json configs[1]
shape: 4 stages x 8 microbatches x 8 sequences x T=1024) on one B200 through the public API
(ckf_run_experiment): a stage failure mid-run recovered by CheckFree (stage 2) or CheckFree+
(stage 1, edge copy), plus the no-failure baseline.  Writes the reference-schema run records
as one JSON summary (loss before/after the failure, spike,
reduction error, measured recovery latency).   python tools/train_124m_demo.py OUT_DIR [ITERS]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_15461_b200 as P

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/train124m"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
fail_at = iters // 2
base = {"block": "llama", "precision": "bf16", "vocab": 50304, "model-dim": 512, "layers": 12, "heads": 8,
        "hidden-dim": 2048, "seq-len": 1024, "stages": 4, "iters": iters, "batch": 64, "microbatches": 8,
        "lr": 6e-4, "eval-interval": 25, "val-size": 16}
runs = {
    "no_failures": ({"strategy": "no-failures"}, []),
    "checkfree_stage2": ({"strategy": "checkfree"}, [(fail_at, 2)]),
    "checkfree_plus_stage1": ({"strategy": "checkfree-plus"}, [(fail_at, 1)]),
}
summary = {}
for name, (over, events) in runs.items():
    cfg = dict(base)
    cfg.update(over)
    trace = "checkfree-trace v1 seed=0 p_hour=0 iter_s=3600 stages=1,2,3,4\n" + "".join(f"{i},{s}\n" for i, s in events)
    t0 = time.time()
    evals, evs, unrec = P.run_experiment(cfg, trace, 1)
    wall = time.time() - t0
    summary[name] = {"config": cfg, "trace": trace, "wall_s": wall, "evals": evals,
                     "events": [{"iter": e[0], "stage": e[1], "action": e[2], "reduction_error": e[3],
                                 "loss_spike": e[4], "recovery_ms": e[5]} for e in evs],
                     "unrecoverable": unrec}
    print(name, f"{wall:.1f}s", "val@0", evals[0][2], "val@end", evals[-1][2],
          [(e[2], round(e[4], 4), round(e[5], 3)) for e in evs], flush=True)
os.makedirs(out, exist_ok=True)
with open(os.path.join(out, "summary.json"), "w") as f:
    json.dump(summary, f, indent=1)
