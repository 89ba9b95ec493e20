"""Cost model re-parameterised with B200 measurements -> one JSON file.

1. per-stage per-microbatch forward / backward seconds MEASURED on the engine for the bench
   workloads (cost.measure_stage_seconds), and the checkpoint path's GPU->pinned-host copy
   bandwidth MEASURED here;
2. CostParams from those (cost.params_b200) on three network profiles: one B200 NVSwitch
   node, the same stages split over two nodes (scale-out NIC between them), and the
   reference's synthetic 5-site WAN (cost_model.cpp:71-99);
3. iteration / recovery time per strategy on each profile;
4. the reference's compare_strategies experiment (experiment.cpp:215-275) on the GPU
   trainer: LLaMA-124M, one shared failure trace per failure rate (5/10/16 % per stage-hour,
   iter_s 120 = the reference default, intermediate stages), target = the validation loss
   the failure-free run reaches at `--target-iter`; each strategy costed on each profile
   (modelled hours) and by the B200's own wall clock.

    python tools/cost_b200.py --out gpurun_out/cost_b200.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

STRATEGIES = ["checkpointing", "redundant", "checkfree", "checkfree-plus"]


def d2h_bandwidth(nbytes=1 << 30, reps=5):
    import torch
    src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    dst = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    best = 0.0
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) / 1e3))
    return best


def measure(wname: str, w: dict):
    import paper_2506_15461_b200 as P
    from paper_2506_15461_b200 import api, cost

    mb_rows = w["rows"] // w["microbatches"]
    spec = api.ModelSpec.llama(w["output_dim"], w["model_dim"], w["layers"], w["heads"], w["hidden_dim"],
                               w["seq_len"], w["stages"], precision=w["precision"],
                               max_tokens=mb_rows * w["seq_len"])
    eng = P.Engine(spec)
    eng.init(1, 3e-4)
    tpm = mb_rows * w["seq_len"]
    f, b, detail = cost.measure_stage_seconds(eng, spec, tpm, w["microbatches"])
    stage_p, emb_p, head_p = eng.stage_params, eng.embed_params, eng.deembed_params
    eng.close()
    # The iteration fuses microbatches into groups, so a lone microbatch's forward overstates
    # the in-iteration forward: time the whole batch's forward in one pass on the same model
    # built for the batch's tokens, and split the measured iteration with that.
    detail["per_microbatch_forward"] = {"fwd_seconds": f, "bwd_seconds": b}
    eng_all = None
    try:
        spec_all = api.ModelSpec.llama(w["output_dim"], w["model_dim"], w["layers"], w["heads"], w["hidden_dim"],
                                       w["seq_len"], w["stages"], precision=w["precision"],
                                       max_tokens=w["rows"] * w["seq_len"])
        eng_all = P.Engine(spec_all)
        eng_all.init(1, 3e-4)
        fa, _, da = cost.measure_stage_seconds(eng_all, spec_all, w["rows"] * w["seq_len"], 1)
        it_stage = detail["iteration_s"] / (w["stages"] * w["microbatches"])
        f = fa / w["microbatches"]
        b = max(it_stage - f, f)
        detail["forward_source"] = "whole-batch forward pass"
        detail["forward_pass_s"] = da["forward_pass_s"]
    except Exception as e:  # the whole-batch model does not fit: keep the per-microbatch split
        detail["forward_source"] = f"per-microbatch forward ({type(e).__name__})"
    finally:
        if eng_all is not None:
            eng_all.close()
    total = w["stages"] * stage_p + emb_p + head_p
    detail.update({"workload": wname, "fwd_seconds": f, "bwd_seconds": b, "stage_params": stage_p,
                   "edge_params": max(emb_p, head_p), "total_params": total})
    return detail


def costs(cost, prof, par, s, interval):
    out = {}
    for strat in STRATEGIES:
        it = cost.iteration_cost(strat, prof, par, interval)
        rec = {}
        for st in range(1, s + 1):
            try:
                rec[st] = cost.recovery_time(strat, prof, par, st, interval)
            except cost.CostError:
                rec[st] = None
        out[strat] = {"iteration": it, "recovery_s": rec}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/cost_b200.json")
    ap.add_argument("--workloads", default="llama-124m,llama-1.5b")
    ap.add_argument("--compare-iters", type=int, default=400)
    ap.add_argument("--target-iter", type=int, default=250)
    ap.add_argument("--rates", default="0.05,0.10,0.16")
    ap.add_argument("--interval", type=int, default=50)
    ap.add_argument("--skip-compare", action="store_true")
    args = ap.parse_args()

    import torch

    import bench
    from paper_2506_15461_b200 import api, cost

    torch.cuda.set_device(0)
    peaks, _ = bench.load_peaks()
    storage_bps = d2h_bandwidth()
    links = dict(hbm_bps=peaks["hbm_gbs"] * 1e9, storage_bps=storage_bps)
    result = {"links": {**links, "nvlink_bps": 900e9, "nvlink_note": "nominal NVLink 5 per direction (1 GPU box)",
                        "nic_bps": 50e9, "storage_note": "measured GPU->pinned host copy (checkpoint path)"},
              "workloads": {}}

    for wname in args.workloads.split(","):
        w = bench.WORKLOADS[wname]
        m = measure(wname, w)
        par = cost.params_b200(m["fwd_seconds"], m["bwd_seconds"], m["tokens_per_microbatch"], w["model_dim"],
                               m["stage_params"], m["edge_params"], m["total_params"], w["microbatches"])
        s = w["stages"]
        profiles = {"b200_node": cost.Profile.b200(s, **links),
                    "b200_2nodes": cost.Profile.b200(s, gpus_per_node=max(1, s // 2), nodes=2, **links),
                    "wan_synthetic": cost.Profile.synthetic(s)}
        m["params"] = vars(par)
        m["costs"] = {pn: costs(cost, p, par, s, args.interval) for pn, p in profiles.items()}
        result["workloads"][wname] = m
        print(wname, json.dumps({k: m[k] for k in ("fwd_seconds", "bwd_seconds", "iteration_s", "per_microbatch_forward")}), flush=True)

    if not args.skip_compare:
        w = bench.WORKLOADS["llama-124m"]
        s = w["stages"]
        cfg = {"block": "llama", "precision": "bf16", "vocab": w["output_dim"], "model-dim": w["model_dim"],
               "layers": w["layers"], "heads": w["heads"], "hidden-dim": w["hidden_dim"], "seq-len": w["seq_len"],
               "stages": s, "iters": args.compare_iters, "batch": w["rows"], "microbatches": w["microbatches"],
               "lr": 6e-4, "eval-interval": 25, "val-size": 16, "checkpoint-interval": args.interval}
        t0 = time.time()
        base = cost.run_record({**cfg, "strategy": "no-failures"},
                               api.generate_trace(0, 0.0, 120.0, args.compare_iters, list(range(1, s + 1))), 0)
        target = next(v for (it, _, v, _, _) in base["evals"] if it >= args.target_iter)
        cfg["target-loss"] = repr(target)
        m = result["workloads"]["llama-124m"]
        par = cost.Params(**m["params"])
        profiles = {"b200_node": cost.Profile.b200(s, **links),
                    "b200_2nodes": cost.Profile.b200(s, gpus_per_node=max(1, s // 2), nodes=2, **links),
                    "wan_synthetic": cost.Profile.synthetic(s)}
        cmp = {"config": cfg, "target_val_loss": target, "no_failures_evals": base["evals"], "rates": {}}
        for rate in [float(r) for r in args.rates.split(",")]:
            trace = api.generate_trace(17, rate, 120.0, args.compare_iters, list(range(2, s)))
            by_prof = cost.compare_strategies(cfg, STRATEGIES, trace, profiles, par, seed=0)
            entry = {"trace": trace, "profiles": {}}
            for pn, rows in by_prof.items():
                entry["profiles"][pn] = {"rows": [vars(r) for r in rows], "table": cost.comparison_table(rows)}
                print(f"p_hour={rate} {pn}\n" + cost.comparison_table(rows), flush=True)
            cmp["rates"][str(rate)] = entry
        cmp["wall_s"] = time.time() - t0
        result["compare_strategies"] = cmp

    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(result, f, indent=1, default=str)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
