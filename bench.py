#!/usr/bin/env python
"""Benchmark of the CheckFree / CheckFree+ pipeline training step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]

One "step" = one pipeline::run_iteration (src/pipeline.cpp:58-95) over one
synthetic batch: every microbatch forward + backward through all stages in
its execution order, gradient accumulation, fused Adam + omega per stage.
N=1 keeps every stage resident on cuda:0 (BASELINE.json configs[1] shape);
N>1 places contiguous stage blocks per rank (stage transfers over NCCL).

Prints ONE JSON line (rank 0).  `value` = tokens/s with inputs resident in HBM,
device time from CUDA events on the engine's stream, max over ranks, L2
flushed (256 MiB memset) between steps outside the timed events.  `e2e` = the
same step through the public API with pinned HOST inputs (H2D inside the timed
region) and the loss/omegas read back.  `roofline` covers the dominant kernel
class, timed live with CUDA events inside the timed region.  `cpu_baseline`
times the reference's own CPU path (oracle/_ref, the unmodified reference
library) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# MEASURED_PEAKS.json is driver-written on the GPU box; when it is absent we use the
# pool's measured values recorded in BASELINE.md §4 (bf16 1632.8 burst / 1361.2
# sustained TFLOP/s, HBM 6544 GB/s) and say so in the JSON ("peak_source").
PEAKS_FALLBACK = {"hbm_gbs": 6544.0, "bf16_tflops": 1632.8, "bf16_tflops_sustained": 1361.2}

# Workloads.  The residual-MLP block is the reference's own model family
# (model.hpp:55-60); "mlp-124m" runs it at the LLaMA-124M pipeline shape
# (d=512, hidden=2048, 12 layers, 4 stages, 8 microbatches, 65,536 rows/iter)
# in the fp32 parity precision.
WORKLOADS = {
    # BASELINE.json configs[1]: LLaMA-124M, 4 stages x 8 microbatches, seq 1024 (8 seqs / microbatch)
    "llama-124m": dict(block="llama", precision="bf16", input_dim=50304, hidden_dim=2048, model_dim=512,
                       output_dim=50304, layers=12, stages=4, microbatches=8, rows=64, seq_len=1024, heads=8),
    # configs[0] shape (tiny LLaMA, 4 stages) -- a parity case, not the headline
    "llama-tiny": dict(block="llama", precision="bf16", input_dim=4096, hidden_dim=768, model_dim=256,
                       output_dim=4096, layers=8, stages=4, microbatches=8, rows=32, seq_len=128, heads=4),
    # configs[2] shape on one GPU (LLaMA-500M, 8 stages)
    "llama-500m": dict(block="llama", precision="bf16", input_dim=50304, hidden_dim=4096, model_dim=1024,
                       output_dim=50304, layers=24, stages=8, microbatches=8, rows=64, seq_len=1024, heads=16),
    # configs[3] model on one GPU (LLaMA-1.5B, 4 stages, T=4096, head_dim 128): one replica's
    # 8 microbatches of one sequence each (the 8-GPU run adds DP2 over 4 pipeline ranks)
    "llama-1.5b": dict(block="llama", precision="bf16", input_dim=50304, hidden_dim=5632, model_dim=2048,
                       output_dim=50304, layers=24, stages=4, microbatches=8, rows=8, seq_len=4096, heads=16),
    "mlp-124m": dict(block="mlp", precision="fp32", input_dim=16, hidden_dim=2048, model_dim=512, output_dim=16,
                     layers=12, stages=4, microbatches=8, rows=65536, seq_len=1, heads=1),
}
# north_star target on one GPU: BASELINE.json configs[2], LLaMA-500M, 8 stages, CheckFree+
DEFAULT_WORKLOAD = "llama-500m"
DEFAULT_STRATEGY = "checkfree-plus"


def flops_per_token(w: dict) -> float:
    """Training FLOPs per row/token (fwd + 2x bwd), algorithmic."""
    if w["block"] == "mlp":
        d, h, L = w["model_dim"], w["hidden_dim"], w["layers"]
        return 6.0 * (w["input_dim"] * d + L * 2 * d * h + d * w["output_dim"])
    d, f, L, V, T = w["model_dim"], w["hidden_dim"], w["layers"], w["output_dim"], w["seq_len"]
    return 6.0 * (L * (4 * d * d + 3 * d * f) + d * V) + 6.0 * L * d * T  # causal attention at half


def load_peaks() -> tuple[dict, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            raw = json.load(f)
        out = dict(PEAKS_FALLBACK)
        for k in out:
            if k in raw and isinstance(raw[k], (int, float)):
                out[k] = float(raw[k])
        return out, "measured"
    return dict(PEAKS_FALLBACK), "BASELINE.md §4 measured peaks (MEASURED_PEAKS.json absent)"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region through NVML (in-process,
    every 50 ms: cheap enough not to perturb the host that launches the step); nvidia-smi
    subprocess polling only when pynvml is unavailable."""

    # nvmlClocksEventReasons bits
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown"}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples: list[tuple[float, float, set]] = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        self.power: list[float] = []
        self.temp: list[float] = []
        # CKF_BENCH_CLOCKS="period_s[,full]" (default 0.1 s, clocks + reasons only; "full" adds power and
        # temperature, whose NVML queries were seen to coincide with slow steps)
        spec = os.environ.get("CKF_BENCH_CLOCKS", "0.1").split(",")
        self.period = float(spec[0])
        self.full = len(spec) > 1 and spec[1] == "full"
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            h = None
            try:
                pr = torch.cuda.get_device_properties(gpu)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(gpu)
            self._nvml = (pynvml, h)
        except Exception:
            self._nvml = None

    def _run(self):
        if self._nvml is not None:
            nv, h = self._nvml
            get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            while not self._stop.is_set():
                try:
                    sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    bits = int(get_reasons(h))
                    self.samples.append((sm, mx, {n for b, n in self.REASONS.items() if bits & b}))
                    if self.full:
                        try:
                            self.power.append(nv.nvmlDeviceGetPowerUsage(h) / 1000.0)
                            self.temp.append(float(nv.nvmlDeviceGetTemperature(h, nv.NVML_TEMPERATURE_GPU)))
                        except Exception:
                            pass
                except Exception:
                    pass
                self._stop.wait(self.period)
            return
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                parts = [x.strip() for x in out.split(",")]
                reasons = {n for n, v in zip(names, parts[2:]) if v.lower() == "active"}
                self.samples.append((float(parts[0]), float(parts[1]), reasons))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted(set().union(*[s[2] for s in self.samples]))
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons, "samples": len(self.samples),
                "sm_mhz_min": min(s[0] for s in self.samples),
                "power_w_median": statistics.median(self.power) if self.power else None,
                "temp_c_max": max(self.temp) if self.temp else None,
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


# ----------------------------------------------------------------------------- reference CPU arm
def ref_sample_kv(w: dict, rows: int) -> dict:
    """Residual-MLP config of the reference at the workload's pipeline shape, `rows` rows per iteration."""
    return {"input-dim": w["input_dim"] if w["block"] == "mlp" else 16,
            "hidden-dim": w["hidden_dim"], "model-dim": w["model_dim"],
            "output-dim": w["output_dim"] if w["block"] == "mlp" else 16,
            "layers": w["layers"], "stages": w["stages"], "batch": rows, "microbatches": w["microbatches"],
            "activation": "tanh", "task": "regression", "strategy": "checkfree", "lr": 3e-4}


def cpu_reference(w: dict, iters: int, rows: int) -> dict:
    """Times the UNMODIFIED reference (oracle/_ref) training loop body on the host cores."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refshim  # noqa: E402  (test/baseline infrastructure only)
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    s_per_iter = refshim.time_train_iterations(ref_sample_kv(w, rows), 1, iters)
    return {"value": rows / s_per_iter, "unit": "tokens/s", "cores": refshim.parallel_threads(),
            "kind": "reference", "s_per_iter": s_per_iter,
            "sample": f"reference residual-MLP block (fp64, OpenMP) at this workload's pipeline shape "
                      f"(d={w['model_dim']}, hidden={w['hidden_dim']}, L={w['layers']}, s={w['stages']}, "
                      f"m={w['microbatches']}), {rows} rows/iteration, {iters} timed iterations after 1 warm-up"}


def run_reference_arm(args, w: dict):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    rows = ref_rows(w)
    # each timed step is one reference iteration at `rows` rows; the number of timed iterations is
    # capped so the whole arm ends within a few minutes at the large workloads (stated in `sample`)
    probe = cpu_reference(w, 1, rows)
    iters = max(1, min(args.steps, int(120.0 / max(probe["s_per_iter"], 1e-3))))
    cb = cpu_reference(w, iters, rows)
    line = {"metric": METRIC, "value": cb["value"], "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": cb["s_per_iter"] * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "config": workload_config(args, w),
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


METRIC = "pipeline train tokens/s"


def placement(world: int, s: int):
    """(pipeline ranks P, replicas R) with P * R = world: contiguous stage blocks per rank,
    data-parallel replicas once every stage has its own GPU."""
    if world <= s and s % world == 0:
        return world, 1
    if world % s == 0:
        return s, world // s
    raise SystemExit(f"{s} stages cannot be placed on {world} GPUs (need world | s or s | world)")


def scaled_workload(w: dict, gpus: int) -> dict:
    """Weak scaling over pipeline ranks: with the stages partitioned over P ranks the step runs
    P x the microbatches (same tokens per microbatch), so every GPU pushes the same token-layers
    per step as the single-GPU run (65,536 tokens x 24 layers at LLaMA-500M) and the 1F1B bubble
    (P-1)/(m+P-1) stays ~10 %.  Data-parallel replicas each add their own batch."""
    P, _ = placement(gpus, w["stages"])
    if P == 1:
        return w
    return dict(w, microbatches=w["microbatches"] * P, rows=w["rows"] * P)


def workload_config(args, w: dict) -> dict:
    P, R = placement(args.gpus, w["stages"])
    cfg = {"parallelism": f"pp{P}" + (f"xdp{R}" if R > 1 else ""),"workload": args.workload, "block": w["block"], "stages": w["stages"],
           "microbatches": w["microbatches"], "layers": w["layers"], "model_dim": w["model_dim"],
           "hidden_dim": w["hidden_dim"], "tokens_per_step": tokens_per_step(w) * R, "seq_len": w["seq_len"],
           "strategy": getattr(args, "strategy", DEFAULT_STRATEGY),
           "schedule": "swapped_half (swapped first/last-stage order at even microbatches) + per-step edge replica "
                       "refresh" if getattr(args, "strategy", DEFAULT_STRATEGY) == "checkfree-plus" else "standard", "placement": f"{w['stages']} stages on {P} pipeline rank(s) x {R} replica(s)",
           "l2": "256 MiB memset between timed steps (outside the events)",
           "pipeline_schedule": ("1F1B (host-planned global op order; transfers on send/recv streams, "
                                 + ("per-link NCCL communicators)" if os.environ.get("CKF_TRANSPORT") == "nccl"
                                    else "peer-memory copies into the next rank's mailbox + device flags)"))
                                if P > 1 else "all stages resident (fused microbatch groups)",
           "bubble_1f1b": (P - 1) / (w["microbatches"] + P - 1) if P > 1 else 0.0}
    if w["block"] == "llama":
        cfg.update(vocab=w["output_dim"], heads=w["heads"])
        # all stages resident on a rank => microbatches sharing an execution order run as
        # one fused pass (Engine::run_iteration; cap 0 = fit to HBM, 1 = per microbatch)
        cfg["microbatch_fusion"] = ("cap " + os.environ["CKF_MB_GROUP"]) if os.environ.get("CKF_MB_GROUP") else (
            "auto (fit to HBM)" if P == 1 else "off (stages partitioned)")
    return cfg


def tokens_per_step(w: dict) -> int:
    return w["rows"] * (w["seq_len"] if w["block"] == "llama" else 1)


# ----------------------------------------------------------------------------- our arm
def make_batch(w: dict, gen, device):
    import torch
    rows = w["rows"]
    if w["block"] == "llama":
        x = torch.randint(0, w["output_dim"], (rows, w["seq_len"] + 1), generator=gen, dtype=torch.int32)
        return x, None
    x = torch.rand((rows, w["input_dim"]), generator=gen, dtype=torch.float64) * 2 - 1
    y = torch.rand((rows, w["output_dim"]), generator=gen, dtype=torch.float64) * 2 - 1
    return x, y


def run_ours(args, w: dict):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2506_15461_b200 as P_
    from paper_2506_15461_b200 import api

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # CKF_BENCH_SAME_GPU=1 (tests only): every rank on cuda:0, gloo for the host plumbing, no NCCL
    # -- the N>1 pipeline path (placement, 1F1B across processes over the peer transport, peer
    # recovery) runs as a FUNCTIONAL check on a one-GPU box; its timings are time-sliced, not
    # performance numbers, and the JSON says so
    same_gpu = world > 1 and os.environ.get("CKF_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    s = w["stages"]
    P, R = placement(world, s)
    if same_gpu and (R > 1 or w["block"] != "llama"):
        raise SystemExit("CKF_BENCH_SAME_GPU covers the LLaMA pipeline without data-parallel replicas")

    mb_rows = w["rows"] // w["microbatches"]
    if w["block"] == "llama":
        spec = api.ModelSpec.llama(w["output_dim"], w["model_dim"], w["layers"], w["heads"], w["hidden_dim"],
                                   w["seq_len"], s, precision=w["precision"], max_tokens=mb_rows * w["seq_len"],
                                   device=local)
    else:
        spec = api.ModelSpec(w["input_dim"], w["hidden_dim"], w["model_dim"], w["output_dim"], w["layers"], s,
                             precision=w["precision"], max_rows=mb_rows, device=local)
    eng = P_.Engine(spec)
    eng.init(1, 3e-4)
    if args.strategy == "redundant":
        eng.set_redundant(True)
    cfp = args.strategy == "checkfree-plus"
    if cfp:
        eng.set_edge_replicas(True)  # trainer.cpp:83-84: E / E^-1 replicas refreshed inside every step
    if same_gpu:
        eng.set_placement(world, rank, [(sid - 1) * P // s for sid in range(1, s + 1)], R)
        eng.enable_peer_transport(w["microbatches"])
        blobs = [None] * world
        dist.all_gather_object(blobs, eng.ipc_export())
        eng.ipc_import(blobs)
    elif world > 1:
        uid = [P_.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        eng.attach_comm(uid[0], world, rank, [(sid - 1) * P // s for sid in range(1, s + 1)], R)
        if P > 1 and w["block"] == "llama" and os.environ.get("CKF_TRANSPORT", "peer") != "nccl":
            # 1F1B stage transfers through peer memory: copies into the next rank's mailbox over
            # NVLink + flags in its HBM (CKF_TRANSPORT=nccl: NCCL send/recv on per-link communicators)
            eng.enable_peer_transport(w["microbatches"])
        eng.exchange_peers()  # CUDA IPC mappings: recovery reads neighbours from the peers' HBM

    orders = np.array(api.build_schedule(w["microbatches"], cfp, s), np.int32)  # pipeline.cpp:41-56
    gen = torch.Generator().manual_seed(1234 + rank // P)  # one batch per replica (weak scaling)
    xh, yh = make_batch(w, gen, local)
    xh, yh = xh.pin_memory(), (yh.pin_memory() if yh is not None else None)
    xd = xh.to(f"cuda:{local}", non_blocking=False)
    yd = yh.to(f"cuda:{local}") if yh is not None else None
    if w["block"] == "mlp" and w["precision"] == "fp32":
        xd, yd = xd.float(), yd.float()
    torch.cuda.synchronize()

    stream = torch.cuda.ExternalStream(eng.stream_ptr(), device=local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def step(it, on_device):
        if on_device:
            r = eng.run_iteration(orders, xd, yd, it, on_device=True)
        else:
            r = eng.run_iteration(orders, xh.numpy(), yh.numpy() if yh is not None else None, it)
        if same_gpu:  # the iteration boundary the NCCL loss / omega all-reduce provides otherwise
            dist.barrier()
        return r

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    per_step = []  # device ms of every timed step, per timed pass (variance check)

    def timed(k, on_device, it0):
        # Device time of each step from the engine's own CUDA events on its stream (first
        # device op of run_iteration .. loss / omega D2H): the L2 flush runs before, outside;
        # host scheduling after the step's final sync is excluded.  The outer a/b events
        # (which also count host gaps at the step boundaries) are kept for comparison.
        evs, dev = [], []
        for i in range(k):
            with torch.cuda.stream(stream):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
            step(it0 + i, on_device)
            dev.append(eng.last_step_ms())
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        per_step.append({"device": [round(x, 3) for x in dev],
                         "outer_events": [round(a.elapsed_time(b), 3) for a, b in evs]})
        return sum(dev)

    it = 1
    for _ in range(args.warmup):
        step(it, True)
        it += 1
    barrier()
    launches0 = eng.kernel_launches()
    with ClockSampler(local) as clk:
        barrier()
        ms_total = timed(args.steps, True, it)
        barrier()
    it += args.steps
    launches = eng.kernel_launches() - launches0

    # e2e through the public API with pinned host buffers (H2D + loss/omega D2H inside),
    # right after the device-resident pass so both see the same thermal / power state
    for _ in range(2):
        step(it, False)
        it += 1
    barrier()
    e2e_total = timed(args.steps, False, it)
    barrier()
    it += args.steps

    # roofline pass: the same K steps again with every tagged launch bracketed by
    # CUDA events on the engine stream (kept out of the headline timing: the
    # per-launch event records add host work to a launch-dense step)
    eng.kernel_timing(True)
    barrier()
    ms_prof = timed(args.steps, True, it)
    barrier()
    it += args.steps
    kstats = {c: eng.kernel_stats(c) for c in api.Engine.KCLASS}
    eng.kernel_timing(False)

    ms = ms_total / args.steps
    e2e_ms = e2e_total / args.steps
    if world > 1:
        t = torch.tensor([ms, e2e_ms], dtype=torch.float64, device="cpu" if same_gpu else f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_ms = t.tolist()

    # stage-recovery latency (trainer.cpp:230-276 semantics, weights + moments + lr + omega), stage 2
    rec = None
    if s >= 3:
        # kill-to-ready latency of an interior stage (CheckFree omega-average, trainer.cpp:230-276):
        # one fused pass -- weights, Fresh moments, zeroed gradient, bf16 shadow -- CUDA events on the
        # replacement GPU's stream; algorithmic bytes 26 per fp32 parameter (read Wp, Wn; write W, m,
        # v, g; bf16 W).  N > 1: the first stage of pipeline rank 1, whose previous neighbour lives on
        # rank 0 -- the kernel reads it from the peer's HBM over NVLink (CUDA IPC mapping); every rank
        # takes part (the recovery is collective) and the latency is the replacement GPU's.
        sid = 2 if P == 1 else min(s - 1, s // P + 1)
        lat = []
        for _ in range(5):
            eng.kill_stage(sid)
            lat.append(eng.recover_stage(sid, reduction_error=False).latency_ms)
            if same_gpu:  # no communicator: share the replacement GPU's latency, fence the peers
                lt = torch.tensor([lat[-1]], dtype=torch.float64)
                dist.all_reduce(lt, op=dist.ReduceOp.MAX)
                lat[-1] = float(lt.item())
        n_stage = eng.stage_params
        pb = 4 if w["precision"] != "fp64" else 8
        nbytes = n_stage * (6 * pb + (2 if w["precision"] == "bf16" else 0))
        med = statistics.median(lat)
        owner = lambda x: (x - 1) * P // s  # noqa: E731
        remote = [n for n in (sid - 1, sid + 1) if owner(n) != owner(sid)]
        rec = {"stage": sid, "stage_params": n_stage, "latency_ms": med, "latency_ms_min": min(lat),
               "bytes": nbytes, "gbs": nbytes / (med / 1e3) / 1e9,
               "neighbours_on_peers": remote,
               "what": "kill -> ready: omega-weighted weights, Fresh m/v, g = 0, bf16 shadow in one kernel"}
        if remote:
            rec["nvlink_ingress_gbs"] = len(remote) * pb * n_stage / (med / 1e3) / 1e9
        if cfp:
            # CheckFree+ first-stage recovery: stage 1 := stage 2, E := its replica (recovery.cpp:90-101)
            el = []
            for _ in range(3 if not same_gpu else 0):  # (the edge replica pull needs NCCL across ranks)
                eng.kill_stage(1)
                el.append(eng.recover_stage(1, mode=P_._native.CKF_REC_EDGE, reduction_error=False).latency_ms)
            rec["edge_stage1_latency_ms"] = statistics.median(el) if el else None

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks, peak_src = load_peaks()
    sweep = recovery_sweep(P_, local, peaks["hbm_gbs"], cpu=not args.no_cpu_baseline) \
        if (world == 1 and not args.no_recovery_sweep) else None
    tok = tokens_per_step(w) * R  # every replica trains on its own batch
    value = tok / (ms / 1e3)
    e2e_value = tok / (e2e_ms / 1e3)
    # dominant kernel class (by device time inside the timed region)
    dom = max(kstats, key=lambda c: kstats[c][0])

    def class_rate(c, v):
        # every class against its own roofline: the tensor classes in TFLOP/s against the sustained
        # bf16 peak, the others in GB/s of algorithmic bytes against the measured copy bandwidth
        cms, cn, cfl, cby = v
        r = {"ms": cms, "launches": cn}
        if cms > 0 and c in ("gemm", "attention") and cfl > 0:
            r.update(tflops=cfl / (cms / 1e3) / 1e12, frac=cfl / (cms / 1e3) / 1e12 / peaks["bf16_tflops_sustained"])
        elif cms > 0 and cby > 0:
            r.update(gbs=cby / (cms / 1e3) / 1e9, frac=cby / (cms / 1e3) / 1e9 / peaks["hbm_gbs"])
        return r
    kms, kn, kfl, kby = kstats[dom]
    if dom in ("gemm", "attention") and w["precision"] == "bf16":
        achieved = kfl / (kms / 1e3) / 1e12
        roof = {"bound": "tensor", "unit": "TFLOP/s", "peak": peaks["bf16_tflops_sustained"]}
    elif dom in ("gemm", "attention"):
        achieved = kfl / (kms / 1e3) / 1e12
        roof = {"bound": "tensor", "unit": "TFLOP/s", "peak": peaks["bf16_tflops_sustained"],
                "note": f"{w['precision']} parity path on CUDA cores, shown against the bf16 tensor peak"}
    else:
        achieved = kby / (kms / 1e3) / 1e9
        roof = {"bound": "hbm", "unit": "GB/s", "peak": peaks["hbm_gbs"]}
    # measured DRAM traffic per launch of the dominant class: ncu capture committed under
    # profiles/ (tools/ncu_traffic.py; same workload, one step's launches)
    traffic, traffic_src = None, None
    # per-workload capture (tools/ncu_traffic.py): r02_<workload>_<class>_dram_traffic.json; the
    # round-1 capture covers llama-124m
    tp = os.path.join(ROOT, "profiles", f"r02_{args.workload}_{dom}_dram_traffic.json")
    if not os.path.exists(tp) and args.workload == "llama-124m":
        tp = os.path.join(ROOT, "profiles", f"r01_{dom}_dram_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj.get("traffic_per_launch_bytes")
        traffic_src = f"profiles/{os.path.basename(tp)} ({tj.get('launches')} launches, ncu dram__bytes_read+write)"
    roof.update(kernel_class=dom, achieved=achieved, frac=achieved / roof["peak"], traffic=traffic,
                traffic_source=traffic_src,
                peak_source=peak_src, launches=kn, share_of_step=kms / ms_prof,
                timing="CUDA events around each launch on the engine stream, separate pass of the same steps",
                per_launch={"ms": kms / max(kn, 1), "flops": kfl / max(kn, 1), "bytes": kby / max(kn, 1)},
                classes={c: class_rate(c, v) for c, v in kstats.items() if v[1]})
    step_tflops = flops_per_token(w) * tok / (ms / 1e3) / 1e12

    if rec is not None:
        rec["frac_hbm"] = rec["gbs"] / peaks["hbm_gbs"]

    h2d = xh.numel() * xh.element_size() + (yh.numel() * yh.element_size() if yh is not None else 0)
    d2h = 8 * (1 + s) + 8 * w["microbatches"]
    cpu, cpu_llama = None, None
    if not args.no_cpu_baseline:
        cpu = cpu_reference(w, 1, ref_rows(w))
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample", "s_per_iter")}
        cpu_llama = cpu_llama_oracle()
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": {"fp32": "f32", "fp64": "f64", "bf16": "bf16"}[w["precision"]],
            "data": "synthetic (seeded random rows/tokens; random-init weights via the counter RNG)",
            "config": workload_config(args, w),
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms},
            "gpu_launches": launches, "roofline": roof, "step_tflops": step_tflops,
            "step_ms": {"timed": per_step[0], "e2e": per_step[-1]},
            "timing": "engine CUDA events per step (first device op .. result D2H), L2 flushed before each step",
            "flops_per_token": flops_per_token(w), "cpu_baseline": cpu, "cpu_baseline_llama_oracle": cpu_llama,
            "clocks": clk.summary(),
            "recovery": rec, "recovery_sweep": sweep}
    if same_gpu:
        line["functional_same_gpu"] = ("CKF_BENCH_SAME_GPU: all ranks time-slice ONE GPU (peer transport over CUDA "
                                       "IPC, gloo host plumbing) -- a functional check of the N>1 path, not a "
                                       "performance number")
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def recovery_sweep(P, local, hbm_peak, cpu=True):
    """BASELINE.json configs[4]: omega-weighted neighbour-average reinit over stage sizes 10M-400M
    params (fp32 masters, recovery.cpp:57-73, omega = (4, 1)).  Two passes per size, L2 flushed
    before each rep, CUDA events: the engine's FUSED recovery (26 B/param: read W_prev, W_next;
    write W, m, v, g; bf16 shadow) and the weights-only average (12 B/param).  Beside each point
    the reference's own recover_checkfree (oracle/_ref, serial as shipped, fp64) on the host."""
    import torch
    dev = f"cuda:{local}"
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = []

    def timeit(fn):
        fn()
        times = []
        for _ in range(5):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        return sorted(times)[len(times) // 2]

    refshim = None
    if cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import refshim  # noqa: F811  (baseline infrastructure only)
    for n in (10_000_000, 12_585_984, 25_000_000, 50_337_792, 100_000_000, 200_000_000, 400_000_000):
        wp = torch.rand(n, device=dev)
        wn = torch.rand(n, device=dev)
        ws = torch.empty(n, device=dev)
        m, v, g = torch.empty(n, device=dev), torch.empty(n, device=dev), torch.empty(n, device=dev)
        wlp = torch.empty(n, device=dev, dtype=torch.bfloat16)
        ms_f = timeit(lambda: P.api.recover_stage_device(wp, wn, ws, m, v, g, 4.0, 1.0, w_bf16=wlp))
        ms_w = timeit(lambda: P.recover_device(wp, wn, ws, 4.0, 1.0))
        pt = {"params": n, "ms": ms_f, "gbs": 26.0 * n / (ms_f / 1e3) / 1e9,
              "frac_hbm": 26.0 * n / (ms_f / 1e3) / 1e9 / hbm_peak, "bytes_per_param": 26,
              "weights_only": {"ms": ms_w, "gbs": 12.0 * n / (ms_w / 1e3) / 1e9,
                               "frac_hbm": 12.0 * n / (ms_w / 1e3) / 1e9 / hbm_peak}}
        if refshim is not None and refshim.available():
            s_ref = refshim.time_recover_checkfree(n, 1)
            pt["cpu_reference"] = {"ms": s_ref * 1e3, "gbs": 24.0 * n / s_ref / 1e9, "cores": 1,
                                   "kind": "reference", "what": "recovery::recover_checkfree, fp64, serial as shipped"}
        out.append(pt)
        del wp, wn, ws, m, v, g, wlp
    torch.cuda.empty_cache()
    return out


def ref_rows(w: dict) -> int:
    """Rows per iteration of the reference arm's bounded sample: >= one row per microbatch and at
    least 32, so per-iteration fixed costs (Adam over the fp64 stage vectors) do not dominate."""
    return max(w["microbatches"], 64 if w["block"] == "mlp" else 32)


def cpu_llama_oracle() -> dict:
    """The LLaMA CPU oracle (oracle/llama_oracle.py, torch fp64 on the host cores) timed on
    BASELINE.json configs[0]: tiny LLaMA (d=256, L=8, H=4, f=768, V=4096, T=128), 4 stages,
    8 microbatches x 4 sequences = 4096 tokens per iteration, one iteration after a warm-up."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import llama_oracle as LO  # noqa: E402  (baseline infrastructure only)
    torch.set_num_threads(os.cpu_count() or 1)
    spec = LO.LSpec(vocab=4096, d=256, layers=8, heads=4, ffn=768, seq_len=128, stages=4)
    model = LO.LModel(spec, 3, 3e-4)
    sched = LO.build_schedule(8, False, 4)
    toks = LO.token_batch(1, 1, 1, 32, 128, 4096)
    LO.run_iteration(model, sched, toks)
    t0 = time.perf_counter()
    LO.run_iteration(model, sched, toks)
    dt = time.perf_counter() - t0
    return {"value": 32 * 128 / dt, "unit": "tokens/s", "cores": torch.get_num_threads(), "kind": "port",
            "s_per_iter": dt, "sample": "LLaMA CPU oracle (torch fp64) on configs[0]: tiny LLaMA, 4 stages, "
                                        "8 microbatches x 4 seq x T=128, 1 timed iteration after 1 warm-up"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=DEFAULT_WORKLOAD)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-recovery-sweep", action="store_true")
    ap.add_argument("--strategy", choices=["checkfree", "checkfree-plus", "redundant"], default=DEFAULT_STRATEGY,
                    help="checkfree-plus: swapped_half orders + per-step edge replica refresh (default); "
                         "redundant: the redundant-computation baseline measured (extra forward per stage, "
                         "post-step replica refresh)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    w = scaled_workload(WORKLOADS[args.workload], args.gpus)
    if args.gpus > 1:
        # NCCL init lines (rank count, transport) on stderr-side logging, for the scaling run's evidence
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.impl == "reference":
        run_reference_arm(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()
