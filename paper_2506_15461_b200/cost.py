"""Cost model and strategy comparison (reference include/ckfree/cost_model.hpp,
src/experiment.cpp:215-300), Python face over the drop-in library's ckfree_cost_* entry
points (dropin/cost_model.cpp).

The accounting itself is the reference's, bit-for-bit (tests/test_cost_model.py); what is
B200-specific is what it is fed:

* ``Profile.b200(...)`` -- stages on B200 GPUs: NVLink 5 / NVSwitch inside a node, the
  scale-out NIC across nodes, a storage site for checkpoints;
* ``params_b200(...)`` -- per-stage per-microbatch forward/backward seconds measured on the
  engine (``measure_stage_seconds``) and the B200 data layout's message sizes.

``compare_strategies`` runs the GPU trainer once per strategy over ONE shared failure trace
(fairness, experiment.cpp:287-296) and costs each run both ways: the modelled wall clock
for the given profile (the reference's ``train_time_h``) and the hours the B200 actually
took (``measured_hours``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

_LIB = None
_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class CostError(RuntimeError):
    pass


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_ROOT, "dropin", "libckfree_b200.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: build it with `make -C dropin` (__graft_entry__.build())")
        L = C.CDLL(path)
        L.ckfree_cost_last_error.restype = C.c_char_p
        d, i, l_, s = C.c_double, C.c_int, C.c_long, C.c_char_p
        dp = C.POINTER(C.c_double)
        L.ckfree_cost_profile_synthetic.argtypes = [i, s, C.c_size_t]
        L.ckfree_cost_profile_b200.argtypes = [i, i, i, dp, s, C.c_size_t]
        L.ckfree_cost_params_b200.argtypes = [d, d, C.c_uint64, C.c_size_t, C.c_uint64, C.c_uint64, C.c_uint64, i, dp]
        L.ckfree_cost_iteration.argtypes = [s, l_, i, s, dp, dp]
        L.ckfree_cost_recovery.argtypes = [s, l_, s, dp, i, dp]
        L.ckfree_cost_train.argtypes = [s, l_, i, s, dp, l_, C.POINTER(C.c_long), C.POINTER(C.c_int), i, dp]
        _LIB = L
    return _LIB


_ERRORS = {1: "config", 2: "parse", 3: "unsupported recovery"}


def _check(rc: int):
    if rc:
        msg = _lib().ckfree_cost_last_error().decode()
        raise CostError(f"{_ERRORS.get(rc, rc)} error: {msg}")


def _dvec(vals):
    return (C.c_double * len(vals))(*vals)


# ----------------------------------------------------------------------------- profile
@dataclass(frozen=True)
class Profile:
    """A "ckfree-net v1" network profile (cost_model.hpp:16-41), kept as its text."""
    text: str

    @classmethod
    def synthetic(cls, num_stages: int) -> "Profile":
        buf = C.create_string_buffer(1 << 16)
        _check(_lib().ckfree_cost_profile_synthetic(num_stages, buf, len(buf)))
        return cls(buf.value.decode())

    @classmethod
    def b200(cls, num_stages: int, gpus_per_node: int = 8, nodes: int = 1, nvlink_bps=900e9, nvlink_latency_s=3e-6,
             nic_bps=50e9, nic_latency_s=10e-6, hbm_bps=7.7e12, storage_bps=25e9, storage_latency_s=1e-3) -> "Profile":
        links = _dvec([nvlink_bps, nvlink_latency_s, nic_bps, nic_latency_s, hbm_bps, storage_bps, storage_latency_s])
        buf = C.create_string_buffer(1 << 20)
        _check(_lib().ckfree_cost_profile_b200(num_stages, gpus_per_node, nodes, links, buf, len(buf)))
        return cls(buf.value.decode())

    @classmethod
    def load(cls, path: str) -> "Profile":
        with open(path) as f:
            return cls(f.read())

    def save(self, path: str) -> None:
        with open(path, "w") as f:
            f.write(self.text)


# ----------------------------------------------------------------------------- params
@dataclass
class Params:
    """CostParams (cost_model.hpp:43-53)."""
    fwd_seconds: float = 1.0
    bwd_seconds: float = 2.0
    activation_bytes: int = 1 << 16
    stage_weight_bytes: int = 1 << 20
    edge_weight_bytes: int = 1 << 14
    full_model_bytes: int = 1 << 22
    num_microbatches: int = 8

    def _pack(self):
        return _dvec([self.fwd_seconds, self.bwd_seconds, self.activation_bytes, self.stage_weight_bytes,
                      self.edge_weight_bytes, self.full_model_bytes, self.num_microbatches])


def params_b200(fwd_seconds: float, bwd_seconds: float, tokens_per_microbatch: int, model_dim: int,
                stage_params: int, edge_params: int, total_params: int, num_microbatches: int) -> Params:
    """CostParams::from_b200: bf16 boundary activations, fp32 masters, fp32 Adam moments."""
    out = (C.c_double * 7)()
    _check(_lib().ckfree_cost_params_b200(fwd_seconds, bwd_seconds, int(tokens_per_microbatch), int(model_dim),
                                          int(stage_params), int(edge_params), int(total_params),
                                          int(num_microbatches), out))
    return Params(out[0], out[1], int(out[2]), int(out[3]), int(out[4]), int(out[5]), int(out[6]))


# ----------------------------------------------------------------------------- accounting
def iteration_cost(strategy: str, profile: Profile, params: Params, checkpoint_interval: int = 100,
                   blocking_upload: bool = False) -> dict:
    out = (C.c_double * 3)()
    _check(_lib().ckfree_cost_iteration(strategy.encode(), checkpoint_interval, int(blocking_upload),
                                        profile.text.encode(), params._pack(), out))
    return {"compute": out[0], "communication": out[1], "checkpoint_overhead": out[2],
            "total": out[0] + out[1] + out[2]}


def recovery_time(strategy: str, profile: Profile, params: Params, failed_stage: int,
                  checkpoint_interval: int = 100) -> float:
    out = C.c_double()
    _check(_lib().ckfree_cost_recovery(strategy.encode(), checkpoint_interval, profile.text.encode(), params._pack(),
                                       failed_stage, C.byref(out)))
    return out.value


def train_time(strategy: str, profile: Profile, params: Params, iterations_to_target: int, events,
               checkpoint_interval: int = 100, blocking_upload: bool = False) -> dict:
    """train_time (cost_model.hpp:91-98); events = [(iteration, stage_id), ...]."""
    n = len(events)
    it = (C.c_long * max(n, 1))(*[e[0] for e in events])
    st = (C.c_int * max(n, 1))(*[e[1] for e in events])
    out = (C.c_double * 6)()
    _check(_lib().ckfree_cost_train(strategy.encode(), checkpoint_interval, int(blocking_upload),
                                    profile.text.encode(), params._pack(), iterations_to_target, it, st, n, out))
    keys = ("compute", "communication", "checkpoint_overhead", "recovery", "rollback_lost", "hours")
    return dict(zip(keys, out))


# ----------------------------------------------------------------------------- measurement
def measure_stage_seconds(engine, spec, tokens_per_microbatch: int, microbatches: int, reps: int = 5,
                          warmup: int = 3, seed: int = 1, forward_engine=None):
    """Per-stage per-microbatch forward and backward seconds of `engine` on the B200.

    forward  = device time of one microbatch's forward through all stages (Engine.eval_loss,
               head and loss included) / stages -- or, with `forward_engine` (the same model
               built for the whole batch's tokens), of the whole batch's forward in one pass
               / (stages x microbatches), which matches the fused microbatch groups the
               training iteration runs;
    backward = device time of one training iteration (Engine.last_step_ms: every microbatch's
               forward + backward and the optimizer step) / (stages x microbatches) - forward.
    Medians over `reps` after `warmup`.  Returns (fwd_s, bwd_s, detail)."""
    import numpy as np
    import torch

    from . import api

    s = spec.num_stages
    mb_rows = tokens_per_microbatch // spec.seq_len
    order = list(range(1, s + 1))
    orders = np.array(api.build_schedule(microbatches, False, s), np.int32)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    toks = torch.randint(0, spec.output_dim, (microbatches * mb_rows, spec.seq_len + 1), generator=gen,
                         device="cuda", dtype=torch.int32)
    one = toks[:mb_rows].contiguous()
    fwd_eng, fwd_x, fwd_units = (engine, one, s) if forward_engine is None else (forward_engine, toks, s * microbatches)
    stream = torch.cuda.ExternalStream(fwd_eng.stream_ptr())
    it, fwd = [], []
    for r in range(warmup + reps):  # training iterations back to back (graph replay settles)
        engine.run_iteration(orders, toks, None, r + 1, on_device=True)
        torch.cuda.synchronize()
        if r >= warmup:
            it.append(engine.last_step_ms() / 1e3)
    for r in range(warmup + reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        fwd_eng.eval_loss(order, fwd_x, on_device=True)
        b.record(stream)
        torch.cuda.synchronize()
        if r >= warmup:
            fwd.append(a.elapsed_time(b) / 1e3)
    f_stage = float(np.median(fwd)) / fwd_units
    it_stage = float(np.median(it)) / (s * microbatches)
    detail = {"forward_pass_s": float(np.median(fwd)), "forward_units": fwd_units, "iteration_s": float(np.median(it)),
              "stages": s, "microbatches": microbatches, "tokens_per_microbatch": tokens_per_microbatch}
    return f_stage, max(it_stage - f_stage, f_stage), detail


# ----------------------------------------------------------------------------- comparison
@dataclass
class CompareRow:
    """experiment.hpp:109-118 + the B200 measured wall clock."""
    strategy: str
    iteration_time_s: float
    slots_to_target: int
    model_iters_to_target: int
    train_time_h: float
    final_val_loss: float
    unrecoverable: bool
    measured_hours: float = 0.0
    breakdown: dict = field(default_factory=dict)


def run_record(cfg: dict, trace_text: str, seed: int) -> dict:
    """run_experiment on the GPU trainer, reduced to what the cost accounting needs
    (RunRecord fields of experiment.hpp:77-107)."""
    from ._native import check, lib

    kv = ";".join(f"{k}={v}" for k, v in cfg.items()).encode()
    buf = C.create_string_buffer(1 << 22)
    check(lib().ckf_run_experiment(kv, trace_text.encode(), seed, buf, len(buf)))
    evals, unrec = [], None
    for ln in buf.value.decode().splitlines():
        p = ln.split(",")
        if p[0] == "E":
            evals.append((int(p[1]), float(p[2]), float(p[3]), float(p[4]), int(p[5])))
        elif p[0] == "U":
            unrec = ln[2:]
    target = float(cfg.get("target-loss", 0) or 0)
    hit = next((e for e in evals if target > 0 and e[2] <= target), None)
    last = evals[-1]
    return {"slots_run": last[0], "model_iterations": last[4], "final_val_loss": last[2], "hours": last[3],
            "slots_to_target": hit[0] if hit else -1, "model_iters_to_target": hit[4] if hit else -1,
            "hours_to_target": hit[3] if hit else -1.0, "unrecoverable": unrec is not None, "evals": evals}


def _trace_events(trace_text: str):
    ev = []
    for ln in trace_text.splitlines()[1:]:
        ln = ln.strip()
        if ln and not ln.startswith("#"):
            a, b = ln.split(",")[:2]
            ev.append((int(a), int(b)))
    return ev


def cost_row(strategy: str, rec: dict, trace_text: str, profile: Profile, params: Params,
             checkpoint_interval: int = 100) -> CompareRow:
    """make_row (experiment.cpp:217-243): the modelled cost stops at the convergence point when
    it was reached (else covers the whole run) and charges only the failures up to it."""
    reached = rec["slots_to_target"] >= 0
    horizon = rec["slots_to_target"] if reached else rec["slots_run"]
    model_iters = rec["model_iters_to_target"] if reached else rec["model_iterations"]
    events = [e for e in _trace_events(trace_text) if e[0] <= horizon]
    per_iter = iteration_cost(strategy, profile, params, checkpoint_interval)
    try:
        tt = train_time(strategy, profile, params, model_iters, events, checkpoint_interval)
    except CostError:  # a failure the strategy cannot recover (e.g. CheckFree on an edge stage)
        tt = {"hours": float("nan")}
    return CompareRow(strategy, per_iter["total"], rec["slots_to_target"], rec["model_iters_to_target"], tt["hours"],
                      rec["final_val_loss"], rec["unrecoverable"],
                      rec["hours_to_target"] if reached else rec["hours"], tt)


def compare_strategies(cfg: dict, strategies, trace_text: str, profile, params: Params,
                       seed: int | None = None):
    """compare_strategies (experiment.cpp:245-275) over the GPU trainer: one run per strategy on
    the SAME trace.  `profile` is one Profile (-> list of rows) or {name: Profile} (-> {name:
    rows}, every profile costing the same runs)."""
    seed = int(cfg.get("seed", 0)) if seed is None else seed
    interval = int(cfg.get("checkpoint-interval", 100))
    recs = [(st, run_record({**cfg, "strategy": st}, trace_text, seed)) for st in strategies]
    profs = profile if isinstance(profile, dict) else {"": profile}
    out = {name: [cost_row(st, rec, trace_text, pr, params, interval) for st, rec in recs]
           for name, pr in profs.items()}
    return out if isinstance(profile, dict) else out[""]


def milestones(evals_off, evals_on, fracs=(0.25, 0.5, 0.75, 0.9)):
    """ablation_swap's milestones (experiment.cpp:370-385): validation-loss levels at fractions
    of the swap-off run's total drop, and the first evaluated iteration at or below each level
    in either run (-1: never).  evals = [(iteration, train, val, ...), ...]."""
    v0, vf = evals_off[0][2], evals_off[-1][2]
    rows = []
    for frac in fracs:
        level = v0 - frac * (v0 - vf)
        first = lambda ev: next((e[0] for e in ev if e[2] <= level), -1)  # noqa: E731
        rows.append({"level": level, "iter_off": first(evals_off), "iter_on": first(evals_on)})
    return rows


def ablation_swap(cfg: dict, seed: int) -> dict:
    """ablation_swap (experiment.cpp:349-386) on the GPU trainer: paired zero-failure runs with
    the standard and the swapped-half schedule, same seed, and the milestone table."""
    s = int(cfg.get("stages", 4))
    base = {k: v for k, v in cfg.items() if k not in ("p-hour", "p-iter", "trace", "target-loss")}
    base["strategy"] = "no-failures"
    from . import api
    empty = api.generate_trace(seed, 0.0, float(cfg.get("iter-seconds", 120.0)), 1, list(range(1, s + 1)))
    off = run_record({**base, "schedule": "standard"}, empty, seed)
    on = run_record({**base, "schedule": "swapped-half"}, empty, seed)
    return {"off": off, "on": on, "milestones": milestones(off["evals"], on["evals"])}


def estimate_delta(engine, x) -> dict:
    """estimate_delta (experiment.cpp:305-345) on the GPU engine, residual-MLP model: for each
    layer, param_ratio = ||W1, W2 of the layer|| / ||all weights (embed, de-embed, stages)|| and
    func_ratio = ||F(x) - F_without_layer(x)|| / ||F(x)|| over the probe rows x (the reference
    draws them from its task's validation set; here the caller passes them).  A layer is
    omitted by zeroing its W2 on the device -- h + act(h W1) 0 = h exactly -- and restored."""
    import numpy as np

    from . import api

    spec = engine.spec
    if spec.block != "mlp":
        raise NotImplementedError("estimate_delta is defined for the reference's residual-MLP blocks")
    s, d, hd = spec.num_stages, spec.model_dim, spec.hidden_dim
    order = list(range(1, s + 1))
    emb, deemb = engine.export_edge(0)[0], engine.export_edge(1)[0]
    stages = [np.array(engine.export_stage(i)[0], np.float64) for i in range(1, s + 1)]
    allw = np.concatenate([np.ravel(emb), np.ravel(deemb)] + stages)
    norm_all = float(np.sqrt(np.dot(allw, allw)))
    full = engine.predict(order, x)
    norm_out = float(np.sqrt(np.sum(full * full)))
    part = api.even_partition(spec.num_layers, s)
    rows, dp, df = [], 0.0, 0.0
    for layer in range(1, spec.num_layers + 1):
        sid = next(i + 1 for i, (a, b) in enumerate(part) if a <= layer <= b)
        off = (layer - part[sid - 1][0]) * 2 * d * hd
        w = stages[sid - 1]
        blk = w[off:off + 2 * d * hd]
        wnorm = float(np.sqrt(np.dot(blk, blk)))
        masked = w.copy()
        masked[off + d * hd:off + 2 * d * hd] = 0.0
        engine.import_stage(sid, w=masked)
        try:
            pred = engine.predict(order, x)
        finally:
            engine.import_stage(sid, w=w)
        diff = float(np.sqrt(np.sum((full - pred) ** 2)))
        row = {"layer": layer, "param_ratio": wnorm / norm_all if norm_all > 0 else 0.0,
               "func_ratio": diff / norm_out if norm_out > 0 else 0.0}
        rows.append(row)
        dp, df = max(dp, row["param_ratio"]), max(df, row["func_ratio"])
    return {"rows": rows, "delta_param": dp, "delta_func": df}


def delta_csv(report: dict) -> str:
    """experiment.cpp:347-354's schema."""
    out = ["# format_version=1", "layer,param_ratio,func_ratio"]
    out += [f"{r['layer']},{r['param_ratio']:.17g},{r['func_ratio']:.17g}" for r in report["rows"]]
    return "\n".join(out) + "\n"


def comparison_csv(rows) -> str:
    """experiment.cpp:277-285's schema + measured_hours."""
    out = ["# format_version=1",
           "strategy,iteration_time_s,iters_to_target,model_iters_to_target,train_time_h,final_val_loss,unrecoverable,"
           "measured_hours"]
    for r in rows:
        out.append(f"{r.strategy},{r.iteration_time_s:.17g},{r.slots_to_target},{r.model_iters_to_target},"
                   f"{r.train_time_h:.17g},{r.final_val_loss:.17g},{int(r.unrecoverable)},{r.measured_hours:.17g}")
    return "\n".join(out) + "\n"


def comparison_table(rows) -> str:
    lines = [f"{'strategy':<20} {'iter time (s)':>16} {'iters to tgt':>16} {'train time (h)':>14} "
             f"{'final val':>14} {'status':>6} {'B200 (h)':>10}"]
    for r in rows:
        lines.append(f"{r.strategy:<20} {r.iteration_time_s:16.3f} {r.slots_to_target:16d} {r.train_time_h:14.3f} "
                     f"{r.final_val_loss:14.6g} {'DEAD' if r.unrecoverable else 'ok':>6} {r.measured_hours:10.5f}")
    return "\n".join(lines) + "\n"
