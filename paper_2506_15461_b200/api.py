"""Python face of the B200 engine, mirroring the reference's operator names
(ckfree::pipeline / ckfree::recovery / harness, /root/reference/proj/include).

Thin: all arithmetic runs in libckf.so's sm_100a kernels via include/ckf.h.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._native import check, lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


# ------------------------------------------------------------- host logic (no GPU)
def generate_trace(seed: int, p_hour: float, iter_s: float, n_iters: int, stages) -> str:
    """failures::generate_trace + serialize_trace (src/failures.cpp:63-95)."""
    arr = (C.c_int * len(stages))(*stages)
    buf = C.create_string_buffer(1 << 22)
    check(lib().ckf_generate_trace(seed, p_hour, iter_s, n_iters, arr, len(stages), buf, len(buf)))
    return buf.value.decode()


def parse_trace(text: str) -> str:
    buf = C.create_string_buffer(max(1 << 16, 4 * len(text)))
    check(lib().ckf_parse_trace(text.encode(), buf, len(buf)))
    return buf.value.decode()


def consecutive_conflicts(text: str):
    out = (C.c_long * 20000)()
    n = C.c_int(0)
    check(lib().ckf_consecutive_conflicts(text.encode(), out, 10000, C.byref(n)))
    return [(out[2 * i], out[2 * i + 1]) for i in range(n.value)]


def hourly_to_per_iteration(p_hour: float, iter_s: float) -> float:
    return lib().ckf_hourly_to_per_iteration(p_hour, iter_s)


def even_partition(layers: int, stages: int):
    out = (C.c_size_t * (2 * stages))()
    check(lib().ckf_even_partition(layers, stages, out))
    return [(out[2 * i], out[2 * i + 1]) for i in range(stages)]


def build_schedule(m: int, swapped_half: bool, s: int):
    out = (C.c_int * (max(m, 1) * s))()
    check(lib().ckf_build_schedule(m, 1 if swapped_half else 0, s, out))
    return [[out[k * s + j] for j in range(s)] for k in range(m)]


PLAN_KINDS = ("embed_fwd", "stage_fwd", "xfer", "head", "stage_bwd", "embed_bwd")


def pipeline_plan(orders, stage_rank, schedule: int = 1, stage_cost=None, head_cost: float = 1.0):
    """Global op sequence of one iteration for a stage -> rank placement (ckf_pipeline_plan_cost);
    schedule 0 sequential, 1 GPipe, 2 1F1B (weighted by stage_cost / head_cost)."""
    orders = np.ascontiguousarray(orders, np.int32)
    m, s = orders.shape
    sr = np.ascontiguousarray(stage_rank, np.int32)
    cap = 8 * m * (s + 4) + 16
    out = np.zeros(6 * cap, np.int32)
    n = C.c_int(0)
    sc = None if stage_cost is None else np.ascontiguousarray(stage_cost, np.float64)
    check(lib().ckf_pipeline_plan_cost(s, m, _ip(orders.reshape(-1)), _ip(sr), schedule,
                                       _dp(sc) if sc is not None else None, head_cost, _ip(out), cap, C.byref(n)))
    return [dict(phase=int(o[0]), mb=int(o[1]), kind=PLAN_KINDS[o[2]], rank=int(o[3]), arg=int(o[4]),
                 aux=int(o[5])) for o in out[:6 * n.value].reshape(-1, 6)]


# ------------------------------------------------------------- L1 seam (kernels.hpp)
def recover_checkfree(w_prev, w_next, omega_prev: float, omega_next: float):
    """recovery::recover_checkfree (src/recovery.cpp:57-73) on the GPU, fp64."""
    wp = np.ascontiguousarray(w_prev, np.float64)
    wn = np.ascontiguousarray(w_next, np.float64)
    if wp.shape != wn.shape:
        raise N.ConfigError(N.CKF_E_CONFIG, "neighbor stage weights differ in shape")
    out = np.empty_like(wp)
    deg = C.c_int(0)
    check(lib().ckf_k_recover_checkfree(_dp(wp), _dp(wn), wp.size, omega_prev, omega_next, _dp(out), C.byref(deg)))
    return out, bool(deg.value)


def counter_uniform(key: int, lo: float, hi: float, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    check(lib().ckf_k_counter_uniform(key, lo, hi, _dp(out), n))
    return out


def adam_update(w, m, v, g, lr, step):
    w, m, v = (np.array(a, np.float64) for a in (w, m, v))
    g = np.ascontiguousarray(g, np.float64)
    check(lib().ckf_k_adam_update(_dp(w), _dp(m), _dp(v), _dp(g), w.size, lr, 0.9, 0.999, 1e-8, step))
    return w, m, v


def sum_squares(x) -> float:
    x = np.ascontiguousarray(x, np.float64)
    out = C.c_double(0)
    check(lib().ckf_k_sum_squares(_dp(x), x.size, C.byref(out)))
    return out.value


def gemm(kind: str, a, b, c, m, k, n):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    c = np.array(c, np.float64)
    fn = {"nn": lib().ckf_k_gemm_nn, "nn_acc": lib().ckf_k_gemm_nn_acc, "nt_acc": lib().ckf_k_gemm_nt_acc,
          "tn_acc": lib().ckf_k_gemm_tn_acc}[kind]
    check(fn(_dp(a), _dp(b), _dp(c), m, k, n))
    return c


def llama_token_batch(data_seed: int, stream: int, index: int, rows: int, T: int, V: int) -> np.ndarray:
    """Counter-RNG token stream of the LLaMA block, generated on the GPU (rows x (T+1) int32)."""
    out = np.zeros((rows, T + 1), np.int32)
    check(lib().ckf_llama_token_batch(data_seed, stream, index, rows, T, V, _ip(out)))
    return out


# ------------------------------------------------------------- device primitives
def recover_device(wp, wn, out, omega_prev, omega_next, old_sq=None, stream=0):
    """omega-weighted recovery on torch CUDA tensors (fp32 / fp64 master weights)."""
    import torch
    dt = {torch.float64: N.CKF_FP64, torch.float32: N.CKF_FP32}[out.dtype]
    check(lib().ckf_recover_device(dt, wp.data_ptr(), wn.data_ptr(), out.data_ptr(), out.numel(), omega_prev,
                                   omega_next, old_sq.data_ptr() if old_sq is not None else None, stream or None))


def recover_stage_device(wp, wn, w, m, v, g, omega_prev, omega_next, w_bf16=None, mp=None, mn=None, vp=None,
                         vn=None, old_sq=None, stream=0):
    """The engine's fused stage recovery (ckf_recover_stage_device) on torch CUDA tensors:
    weights, moments (Fresh, or omega-weighted when mp/mn/vp/vn are given), g = 0, bf16 shadow and
    the optional reduction error in ONE pass.  The neighbour tensors may live in a peer's HBM."""
    import torch
    dt = {torch.float64: N.CKF_FP64, torch.float32: N.CKF_FP32}[w.dtype]
    avg = mp is not None
    ptr = (lambda t: t.data_ptr() if t is not None else None)
    check(lib().ckf_recover_stage_device(dt, ptr(wp), ptr(wn), ptr(mp), ptr(mn), ptr(vp), ptr(vn), ptr(w), ptr(m),
                                         ptr(v), ptr(g), ptr(w_bf16), w.numel(), omega_prev, omega_next,
                                         1 if avg else 0, ptr(old_sq), stream or None))


def adam_device(w, m, v, g, lr, step, grad_scale=1.0, zero_grad=False, w_bf16=None, omega=None, stream=0):
    import math
    import torch
    dt = {torch.float64: N.CKF_FP64, torch.float32: N.CKF_FP32}[w.dtype]
    bc1 = 1.0 - math.pow(0.9, step)
    bc2 = 1.0 - math.pow(0.999, step)
    check(lib().ckf_adam_device(dt, w.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(),
                                w_bf16.data_ptr() if w_bf16 is not None else None, w.numel(), lr, bc1, bc2,
                                grad_scale, 1 if zero_grad else 0, omega.data_ptr() if omega is not None else None,
                                stream or None))


# ------------------------------------------------------------- engine
@dataclass
class ModelSpec:
    """ModelSpec (model.hpp:32-53) + the LLaMA shape keys."""
    input_dim: int = 16
    hidden_dim: int = 64
    model_dim: int = 32
    output_dim: int = 16
    num_layers: int = 8
    num_stages: int = 4
    activation: str = "tanh"
    task: str = "regression"
    block: str = "mlp"
    precision: str = "fp64"
    n_heads: int = 1
    seq_len: int = 1
    max_rows: int = 256
    device: int = 0

    @staticmethod
    def llama(vocab, d, layers, heads, ffn, seq_len, stages, precision="bf16", max_tokens=8192, device=0):
        return ModelSpec(vocab, ffn, d, vocab, layers, stages, "identity", "classification", "llama", precision,
                         heads, seq_len, max_tokens, device)


class Engine:
    """Device-resident stages + edges on one GPU (include/ckf.h section 3)."""

    def __init__(self, spec: ModelSpec):
        self.spec = spec
        d = N.ModelDesc()
        d.block = N.CKF_BLOCK_LLAMA if spec.block == "llama" else N.CKF_BLOCK_MLP
        d.precision = {"fp64": N.CKF_FP64, "fp32": N.CKF_FP32, "bf16": N.CKF_BF16}[spec.precision]
        d.activation = N.CKF_ACT[spec.activation]
        d.task = N.CKF_TASK[spec.task]
        d.input_dim, d.hidden_dim, d.model_dim, d.output_dim = spec.input_dim, spec.hidden_dim, spec.model_dim, \
            spec.output_dim
        d.num_layers, d.num_stages, d.n_heads, d.seq_len = spec.num_layers, spec.num_stages, spec.n_heads, spec.seq_len
        d.partition = None
        d.max_rows = spec.max_rows
        d.device = spec.device
        self._h = C.c_void_p()
        check(lib().ckf_engine_create(C.byref(d), C.byref(self._h)))
        sp, ep, dp = C.c_size_t(), C.c_size_t(), C.c_size_t()
        check(lib().ckf_engine_param_counts(self._h, C.byref(sp), C.byref(ep), C.byref(dp)))
        self.stage_params, self.embed_params, self.deembed_params = sp.value, ep.value, dp.value

    def close(self):
        if self._h:
            check(lib().ckf_engine_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def init(self, seed: int, lr: float):
        check(lib().ckf_engine_init(self._h, seed, lr))

    def run_iteration(self, orders, x, y, iteration: int, on_device: bool = False):
        orders = np.ascontiguousarray(orders, np.int32).reshape(-1)
        m = orders.size // self.spec.num_stages
        loss = C.c_double(0)
        om = np.zeros(self.spec.num_stages, np.float64)
        xp, yp, rows = self._inputs(x, y, on_device)
        check(lib().ckf_engine_run_iteration(self._h, _ip(orders), m, xp, yp, rows, 1 if on_device else 0, iteration,
                                             C.byref(loss), _dp(om)))
        return loss.value, om

    def _inputs(self, x, y, on_device):
        if on_device:
            return x.data_ptr(), (y.data_ptr() if y is not None else None), x.shape[0]
        if self.spec.block == "llama":
            self._x = np.ascontiguousarray(x, np.int32)
            return self._x.ctypes.data, None, self._x.shape[0]
        self._x = np.ascontiguousarray(x, np.float64)
        self._y = np.ascontiguousarray(y, np.float64)
        return self._x.ctypes.data, self._y.ctypes.data, self._x.shape[0]

    def eval_loss(self, order, x, y=None, on_device=False):
        order = np.ascontiguousarray(order, np.int32)
        xp, yp, rows = self._inputs(x, y, on_device)
        out = C.c_double(0)
        check(lib().ckf_engine_eval_loss(self._h, _ip(order), xp, yp, rows, 1 if on_device else 0, C.byref(out)))
        return out.value

    def accumulate(self, order, x, y=None, on_device=False) -> float:
        """One microbatch forward + backward accumulating gradients (no optimizer step)."""
        order = np.ascontiguousarray(order, np.int32)
        xp, yp, rows = self._inputs(x, y, on_device)
        out = C.c_double(0)
        check(lib().ckf_engine_accumulate(self._h, _ip(order), xp, yp, rows, 1 if on_device else 0, C.byref(out)))
        return out.value

    def zero_grad(self):
        check(lib().ckf_engine_zero_grad(self._h))

    def export_grad(self, which: str, stage: int = 0) -> np.ndarray:
        n = {"embed": self.embed_params, "deembed": self.deembed_params, "stage": self.stage_params}[which]
        g = np.zeros(n)
        check(lib().ckf_engine_export_grad(self._h, {"embed": 0, "deembed": 1, "stage": 2}[which], stage, _dp(g)))
        return g

    def predict(self, order, x):
        order = np.ascontiguousarray(order, np.int32)
        x = np.ascontiguousarray(x, np.float64)
        pred = np.zeros((x.shape[0], self.spec.output_dim), np.float64)
        check(lib().ckf_engine_predict(self._h, _ip(order), _dp(x), x.shape[0], _dp(pred)))
        return pred

    def refresh_edge_replicas(self):
        check(lib().ckf_engine_refresh_edge_replicas(self._h))

    def kill_stage(self, stage: int):
        check(lib().ckf_engine_kill_stage(self._h, stage))

    def recover_stage(self, stage, mode=N.CKF_REC_CHECKFREE, moments=N.CKF_MOM_FRESH, lr_bump=1.1, reinit_seed=0,
                      reduction_error=False):
        r = N.RecoveryReport()
        check(lib().ckf_engine_recover_stage(self._h, stage, mode, moments, lr_bump, reinit_seed,
                                             1 if reduction_error else 0, C.byref(r)))
        return r

    def export_stage(self, stage):
        w, m, v = (np.zeros(self.stage_params) for _ in range(3))
        check(lib().ckf_engine_export_stage(self._h, stage, _dp(w), _dp(m), _dp(v)))
        return w, m, v

    def import_stage(self, stage, w=None, m=None, v=None):
        arrs = [None if a is None else np.ascontiguousarray(a, np.float64) for a in (w, m, v)]
        check(lib().ckf_engine_import_stage(self._h, stage, *[None if a is None else _dp(a) for a in arrs]))

    def export_edge(self, which):
        n = self.embed_params if which == 0 else self.deembed_params
        w, m, v = (np.zeros(n) for _ in range(3))
        check(lib().ckf_engine_export_edge(self._h, which, _dp(w), _dp(m), _dp(v)))
        return w, m, v

    def import_edge(self, which, w=None, m=None, v=None):
        arrs = [None if a is None else np.ascontiguousarray(a, np.float64) for a in (w, m, v)]
        check(lib().ckf_engine_import_edge(self._h, which, *[None if a is None else _dp(a) for a in arrs]))

    def scalars(self, stage):
        om, lr, st = C.c_double(), C.c_double(), C.c_long()
        check(lib().ckf_engine_get_scalars(self._h, stage, C.byref(om), C.byref(lr), C.byref(st)))
        return om.value, lr.value, st.value

    def set_scalars(self, stage, omega, lr, step):
        check(lib().ckf_engine_set_scalars(self._h, stage, omega, lr, step))

    def attach_comm(self, uid: bytes, nranks: int, rank: int, stage_rank, replicas: int = 1):
        """Multi-GPU placement: stage_rank = pipeline rank per stage; nranks = replicas * pipeline ranks."""
        sr = np.ascontiguousarray(stage_rank, np.int32)
        buf = C.create_string_buffer(uid, 128)
        check(lib().ckf_engine_attach_comm_dp(self._h, buf, nranks, rank, _ip(sr), replicas))

    def set_placement(self, nranks: int, rank: int, stage_rank, replicas: int = 1):
        """Stage -> rank ownership without a communicator (attach_comm = this + NCCL)."""
        sr = np.ascontiguousarray(stage_rank, np.int32)
        check(lib().ckf_engine_set_placement(self._h, nranks, rank, _ip(sr), replicas))

    def ipc_export(self) -> bytes:
        """CUDA IPC handles of this rank's stage buffers (peer recovery over NVLink)."""
        buf = C.create_string_buffer(1 << 16)
        n = C.c_size_t(0)
        check(lib().ckf_engine_ipc_export(self._h, buf, len(buf), C.byref(n)))
        return buf.raw[:n.value]

    def ipc_import(self, blobs):
        """Maps the other ranks' stages (blobs from every rank's ipc_export; own entries skipped)."""
        data = b"".join(blobs)
        buf = C.create_string_buffer(data, max(1, len(data)))
        check(lib().ckf_engine_ipc_import(self._h, buf, len(data)))

    def enable_peer_transport(self, max_microbatches: int):
        """Stage transfers through peer memory (mailbox + flags, CUDA IPC) instead of NCCL;
        call on every rank before the IPC exchange."""
        check(lib().ckf_engine_enable_peer_transport(self._h, max_microbatches))

    def plan_cost(self):
        """(per-stage forward costs, head cost) the engine's 1F1B plan is simulated with."""
        sc = np.zeros(self.spec.num_stages, np.float64)
        h = C.c_double()
        check(lib().ckf_engine_plan_cost(self._h, _dp(sc), C.byref(h)))
        return sc, h.value

    def exchange_peers(self):
        """Collective (after attach_comm): maps every other rank's stages for peer recovery."""
        check(lib().ckf_engine_exchange_peers(self._h))

    def sync(self):
        check(lib().ckf_engine_sync(self._h))

    def set_redundant(self, on: bool):
        """Redundant-computation baseline: extra forward per stage + post-step replica refresh."""
        check(lib().ckf_engine_set_redundant(self._h, 1 if on else 0))

    def last_step_ms(self) -> float:
        """Device time of the last run_iteration (CUDA events on the engine stream)."""
        ms = C.c_float()
        check(lib().ckf_engine_last_step_ms(self._h, C.byref(ms)))
        return ms.value

    def set_edge_replicas(self, on: bool):
        """CheckFree+: refresh the edge replicas at the end of every run_iteration (trainer.cpp:83-84)."""
        check(lib().ckf_engine_set_edge_replicas(self._h, 1 if on else 0))

    def set_group_cap(self, cap: int):
        """Microbatch fusion cap (0 = fit to HBM, 1 = one microbatch per pass)."""
        check(lib().ckf_engine_set_group_cap(self._h, cap))

    def set_schedule(self, mode: int):
        """0 = forward+backward per microbatch, 1 = GPipe (all forwards, then all backwards)."""
        check(lib().ckf_engine_set_schedule(self._h, mode))

    def hop_log(self, stage_rank=None):
        """Enable (stage_rank given) or read back the virtual-placement transfer log [(src, dst, bytes)]."""
        if stage_rank is not None:
            self._vr = np.ascontiguousarray(stage_rank, np.int32)
            check(lib().ckf_engine_hop_log(self._h, int(self._vr.max()) + 1, _ip(self._vr)))
            return None
        out = (C.c_long * (3 * 65536))()
        n = C.c_int(0)
        check(lib().ckf_engine_get_hop_log(self._h, out, 65536, C.byref(n)))
        return [(out[3 * i], out[3 * i + 1], out[3 * i + 2]) for i in range(n.value)]

    def kernel_launches(self) -> int:
        return lib().ckf_engine_kernel_launches(self._h)

    def stream_ptr(self) -> int:
        """cudaStream_t the engine launches on (wrap with torch.cuda.ExternalStream for event timing)."""
        s = C.c_void_p()
        check(lib().ckf_engine_stream(self._h, C.byref(s)))
        return s.value or 0

    def kernel_timing(self, enable: bool):
        check(lib().ckf_engine_kernel_timing(self._h, 1 if enable else 0))

    KCLASS = {"gemm": 0, "attention": 1, "adam": 2, "recovery": 3, "norm": 4, "loss": 5, "transfer": 6}

    def kernel_stats(self, cls: str):
        """(ms, launches, algorithmic flops, algorithmic bytes) summed since kernel_timing(True)."""
        ms, n, fl, by = C.c_double(), C.c_long(), C.c_double(), C.c_double()
        check(lib().ckf_engine_kernel_stats(self._h, self.KCLASS[cls], C.byref(ms), C.byref(n), C.byref(fl),
                                            C.byref(by)))
        return ms.value, n.value, fl.value, by.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().ckf_nccl_unique_id(buf, 128))
    return buf.raw


# ------------------------------------------------------------- trainer
def run_experiment(cfg: dict, trace_text: str, seed: int, comm=None):
    """harness::run_experiment (src/trainer.cpp:314-322) on the GPU engine.
    comm = (nccl_uid, nranks, rank, replicas): this process is one rank of a multi-GPU run
    (torchrun, one process per GPU; every rank passes rank 0's nccl_unique_id()).
    Returns (evals[(iter, train, val)], events[(iter, stage, action, red, spike, ms)], unrecoverable_reason|None)."""
    kv = ";".join(f"{k}={v}" for k, v in cfg.items()).encode()
    buf = C.create_string_buffer(1 << 22)
    if comm is None:
        check(lib().ckf_run_experiment(kv, trace_text.encode(), seed, buf, len(buf)))
    else:
        uid, nranks, rank, replicas = comm
        ub = C.create_string_buffer(uid, 128)
        check(lib().ckf_run_experiment_rank(kv, trace_text.encode(), seed, ub, nranks, rank, replicas, buf, len(buf)))
    evals, events, unrec = [], [], None
    for ln in buf.value.decode().splitlines():
        p = ln.split(",")
        if p[0] == "E":
            evals.append((int(p[1]), float(p[2]), float(p[3])))  # p[4]: measured wall hours
        elif p[0] == "F":
            events.append((int(p[1]), int(p[2]), p[3], float(p[4]), float(p[5]), float(p[6])))
        elif p[0] == "U":
            unrec = ln[2:]
    return evals, events, unrec


def run_experiment_to_dir(cfg: dict, trace_text: str, seed: int, out_dir: str):
    """harness::run_experiment_to_dir (src/experiment.cpp:202-213): metrics.csv, events.csv,
    summary.json, config.resolved in the reference's schema."""
    kv = ";".join(f"{k}={v}" for k, v in cfg.items()).encode()
    check(lib().ckf_run_experiment_to_dir(kv, trace_text.encode(), seed, out_dir.encode()))
