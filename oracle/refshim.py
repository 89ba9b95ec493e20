"""ctypes wrapper over oracle/_ref/libckfree_oracle.so -- the UNMODIFIED reference
library (/root/reference/proj/src) plus ref_shim.cpp.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's reference / cpu_baseline legs, as the checker and the CPU baseline.
The product path (paper_2506_15461_b200) never imports anything under oracle/.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libckfree_oracle.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run `make -C oracle`)")
        L = C.CDLL(LIB_PATH)
        u64, dbl, sz, i32, lng = C.c_uint64, C.c_double, C.c_size_t, C.c_int, C.c_long
        dp, ip, cp = C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_char_p
        L.ref_last_error.restype = cp
        L.ref_mix64.restype = u64
        L.ref_mix64.argtypes = [u64]
        L.ref_derive_key.restype = u64
        L.ref_derive_key.argtypes = [u64, u64, u64, u64]
        L.ref_unit_at.restype = dbl
        L.ref_unit_at.argtypes = [u64, u64, u64, u64]
        L.ref_counter_uniform.argtypes = [u64, dbl, dbl, dp, sz]
        L.ref_hourly_to_per_iteration.restype = dbl
        L.ref_hourly_to_per_iteration.argtypes = [dbl, dbl]
        L.ref_generate_trace.argtypes = [u64, dbl, dbl, lng, ip, i32, cp, sz]
        L.ref_parse_trace.argtypes = [cp, cp, sz]
        L.ref_consecutive_conflicts.argtypes = [cp, C.POINTER(C.c_long), i32, ip]
        L.ref_even_partition.argtypes = [sz, sz, C.POINTER(C.c_size_t)]
        L.ref_build_schedule.argtypes = [i32, i32, i32, ip]
        L.ref_recover_checkfree.argtypes = [dp, dp, sz, dbl, dbl, dp, ip]
        L.ref_reduction_error.argtypes = [dp, dp, dp, sz, dbl, dbl, dp]
        L.ref_bump_lr.restype = dbl
        L.ref_bump_lr.argtypes = [dbl, dbl]
        L.ref_time_recover_checkfree.restype = dbl
        L.ref_time_recover_checkfree.argtypes = [sz, i32]
        L.ref_sum_squares.restype = dbl
        L.ref_sum_squares.argtypes = [dp, sz]
        L.ref_sum_squared_diff.restype = dbl
        L.ref_sum_squared_diff.argtypes = [dp, dp, sz]
        L.ref_adam_update.argtypes = [dp, dp, dp, dp, sz, dbl, lng]
        L.ref_gemm.argtypes = [i32, dp, dp, dp, sz, sz, sz]
        L.ref_init_model_flat.argtypes = [cp, u64, dp, sz, C.POINTER(C.c_size_t)]
        L.ref_batch.argtypes = [cp, u64, lng, sz, dp, dp]
        L.ref_run_iteration.argtypes = [cp, u64, i32, dp, dp, sz, lng, dp, dp, dp]
        L.ref_run_experiment.argtypes = [cp, cp, u64, cp, sz, cp, sz]
        L.ref_run_experiment_full.argtypes = [cp, cp, u64, cp, sz]
        L.ref_time_train_iterations.restype = dbl
        L.ref_time_train_iterations.argtypes = [cp, u64, i32]
        L.ref_parallel_threads.restype = i32
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _check(rc: int):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {lib().ref_last_error().decode()}")


def kv(cfg: dict) -> bytes:
    return ";".join(f"{k}={v}" for k, v in cfg.items()).encode()


def mix64(x): return lib().ref_mix64(x)
def derive_key(s, a=0, b=0, c=0): return lib().ref_derive_key(s, a, b, c)
def unit_at(s, a, b=0, c=0): return lib().ref_unit_at(s, a, b, c)


def counter_uniform(key, lo, hi, n):
    out = np.empty(n, np.float64)
    lib().ref_counter_uniform(key, lo, hi, _dp(out), n)
    return out


def hourly_to_per_iteration(p, s): return lib().ref_hourly_to_per_iteration(p, s)


def generate_trace(seed, p_hour, iter_s, n_iters, stages) -> str:
    arr = (C.c_int * len(stages))(*stages)
    buf = C.create_string_buffer(1 << 22)
    _check(lib().ref_generate_trace(seed, p_hour, iter_s, n_iters, arr, len(stages), buf, len(buf)))
    return buf.value.decode()


def parse_trace(text: str) -> str:
    buf = C.create_string_buffer(1 << 22)
    _check(lib().ref_parse_trace(text.encode(), buf, len(buf)))
    return buf.value.decode()


def even_partition(L, s):
    out = (C.c_size_t * (2 * s))()
    lib().ref_even_partition(L, s, out)
    return [(out[2 * i], out[2 * i + 1]) for i in range(s)]


def build_schedule(m, swapped_half, s):
    out = (C.c_int * (m * s))()
    _check(lib().ref_build_schedule(m, 1 if swapped_half else 0, s, out))
    return [[out[k * s + j] for j in range(s)] for k in range(m)]


def recover_checkfree(wp, wn, op, on):
    wp = np.ascontiguousarray(wp, np.float64)
    wn = np.ascontiguousarray(wn, np.float64)
    out = np.empty_like(wp)
    deg = C.c_int(0)
    _check(lib().ref_recover_checkfree(_dp(wp), _dp(wn), wp.size, op, on, _dp(out), C.byref(deg)))
    return out, bool(deg.value)


def reduction_error(wp, wf, wn, op, on):
    wp, wf, wn = (np.ascontiguousarray(a, np.float64) for a in (wp, wf, wn))
    out = C.c_double(0)
    _check(lib().ref_reduction_error(_dp(wp), _dp(wf), _dp(wn), wp.size, op, on, C.byref(out)))
    return out.value


def sum_squares(x):
    x = np.ascontiguousarray(x, np.float64)
    return lib().ref_sum_squares(_dp(x), x.size)


def adam_update(w, m, v, g, lr, step):
    w, m, v = (np.array(a, np.float64) for a in (w, m, v))
    g = np.ascontiguousarray(g, np.float64)
    lib().ref_adam_update(_dp(w), _dp(m), _dp(v), _dp(g), w.size, lr, step)
    return w, m, v


def init_model_flat(cfg: dict, seed: int) -> np.ndarray:
    cap = 1 << 26
    out = np.empty(cap, np.float64)
    n = C.c_size_t(0)
    _check(lib().ref_init_model_flat(kv(cfg), seed, _dp(out), cap, C.byref(n)))
    return out[: n.value].copy()


def batch(cfg: dict, run_seed: int, index: int, rows: int):
    x = np.empty(rows * int(cfg["input-dim"]), np.float64)
    ycols = int(cfg["output-dim"]) if cfg.get("task", "regression") == "regression" else 1
    y = np.empty(rows * ycols, np.float64)
    _check(lib().ref_batch(kv(cfg), run_seed, index, rows, _dp(x), _dp(y)))
    return x.reshape(rows, -1), y.reshape(rows, -1)


def run_iteration(cfg: dict, seed: int, swapped_half: bool, x, y, iteration: int, n_params: int):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    loss = C.c_double(0)
    om = np.zeros(int(cfg["stages"]), np.float64)
    flat = np.zeros(n_params, np.float64)
    _check(lib().ref_run_iteration(kv(cfg), seed, 1 if swapped_half else 0, _dp(x), _dp(y), x.shape[0],
                                   iteration, C.byref(loss), _dp(om), _dp(flat)))
    return loss.value, om, flat


def run_experiment(cfg: dict, trace_text: str, seed: int):
    m = C.create_string_buffer(1 << 22)
    e = C.create_string_buffer(1 << 22)
    _check(lib().ref_run_experiment(kv(cfg), trace_text.encode(), seed, m, len(m), e, len(e)))
    return m.value.decode(), e.value.decode()


def run_experiment_full(cfg: dict, trace_text: str, seed: int) -> str:
    buf = C.create_string_buffer(1 << 22)
    _check(lib().ref_run_experiment_full(kv(cfg), trace_text.encode(), seed, buf, len(buf)))
    return buf.value.decode()


def time_train_iterations(cfg: dict, seed: int, iters: int) -> float:
    t = lib().ref_time_train_iterations(kv(cfg), seed, iters)
    if t < 0:
        raise RuntimeError(lib().ref_last_error().decode())
    return t


def time_recover_checkfree(n: int, reps: int) -> float:
    return lib().ref_time_recover_checkfree(n, reps)


def parallel_threads() -> int:
    return lib().ref_parallel_threads()
