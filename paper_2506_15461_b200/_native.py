"""ctypes binding of include/ckf.h (libckf.so, built in-tree by build.py).

The product path: every call below runs this package's own sm_100a kernels.
There is no CPU fallback -- if libckf.so is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CKF_LIB_PATH: an alternative build of the same library (A/B timing tools only)
LIB_PATH = os.environ.get("CKF_LIB_PATH") or os.path.join(HERE, "libckf.so")

CKF_OK, CKF_E_CONFIG, CKF_E_DIVERGENCE, CKF_E_USAGE, CKF_E_PARSE, CKF_E_UNSUPPORTED_RECOVERY, CKF_E_CUDA, \
    CKF_E_NCCL = range(8)
CKF_FP64, CKF_FP32, CKF_BF16 = 0, 1, 2
CKF_BLOCK_MLP, CKF_BLOCK_LLAMA = 0, 1
CKF_ACT = {"tanh": 0, "relu": 1, "identity": 2}
CKF_TASK = {"regression": 0, "classification": 1}
CKF_REC_CHECKFREE, CKF_REC_UNIFORM, CKF_REC_COPY_PREV, CKF_REC_RANDOM, CKF_REC_EDGE = range(5)
CKF_MOM_FRESH, CKF_MOM_AVERAGED = 0, 1


class CkfError(RuntimeError):
    """Mirrors the reference's exception family (include/ckfree/errors.hpp)."""

    def __init__(self, code: int, msg: str, iteration: int = -1):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.iteration = iteration


class ConfigError(CkfError): pass
class NumericDivergenceError(CkfError): pass
class UsageError(CkfError): pass
class ParseError(CkfError): pass
class UnsupportedRecoveryError(CkfError): pass
class CudaError(CkfError): pass


_ERR = {CKF_E_CONFIG: ConfigError, CKF_E_DIVERGENCE: NumericDivergenceError, CKF_E_USAGE: UsageError,
        CKF_E_PARSE: ParseError, CKF_E_UNSUPPORTED_RECOVERY: UnsupportedRecoveryError, CKF_E_CUDA: CudaError,
        CKF_E_NCCL: CudaError}


class ModelDesc(C.Structure):
    _fields_ = [("block", C.c_int), ("precision", C.c_int), ("activation", C.c_int), ("task", C.c_int),
                ("input_dim", C.c_size_t), ("hidden_dim", C.c_size_t), ("model_dim", C.c_size_t),
                ("output_dim", C.c_size_t), ("num_layers", C.c_size_t), ("num_stages", C.c_size_t),
                ("n_heads", C.c_size_t), ("seq_len", C.c_size_t), ("partition", C.POINTER(C.c_size_t)),
                ("max_rows", C.c_size_t), ("device", C.c_int)]


class RecoveryReport(C.Structure):
    _fields_ = [("degenerate", C.c_int), ("reduction_error", C.c_double), ("latency_ms", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    i, sz, dbl, u64, lng = C.c_int, C.c_size_t, C.c_double, C.c_uint64, C.c_long
    dp, vp, ip, cp = C.POINTER(C.c_double), C.c_void_p, C.POINTER(C.c_int), C.c_char_p
    eng = C.c_void_p
    sig = {
        "ckf_last_error": (cp, []), "ckf_last_error_iteration": (lng, []), "ckf_version": (i, []),
        "ckf_device_count": (i, [ip]),
        "ckf_generate_trace": (i, [u64, dbl, dbl, lng, ip, i, cp, sz]), "ckf_parse_trace": (i, [cp, cp, sz]),
        "ckf_consecutive_conflicts": (i, [cp, C.POINTER(lng), i, ip]),
        "ckf_hourly_to_per_iteration": (dbl, [dbl, dbl]),
        "ckf_even_partition": (i, [sz, sz, C.POINTER(sz)]), "ckf_build_schedule": (i, [i, i, i, ip]),
        "ckf_pipeline_plan": (i, [i, i, ip, ip, i, ip, i, ip]),
        "ckf_pipeline_plan_cost": (i, [i, i, ip, ip, i, dp, dbl, ip, i, ip]),
        "ckf_k_gemm_nn": (i, [dp, dp, dp, sz, sz, sz]), "ckf_k_gemm_nn_acc": (i, [dp, dp, dp, sz, sz, sz]),
        "ckf_k_gemm_nt_acc": (i, [dp, dp, dp, sz, sz, sz]), "ckf_k_gemm_tn_acc": (i, [dp, dp, dp, sz, sz, sz]),
        "ckf_k_add_inplace": (i, [dp, dp, sz]), "ckf_k_axpy": (i, [dbl, dp, dp, sz]), "ckf_k_scale": (i, [dbl, dp, sz]),
        "ckf_k_apply_activation": (i, [i, dp, dp, sz]), "ckf_k_activation_backward": (i, [i, dp, dp, dp, sz]),
        "ckf_k_sum_squares": (i, [dp, sz, dp]), "ckf_k_sum_squared_diff": (i, [dp, dp, sz, dp]),
        "ckf_k_adam_update": (i, [dp, dp, dp, dp, sz, dbl, dbl, dbl, dbl, lng]),
        "ckf_k_mse_loss_grad": (i, [dp, dp, sz, sz, dp, dp]),
        "ckf_k_softmax_xent_loss_grad": (i, [dp, ip, sz, sz, dp, dp]),
        "ckf_k_recover_checkfree": (i, [dp, dp, sz, dbl, dbl, dp, ip]),
        "ckf_k_counter_uniform": (i, [u64, dbl, dbl, dp, sz]),
        "ckf_recover_device": (i, [i, vp, vp, vp, sz, dbl, dbl, vp, vp]),
        "ckf_gemm_bf16": (i, [i, i, i, vp, i, i, vp, i, i, vp, i, i, C.c_float, i, vp]),
        "ckf_xent_bf16": (i, [vp, vp, C.c_size_t, C.c_size_t, C.c_float, i, vp, vp]),
        "ckf_lm_head_xent_workspace": (C.c_size_t, [sz, sz, sz]),
        "ckf_lm_head_xent": (i, [vp, vp, vp, sz, sz, sz, C.c_float, i, vp, vp, vp, vp, vp, vp, vp, vp]),
        "ckf_gemm_bf16_aux": (i, [i, i, i, vp, i, i, vp, i, i, vp, i, i, C.c_float, i, vp, i, vp]),
        "ckf_attention_fwd": (i, [vp, sz, sz, sz, sz, vp, vp, i, vp]),
        "ckf_attention_bwd": (i, [vp, vp, vp, vp, sz, sz, sz, sz, vp, vp, i, vp]),
        "ckf_llama_token_batch": (i, [u64, u64, u64, sz, sz, sz, ip]),
        "ckf_llama_rmsnorm_fwd": (i, [vp, vp, sz, sz, vp, vp, vp, vp]),
        "ckf_llama_rmsnorm_bwd": (i, [vp, vp, vp, vp, sz, sz, vp, vp, vp, vp]),
        "ckf_llama_rope": (i, [vp, sz, sz, sz, sz, i, vp]),
        "ckf_llama_swiglu_fwd": (i, [vp, sz, sz, vp, vp]), "ckf_llama_swiglu_bwd": (i, [vp, vp, sz, sz, vp, vp]),
        "ckf_llama_embed_fwd": (i, [vp, sz, vp, sz, vp, vp]), "ckf_llama_embed_bwd": (i, [vp, sz, vp, sz, vp, vp]),
        "ckf_gemm_qkv_rope": (i, [i, i, vp, vp, vp, sz, sz, vp]),
        "ckf_gemm_o_dgrad_dsum": (i, [i, i, vp, vp, vp, vp, vp, sz, sz, vp]),
        "ckf_adam_device": (i, [i, vp, vp, vp, vp, vp, sz, dbl, dbl, dbl, dbl, i, vp, vp]),
        "ckf_engine_create": (i, [C.POINTER(ModelDesc), C.POINTER(eng)]), "ckf_engine_destroy": (i, [eng]),
        "ckf_engine_param_counts": (i, [eng, C.POINTER(sz), C.POINTER(sz), C.POINTER(sz)]),
        "ckf_engine_init": (i, [eng, u64, dbl]),
        "ckf_engine_set_schedule": (i, [eng, i]), "ckf_engine_set_group_cap": (i, [eng, i]),
        "ckf_engine_last_step_ms": (i, [eng, C.POINTER(C.c_float)]),
        "ckf_engine_set_redundant": (i, [eng, i]), "ckf_engine_set_edge_replicas": (i, [eng, i]),
        "ckf_nccl_unique_id": (i, [vp, sz]), "ckf_engine_attach_comm": (i, [eng, vp, i, i, ip]),
        "ckf_engine_attach_comm_dp": (i, [eng, vp, i, i, ip, i]),
        "ckf_engine_set_placement": (i, [eng, i, i, ip, i]),
        "ckf_engine_ipc_export": (i, [eng, vp, sz, C.POINTER(sz)]), "ckf_engine_ipc_import": (i, [eng, vp, sz]),
        "ckf_engine_exchange_peers": (i, [eng]),
        "ckf_engine_plan_cost": (i, [eng, dp, dp]), "ckf_engine_enable_peer_transport": (i, [eng, i]),
        "ckf_recover_stage_device": (i, [i, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, dbl, dbl, i, vp, vp]),
        "ckf_engine_run_iteration": (i, [eng, ip, i, vp, vp, sz, i, lng, dp, dp]),
        "ckf_engine_eval_loss": (i, [eng, ip, vp, vp, sz, i, dp]),
        "ckf_engine_predict": (i, [eng, ip, dp, sz, dp]),
        "ckf_engine_accumulate": (i, [eng, ip, vp, vp, sz, i, dp]), "ckf_engine_zero_grad": (i, [eng]),
        "ckf_engine_export_grad": (i, [eng, i, i, dp]),
        "ckf_engine_refresh_edge_replicas": (i, [eng]), "ckf_engine_kill_stage": (i, [eng, i]),
        "ckf_engine_recover_stage": (i, [eng, i, i, i, dbl, u64, i, C.POINTER(RecoveryReport)]),
        "ckf_engine_export_stage": (i, [eng, i, dp, dp, dp]), "ckf_engine_import_stage": (i, [eng, i, dp, dp, dp]),
        "ckf_engine_export_edge": (i, [eng, i, dp, dp, dp]), "ckf_engine_import_edge": (i, [eng, i, dp, dp, dp]),
        "ckf_engine_get_scalars": (i, [eng, i, dp, dp, C.POINTER(lng)]),
        "ckf_engine_set_scalars": (i, [eng, i, dbl, dbl, lng]),
        "ckf_engine_get_edge_scalars": (i, [eng, dp, C.POINTER(lng), C.POINTER(lng)]),
        "ckf_engine_set_edge_scalars": (i, [eng, dbl, lng, lng]),
        "ckf_engine_kernel_launches": (lng, [eng]), "ckf_engine_sync": (i, [eng]),
        "ckf_engine_stream": (i, [eng, C.POINTER(C.c_void_p)]), "ckf_engine_kernel_timing": (i, [eng, i]),
        "ckf_engine_kernel_stats": (i, [eng, i, dp, C.POINTER(lng), dp, dp]),
        "ckf_run_experiment": (i, [cp, cp, u64, cp, sz]),
        "ckf_run_experiment_to_dir": (i, [cp, cp, u64, cp]),
        "ckf_run_experiment_rank": (i, [cp, cp, u64, vp, i, i, i, cp, sz]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc: int):
    if rc != CKF_OK:
        L = lib()
        raise _ERR.get(rc, CkfError)(rc, L.ckf_last_error().decode(), L.ckf_last_error_iteration())


def exported_symbols_from_header() -> list[str]:
    import re
    hdr = os.path.join(os.path.dirname(HERE), "include", "ckf.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(ckf_\w+)\s*\(", text)))
