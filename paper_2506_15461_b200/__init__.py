"""B200-native CheckFree / CheckFree+ pipeline training and stage recovery
(arXiv 2506.15461), behind the reference's stage / pipeline / recovery API.

libckf.so (sm_100a kernels + engine, C-ABI in include/ckf.h) is the product;
this package is its Python face.  Importing fails loudly if the library was
not built -- there is no CPU fallback.
"""
from ._native import (CkfError, ConfigError, NumericDivergenceError, ParseError, UnsupportedRecoveryError,  # noqa
                      UsageError, lib)
from .api import (Engine, ModelSpec, adam_device, adam_update, counter_uniform, gemm, nccl_unique_id,  # noqa
                  recover_checkfree, recover_device, run_experiment, sum_squares)

lib()  # load now: a missing/unbuilt libckf.so is an ImportError, never a silent fallback
