#!/usr/bin/env python
"""Split-K sweep for the weight-gradient shapes (run with CKF_GEMM_SPLITS=<n> in the environment)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_15461_b200  # noqa
from paper_2506_15461_b200._native import check, lib
from gemm_layouts import t  # noqa
for (M, N, K) in [(512, 4096, 8192), (2048, 512, 8192), (512, 1536, 8192), (512, 512, 8192)]:
    A = torch.randn((K, M), device="cuda").bfloat16()
    B = torch.randn((K, N), device="cuda").bfloat16()
    C = torch.zeros((M, N), device="cuda")
    for bn in (128, 256):
        ms = t(lambda: check(lib().ckf_gemm_bf16(M, N, K, A.data_ptr(), M, 1, B.data_ptr(), N, 1, C.data_ptr(), N, 2, 1.0, bn, None)))
        print(json.dumps({"splits": os.environ.get("CKF_GEMM_SPLITS", "auto"), "M": M, "N": N, "K": K, "bn": bn, "us": round(ms * 1e3, 1), "tflops": round(2.0 * M * N * K / ms / 1e9, 1)}), flush=True)
