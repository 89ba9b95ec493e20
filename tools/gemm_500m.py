#!/usr/bin/env python
"""Times every GEMM family of the LLaMA-500M step (one CheckFree+ order-class group = 32,768
tokens, as the step runs them) with CUDA events; one JSON line per family (us, TFLOP/s)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402
import tensor_counter as TC  # noqa: E402

only = [x for x in sys.argv[1:] if not x.startswith('--')]
out = {}
for (name, M, N, K, a_mn, b_mn, epi) in TC.SHAPES:
    if only and name not in only:
        continue
    if M == TC.T_:
        M //= 2
    elif K == TC.T_:
        K //= 2
    keep, fn = TC.gemm_call(M, N, K, a_mn, b_mn, epi)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        fn()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / 20 * 1e3
    out[name] = {"us": round(us, 1), "tflops": round(2.0 * M * N * K / us / 1e6, 1)}
    if "--cublas" in sys.argv:  # the same product through torch.matmul (cuBLAS), plain bf16 output
        A, B = keep[0], keep[1]
        x = A.t() if a_mn else A
        y = B if b_mn else B.t()
        for _ in range(3):
            torch.matmul(x, y)
        torch.cuda.synchronize()
        a.record()
        for _ in range(20):
            torch.matmul(x, y)
        b.record()
        torch.cuda.synchronize()
        cu = a.elapsed_time(b) / 20 * 1e3
        out[name]["cublas_us"] = round(cu, 1)
        out[name]["vs_cublas"] = round(cu / us, 3)
    del keep
print(json.dumps(out), flush=True)
