#!/usr/bin/env python
"""One launch of named GEMM families of the LLaMA-500M step between cudaProfilerStart / Stop
(warm-up outside), for ncu --profile-from-start off.  Usage: gemm_one.py name [name ...]
(names from tools/tensor_counter.py SHAPES)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402
import tensor_counter as TC  # noqa: E402

want = sys.argv[1:]
calls, keep = [], []
for (name, M, N, K, a_mn, b_mn, epi) in TC.SHAPES:
    if name in want:
        k, fn = TC.gemm_call(M // 2, N, K, a_mn, b_mn, epi) if M == TC.T_ else TC.gemm_call(M, N, K // 2, a_mn, b_mn, epi)
        keep.append(k)
        calls.append(fn)
for fn in calls:
    fn()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for fn in calls:
    fn()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
