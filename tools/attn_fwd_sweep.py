#!/usr/bin/env python
"""Times the tcgen05 attention forward at the benched shapes (one configuration per process:
CKF_ATTN_FWD_NG / CKF_ATTN_POLY are read once).  Prints one JSON line per shape."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_15461_b200  # noqa
from paper_2506_15461_b200._native import check, lib


def bench(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it


shapes = [(64, 1024, 16, 64), (32, 1024, 16, 64), (64, 1024, 8, 64), (16, 4096, 16, 128), (32, 2048, 16, 128)]
for (B, T, H, hd) in shapes:
    qkv = torch.randn(B * T, 3 * H * hd, device="cuda").bfloat16()
    o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B * H * T, device="cuda")
    flops = 2.0 * B * H * T * T * hd
    ms = bench(lambda: check(lib().ckf_attention_fwd(qkv.data_ptr(), B, T, H, hd, o.data_ptr(), lse.data_ptr(), 2, None)))
    print(json.dumps({"shape": [B, T, H, hd], "ng": os.environ.get("CKF_ATTN_FWD_NG", "default"),
                      "poly": os.environ.get("CKF_ATTN_POLY", "default"), "fwd_us": ms * 1e3,
                      "tflops": flops / ms / 1e9}), flush=True)
