#!/usr/bin/env python
"""Attention backward time vs the dS^T scratch budget per pass (CKF_ATTN_DS_BYTES, read once per
process: run one process per budget).  Usage: CKF_ATTN_DS_BYTES=N python tools/attn_ds_chunk.py"""
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


for (B, T, H, hd) in [(64, 1024, 16, 64), (32, 1024, 16, 64), (16, 4096, 16, 128)]:
    qkv = torch.randn(B * T, 3 * H * hd, device="cuda").bfloat16()
    o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B * H * T, device="cuda")
    dout = torch.randn(B * T, H * hd, device="cuda").bfloat16()
    dqkv = torch.empty_like(qkv)
    D = torch.empty(B * H * T, device="cuda")
    check(lib().ckf_attention_fwd(qkv.data_ptr(), B, T, H, hd, o.data_ptr(), lse.data_ptr(), 2, None))
    ms = bench(lambda: check(lib().ckf_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(),
                                                     B, T, H, hd, dqkv.data_ptr(), D.data_ptr(), 0, None)))
    print(json.dumps({"ds_bytes": os.environ.get("CKF_ATTN_DS_BYTES", "default"), "shape": [B, T, H, hd],
                      "bwd_us": round(ms * 1e3, 1)}), flush=True)
