#!/usr/bin/env python
"""Times the attention kernels at the LLaMA-124M microbatch shape (B=8, T=1024, H=8, hd=64)."""
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

for (B, T, H, hd) in [(64, 1024, 8, 64), (8, 1024, 8, 64), (64, 1024, 16, 64), (16, 4096, 16, 128)]:
    qkv = torch.randn(B * T, 3 * H * hd, device="cuda").bfloat16()
    o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B * H * T, device="cuda")
    dout = torch.randn(B * T, H * hd, device="cuda").bfloat16()
    dqkv = torch.empty_like(qkv)
    D = torch.empty(B * H * T, device="cuda")
    flops = 2.0 * B * H * T * T * hd  # causal half of 4 T^2 hd
    res = {"shape": [B, T, H, hd]}
    for impl in (1, 2):
        if impl == 2 and hd not in (64, 128):
            continue
        ms = bench(lambda: check(lib().ckf_attention_fwd(qkv.data_ptr(), B, T, H, hd, o.data_ptr(), lse.data_ptr(), impl, None)))
        res[f"fwd_impl{impl}_us"] = ms * 1e3
        res[f"fwd_impl{impl}_tflops"] = flops / ms / 1e9
    ms = bench(lambda: check(lib().ckf_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(), B, T, H, hd, dqkv.data_ptr(), D.data_ptr(), 0, None)))
    res["bwd_us"] = ms * 1e3
    res["bwd_tflops"] = 2.5 * flops / ms / 1e9
    print(json.dumps(res), flush=True)
