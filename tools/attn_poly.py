#!/usr/bin/env python
"""Attention forward (and backward) time and accuracy at the LLaMA-500M / 1.5B shapes for one
CKF_ATTN_POLY / CKF_ATTN_BWD_POLY setting (set in the environment; the kernels read it once).
Prints one JSON line: us and TFLOP/s (causal-half FLOPs), max / Frobenius error vs fp32 torch."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_15461_b200  # noqa: E402,F401
from paper_2506_15461_b200._native import check, lib  # noqa: E402

L = lib()


def bench(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


out = {"poly": os.environ.get("CKF_ATTN_POLY"), "bwd_poly": os.environ.get("CKF_ATTN_BWD_POLY")}
for (B, T, H, hd) in [(64, 1024, 16, 64), (16, 4096, 16, 128)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    qkv = (torch.randn(B * T, 3 * H * hd, device="cuda", generator=g) * 1.5).bfloat16()
    o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B * H * T, device="cuda")
    dout = torch.randn(B * T, H * hd, device="cuda", generator=g).bfloat16()
    dqkv = torch.empty_like(qkv)
    D = torch.empty(B * H * T, device="cuda")
    fl = 2.0 * B * H * T * T * hd
    f_us = bench(lambda: check(L.ckf_attention_fwd(qkv.data_ptr(), B, T, H, hd, o.data_ptr(), lse.data_ptr(), 2, None)))
    b_us = bench(lambda: check(L.ckf_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(), B, T,
                                                   H, hd, dqkv.data_ptr(), D.data_ptr(), 0, None)))
    # accuracy on the first 2 sequences vs fp32 SDPA
    bs = 2
    x = qkv[:bs * T].float().view(bs, T, 3, H, hd)
    q, k, v = (x[:, :, i].transpose(1, 2).requires_grad_(True) for i in range(3))
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
    ref_o = ref.detach().transpose(1, 2).reshape(bs * T, H * hd)
    got_o = o[:bs * T].float()
    ref.backward(dout[:bs * T].float().view(bs, T, H, hd).transpose(1, 2))
    ref_d = torch.cat([t.grad.transpose(1, 2).reshape(bs * T, H * hd) for t in (q, k, v)], 1)
    got_d = dqkv[:bs * T].float()
    out[f"hd{hd}"] = {"fwd_us": f_us, "fwd_tflops": fl / f_us / 1e6, "bwd_us": b_us, "bwd_tflops": 2.5 * fl / b_us / 1e6,
                      "fwd_rel": float((got_o - ref_o).norm() / ref_o.norm()),
                      "fwd_maxabs": float((got_o - ref_o).abs().max()),
                      "bwd_rel": float((got_d - ref_d).norm() / ref_d.norm())}
print(json.dumps(out), flush=True)
