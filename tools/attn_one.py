#!/usr/bin/env python
"""One attention fwd + bwd (for ncu).  Shape from argv: B T H hd (default: the LLaMA-124M microbatch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_15461_b200  # noqa
from paper_2506_15461_b200._native import check, lib
B, T, H, hd = (int(a) for a in sys.argv[1:5]) if len(sys.argv) > 4 else (8, 1024, 8, 64)
qkv = torch.randn(B * T, 3 * H * hd, device="cuda").bfloat16()
o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device="cuda")
lse = torch.empty(B * H * T, device="cuda")
dout = torch.randn(B * T, H * hd, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv)
D = torch.empty(B * H * T, device="cuda")
for _ in range(3):
    check(lib().ckf_attention_fwd(qkv.data_ptr(), B, T, H, hd, o.data_ptr(), lse.data_ptr(), 2, None))
    check(lib().ckf_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(), B, T, H, hd, dqkv.data_ptr(), D.data_ptr(), 2, None))
torch.cuda.synchronize()
