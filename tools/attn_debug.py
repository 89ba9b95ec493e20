#!/usr/bin/env python
"""CKF_ATTN_DEBUG=1 python tools/attn_debug.py: per-CTA phase timings of the tcgen05 attention forward."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2506_15461_b200  # noqa
from paper_2506_15461_b200._native import check, lib
B, T, H, hd = (int(os.environ.get(k, v)) for k, v in (('B', 64), ('T', 1024), ('H', 8), ('HD', 64)))
qkv = torch.randn(B * T, 3 * H * hd, device="cuda").bfloat16()
o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device="cuda")
lse = torch.empty(B * H * T, device="cuda")
for _ in range(3):
    check(lib().ckf_attention_fwd(qkv.data_ptr(), B, T, H, hd, o.data_ptr(), lse.data_ptr(), 2, None))
torch.cuda.synchronize()
n = (T // 128) * B * H
buf = (C.c_longlong * (8 * n))()
L = lib()
L.ckf_debug_attn_fwd_timings.argtypes = [C.POINTER(C.c_longlong), C.c_int]
check(L.ckf_debug_attn_fwd_timings(buf, n))
a = np.array(buf[:]).reshape(n, 8)
t0 = a[:, 6].min()
print("ctas", n, "cycles: total(max)", a[:, 4].max(), "mean", a[:, 4].mean())
for nk in sorted(set(a[:, 0])):
    s = a[a[:, 0] == nk]
    print(f"nkb={nk:3d} n={len(s):4d} first_S={s[:,1].mean():8.0f} wait_S={s[:,2].mean():8.0f} wait_P={s[:,3].mean():8.0f} "
          f"total={s[:,4].mean():8.0f} per_tile={(s[:,4]-s[:,1]).mean()/nk:7.0f} start={((s[:,6]-t0)/1e3).mean():8.1f}k")

# backward dK/dV kernel (timings at offset 32768 CTAs)
dout = torch.randn(B * T, H * hd, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv)
Dd = torch.empty(B * H * T, device="cuda")
for _ in range(3):
    check(lib().ckf_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(), B, T, H, hd,
                                  dqkv.data_ptr(), Dd.data_ptr(), 2, None))
torch.cuda.synchronize()
buf2 = (C.c_longlong * (8 * 32768 + 16 * 148))()
check(L.ckf_debug_attn_fwd_timings(buf2, 32768 + 2 * 148))
a = np.array(buf2[8 * 32768:]).reshape(148, 16)
t = a[:, 0].sum()
print(f"dkdv (persistent, 148 CTAs): tiles/CTA {a[:,0].mean():.1f}  total cycles {a[:,5].mean():.0f}  per tile {a[:,5].sum()/t:.0f}")
print(f"  softmax per tile: wait S {a[:,1].sum()/t:.0f}  wait pd_free {a[:,2].sum()/t:.0f}  compute {a[:,3].sum()/t:.0f} "
      f"(of which TMEM loads {a[:,6].sum()/t:.0f})  store phase {a[:,7].sum()/t:.0f}  "
      f"epilogue/unit-share {a[:,4].sum()/t:.0f}")
print(f"  MMA per tile: issue_s(+waits) {a[:,8].sum()/t:.0f}  acc_free wait {a[:,9].sum()/t:.0f}  pd_full wait {a[:,10].sum()/t:.0f}")
