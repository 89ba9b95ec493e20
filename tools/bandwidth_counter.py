#!/usr/bin/env python
"""HBM evidence for the bandwidth kernels at the LLaMA-500M step's sizes (one CheckFree+ order-class
group = 32,768 tokens; d = 1024, f = 4096, V = 50,304; one 50.3 M-parameter stage): ONE launch of
each between cudaProfilerStart / Stop (warm-ups outside), for

    ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        python tools/bandwidth_counter.py

Algorithmic bytes per launch (the minimum each op must move) go to gpurun_out/bandwidth_bytes.json
in launch order (tools/bandwidth_table.py joins them)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_15461_b200 as P  # noqa: E402
from paper_2506_15461_b200._native import check, lib  # noqa: E402

L = lib()
M, d, f, V, NP = 32768, 1024, 4096, 50304, 50_337_792
dev = "cuda"
ops = []  # (name, n_kernels, algorithmic bytes, fn)

x = torch.randn(M, d, device=dev)
g = torch.ones(d, device=dev)
y = torch.empty(M, d, device=dev, dtype=torch.bfloat16)
rstd = torch.empty(M, device=dev)
xc = torch.empty_like(x)
ops.append(("rmsnorm_fwd", 1, M * d * (4 + 2 + 4) + M * 4,
            lambda: check(L.ckf_llama_rmsnorm_fwd(x.data_ptr(), g.data_ptr(), M, d, y.data_ptr(), rstd.data_ptr(),
                                                  xc.data_ptr(), None))))
dy = torch.randn(M, d, device=dev)
dh = torch.zeros(M, d, device=dev)
dhb = torch.empty(M, d, device=dev, dtype=torch.bfloat16)
gg = torch.zeros(d, device=dev)
ops.append(("rmsnorm_bwd + gain fold", 2, M * d * (4 + 4 + 4 + 4 + 2) + M * 4,
            lambda: check(L.ckf_llama_rmsnorm_bwd(dy.data_ptr(), x.data_ptr(), g.data_ptr(), rstd.data_ptr(), M, d,
                                                  dh.data_ptr(), dhb.data_ptr(), gg.data_ptr(), None))))
qkv = torch.randn(M, 3 * d, device=dev).bfloat16()
ops.append(("rope (inverse, q and k)", 1, M * 2 * d * 2 * 2,
            lambda: check(L.ckf_llama_rope(qkv.data_ptr(), M, 1024, d, d // 64, 1, None))))
gu = torch.randn(M, 2 * f, device=dev).bfloat16()
a = torch.empty(M, f, device=dev, dtype=torch.bfloat16)
ops.append(("swiglu_fwd (standalone)", 1, M * f * (4 + 2),
            lambda: check(L.ckf_llama_swiglu_fwd(gu.data_ptr(), M, f, a.data_ptr(), None))))
dgu = torch.empty_like(gu)
ops.append(("swiglu_bwd (standalone)", 1, M * f * (4 + 2 + 4),
            lambda: check(L.ckf_llama_swiglu_bwd(gu.data_ptr(), a.data_ptr(), M, f, dgu.data_ptr(), None))))
logits = torch.randn(M // 4, V, device=dev).bfloat16()
lab = torch.randint(0, V, (M // 4,), device=dev, dtype=torch.int32)
rl = torch.empty(M // 4, device=dev, dtype=torch.float64)
ops.append(("cross-entropy + gradient (8,192 rows)", 1, (M // 4) * V * 4,
            lambda: check(L.ckf_xent_bf16(logits.data_ptr(), lab.data_ptr(), M // 4, V, 1.0, 1, rl.data_ptr(), None))))
w, m_, v_, gr = (torch.rand(NP, device=dev) for _ in range(4))
wl = torch.empty(NP, device=dev, dtype=torch.bfloat16)
om = torch.zeros(1, device=dev, dtype=torch.float64)
ops.append(("fused Adam + omega (+ bf16 shadow, g zeroed)", 2, NP * (4 * 4 + 4 * 4 + 2),
            lambda: P.api.adam_device(w, m_, v_, gr, 3e-4, 10, 1.0 / 8, True, wl, om)))
t6 = [torch.rand(NP, device=dev) for _ in range(6)]
ops.append(("fused stage recovery", 1, NP * 26,
            lambda: P.api.recover_stage_device(t6[0], t6[1], t6[2], t6[3], t6[4], t6[5], 4.0, 1.0, w_bf16=wl)))
tok = torch.randint(0, V, (M,), device=dev, dtype=torch.int32)
E = torch.randn(V, d, device=dev)
h = torch.empty(M, d, device=dev)
ops.append(("embedding gather", 1, M * d * 8 + M * 4,
            lambda: check(L.ckf_llama_embed_fwd(tok.data_ptr(), M, E.data_ptr(), d, h.data_ptr(), None))))

for _, _, _, fn in ops:
    fn()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _, _, _, fn in ops:
    fn()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
os.makedirs("gpurun_out", exist_ok=True)
json.dump([{"name": n, "kernels": k, "bytes": b} for n, k, b, _ in ops], open("gpurun_out/bandwidth_bytes.json", "w"),
          indent=1)
