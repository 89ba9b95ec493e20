"""Times the LLaMA head loss kernel (ckf_xent_bf16) at the LLaMA-124M step shape (65,536 rows x
50,304 vocabulary, bf16 logits, gradient in place); CUDA events, HBM GB/s of read + write."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_15461_b200._native import check, lib
rows, V = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (65536, 50304)))
x = (torch.randn(rows, V, device="cuda") * 3).bfloat16()
lab = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
loss = torch.zeros(rows, device="cuda", dtype=torch.float64)
f = lambda: check(lib().ckf_xent_bf16(x.data_ptr(), lab.data_ptr(), rows, V, 1.0 / rows, 1, loss.data_ptr(), None))
for _ in range(3): f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
e0.record()
for _ in range(n): f()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(json.dumps({"rows": rows, "V": V, "ms": ms, "gbs": 2 * rows * V * 2 / ms / 1e6}))
