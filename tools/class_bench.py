import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2506_15461_b200 as P
from paper_2506_15461_b200 import api
# one LLaMA-124M iteration, kernel timing classes (norm class) via the engine
w = dict(vocab=50304, d=512, layers=12, heads=8, ffn=2048, T=1024, s=4, m=8, rows=64)
spec = api.ModelSpec.llama(w["vocab"], w["d"], w["layers"], w["heads"], w["ffn"], w["T"], w["s"], max_tokens=8 * 1024)
eng = P.Engine(spec); eng.init(1, 3e-4)
import numpy as np
orders = np.array(api.build_schedule(8, False, 4), np.int32)
x = torch.randint(0, 50304, (64, 1025), device="cuda", dtype=torch.int32)
for i in range(4): eng.run_iteration(orders, x, None, i + 1, on_device=True)
eng.kernel_timing(True)
for i in range(5): eng.run_iteration(orders, x, None, i + 10, on_device=True)
print(json.dumps({c: eng.kernel_stats(c) for c in ("norm", "gemm", "attention", "loss")}))
