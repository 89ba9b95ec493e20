#!/usr/bin/env python
"""Same GEMM shape, every operand layout: isolates the cost of MN-major operands (wgrad)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_15461_b200  # noqa
from paper_2506_15461_b200._native import check, lib

def t(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it

if __name__ == "__main__":
  for (M, N, K, epi) in [(512, 4096, 8192, 2), (2048, 512, 8192, 2), (4096, 4096, 4096, 1), (8192, 1536, 512, 0)]:
      for a_mn in (0, 1):
          for b_mn in (0, 1):
              A = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
              B = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
              C = torch.zeros((M, N), device="cuda", dtype=torch.bfloat16 if epi == 0 else torch.float32)
              for bn in (128, 256):
                  ms = t(lambda: check(lib().ckf_gemm_bf16(M, N, K, A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn, C.data_ptr(), N, epi, 1.0, bn, None)))
                  print(json.dumps({"M": M, "N": N, "K": K, "a_mn": a_mn, "b_mn": b_mn, "bn": bn, "epi": epi, "us": round(ms * 1e3, 1), "tflops": round(2.0 * M * N * K / ms / 1e9, 1)}), flush=True)
