#!/usr/bin/env python
"""Times the tcgen05 bf16 GEMM (ckf_gemm_bf16) at the LLaMA stage shapes against
torch.matmul (cuBLAS) on the same operands; CUDA events, L2-resident operands."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_15461_b200  # noqa
from paper_2506_15461_b200._native import check, lib

SHAPES = [  # (name, M, N, K, a_mn, b_mn, epi): one fused LLaMA-124M step (65,536 tokens)
    ("qkv_fwd", 65536, 1536, 512, 0, 1, 0), ("o_fwd", 65536, 512, 512, 0, 1, 2), ("gu_fwd", 65536, 4096, 512, 0, 1, 0),
    ("down_fwd", 65536, 512, 2048, 0, 1, 2), ("down_dgrad", 65536, 2048, 512, 0, 0, 0),
    ("gu_dgrad", 65536, 512, 4096, 0, 0, 1), ("o_dgrad", 65536, 512, 512, 0, 0, 0),
    ("qkv_dgrad", 65536, 512, 1536, 0, 0, 1),
    ("qkv_wgrad", 512, 1536, 65536, 1, 1, 2), ("o_wgrad", 512, 512, 65536, 1, 1, 2),
    ("gu_wgrad", 512, 4096, 65536, 1, 1, 2), ("down_wgrad", 2048, 512, 65536, 1, 1, 2),
    ("lmhead_fwd", 65536, 50304, 512, 0, 1, 0), ("lmhead_dgrad", 65536, 512, 50304, 0, 0, 1),
    ("lmhead_wgrad", 512, 50304, 65536, 1, 1, 2),
    ("sq8192", 8192, 8192, 8192, 0, 1, 0),
    # fused SwiGLU epilogues (compare with gu_fwd / down_dgrad above)
    ("gu_fwd_swiglu", 65536, 4096, 512, 0, 1, 3), ("down_dgrad_swiglu", 65536, 2048, 512, 0, 0, 4),
    # LLaMA-500M (one CheckFree+ group of 32,768 tokens)
    ("down_dgrad_500m", 32768, 4096, 1024, 0, 0, 0), ("down_dgrad_swiglu_500m", 32768, 4096, 1024, 0, 0, 4),
    ("gu_fwd_swiglu_500m", 32768, 8192, 1024, 0, 1, 3), ("o_fwd_500m", 32768, 1024, 1024, 0, 1, 2),
    ("qkv_fwd_500m", 32768, 3072, 1024, 0, 1, 0), ("down_fwd_500m", 32768, 1024, 4096, 0, 1, 2),
    ("gu_dgrad_500m", 32768, 1024, 8192, 0, 0, 1), ("qkv_dgrad_500m", 32768, 1024, 3072, 0, 0, 1),
]

def run(name, M, N, K, a_mn, b_mn, epi, bn=0, iters=20):
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
    cw = 2 * N if epi == 4 else N
    C = torch.zeros((M, cw), device="cuda", dtype=torch.bfloat16 if epi in (0, 3, 4) else torch.float32)
    aux = (torch.zeros((M, N // 2), device="cuda", dtype=torch.bfloat16) if epi == 3 else
           torch.randn((M, 2 * N), device="cuda").bfloat16() if epi == 4 else None)
    f = lambda: check(lib().ckf_gemm_bf16_aux(M, N, K, A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn,
                                              C.data_ptr(), cw, epi, 1.0, bn, aux.data_ptr() if aux is not None else None,
                                              aux.shape[1] if aux is not None else 0, None))
    a = A.t() if a_mn else A
    b = B if b_mn else B.t()
    g = lambda: torch.matmul(a, b)
    res = {}
    for tag, fn in (("ours", f), ("cublas", g)):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters): fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        res[tag] = (ms, 2.0 * M * N * K / ms / 1e9)
    print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "bn": bn, "ours_ms": res["ours"][0],
                      "ours_tflops": res["ours"][1], "cublas_ms": res["cublas"][0], "cublas_tflops": res["cublas"][1]}))

if __name__ == "__main__":
    only = [a for a in sys.argv[1:] if not a.startswith("-")]
    for s in SHAPES:
        if only and s[0] not in only:
            continue
        run(*s)
        if "--bn" in sys.argv:
            for bn in (128, 256):
                run(*s, bn=bn)
