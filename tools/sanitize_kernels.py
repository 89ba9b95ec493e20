#!/usr/bin/env python
"""Small launches of every sm_100a kernel family for compute-sanitizer
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_kernels.py

tcgen05 GEMM (all epilogues, ragged tails, split-K), tcgen05 attention forward / backward
(head_dim 64 and 128), fused stage recovery, the LLaMA bandwidth kernels, and two engine
iterations of a small LLaMA model (fused groups, deferred W pass, CUDA-graph capture).
Each step prints a line; the sanitizer's summary goes to its own log."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_15461_b200 as P  # noqa: E402
from paper_2506_15461_b200._native import check, lib  # noqa: E402

L = lib()
dev = "cuda"


def gemm(M, N, K, a_mn, b_mn, epi):
    A = torch.randn((K, M) if a_mn else (M, K), device=dev).bfloat16()
    B = torch.randn((K, N) if b_mn else (N, K), device=dev).bfloat16()
    cw = 2 * N if epi == 4 else N
    C = torch.zeros((M, cw), device=dev, dtype=torch.bfloat16 if epi in (0, 3, 4) else torch.float32)
    aux = (torch.zeros((M, N // 2), device=dev, dtype=torch.bfloat16) if epi == 3 else
           torch.randn((M, 2 * N), device=dev).bfloat16() if epi == 4 else None)
    check(L.ckf_gemm_bf16_aux(M, N, K, A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn, C.data_ptr(),
                              cw, epi, 1.0, 0, aux.data_ptr() if aux is not None else None,
                              aux.shape[1] if aux is not None else 0, None))
    torch.cuda.synchronize()


for shape in [(256, 512, 256, 0, 1, 0), (300, 200, 136, 0, 0, 1), (512, 384, 4096, 1, 1, 2), (1024, 1024, 256, 0, 1, 3),
              (1024, 512, 256, 0, 0, 4), (256, 1024, 16384, 1, 1, 2)]:
    gemm(*shape)
    print("gemm", shape, flush=True)

for (B, T, H, hd) in [(2, 256, 2, 64), (1, 256, 2, 128)]:
    qkv = torch.randn(B * T, 3 * H * hd, device=dev).bfloat16()
    o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(B * H * T, device=dev)
    dout = torch.randn(B * T, H * hd, device=dev).bfloat16()
    dqkv = torch.empty_like(qkv)
    D = torch.empty(B * H * T, device=dev)
    check(L.ckf_attention_fwd(qkv.data_ptr(), B, T, H, hd, o.data_ptr(), lse.data_ptr(), 2, None))
    check(L.ckf_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(), B, T, H, hd,
                              dqkv.data_ptr(), D.data_ptr(), 0, None))
    # the RoPE backward fused into the dK / dQ epilogues (CKF_ATTN_ROPE_BWD)
    check(L.ckf_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(), B, T, H, hd,
                              dqkv.data_ptr(), D.data_ptr(), 2 | 16, None))
    # the O-projection dgrad with the attention backward's D in its epilogue, and the QKV GEMM with RoPE
    d_ = H * hd
    W = torch.randn(d_, d_, device=dev).bfloat16()
    dO = torch.empty(B * T, d_, device=dev, dtype=torch.bfloat16)
    check(L.ckf_gemm_o_dgrad_dsum(B * T, d_, dout.data_ptr(), W.data_ptr(), dO.data_ptr(), o.data_ptr(), D.data_ptr(),
                                  T, H, None))
    Wq = torch.randn(d_, 3 * d_, device=dev).bfloat16()
    check(L.ckf_gemm_qkv_rope(B * T, d_, o.data_ptr(), Wq.data_ptr(), qkv.data_ptr(), T, H, None))
    torch.cuda.synchronize()
    print("attention", (B, T, H, hd), flush=True)

for dt in (torch.float32, torch.float64):
    n = 100_003
    t = [torch.rand(n, device=dev, dtype=dt) for _ in range(10)]
    wlp = torch.empty(n, device=dev, dtype=torch.bfloat16) if dt == torch.float32 else None
    sq = torch.zeros(1, device=dev, dtype=torch.float64)
    P.api.recover_stage_device(t[0], t[1], t[2], t[3], t[4], t[5], 4.0, 1.0, w_bf16=wlp, old_sq=sq)
    P.api.recover_stage_device(t[0], t[1], t[2], t[3], t[4], t[5], 4.0, 1.0, w_bf16=wlp, mp=t[6], mn=t[7], vp=t[8],
                               vn=t[9])
    torch.cuda.synchronize()
    print("recovery", dt, flush=True)

for d in (512, 1024, 2048):
    rows = 300
    x = torch.randn(rows, d, device=dev)
    g = torch.ones(d, device=dev)
    y = torch.empty(rows, d, device=dev, dtype=torch.bfloat16)
    r = torch.empty(rows, device=dev)
    check(L.ckf_llama_rmsnorm_fwd(x.data_ptr(), g.data_ptr(), rows, d, y.data_ptr(), r.data_ptr(), None, None))
    dh = torch.zeros(rows, d, device=dev)
    gg = torch.zeros(d, device=dev)
    check(L.ckf_llama_rmsnorm_bwd(x.data_ptr(), x.data_ptr(), g.data_ptr(), r.data_ptr(), rows, d, dh.data_ptr(),
                                  None, gg.data_ptr(), None))
    qkv = torch.randn(256, 3 * d, device=dev).bfloat16()
    check(L.ckf_llama_rope(qkv.data_ptr(), 256, 128, d, d // 64, 0, None))
    gu = torch.randn(256, 2 * d, device=dev).bfloat16()
    a = torch.empty(256, d, device=dev, dtype=torch.bfloat16)
    check(L.ckf_llama_swiglu_fwd(gu.data_ptr(), 256, d, a.data_ptr(), None))
    dgu = torch.empty_like(gu)
    check(L.ckf_llama_swiglu_bwd(gu.data_ptr(), a.data_ptr(), 256, d, dgu.data_ptr(), None))
    torch.cuda.synchronize()
    print("llama kernels d", d, flush=True)

spec = P.api.ModelSpec.llama(512, 128, 4, 2, 256, 128, 4, max_tokens=2 * 128)
e = P.Engine(spec)
e.init(3, 1e-3)
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
for it in (1, 2, 3):
    toks = P.api.llama_token_batch(5, 1, it, 8, 128, 512)
    e.run_iteration(P.api.build_schedule(4, it == 2, 4), toks, None, it)
e.kill_stage(2)
e.recover_stage(2)
e.close()
print("engine iterations + recovery", flush=True)
