"""Times torch SDPA backends (cuDNN / flash / efficient) at the LLaMA-124M attention shape, as a
ceiling reference for our tcgen05 attention kernels (tools/attn_bench.py)."""
import torch, json, sys
from torch.nn.attention import sdpa_kernel, SDPBackend
B, H, T, D = [int(x) for x in (sys.argv[1:] or ["64", "8", "1024", "64"])]
q, k, v = [torch.randn(B, H, T, D, device="cuda", dtype=torch.bfloat16, requires_grad=True) for _ in range(3)]
flops_f = 4 * B * H * T * T * D / 2
for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
    try:
        with sdpa_kernel(be):
            o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
            g = torch.randn_like(o)
            for _ in range(3):
                o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True); o.backward(g)
            torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            n = 10; tf = tb = 0.0
            for _ in range(n):
                e[0].record(); o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True); e[1].record()
                o.backward(g); e[2].record(); torch.cuda.synchronize()
                tf += e[0].elapsed_time(e[1]); tb += e[1].elapsed_time(e[2])
            tf /= n; tb /= n
            print(json.dumps({"backend": str(be), "shape": [B, H, T, D], "fwd_us": tf * 1e3, "fwd_tflops": flops_f / tf / 1e9,
                              "bwd_us": tb * 1e3, "bwd_tflops": 2.5 * flops_f / tb / 1e9}))
    except Exception as ex:
        print(json.dumps({"backend": str(be), "error": str(ex)[:200]}))
