#!/usr/bin/env python
"""Fused stage recovery (26 B/param fp32) time at small stage sizes for the current
CKF_RECOVER_U / CKF_RECOVER_BPS; L2 flushed before each rep."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_15461_b200 as P  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {"U": os.environ.get("CKF_RECOVER_U"), "BPS": os.environ.get("CKF_RECOVER_BPS")}
for n in (10_000_000, 12_585_984, 25_000_000, 50_337_792, 100_000_000):
    t = [torch.rand(n, device="cuda") for _ in range(6)]
    wlp = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    fn = lambda: P.api.recover_stage_device(t[0], t[1], t[2], t[3], t[4], t[5], 4.0, 1.0, w_bf16=wlp)  # noqa: E731
    fn()
    ts = []
    for _ in range(9):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[4]
    out[str(n)] = {"us": round(ms * 1e3, 1), "frac": round(26.0 * n / (ms / 1e3) / 1e9 / 6463.3, 3)}
    del t, wlp
print(json.dumps(out), flush=True)
