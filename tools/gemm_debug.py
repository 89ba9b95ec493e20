#!/usr/bin/env python
"""CKF_GEMM_DEBUG=1 python tools/gemm_debug.py SHAPE: per-CTA phase cycles of one tcgen05 GEMM launch
(producer waiting for free stages, MMA waiting for data / for a free accumulator, epilogue waiting
for a full accumulator), averaged over CTAs, as fractions of the kernel's cycles."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gemm_bench as GB  # noqa
from paper_2506_15461_b200._native import check, lib
name = sys.argv[1]
s = next(x for x in GB.SHAPES if x[0] == name)
GB.run(*s, iters=3)
L = lib()
L.ckf_debug_gemm_timings.argtypes = [C.POINTER(C.c_longlong), C.c_int]
buf = (C.c_longlong * (8 * 148))()
check(L.ckf_debug_gemm_timings(buf, 148))
a = np.array(buf[:]).reshape(148, 8).astype(float)
tot = a[:, 4].mean()
print(f"{name}: cycles {tot:.0f}  producer-empty-wait {a[:,0].mean()/tot:.2f}  mma-full-wait {a[:,1].mean()/tot:.2f}  "
      f"mma-tempty-wait {a[:,2].mean()/tot:.2f}  epilogue-tfull-wait {a[:,3].mean()/tot:.2f}")
