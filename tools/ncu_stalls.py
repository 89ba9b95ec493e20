#!/usr/bin/env python
"""Warp-stall breakdown of one kernel from an ncu report (--set full --import-source on):
totals per stall reason, and the top SASS instructions by stall samples with their main reasons.
  python tools/ncu_stalls.py REPORT.ncu-rep [top_n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {r: 0 for r in reasons}
lines = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    m = dict(zip(hdr, r))
    s = {k: int(m[k] or 0) for k in reasons}
    for k in reasons:
        tot[k] += s[k]
    n = int(m["Warp Stall Sampling (All Samples)"] or 0)
    lines.append((n, m["Address"][-5:], m["Source"].strip(), s))
allS = sum(tot.values())
print(f"{rep}: {allS} stall samples")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v:
        print(f"  {k[6:]:<18} {100.0 * v / allS:5.1f} %")
print("top instructions:")
for n, a, src, s in sorted(lines, key=lambda x: -x[0])[:top]:
    main = ", ".join(f"{k[6:]} {v}" for k, v in sorted(s.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"  {100.0 * n / allS:5.1f} %  {a}  {src[:60]:<60}  {main}")

# per CUDA source line (needs -lineinfo): samples and the top reasons
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
idx = hdr.index("Warp Stall Sampling (All Samples)")
rcols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
L = []
for r in rows[hi + 1:]:
    if len(r) != len(hdr) or r[2] != "-":  # CUDA-line rows carry "-" in the SASS address column
        continue
    n = int(r[idx] or 0)
    why = sorted(((int(r[i] or 0), h[6:]) for i, h in rcols), reverse=True)[:3]
    L.append((n, r[0], r[1].strip(), ", ".join(f"{w} {v}" for v, w in why if v)))
print("top CUDA lines:")
for n, ln, src, why in sorted(L, reverse=True)[:top]:
    print(f"  {100.0 * n / allS:5.1f} %  L{ln:<5} {src[:70]:<70}  {why}")
