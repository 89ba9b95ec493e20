#!/usr/bin/env python
"""Top SASS instructions by warp-stall samples from an ncu report (--page source --csv)."""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
si = hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r[si].isdigit()]
tot = sum(int(r[si] or 0) for r in body)
top = sorted(body, key=lambda r: -int(r[si] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
print(f"total samples {tot}")
for r in top:
    print(f"{int(r[si]):7d} {int(r[si]) / tot:6.1%}  {r[0][-5:]}  {r[1].strip()[:90]}")
