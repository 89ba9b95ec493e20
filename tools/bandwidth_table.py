#!/usr/bin/env python
"""Joins tools/bandwidth_counter.py's ncu CSV (one row per launch and metric) with its algorithmic
bytes: per op, time, algorithmic GB/s and fraction of the measured HBM peak, ncu DRAM bytes.
Usage: bandwidth_table.py ncu.csv bandwidth_bytes.json out.json [hbm_gbs]"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ID, KN, MN, MV = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
per = {}
for r in rows[hi + 1:]:
    if r and r[0].isdigit():
        dct = per.setdefault(int(r[ID]), {"kernel": r[KN][:60]})
        try:
            dct[r[MN]] = float(r[MV].replace(",", ""))
        except ValueError:
            pass
launches = [per[k] for k in sorted(per)]
ops = json.load(open(sys.argv[2]))
peak = float(sys.argv[4]) if len(sys.argv) > 4 else 6463.3
out, i = [], 0
for op in ops:
    grp = launches[i:i + op["kernels"]]
    i += op["kernels"]
    t = sum(x.get("gpu__time_duration.sum", 0) for x in grp) * 1e-9
    dram = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in grp)
    gbs = op["bytes"] / t / 1e9
    out.append({"op": op["name"], "kernels": [x["kernel"] for x in grp], "time_us": t * 1e6,
                "algorithmic_bytes": op["bytes"], "dram_bytes": dram, "gbs": gbs, "frac_hbm": gbs / peak})
json.dump(out, open(sys.argv[3], "w"), indent=1)
for r in out:
    print(f"{r['op']:48s} {r['time_us']:9.1f} us {r['gbs']:7.0f} GB/s {r['frac_hbm']:.3f}  dram/alg "
          f"{r['dram_bytes'] / r['algorithmic_bytes']:.3f}")
