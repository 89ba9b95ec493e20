#!/usr/bin/env python
"""DRAM traffic per GEMM launch from an ncu CSV capture
(--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum), written to
profiles/r0N_<workload>_gemm_dram_traffic.json for bench.py's roofline.traffic.
Usage: ncu_traffic.py capture.csv out.json "<command that produced it>" """
import csv, json, sys, re, collections

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
hdr = next(r for r in csv.reader(open(sys.argv[1])) if r and r[0] == "ID")
mi, vi, ki = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Kernel Name")
units = hdr.index("Metric Unit")
per = collections.defaultdict(dict)
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1024 ** 2, "GB": 1024 ** 3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
for r in rows:
    v = float(r[vi].replace(",", "")) * scale.get(r[units], 1.0)
    per[r[0]][r[mi]] = v
    per[r[0]]["kernel"] = re.sub(r"\(.*", "", r[ki])
launches = [p for p in per.values() if "gemm_kernel" in p["kernel"]]
rd = sum(p.get("dram__bytes_read.sum", 0) for p in launches)
wr = sum(p.get("dram__bytes_write.sum", 0) for p in launches)
t = sum(p.get("gpu__time_duration.sum", 0) for p in launches)
out = {"kernel_class": "gemm", "launches": len(launches), "dram_read_bytes": rd, "dram_write_bytes": wr,
       "traffic_per_launch_bytes": (rd + wr) / max(1, len(launches)),
       "ncu_time_s": t, "note": "ncu cold-cache serialised replay; one bench step's GEMM launches",
       "command": sys.argv[3] if len(sys.argv) > 3 else ""}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out))
