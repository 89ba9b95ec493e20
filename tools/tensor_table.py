#!/usr/bin/env python
"""Joins an ncu CSV of tools/tensor_counter.py (one row per kernel launch, --csv --page raw)
with its FLOP sidecar: per launch group, tensor-pipe utilisation by counter vs by FLOP / time
at the clock ncu measured (dense bf16: 8192 FLOP / clk / SM x 148 SMs).
Usage: tensor_table.py ncu.csv tensor_flops.json out.json"""
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1]))]
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hdr_i]
ID, KN, MN, MV = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
# ncu --csv (details page) prints one row per (launch, metric): pivot to one dict per launch
per = {}
for r in rows[hdr_i + 1:]:
    if not r or not r[0].isdigit():
        continue
    d = per.setdefault(int(r[ID]), {"Kernel Name": r[KN]})
    try:
        d[r[MN]] = float(r[MV].replace(",", ""))
    except ValueError:
        d[r[MN]] = None
data = [per[k] for k in sorted(per)]
hdr = None
launches = json.load(open(sys.argv[2]))


def val(r, m):
    return r.get(m)


# map launches: attention backward = 3 kernels (dsum, dK/dV, dQ); everything else 1
out, i = [], 0
for L in launches:
    n = 3 if L["kernel"].startswith("attn_bwd") else 1
    grp = data[i:i + n]
    i += n
    t = sum(val(r, "gpu__time_duration.sum") or 0 for r in grp) * 1e-9  # ns
    clk = max(val(r, "sm__cycles_elapsed.avg.per_second") or 0 for r in grp)
    ops = sum(val(r, "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32.sum") or 0 for r in grp)
    w = [val(r, "gpu__time_duration.sum") or 0 for r in grp]
    def wavg(m):
        vs = [val(r, m) for r in grp]
        if any(v is None for v in vs):
            return None
        return sum(a * b for a, b in zip(vs, w)) / max(sum(w), 1e-30)
    peak = 8192.0 * 148 * clk
    rec = {"name": L["name"], "kernels": [r["Kernel Name"][:60] for r in grp], "time_us": t * 1e6,
           "sm_clock_mhz": clk / 1e6, "flops": L["flops"], "tflops": L["flops"] / t / 1e12,
           "frac_by_flops_at_clock": L["flops"] / t / peak,
           "hmma_cycles_active_pct": wavg("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed"),
           "tensor_cycles_active_pct": wavg("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
           "hmma_inst": sum(val(r, "sm__inst_executed_pipe_tensor_subpipe_hmma.sum") or 0 for r in grp)}
    out.append(rec)
json.dump(out, open(sys.argv[3], "w"), indent=1)
for r in out:
    print(f"{r['name']:20s} {r['time_us']:9.1f} us {r['tflops']:7.1f} TF/s  by-flop {r['frac_by_flops_at_clock']:.3f}"
          f"  hmma-cycles {r['hmma_cycles_active_pct']}  tensor-cycles {r['tensor_cycles_active_pct']}"
          f"  hmma-inst {r['hmma_inst']:.0f}")
