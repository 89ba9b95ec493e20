#!/usr/bin/env python
"""Key metrics per profiled kernel from an ncu report (ncu -i ... --page raw --csv)."""
import csv
import io
import subprocess
import sys

KEYS = {
    "time_us": "gpu__time_duration.sum",
    "dram_rd_MB": "dram__bytes_read.sum",
    "dram_wr_MB": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct2": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "hmma_pct": "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "tensor_mem_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread",
    "occupancy": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "grid": "launch__grid_size",
    "smem_KB": "launch__shared_mem_per_block_dynamic",
}


def main():
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:70]
        vals = {k: r[hdr.index(m)] for k, m in KEYS.items() if m in hdr}
        print(name, " ".join(f"{k}={v}" for k, v in vals.items()))


if __name__ == "__main__":
    main()
