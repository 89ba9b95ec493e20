#!/bin/bash
# Round-2 profiling pass of the headline workload (LLaMA-500M, 8 stages, CheckFree+) on ONE GPU.
#   1. launch list of one step (ncu, one metric, cold-cache serialised) -> per-kernel shares
#   2. DRAM bytes of every GEMM launch of one step -> roofline.traffic for bench.py
#   3. ncu --set full of the top GEMM families and both attention kernels (source-mapped)
set -u
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-recovery-sweep"
O=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 3200 --csv --log-file $O/r02_launches.csv $B \
    > $O/r02_launches.log 2>&1
python tools/ncu_summary.py $O/r02_launches.csv --window xent_combine_kernel:2 > $O/r02_launches.txt 2>&1
# one step's GEMM launches (the first eager step: 24 layers / 8 stages / 2 order classes)
NG=$(grep -c "gemm_kernel" <(python - <<'PY'
import csv, re
rows=[r for r in csv.reader(open("gpurun_out/r02_launches.csv")) if len(r) > 10 and r[0] != "ID"]
idx=[i for i, r in enumerate(rows) if "xent_combine_kernel" in r[4]]
for r in rows[idx[0]:idx[2]]:
    print(r[4])
PY
))
echo "gemm launches per step: $NG"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:gemm_kernel -c $NG --csv --log-file $O/r02_gemm_traffic.csv $B > $O/r02_gemm_traffic.log 2>&1
python tools/ncu_traffic.py $O/r02_gemm_traffic.csv $O/r02_llama-500m_gemm_dram_traffic.json "$B (first step, $NG GEMM launches)"
# (demangled names read "gemm_kernel<(int)256, (bool)0, ...": "." matches the parentheses)
KLIST=("gemm_kernel<.int.256, .bool.0, .bool.1, .int.3" "gemm_kernel<.int.256, .bool.0, .bool.0, .int.4"
       "gemm_kernel<.int.256, .bool.1, .bool.1, .int.2" "gemm_kernel<.int.256, .bool.0, .bool.1, .int.5"
       attn_fwd_tc attn_dkdv attn_dq_gemm)
[ -n "${ONLY_GEMM:-}" ] && KLIST=("${KLIST[@]:0:4}")
for K in "${KLIST[@]}"; do
  T=$(echo "$K" | tr -c 'a-zA-Z0-9' '_')
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:${K}" -s 2 -c 1 -o $O/r02_full_$T -f $B \
      > $O/r02_full_$T.log 2>&1
  python tools/ncu_metrics.py $O/r02_full_$T.ncu-rep > $O/r02_full_$T.txt 2>&1
done
