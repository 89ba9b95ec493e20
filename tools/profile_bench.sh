#!/bin/bash
# Profiling pass for the bench workload (run under gpurun on ONE GPU).
#   1. launch list of one warm step (ncu, one metric, cold-cache serialised)
#   2. ncu --set full of the top kernels (GEMM, attention, norm-class)
# Outputs land in gpurun_out/; summaries are copied into profiles/ by hand.
set -u
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-recovery-sweep"
TAG=${1:-prof}
ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-0} -c ${COUNT:-3000} --csv \
    --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_launches.log 2>&1
# one training step: from one head-loss launch to the next (backward, Adam, next forward)
python tools/ncu_summary.py gpurun_out/${TAG}_launches.csv --window xent_pipe_kernel > gpurun_out/${TAG}_launches.txt 2>&1
for K in ${KERNELS:-gemm_kernel attn_ rmsnorm swiglu}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s ${KSKIP:-40} -c ${KCOUNT:-4} \
      -o gpurun_out/${TAG}_$K -f $B > gpurun_out/${TAG}_$K.log 2>&1
done
