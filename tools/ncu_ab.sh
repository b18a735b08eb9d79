#!/bin/bash
# Clock-independent A/B: tensor-pipe active % and issue stats per kernel variant.
# tools/ncu_ab.sh "<env>;<env>" workload   -> gpurun_out/ab_<workload>_<i>.csv
IFS=';' read -ra VARS <<< "$1"; w=$2
M=sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,gpu__time_duration.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active
mkdir -p gpurun_out
i=0
for v in "${VARS[@]}"; do
  i=$((i+1))
  env $v timeout 300 python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 || { echo "plain run failed for $v"; continue; }
  echo "$v" > gpurun_out/ab_${w}_$i.txt
  env $v timeout 600 ncu --metrics $M --clock-control none -k regex:attn_fwd -s 3 -c 1 --csv --log-file gpurun_out/ab_${w}_$i.csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
