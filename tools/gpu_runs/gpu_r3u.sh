#!/bin/bash
# C4 evidence for the final D=128 build: plain run, launch list, ncu --set full
mkdir -p gpurun_out
T=gpurun_out/r3u
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
$CMD > ${T}_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3u_launches.csv $CMD > ${T}_ncu_launch.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/r3u_c4 $CMD > ${T}_ncu.log 2>&1
echo "ncu rc=$?"; tail -c 300 ${T}_plain.log
