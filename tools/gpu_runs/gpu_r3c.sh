#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r3c
F="--set full --clock-control none --import-source on"
timeout 300 python tools/ncu_kernels.py tf32 > ${T}_plain.log 2>&1 || { echo plain failed; tail ${T}_plain.log; exit 1; }
timeout 600 ncu $F -k regex:attn_fwd_tf32 -s 2 -c 1 -o ${T}_tf32 python tools/ncu_kernels.py tf32 > ${T}_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${T}_launches.csv python tools/ncu_kernels.py tf32 > /dev/null 2>&1; echo "launch rc=$?"
