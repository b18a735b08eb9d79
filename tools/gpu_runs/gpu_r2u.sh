#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2u
timeout 1500 python tools/soak.py 3000 21 bf16 > ${T}_soak_bf16.txt 2>&1; echo "rc=$?" >> ${T}_soak_bf16.txt
timeout 900 python tools/soak.py 800 22 fp32 > ${T}_soak_fp32.txt 2>&1; echo "rc=$?" >> ${T}_soak_fp32.txt
tail -3 ${T}_soak_bf16.txt ${T}_soak_fp32.txt
