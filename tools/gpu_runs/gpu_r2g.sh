#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2g
timeout 40 ./tools/tf32_kernel_probe_plain 128 64 > ${T}_tf32.txt 2>&1; echo "plain-probe rc=$?" >> ${T}_tf32.txt
timeout 40 ./tools/tf32_kernel_probe 128 64 >> ${T}_tf32.txt 2>&1; echo "bounded-probe rc=$?" >> ${T}_tf32.txt
timeout 40 ./tools/tf32_abi_probe 128 64 >> ${T}_tf32.txt 2>&1; echo "abi-probe rc=$?" >> ${T}_tf32.txt
DMHA_FP32_SIMT=1 timeout 40 ./tools/tf32_abi_probe 128 64 >> ${T}_tf32.txt 2>&1; echo "abi-probe simt rc=$?" >> ${T}_tf32.txt
bash tools/ab.sh "DMHA_ALT=0;DMHA_ALT=1" C4 > ${T}_ab.txt 2>&1
TD=128 TL=32768 timeout 120 python tools/trace.py > ${T}_trace128.txt 2>&1
cat ${T}_tf32.txt ${T}_ab.txt; grep -h "period\|WG0 per" ${T}_trace128.txt
