#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2k
bash tools/ab.sh "DMHA_KV_SPLIT=1;DMHA_KV_SPLIT=0" C2 > ${T}_ab.txt 2>&1
bash tools/ab.sh "DMHA_KV_SPLIT=1" C2x4 C5nc C5s >> ${T}_ab.txt 2>&1
TD=64 TL=16384 timeout 120 python tools/trace.py > ${T}_trace64_c2.txt 2>&1
cat ${T}_ab.txt; grep -h "period" ${T}_trace64_c2.txt
