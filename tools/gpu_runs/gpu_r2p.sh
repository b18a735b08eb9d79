#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2p
for L in 32768 131072; do
  DMHA_LIB=paper_2302_06218_b200/ab/tr/libdmha.so TPHASES=1 TD=64 TL=$L timeout 120 python tools/trace.py > ${T}_trace64_$L.txt 2>&1
done
TL=131072 TH=16 TD=64 TC=1 timeout 120 python tools/cta_timeline.py > ${T}_cta64.txt 2>&1
grep -h "period\|split softmax" ${T}_trace64_*.txt; cat ${T}_cta64.txt
