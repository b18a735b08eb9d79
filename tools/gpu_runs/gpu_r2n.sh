#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2n
A=paper_2302_06218_b200/ab
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/ef1/libdmha.so;DMHA_LIB=$A/ef2/libdmha.so;DMHA_ALT=1" C4 C3 > ${T}_ab.txt 2>&1
bash tools/ab.sh "DMHA_LIB=$A/ef2/libdmha.so DMHA_ALT=1" C4 >> ${T}_ab.txt 2>&1
for v in ef1 ef2; do DMHA_LIB=$A/$v/libdmha.so TD=128 TL=32768 timeout 120 python tools/trace.py > ${T}_trace_$v.txt 2>&1; done
cat ${T}_ab.txt; grep -h "period\|WG0 per" ${T}_trace*.txt
