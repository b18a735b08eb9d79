#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2s
A=paper_2302_06218_b200/ab
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/s104/libdmha.so;DMHA_ALT=0" C5s C2 > ${T}_ab.txt 2>&1
cat ${T}_ab.txt
