#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2q
A=paper_2302_06218_b200/ab
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/nostamp/libdmha.so;DMHA_LIB=$A/old1a3/libdmha.so;DMHA_ALT=0" C5s C2 C4 > ${T}_ab.txt 2>&1
cat ${T}_ab.txt
