#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2v
A=paper_2302_06218_b200/ab
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/k2v2/libdmha.so;DMHA_LIB=$A/k4v3/libdmha.so;DMHA_LIB=$A/k4v4/libdmha.so;DMHA_LIB=$A/k5v5/libdmha.so;DMHA_ALT=0" C5s C2 > ${T}_ab.txt 2>&1
cat ${T}_ab.txt
