#!/bin/bash
# probe: ceiling of removing the row max (constant stabiliser, N(0,1) data)
mkdir -p gpurun_out
T=gpurun_out/r2y
A=paper_2302_06218_b200/ab
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/nomax/libdmha.so;DMHA_ALT=0;DMHA_LIB=$A/nomax/libdmha.so" C4 C5s C2 > ${T}_ab.txt 2>&1
cat ${T}_ab.txt
