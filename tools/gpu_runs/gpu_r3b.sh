#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r3b
A=paper_2302_06218_b200/ab
for shape in "16384 8 64 0" "65536 2 64 0" "16384 8 128 0" "65536 2 128 0"; do
  for v in f1 f2 default f8 f16 f100000; do
    if [ $v = default ]; then L=""; else L="DMHA_LIB=$A/$v/libdmha.so"; fi
    echo -n "$v: "; env $L timeout 300 python tools/tf32_flush_sweep.py $shape 2>&1 | tail -1
  done
done > ${T}_sweep.txt
cat ${T}_sweep.txt
