#!/bin/bash
# 3xTF32 knobs: ring depths and flush interval (C2f shape D=64, and D=128)
A=paper_2302_06218_b200/ab
for shape in "16384 8 64 0" "16384 8 128 0"; do
  for v in default k2v2 k2v3 f8 f2 default; do
    if [ $v = default ]; then L=""; else L="DMHA_LIB=$A/$v/libdmha.so"; fi
    echo -n "$v: "; env $L timeout 300 python tools/tf32_flush_sweep.py $shape 2>&1 | tail -1
  done
done
