#!/bin/bash
A=paper_2302_06218_b200/ab
for shape in "16384 8 64 0" "16384 8 128 0" "65536 2 64 1"; do
  for v in default k3v2f8 k2v2f8 k2v2f16 k2v2f8; do
    if [ $v = default ]; then L=""; else L="DMHA_LIB=$A/$v/libdmha.so"; fi
    echo -n "$v: "; env $L timeout 300 python tools/tf32_flush_sweep.py $shape 2>&1 | tail -1
  done
done
