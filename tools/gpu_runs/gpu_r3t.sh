#!/bin/bash
A=paper_2302_06218_b200/ab
for v in default gsleep default gsleep; do
  if [ $v = default ]; then L=""; else L="DMHA_LIB=$A/$v/libdmha.so"; fi
  echo "== $v"; env $L timeout 300 python tools/gemm_time.py
done
