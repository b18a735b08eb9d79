#!/bin/bash
# mbarrier suspend-time hint A/B (polling is 23 % of C4's instructions)
A=paper_2302_06218_b200/ab
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/hint10m/libdmha.so;DMHA_LIB=$A/hint1u/libdmha.so;DMHA_ALT=0;DMHA_LIB=$A/hint10m/libdmha.so" C4 C5s C2
for v in default hint10m hint1u; do
  if [ $v = default ]; then L=""; else L="DMHA_LIB=$A/$v/libdmha.so"; fi
  echo -n "$v: "; env $L timeout 300 python tools/tf32_flush_sweep.py 16384 8 64 0 2>&1 | tail -1
done
