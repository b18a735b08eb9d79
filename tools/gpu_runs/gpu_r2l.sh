#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2l
for cfg in "16384 8 64 0" "65536 8 64 0" "16384 8 64 1" "32768 16 128 0"; do
  set -- $cfg
  TL=$1 TH=$2 TD=$3 TC=$4 timeout 120 python tools/cta_timeline.py >> ${T}_cta.txt 2>&1
  DMHA_KV_SPLIT=0 TL=$1 TH=$2 TD=$3 TC=$4 timeout 120 python tools/cta_timeline.py >> ${T}_cta.txt 2>&1
done
cat ${T}_cta.txt
