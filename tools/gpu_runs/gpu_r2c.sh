#!/bin/bash
# round-2 call 3: tf32 MMA probe, A/B knobs, kernel timelines, one ncu capture (C3, D=128)
mkdir -p gpurun_out
T=gpurun_out/r2c
timeout 60 ./tools/tf32_mma_probe > ${T}_tf32mma.txt 2>&1; echo "rc=$?" >> ${T}_tf32mma.txt
bash tools/ab.sh "DMHA_SPEC=1;DMHA_SPEC=0" C5s C2 > ${T}_ab.txt 2>&1
bash tools/ab.sh "DMHA_EMU=1;DMHA_EMU=2;DMHA_SPEC=1" C4 >> ${T}_ab.txt 2>&1
for sp in 1 0; do
  DMHA_SPEC=$sp TD=128 TL=32768 timeout 120 python tools/trace.py > ${T}_trace128_spec$sp.txt 2>&1
  DMHA_SPEC=$sp TD=64 TL=32768 timeout 120 python tools/trace.py > ${T}_trace64_spec$sp.txt 2>&1
done
CMD="python bench.py --workload C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
$CMD > ${T}_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 \
    -o gpurun_out/r2c_c3 $CMD > ${T}_ncu.log 2>&1
echo "ncu rc=$?" >> ${T}_ncu.log
cat ${T}_tf32mma.txt ${T}_ab.txt; tail -4 ${T}_trace*.txt; tail -3 ${T}_ncu.log
