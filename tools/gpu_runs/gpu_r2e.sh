#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2e
for a in "128 64" "512 64" "256 128"; do timeout 60 ./tools/tf32_kernel_probe $a >> ${T}_tf32k.txt 2>&1; echo "probe $a rc=$?" >> ${T}_tf32k.txt; done
timeout 900 python -m pytest tests/test_gpu_peer.py -q -x > ${T}_peer.log 2>&1; echo "peer rc=$?" >> ${T}_peer.log
for a in 1 0; do DMHA_ALT=$a TD=128 TL=32768 timeout 120 python tools/trace.py > ${T}_trace128_alt$a.txt 2>&1; done
CMD="python bench.py --workload C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
$CMD > ${T}_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 \
    -o gpurun_out/r2e_c3 $CMD > ${T}_ncu.log 2>&1
echo "ncu rc=$?" >> ${T}_ncu.log
cat ${T}_tf32k.txt; tail -15 ${T}_peer.log; grep -h "period\|WG" ${T}_trace*.txt; tail -2 ${T}_ncu.log
