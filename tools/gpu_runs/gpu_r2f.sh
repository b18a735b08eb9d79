#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2f
bash tools/ab.sh "DMHA_ALT=1;DMHA_ALT=0" C4 C3 > ${T}_ab.txt 2>&1
for a in 1 0; do DMHA_ALT=$a TD=128 TL=32768 timeout 120 python tools/trace.py > ${T}_trace128_alt$a.txt 2>&1; done
for c in p1_small p1_c1 emu_p3 p1_d128_causal; do timeout 60 python tools/tf32_probe.py $c >> ${T}_tf32.txt 2>&1; echo "tf32 $c rc=$?" >> ${T}_tf32.txt; done
timeout 1500 python -m pytest tests -m gpu -q > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
cat ${T}_ab.txt; grep -h "period\|WG" ${T}_trace*.txt; cat ${T}_tf32.txt; tail -5 ${T}_pytest.log
