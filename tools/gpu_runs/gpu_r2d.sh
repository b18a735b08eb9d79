#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2d
bash tools/ab.sh "DMHA_ALT=1;DMHA_ALT=0" C4 C3 > ${T}_ab.txt 2>&1
bash tools/ab.sh "DMHA_SPEC=0" C5s C2 >> ${T}_ab.txt 2>&1
for a in 1 0; do DMHA_ALT=$a TD=128 TL=32768 timeout 120 python tools/trace.py > ${T}_trace128_alt$a.txt 2>&1; done
timeout 1200 python -m pytest tests -m gpu -q -k "not fp32 and not tf32" > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
cat ${T}_ab.txt; grep -h period ${T}_trace*.txt; tail -3 ${T}_pytest.log
