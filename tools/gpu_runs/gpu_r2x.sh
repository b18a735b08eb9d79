#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2x
timeout 1500 python -m pytest tests -m gpu -q -x > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
bash tools/ab.sh "DMHA_ALT=0" C4 C5s > ${T}_ab.txt 2>&1
tail -15 ${T}_pytest.log; cat ${T}_ab.txt
