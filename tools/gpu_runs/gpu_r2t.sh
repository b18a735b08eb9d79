#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2t
A=paper_2302_06218_b200/ab
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "64" > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/wi0/libdmha.so;DMHA_ALT=0;DMHA_LIB=$A/wi0/libdmha.so" C5s C2 > ${T}_ab.txt 2>&1
tail -2 ${T}_pytest.log; cat ${T}_ab.txt
