#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2m
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "kv_split or workspace or fault or small" > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
bash tools/ab.sh "DMHA_SPLIT_MERGE=1;DMHA_SPLIT_MERGE=0;DMHA_KV_SPLIT=0" C2 C2c > ${T}_ab.txt 2>&1
tail -3 ${T}_pytest.log; cat ${T}_ab.txt
