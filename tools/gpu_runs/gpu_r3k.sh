#!/bin/bash
# soak the rewritten 3xTF32 kernel + the new fp32 ring parity tests
mkdir -p gpurun_out
T=gpurun_out/r3k
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "fp32" > ${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 ${T}_pytest.log
timeout 1200 python tools/soak.py 1000 31 fp32 > ${T}_soak_fp32.txt 2>&1; echo "rc=$?" >> ${T}_soak_fp32.txt
tail -3 ${T}_soak_fp32.txt
