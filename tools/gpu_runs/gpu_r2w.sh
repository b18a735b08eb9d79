#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2w
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "graph or headpar or workspace" > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
tail -25 ${T}_pytest.log
