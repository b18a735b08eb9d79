#!/bin/bash
# D=64 default now split S/PV issuers: the whole GPU suite + the D=64 bench lines
mkdir -p gpurun_out
T=gpurun_out/r4i
timeout 2400 python -m pytest tests -m gpu -q > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
tail -3 ${T}_pytest.log
bash tools/ab.sh "DMHA_ALT=0;DMHA_ALT=0" C2 C2c C5s
