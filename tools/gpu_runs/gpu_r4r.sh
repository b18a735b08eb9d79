#!/bin/bash
# D=64: S issuer + one PV issuer per Q tile (4) with the fused combine / KV split allowed
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "env or fused or ring" 2>&1 | tail -2
DMHA_ISSUERS=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "ring or split or fused" 2>&1 | tail -2
bash tools/ab.sh "DMHA_ISSUERS=3;DMHA_ISSUERS=4;DMHA_ISSUERS=4 DMHA_KV_SPLIT=0;DMHA_ISSUERS=3 DMHA_KV_SPLIT=0;DMHA_ISSUERS=3;DMHA_ISSUERS=4" C2 C2c C5s
