#!/bin/bash
# D=64: 32-bit key limit (no spill) vs the previous build
A=paper_2302_06218_b200/ab
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/old/libdmha.so;DMHA_ALT=0;DMHA_LIB=$A/old/libdmha.so" C5s C2 C2c
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x -k "not fp32" 2>&1 | tail -2
