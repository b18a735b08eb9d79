#!/bin/bash
A=paper_2302_06218_b200/ab
DMHA_LIB=$A/heavy/libdmha.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "split or small or causal" 2>&1 | tail -2
bash tools/ab.sh "DMHA_ALT=0;DMHA_LIB=$A/heavy/libdmha.so;DMHA_KV_SPLIT=0;DMHA_ALT=0;DMHA_LIB=$A/heavy/libdmha.so" C2c C2
