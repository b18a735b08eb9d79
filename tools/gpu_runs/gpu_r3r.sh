#!/bin/bash
# confirm: D=128 sleeps on barriers, D=64 polls (default build), vs the previous commit's numbers
bash tools/ab.sh "DMHA_ALT=0;DMHA_ALT=0;DMHA_ALT=0" C4 C5s C2 C3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not fp32" 2>&1 | tail -2
