#!/bin/bash
# trace-free product build: bench A/B reference points, parity, and the trace tool's own build
bash tools/ab.sh "DMHA_ALT=0;DMHA_ALT=0" C4 C5s C2 C3
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x -k "not fp32" 2>&1 | tail -2
timeout 600 python tools/trace.py 2>&1 | tail -4
