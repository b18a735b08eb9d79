#!/bin/bash
# comparators and our final build on the same box
mkdir -p gpurun_out
timeout 1500 python tools/comparators.py > gpurun_out/r4t_comparators.jsonl 2> gpurun_out/r4t_comparators.err; echo "rc=$?"
bash tools/ab.sh "DMHA_ALT=0;DMHA_ALT=0" C4 C5s C2 C2c
python3 -c "
import json
for l in open('gpurun_out/r4t_comparators.jsonl'):
    try:
        d=json.loads(l); print(d.get('config') or d.get('workload'), d.get('impl') or d.get('name'), round(d.get('tflops',0),1), d.get('sm_mhz') or d.get('clk'))
    except Exception as e: pass
"
