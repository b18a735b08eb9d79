#!/bin/bash
# A/B kernel variants on one GPU: tools/ab.sh "<env settings>;..." workload...
# e.g. tools/ab.sh "DMHA_EMU=0;DMHA_EMU=2" C4 C2
IFS=';' read -ra VARS <<< "$1"; shift
for w in "$@"; do
  for v in "${VARS[@]}"; do
    r=$(env $v timeout 300 python bench.py --workload $w --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary 2>&1 | tail -1)
    echo "$w [$v] $(echo "$r" | python3 -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d["value"],1), "TF/s", round(d["ms_per_step"],3), "ms frac", round(d["roofline"]["frac"],3), "clk", d["clocks"]["sm_mhz"])
except Exception as e: print("FAILED", e)')"
  done
done
