#!/bin/bash
# D=64 issuer schedule on the final build: 2 (one per Q tile, current default) vs 3 (S / PV split)
bash tools/ab.sh "DMHA_ISSUERS=2;DMHA_ISSUERS=3;DMHA_ISSUERS=2;DMHA_ISSUERS=3" C2 C2c C5s C5nc
for v in 2 3; do
  echo -n "C5 full iss=$v: "; DMHA_ISSUERS=$v timeout 600 python bench.py --workload C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), d['clocks']['sm_mhz'])"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "env" 2>&1 | tail -2
