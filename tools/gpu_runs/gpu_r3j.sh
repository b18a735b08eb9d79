#!/bin/bash
python tools/host_overhead.py fp32; python tools/host_overhead.py bf16
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
python bench.py --workload C1 --steps 20 --no-secondary 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C1', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'])"
