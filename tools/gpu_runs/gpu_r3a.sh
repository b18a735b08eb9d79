#!/bin/bash
# pipelined 3xTF32 kernel: bounded-wait build first (a protocol bug traps, never hangs)
mkdir -p gpurun_out
T=gpurun_out/r3a
DMHA_LIB=paper_2302_06218_b200/ab/tf32b/libdmha.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fp32" > ${T}_bounded.log 2>&1
echo "bounded rc=$?"; tail -15 ${T}_bounded.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -k "fp32 or workspace or C1 or c1" > ${T}_default.log 2>&1
echo "default rc=$?"; tail -8 ${T}_default.log
timeout 300 python bench.py --workload C2f --steps 10 --warmup 3 --no-secondary --no-cpu-baseline > ${T}_c2f.json 2> ${T}_c2f.err
tail -c 700 ${T}_c2f.json; tail -3 ${T}_c2f.err
timeout 300 python bench.py --workload C1 --steps 20 --warmup 3 --no-secondary --no-cpu-baseline > ${T}_c1.json 2> ${T}_c1.err
python3 -c "import json;d=json.loads(open('${T}_c1.json').read().strip().splitlines()[-1]);print('C1', d['value'], d['ms_per_step'], d['roofline']['frac'])"
