#!/bin/bash
# final validation of the committed state: every GPU test, smoke, bench lines
mkdir -p gpurun_out
T=gpurun_out/r3w
timeout 2400 python -m pytest tests -m gpu -q > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${T}_smoke.log 2>&1
python bench.py > ${T}_bench_c4.json 2> ${T}_bench_c4.err
python bench.py --workload C1 --steps 20 --no-secondary > ${T}_bench_c1.json 2> ${T}_bench_c1.err
python bench.py --workload C2f --steps 10 --no-secondary > ${T}_bench_c2f.json 2> ${T}_bench_c2f.err
python bench.py --workload C2 --steps 20 --no-secondary > ${T}_bench_c2.json 2> ${T}_bench_c2.err
tail -3 ${T}_pytest.log; tail -2 ${T}_smoke.log
for f in c4 c1 c2f c2; do python3 -c "
import json
d=json.loads(open('${T}_bench_$f.json').read().strip().splitlines()[-1])
s=d.get('secondary') or {}
print('$f', round(d['value'],2), d['unit'], 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2) if d.get('e2e') else None, 'launches', d.get('gpu_launches'), 'clk', d['clocks']['sm_mhz'], 'C5', round(s['C5']['value'],1) if 'C5' in s else None)"; done
