#!/bin/bash
# full validation of the committed state
mkdir -p gpurun_out
T=gpurun_out/r3g
timeout 2400 python -m pytest tests -m gpu -q > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${T}_smoke.log 2>&1
python bench.py > ${T}_bench_c4.json 2> ${T}_bench_c4.err
python bench.py --workload C1 --steps 20 --no-secondary > ${T}_bench_c1.json 2> ${T}_bench_c1.err
python bench.py --workload C2f --steps 10 --no-secondary > ${T}_bench_c2f.json 2> ${T}_bench_c2f.err
tail -3 ${T}_pytest.log; cat ${T}_smoke.log | tail -2
for f in c4 c1 c2f; do python3 -c "
import json
d=json.loads(open('${T}_bench_$f.json').read().strip().splitlines()[-1])
print('$f', round(d['value'],2), d['unit'], 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2) if d.get('e2e') else None, 'launches', d.get('gpu_launches'))"; done
