#!/bin/bash
# last check of the exact final tree: every GPU test, smoke, the default bench line
mkdir -p gpurun_out
T=gpurun_out/r4v
timeout 2400 python -m pytest tests -m gpu -q > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${T}_smoke.log 2>&1
python bench.py > ${T}_bench_c4.json 2> ${T}_bench_c4.err
tail -3 ${T}_pytest.log; tail -1 ${T}_smoke.log
python3 -c "
import json
d=json.loads(open('${T}_bench_c4.json').read().strip().splitlines()[-1])
print('c4', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), 'clk', d['clocks'], 'C5', round(d['secondary']['C5']['value'],1))"
