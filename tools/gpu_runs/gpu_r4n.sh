#!/bin/bash
# bench lines of the final product build (D = 64 split issuers)
mkdir -p gpurun_out
T=gpurun_out/r4n
python bench.py > ${T}_bench_c4.json 2> ${T}_bench_c4.err
python bench.py --workload C2 --steps 20 --no-secondary > ${T}_bench_c2.json 2> ${T}_bench_c2.err
python bench.py --workload C2c --steps 20 --no-secondary > ${T}_bench_c2c.json 2> ${T}_bench_c2c.err
for f in c4 c2 c2c; do python3 -c "
import json
d=json.loads(open('${T}_bench_$f.json').read().strip().splitlines()[-1])
s=d.get('secondary') or {}
print('$f', round(d['value'],2), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2) if d.get('e2e') else None, 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'], 'C5', round(s['C5']['value'],1) if 'C5' in s else None)"; done
