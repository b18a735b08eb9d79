#!/bin/bash
# final validation of the trace-free product build + C4 / C5s ncu evidence
mkdir -p gpurun_out
T=gpurun_out/r4f
timeout 2400 python -m pytest tests -m gpu -q > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${T}_smoke.log 2>&1
python bench.py > ${T}_bench_c4.json 2> ${T}_bench_c4.err
python bench.py --workload C1 --steps 20 --no-secondary > ${T}_bench_c1.json 2> ${T}_bench_c1.err
python bench.py --workload C2f --steps 10 --no-secondary > ${T}_bench_c2f.json 2> ${T}_bench_c2f.err
python bench.py --workload C2 --steps 20 --no-secondary > ${T}_bench_c2.json 2> ${T}_bench_c2.err
python bench.py --workload C2c --steps 20 --no-secondary > ${T}_bench_c2c.json 2> ${T}_bench_c2c.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
$CMD > ${T}_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4f_launches.csv $CMD > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/r4f_c4 $CMD > ${T}_ncu.log 2>&1
echo "ncu c4 rc=$?"
CMD5="python bench.py --workload C5s --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
$CMD5 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/r4f_c5s $CMD5 > ${T}_ncu5.log 2>&1
echo "ncu c5s rc=$?"
tail -3 ${T}_pytest.log; tail -1 ${T}_smoke.log
for f in c4 c1 c2f c2 c2c; do python3 -c "
import json
d=json.loads(open('${T}_bench_$f.json').read().strip().splitlines()[-1])
s=d.get('secondary') or {}
print('$f', round(d['value'],2), d['unit'], 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2) if d.get('e2e') else None, 'launches', d.get('gpu_launches'), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'], 'C5', round(s['C5']['value'],1) if 'C5' in s else None)"; done
