#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2r
python bench.py > ${T}_bench_c4.json 2> ${T}_bench_c4.err
python bench.py --workload C5 --steps 3 --warmup 3 --no-secondary > ${T}_bench_c5.json 2> ${T}_bench_c5.err
python bench.py --workload C2 --steps 20 --no-secondary > ${T}_bench_c2.json 2> ${T}_bench_c2.err
python bench.py --workload C2c --steps 20 --no-secondary > ${T}_bench_c2c.json 2> ${T}_bench_c2c.err
timeout 1200 python tools/bench_steps.py --out gpurun_out/r2r_steps.json > ${T}_steps.log 2>&1
for L in 32768 131072; do
  DMHA_LIB=paper_2302_06218_b200/ab/tr/libdmha.so TPHASES=1 TD=64 TL=$L timeout 120 python tools/trace.py > ${T}_trace64_$L.txt 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -k "parity or large or fuzz" > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
tail -c 250 ${T}_bench_c4.json; tail -c 250 ${T}_bench_c5.json; grep -h "period\|split softmax" ${T}_trace64_*.txt; tail -2 ${T}_pytest.log
