#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2o
timeout 1500 python -m pytest tests -m gpu -q > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
python bench.py > ${T}_bench_c4.json 2> ${T}_bench_c4.err
python bench.py --workload C5 --steps 3 --warmup 3 --no-secondary > ${T}_bench_c5.json 2> ${T}_bench_c5.err
timeout 1200 python tools/bench_steps.py --out gpurun_out/r2o_steps.json > ${T}_steps.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > ${T}_smoke.log 2>&1; echo "smoke rc=$?" >> ${T}_smoke.log
tail -3 ${T}_pytest.log; tail -c 300 ${T}_bench_c4.json; tail -c 300 ${T}_bench_c5.json; tail -2 ${T}_smoke.log
