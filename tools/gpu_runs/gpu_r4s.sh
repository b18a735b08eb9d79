#!/bin/bash
# final: per-step table with the final build, then the whole GPU suite + smoke
mkdir -p gpurun_out
T=gpurun_out/r4s
timeout 1500 python tools/bench_steps.py --out gpurun_out/r4s_steps.json > ${T}_steps.log 2>&1; echo "steps rc=$?" >> ${T}_steps.log
timeout 2400 python -m pytest tests -m gpu -q > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${T}_smoke.log 2>&1
tail -2 ${T}_steps.log; tail -3 ${T}_pytest.log; tail -1 ${T}_smoke.log
