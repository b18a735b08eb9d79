#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2h
timeout 40 ./tools/tf32_abi_probe 128 64 > ${T}_tf32.txt 2>&1; echo "abi-probe rc=$?" >> ${T}_tf32.txt
timeout 40 ./tools/tf32_abi_probe 1000 128 >> ${T}_tf32.txt 2>&1; echo "abi-probe d128 rc=$?" >> ${T}_tf32.txt
if grep -q "HANG" ${T}_tf32.txt; then echo "tf32 still hangs; skipping fp32 tests" >> ${T}_tf32.txt; K='not fp32 and not tf32'; else K=''; fi
timeout 1500 python -m pytest tests -m gpu -q ${K:+-k "$K"} > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
timeout 2400 python tools/max_len.py --out gpurun_out/r2h_max_len.json > ${T}_maxlen.log 2>&1; echo "maxlen rc=$?" >> ${T}_maxlen.log
cat ${T}_tf32.txt; tail -4 ${T}_pytest.log; tail -4 ${T}_maxlen.log | cut -c1-400
