#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r2i
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > ${T}_smi.txt 2>&1
python bench.py > ${T}_bench_c4.json 2> ${T}_bench_c4.err; echo "rc=$?" >> ${T}_bench_c4.err
python bench.py --workload C1 --steps 20 --no-secondary > ${T}_bench_c1.json 2> ${T}_bench_c1.err
python bench.py --workload C2 --steps 20 --no-secondary > ${T}_bench_c2.json 2> ${T}_bench_c2.err
python bench.py --workload C2c --steps 20 --no-secondary > ${T}_bench_c2c.json 2> ${T}_bench_c2c.err
DMHA_LIB=paper_2302_06218_b200/ab/r176/libdmha.so bash tools/ab.sh "DMHA_ALT=0" C4 > ${T}_ab.txt 2>&1
bash tools/ab.sh "DMHA_ALT=0" C4 >> ${T}_ab.txt 2>&1
timeout 1200 python tools/bench_steps.py --out gpurun_out/r2i_steps.json > ${T}_steps.log 2>&1; echo "steps rc=$?" >> ${T}_steps.log
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
$CMD > ${T}_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launches.csv $CMD > ${T}_ncu_launch.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/r2i_c4 $CMD > ${T}_ncu.log 2>&1
echo "ncu rc=$?" >> ${T}_ncu.log
tail -c 400 ${T}_bench_c4.json; cat ${T}_ab.txt; tail -3 ${T}_steps.log; tail -2 ${T}_ncu.log
