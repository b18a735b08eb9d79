#!/bin/bash
# One gpurun call: GPU tests, the default bench line, optional A/B.
# usage: tools/gpu_check.sh <tag> [pytest-args] ; env AB="<env;env>" ABW="C5s C2"
tag=${1:-run}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt 2>&1
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q ${@:-} > gpurun_out/${tag}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
fi
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
  echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
fi
if [ -n "$AB" ]; then
  bash tools/ab.sh "$AB" ${ABW:-C5s} > gpurun_out/${tag}_ab.txt 2>&1
fi
tail -3 gpurun_out/${tag}_pytest.log 2>/dev/null; tail -c 600 gpurun_out/${tag}_bench.json 2>/dev/null; cat gpurun_out/${tag}_ab.txt 2>/dev/null
