#!/bin/bash
# round-2 call: fp32-path isolation, GPU suite without the fp32 tests, A/B, comparators
mkdir -p gpurun_out
T=gpurun_out/r2b
for c in p1_small p1_c1 p1_ragged_causal p1_d128 p1_d128_causal emu_p2 emu_p3 bf16_emu_p3; do
  timeout 60 python tools/tf32_probe.py $c >> ${T}_tf32.txt 2>&1; echo "tf32 $c rc=$?" >> ${T}_tf32.txt
  DMHA_FP32_SIMT=1 timeout 60 python tools/tf32_probe.py $c >> ${T}_tf32.txt 2>&1; echo "simt $c rc=$?" >> ${T}_tf32.txt
done
timeout 1200 python -m pytest tests -m gpu -q -k "not fp32 and not tf32" > ${T}_pytest.log 2>&1; echo "pytest rc=$?" >> ${T}_pytest.log
bash tools/ab.sh "DMHA_SPEC=1;DMHA_SPEC=0;DMHA_PS=1" C4 > ${T}_ab.txt 2>&1
bash tools/ab.sh "DMHA_EMU=0;DMHA_EMU=1;DMHA_EMU=2" C5s C2 >> ${T}_ab.txt 2>&1
timeout 600 python tools/comparators.py C4 C5s C2 C2c > ${T}_comp.txt 2>&1
tail -5 ${T}_pytest.log; cat ${T}_tf32.txt ${T}_ab.txt ${T}_comp.txt
