#!/bin/bash
# MMA + TMA ceiling of the 3xTF32 kernel (softmax skipped; output garbage)
A=paper_2302_06218_b200/ab
M=sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum
for v in default probe; do
  if [ $v = default ]; then L=""; else L="DMHA_LIB=$A/$v/libdmha.so"; fi
  echo "== $v"
  env $L timeout 600 ncu --metrics $M --clock-control none -k regex:attn_fwd_tf32 -s 2 -c 1 python tools/ncu_kernels.py tf32 2>&1 | grep -E "tensor|duration"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fp32 or workspace" 2>&1 | tail -2
for shape in "16384 8 64 0" "16384 8 128 0"; do timeout 300 python tools/tf32_flush_sweep.py $shape 2>&1 | tail -1; done
