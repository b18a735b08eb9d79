#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r3d
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fp32 or workspace" > ${T}_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 ${T}_pytest.log
for shape in "16384 8 64 0" "16384 8 64 1" "16384 8 128 0" "65536 2 64 0"; do
  timeout 300 python tools/tf32_flush_sweep.py $shape 2>&1 | tail -1
done
timeout 600 ncu --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:attn_fwd_tf32 -s 2 -c 1 python tools/ncu_kernels.py tf32 2>&1 | grep -E "tensor|duration|per_second"
