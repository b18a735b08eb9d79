#!/bin/bash
# round-2 ncu --set full captures of the non-C4 kernels: D=64 north-star attention
# (C5s), 3xTF32 attention, tcgen05 GEMM, head-parallel pack/unpack, LSE combine
mkdir -p gpurun_out
T=gpurun_out/r2z
F="--set full --clock-control none --import-source on"
CMD="python bench.py --workload C5s --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
$CMD > ${T}_c5s_plain.log 2>&1 && timeout 600 ncu $F -k regex:attn_fwd -s 3 -c 1 -o ${T}_c5s $CMD > ${T}_c5s_ncu.log 2>&1
echo "c5s rc=$?"
for k in tf32:attn_fwd_tf32 gemm:gemm headpar:pack_qkv combine:lse_combine; do
  m=${k%%:*}; re=${k##*:}
  timeout 300 python tools/ncu_kernels.py $m > ${T}_${m}_plain.log 2>&1 || { echo "$m plain failed"; tail -5 ${T}_${m}_plain.log; continue; }
  timeout 600 ncu $F -k regex:$re -s 2 -c 1 -o ${T}_$m python tools/ncu_kernels.py $m > ${T}_${m}_ncu.log 2>&1
  echo "$m rc=$?"
done
ls -la gpurun_out/ | grep r2z
