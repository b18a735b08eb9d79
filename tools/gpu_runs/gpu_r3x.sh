#!/bin/bash
# bf16 soak of the final build (D = 128 now sleeps on its barriers)
mkdir -p gpurun_out
timeout 1500 python tools/soak.py 2000 57 bf16 > gpurun_out/r3x_soak_bf16.txt 2>&1; echo "rc=$?" >> gpurun_out/r3x_soak_bf16.txt
tail -2 gpurun_out/r3x_soak_bf16.txt
