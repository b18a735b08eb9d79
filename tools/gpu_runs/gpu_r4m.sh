#!/bin/bash
# §8(d) max-L with the final product build
mkdir -p gpurun_out
timeout 3000 python tools/max_len.py --out gpurun_out/r4m_max_len.json > gpurun_out/r4m_max_len.log 2>&1; echo "rc=$?" >> gpurun_out/r4m_max_len.log
tail -12 gpurun_out/r4m_max_len.log
