#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tf32x3_and_simt" 2>&1 | tail -4
