#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "empty_shards" 2>&1 | tail -15
