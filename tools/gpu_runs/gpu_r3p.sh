#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "host" 2>&1 | tail -4
