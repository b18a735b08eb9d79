#!/bin/bash
python tools/host_overhead.py fp32; python tools/host_overhead.py bf16
