#!/bin/bash
timeout 600 python tools/trace.py 2>&1 | tail -6
