#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
HK_TC=1 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for cfg in c1 c2 c3; do timeout 900 python tools/gpu_timing.py $cfg 2>&1 | head -2; done
