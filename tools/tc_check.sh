#!/bin/bash
HK_TC=1 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for tc in 1 0; do echo "== HK_TC=$tc"; for cfg in c1 c2 c3; do HK_TC=$tc timeout 900 python tools/gpu_timing.py $cfg 2>&1 | head -2; done; done
