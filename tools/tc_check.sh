#!/bin/bash
HK_TC=1 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for tc in 1 0; do echo "== HK_TC=$tc"; HK_TC=$tc timeout 600 python tools/gpu_timing.py c2 2>&1 | head -2; HK_TC=$tc timeout 900 python tools/gpu_timing.py c3 2>&1 | head -2; done
