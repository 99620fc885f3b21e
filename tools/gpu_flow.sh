#!/bin/bash
for d in 1 2; do echo "depth=$d"; for c in c1 c2 c3; do HK_LA_DEPTH=$d timeout 300 python tools/gpu_timing.py $c 2>/dev/null | head -1; done; done
